#!/bin/bash
O=gpurun_out/stress; mkdir -p $O
timeout 900 python tests/stress_tc.py 120 11 smallc > $O/smallc.txt 2>&1; echo "rc=$?" >> $O/smallc.txt
timeout 1200 python tests/stress_tc.py 200 12 > $O/default.txt 2>&1; echo "rc=$?" >> $O/default.txt
timeout 1200 python tests/stress_tc.py 160 13 wide > $O/wide.txt 2>&1; echo "rc=$?" >> $O/wide.txt
