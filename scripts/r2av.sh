#!/bin/bash
O=gpurun_out/r2av; mkdir -p $O
timeout 120 python tests/scbwd_tl.py > $O/plain.txt 2>&1
PT_B200_SCBWD_DBG=16 timeout 120 python tests/scbwd_tl.py > $O/tl.txt 2>&1
SPECS='[[2,3,38,44,64,3,3,1,1,1,1],[2,1,20,40,48,5,5,2,2,1,1],[3,2,18,36,32,3,5,1,2,1,1],[2,3,224,224,64,3,3,1,1,1,1]]'
timeout 300 python tests/engine_check.py "$SPECS" > $O/check.txt 2>&1; echo "rc=$?" >> $O/check.txt
cat $O/plain.txt; tail -c 300 $O/check.txt
