#!/bin/bash
O=gpurun_out/r2x; mkdir -p $O
PT_B200_SCX16=1 CUDA_LAUNCH_BLOCKING=1 timeout 60 python tests/scbwd_debug.py dgrad > $O/dgrad16.txt 2>&1; echo "rc=$?" >> $O/dgrad16.txt
PT_B200_SCX16=1 CUDA_LAUNCH_BLOCKING=1 timeout 60 python tests/scbwd_debug.py both big > $O/both16.txt 2>&1; echo "rc=$?" >> $O/both16.txt
