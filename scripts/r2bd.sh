#!/bin/bash
O=gpurun_out/r2bd; mkdir -p $O
SPECS='[[2,3,20,20,32,3,3,1,1,1,1],[1,1,20,40,48,5,5,2,2,1,1],[3,2,18,36,32,3,5,1,2,1,1],[2,3,224,224,64,3,3,1,1,1,1]]'
PT_B200_SCBWD_A32=1 timeout 300 python tests/engine_check.py "$SPECS" > $O/check.txt 2>&1; echo "rc=$?" >> $O/check.txt
for a in 0 1; do echo "a32=$a $(PT_B200_SCBWD_A32=$a timeout 120 python tests/scbwd_tl.py 2>&1 | grep 'rep 2')"; done > $O/t.txt
cat $O/t.txt; tail -c 400 $O/check.txt
