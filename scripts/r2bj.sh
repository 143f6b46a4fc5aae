#!/bin/bash
O=gpurun_out/r2bj; mkdir -p $O
SPECS='[[2,3,63,63,64,11,11,2,2,4,4],[2,3,67,67,96,11,11,0,0,4,4],[2,48,20,20,64,3,3,1,1,1,1],[2,40,18,22,72,5,5,2,2,1,1],[1,3,227,227,64,11,11,2,2,4,4]]'
timeout 300 python tests/engine_check.py "$SPECS" > $O/check.txt 2>&1; echo "rc=$?" >> $O/check.txt
PT_B200_HCONV=1 timeout 300 python tests/engine_check.py "$SPECS" > $O/check_h.txt 2>&1; echo "rc=$?" >> $O/check_h.txt
tail -c 200 $O/check.txt; tail -c 200 $O/check_h.txt
timeout 900 bash scripts/ab.sh PT_B200_HCONV_KSKIP "alexnet overfeat" 3 > $O/ab.txt 2>&1
cat $O/ab.txt
