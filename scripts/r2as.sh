#!/bin/bash
O=gpurun_out/r2as; mkdir -p $O; : > $O/t.txt
for d in 0 1 15; do
  echo "dbg=$d" >> $O/t.txt
  PT_B200_GFOLD_DBG=$d timeout 60 python tests/gfold_probe.py 128 3 128 128 96 11 11 0 0 3 2>&1 | grep -E "rep 2|normwise" >> $O/t.txt
  PT_B200_GFOLD_DBG=$d timeout 60 python tests/gfold_probe.py 2 3 128 128 96 11 11 0 0 3 2>&1 | grep "rep 2" >> $O/t.txt
done
SPECS='[[3,3,40,40,96,11,11,0,0,1,1],[1,1,50,37,40,9,7,3,2,1,1],[2,2,33,100,64,5,13,2,6,1,1],[3,3,19,22,16,2,3,1,1,1,1],[2,3,44,70,72,13,9,6,4,1,1],[5,4,26,36,24,5,5,0,4,1,1],[2,3,20,302,32,3,3,1,1,1,1],[2,3,128,128,96,11,11,0,0,1,1]]'
timeout 300 python tests/engine_check.py "$SPECS" > $O/check.txt 2>&1; echo "rc=$?" >> $O/check.txt
timeout 300 ncu --set full --import-source on --clock-control none -k regex:umma_gfold -c 1 -o $O/full python tests/gfold_probe.py 128 3 128 128 96 11 11 0 0 1 > /dev/null 2>&1
cat $O/t.txt
