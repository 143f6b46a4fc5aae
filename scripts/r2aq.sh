#!/bin/bash
# gfold (small-C gradCol + fold dgrad): parity on its edge geometries, then an A/B on convnet
O=gpurun_out/r2aq; mkdir -p $O
for a in "3 3 40 40 96 11 11 0 0" "2 3 128 128 96 11 11 0 0" "3 3 19 22 16 2 3 1 1"; do
  timeout 120 python tests/gfold_probe.py $a 2 >> $O/probe.txt 2>&1; echo "rc=$?" >> $O/probe.txt
done
timeout 120 python tests/gfold_probe.py 128 3 128 128 96 11 11 0 0 4 >> $O/probe.txt 2>&1; echo "rc=$?" >> $O/probe.txt
cat $O/probe.txt
SPECS='[[3,3,40,40,96,11,11,0,0,1,1],[1,1,50,37,40,9,7,3,2,1,1],[2,2,33,100,64,5,13,2,6,1,1],[3,3,19,22,16,2,3,1,1,1,1],[2,3,44,70,72,13,9,6,4,1,1],[5,4,26,36,24,5,5,0,4,1,1],[2,3,20,302,32,3,3,1,1,1,1],[2,3,128,128,96,11,11,0,0,1,1]]'
timeout 300 python tests/engine_check.py "$SPECS" > $O/check.txt 2>&1; echo "rc=$?" >> $O/check.txt
tail -c 1500 $O/check.txt
timeout 300 ncu --set full --import-source on --clock-control none -k regex:umma_gfold -c 1 -o $O/gfold_l1 python tests/gfold_probe.py 128 3 128 128 96 11 11 0 0 1 > $O/ncu.txt 2>&1
