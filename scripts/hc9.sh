#!/bin/bash
OUT=gpurun_out/hc9; mkdir -p $OUT
for g in 2 4; do
PT_B200_HCONV_GROUP_MAX=$g timeout 600 ncu --set full --clock-control none --import-source on -k regex:umma_hconv -s 1 -c 1 -o $OUT/L1_dgrad_g$g python tests/prof_one.py --layer L1 --pass dgrad --iters 2 > /dev/null 2>&1
ncu -i $OUT/L1_dgrad_g$g.ncu-rep --page source --csv --print-source sass > $OUT/L1_dgrad_g${g}_src.csv 2>/dev/null
done
