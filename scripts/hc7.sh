#!/bin/bash
OUT=gpurun_out/hc7; mkdir -p $OUT
PT_B200_HCONV=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:umma_hconv -s 1 -c 1 -o $OUT/L3_dgrad_h python tests/prof_one.py --layer L3 --pass dgrad --iters 2 > /dev/null 2>&1
PT_B200_HCONV=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:umma_hconv -s 1 -c 1 -o $OUT/L2_fwd_h python tests/prof_one.py --layer L2 --pass fwd --iters 2 > /dev/null 2>&1
for f in $OUT/*.ncu-rep; do ncu -i $f --page source --csv --print-source sass > ${f%.ncu-rep}_src.csv 2>/dev/null; done
