#!/bin/bash
OUT=gpurun_out/hc4; mkdir -p $OUT
PT_B200_HCONV=1 timeout 300 python tests/gpu_probe.py > $OUT/probe_h.log 2>&1
PT_B200_HCONV=1 bash scripts/ncu_top.sh hc4 "L2:fwd:umma_hconv"
PT_B200_HCONV=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:umma_conv -s 1 -c 1 -o $OUT/convnet_L2_fwd_im2col python tests/prof_one.py --layer L2 --pass fwd --iters 2 > /dev/null 2>&1
for f in $OUT/*.ncu-rep; do ncu -i $f --page source --csv --print-source sass > ${f%.ncu-rep}_src.csv 2>/dev/null; done
