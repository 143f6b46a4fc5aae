#!/bin/bash
# Round evidence: bench line, launch list of the same command, ncu --set full of the top launches.
TAG=${1:-r1}
OUT=gpurun_out/ev_$TAG; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 900 python bench.py > $OUT/bench_convnet.json 2> $OUT/bench_convnet.err
for wl in alexnet vgga overfeat; do timeout 300 python bench.py --workload $wl --no-cpu-baseline > $OUT/bench_$wl.json 2>> $OUT/bench.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
   python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
KEEP="convnet_L2_dgrad convnet_L2_wgrad" bash scripts/ncu_top.sh ev_$TAG "L2:dgrad:umma_hconv" "L2:fwd:umma_hconv" "L2:wgrad:umma_hwgrad" "L1:dgrad:umma_hconv" \
   "L1:wgrad:umma_swgrad" "L1:fwd:umma_rowconv" "L3:dgrad:umma_conv" "L3:wgrad:umma_hwgrad" "L1:bwd:nchw_to_nhwc" \
   "c1:fwd:umma_rowconv:vgga" "c1:wgrad:umma_swgrad:vgga" "c1:fwd:umma_hconv:alexnet"
