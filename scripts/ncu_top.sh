#!/bin/bash
# ncu --set full captures of the hot kernels, one pass per capture (1 GPU).
# usage: gpurun --timeout 1800 -- bash scripts/ncu_top.sh TAG "layer:pass:kregex" ...
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
for spec in "$@"; do
  IFS=: read layer pass kre wl <<< "$spec"
  wl=${wl:-convnet}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kre -s 1 -c 1 \
     -o $OUT/${wl}_${layer}_${pass} python tests/prof_one.py --workload $wl --layer $layer --pass $pass --iters 2 \
     > $OUT/${wl}_${layer}_${pass}.log 2>&1
  echo "$spec rc=$?"
done
