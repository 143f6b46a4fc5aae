#!/bin/bash
O=gpurun_out/r2an; mkdir -p $O
for wl in alexnet convnet vgga overfeat; do
  for v in force def; do
    if [ $v = force ]; then E="PT_B200_HCONV=1"; else E="PT_B200_X=0"; fi
    env $E timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-e2e > $O/${wl}_$v.json 2>>$O/err.txt
  done
done
