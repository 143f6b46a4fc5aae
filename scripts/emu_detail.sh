#!/bin/bash
O=gpurun_out/emu; mkdir -p $O
for spec in "alexnet 8" "vgga 8" "overfeat 8" "convnet 8"; do set -- $spec
  timeout 300 python bench.py --workload $1 --emulate-ranks $2 --no-cpu-baseline --no-e2e --no-alexnet > $O/${1}_g$2.json 2>>$O/err.txt
done
