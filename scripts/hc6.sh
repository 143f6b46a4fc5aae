#!/bin/bash
OUT=gpurun_out/hc6; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log; tail -3 $OUT/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
bash scripts/ncu_top.sh hc6 "L1:fwd:umma_rowconv" "L1:wgrad:umma_wgrad" "L2:wgrad:umma_wgrad" "L2:dgrad:umma_hconv"
for f in $OUT/*.ncu-rep; do ncu -i $f --page source --csv --print-source sass > ${f%.ncu-rep}_src.csv 2>/dev/null; done
