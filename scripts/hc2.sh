#!/bin/bash
OUT=gpurun_out/hc2; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -5 $OUT/pytest_gpu.log
bash scripts/ncu_top.sh hc2 "L2:dgrad:umma_hconv" "L2:fwd:umma_hconv"
for f in $OUT/*.ncu-rep; do ncu -i $f --page source --csv --print-source sass > ${f%.ncu-rep}_src.csv 2>/dev/null; done
