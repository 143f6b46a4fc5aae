#!/bin/bash
O=gpurun_out/r2af; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_engines.py tests/test_gpu_workloads.py tests/test_gpu_fullsize.py tests/test_gpu_conv.py -q -rf -x -k "hwgrad or default or workloads or fullsize or wgrad" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
bash scripts/ab.sh PT_B200_HWGRAD_VERT "convnet alexnet" 2 > $O/ab.txt 2>&1
for v in 1 0; do PT_B200_HWGRAD_VERT=$v timeout 300 python bench.py --no-cpu-baseline --no-e2e > $O/bench_v$v.json 2>>$O/err.txt; done
