#!/bin/bash
# wrap-around position rows: parity (engine tests, full-size, workloads) + A/B timing
O=gpurun_out/r2y; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_engines.py tests/test_gpu_fullsize.py tests/test_gpu_workloads.py tests/test_gpu_conv.py tests/test_gpu_dp.py -q -rf -x > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for w in 1 0; do
  PT_B200_HCONV_WRAP=$w timeout 300 python bench.py --no-cpu-baseline --no-e2e > $O/bench_convnet_w$w.json 2>> $O/bench.err
  PT_B200_HCONV_WRAP=$w timeout 300 python bench.py --workload alexnet --no-cpu-baseline --no-e2e > $O/bench_alexnet_w$w.json 2>> $O/bench.err
done
