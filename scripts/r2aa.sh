#!/bin/bash
O=gpurun_out/r2ab; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_engines.py tests/test_gpu_fullsize.py tests/test_gpu_workloads.py tests/test_gpu_conv.py tests/test_gpu_dp.py -q -rf -x -k "default or no-s2d or alexnet or overfeat or stride or s2d or c1" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
timeout 300 python bench.py --workload alexnet --no-cpu-baseline --no-e2e > $O/bench_alexnet.json 2>> $O/bench.err
timeout 300 python bench.py --workload overfeat --no-cpu-baseline --no-e2e > $O/bench_overfeat.json 2>> $O/bench.err
