#!/bin/bash
O=gpurun_out/r2v; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_dp.py tests/test_gpu_fullsize.py tests/test_gpu_workloads.py tests/test_gpu_engines.py -q -rf -k "vgga or default or scbwd" > $O/gpu_tests.txt 2>&1; echo "rc=$?" >> $O/gpu_tests.txt
timeout 300 python bench.py --workload vgga --no-cpu-baseline --no-e2e > $O/bench_vgga.json 2> $O/bench.err
