#!/bin/bash
# 3xTF32 parity + bench legs; Winograd vs implicit GEMM timing probe
O=gpurun_out/r2h; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_3xtf32.py -q -rf -x > $O/tests_3x.txt 2>&1; echo "rc=$?" >> $O/tests_3x.txt
timeout 300 python bench.py --math 3xtf32 --no-cpu-baseline --no-e2e > $O/bench_convnet_3x.json 2> $O/bench_3x.err
timeout 300 python bench.py --workload alexnet --math 3xtf32 --no-cpu-baseline --no-e2e > $O/bench_alexnet_3x.json 2>> $O/bench_3x.err
timeout 300 python tests/wino_probe.py > $O/winograd_vs_implicit.jsonl 2> $O/wino.err
