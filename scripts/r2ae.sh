#!/bin/bash
O=gpurun_out/r2ae; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_workloads.py tests/test_gpu_fullsize.py tests/test_gpu_conv.py -q -rf -x > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for r in 1 0; do for wl in alexnet vgga overfeat convnet; do
  PT_B200_CONV_REBALANCE=$r timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-e2e > $O/bench_${wl}_r$r.json 2>> $O/bench.err
done; done
