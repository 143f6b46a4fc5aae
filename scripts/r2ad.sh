#!/bin/bash
O=gpurun_out/r2ad; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_workloads.py tests/test_gpu_conv.py -q -rf -x > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for wl in alexnet convnet; do timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-e2e > $O/bench_$wl.json 2>> $O/bench.err; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"wgrad" -c 12 --csv --log-file $O/l.csv python bench.py --workload alexnet --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
