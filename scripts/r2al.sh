#!/bin/bash
O=gpurun_out/r2al; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_engines.py tests/test_gpu_fullsize.py tests/test_gpu_workloads.py tests/test_gpu_conv.py -q -rf -x -k "default or no-s2d or alexnet or overfeat or stride or s2d or c1" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"d2s|s2d" -c 10 --csv --log-file $O/l.csv python bench.py --workload alexnet --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for wl in alexnet overfeat; do timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-e2e > $O/bench_$wl.json 2>>$O/err.txt; done
