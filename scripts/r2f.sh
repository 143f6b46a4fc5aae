#!/bin/bash
# round-2 baseline evidence: GPU tests, smoke, bench lines (convnet/alexnet/vgga/overfeat), launch list
O=gpurun_out/r2f; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -rf > $O/gpu_tests.txt 2>&1; echo "pytest rc=$?" >> $O/gpu_tests.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 600 python bench.py > $O/bench_convnet.json 2> $O/bench_convnet.err
for wl in alexnet vgga overfeat; do timeout 300 python bench.py --workload $wl --no-cpu-baseline > $O/bench_$wl.json 2>> $O/bench.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
   python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
