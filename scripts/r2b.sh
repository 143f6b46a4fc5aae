#!/bin/bash
# round-2 check: DP tests, default bench line, AlexNet strong-scaling projections on one GPU
set -x
python -m pytest tests/test_gpu_dp.py -q -rf > gpurun_out/r2b_dp.txt 2>&1
python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
for g in 1 2 4 8; do
  python bench.py --workload alexnet --emulate-ranks $g --no-e2e --no-cpu-baseline --no-alexnet > gpurun_out/r2b_alex_emu$g.json 2>>gpurun_out/r2b_bench.err
done
python bench.py --workload vgga --emulate-ranks 8 --no-e2e --no-cpu-baseline --no-alexnet > gpurun_out/r2b_vgga_emu8.json 2>>gpurun_out/r2b_bench.err
python bench.py --workload vgga --no-e2e --no-cpu-baseline --no-alexnet > gpurun_out/r2b_vgga.json 2>>gpurun_out/r2b_bench.err
