#!/bin/bash
# launch lists for the given workloads
for wl in "$@"; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ll_$wl.csv python bench.py --workload $wl --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
