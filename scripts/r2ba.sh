#!/bin/bash
O=gpurun_out/r2ba; mkdir -p $O
timeout 1500 bash scripts/ab.sh BENCH_BWD_STREAMS "convnet alexnet vgga overfeat" 2 > $O/ab.txt 2>&1
cat $O/ab.txt
