#!/bin/bash
O=gpurun_out/r2ax; mkdir -p $O
timeout 900 bash scripts/ab.sh BENCH_ONE_GRAPH "convnet alexnet" 3 > $O/ab.txt 2>&1
cat $O/ab.txt
