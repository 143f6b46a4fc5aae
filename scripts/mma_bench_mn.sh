#!/bin/bash
# MN-major vs K-major tf32 MMA issue rate (tests/mma_bench.cu shift modes 4, 7, 8, 9)
B=tests/mma_bench
for mode in 4 7 8 9; do for n in 64 128 256; do timeout 20 $B $n 2 1000000 $mode 20000; done; done
for mode in 4 7 9; do timeout 20 $B 128 1 1000000 $mode 20000; done
