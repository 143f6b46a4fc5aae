#!/bin/bash
B=tests/mma_bench
for n in 64 96 128 160 192 224 256; do timeout 20 $B $n 2 1000000 4 20000; done
