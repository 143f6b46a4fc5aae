#!/bin/bash
B=tests/mma_bench
for cg in 2 1; do for n in 64 128 256; do for sh in 0 3 4; do timeout 20 $B $n $cg 1000000 $sh; done; done; done
