#!/bin/bash
B=tests/mma_bench
for n in 96 128; do for sh in 4 5 6; do timeout 20 $B $n 2 1000000 $sh 19998; done; done
