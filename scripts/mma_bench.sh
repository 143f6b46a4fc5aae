#!/bin/bash
# tcgen05 kind::tf32 cycles per MMA: CTA pairs (M=256) and single CTAs (M=128) over N
B=tests/mma_bench
for cg in 2 1; do
  for n in ${NS:-16 32 48 64 96 128 160 192 224 256}; do timeout 20 $B $n $cg 1000000 4 20000; done
done
