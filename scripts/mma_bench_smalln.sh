B=tests/mma_bench
for mode in 4 7 9; do for n in 16 32 48 64; do timeout 20 $B $n 1 1000000 $mode 20000; done; done
