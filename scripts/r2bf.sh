#!/bin/bash
O=gpurun_out/r2bf; mkdir -p $O
timeout 1500 bash scripts/ab.sh PT_B200_STRIP64 "convnet alexnet overfeat" 3 > $O/ab.txt 2>&1
cat $O/ab.txt
