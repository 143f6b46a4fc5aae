#!/bin/bash
O=gpurun_out/r2az; mkdir -p $O
timeout 1200 bash scripts/ab.sh PT_B200_PREPACK "convnet alexnet" 4 > $O/ab.txt 2>&1
cat $O/ab.txt
