#!/bin/bash
O=gpurun_out/r2bb; mkdir -p $O
timeout 1500 bash scripts/ab.sh PT_B200_FWD_FORK "convnet alexnet vgga overfeat" 2 > $O/ab.txt 2>&1
cat $O/ab.txt
