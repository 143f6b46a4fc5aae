#!/bin/bash
# fused small-C backward plan sweep (band rows j, derived-ring depth): VGG-A conv1 combined backward
O=gpurun_out/scbwd_sweep; mkdir -p $O; : > $O/t.txt
for rep in 1 2; do for j in 3 4 5; do for sd in 0 2; do
  echo "j=$j sd=$sd $(PT_B200_SCBWD_J=$j PT_B200_SCBWD_SD=$sd timeout 120 python tests/scbwd_tl.py 2>&1 | grep 'rep 2')" >> $O/t.txt
done; done; done
cat $O/t.txt
