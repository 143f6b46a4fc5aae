#!/bin/bash
for m in 0 2 3; do
  for pass in fwd dgrad; do
    PT_B200_HCONV=1 PT_B200_HCONV_EXP=$m timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:umma_hconv --csv python tests/prof_one.py --layer L2 --pass $pass --iters 3 2>&1 | grep -E "gpu__time" | tail -1 | awk -F, '{print $NF}' | sed "s/^/mode $m $pass: /"
  done
done
