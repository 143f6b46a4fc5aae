#!/bin/bash
for ex in 0 4; do
  for L in "L2 fwd" "L3 dgrad"; do
    set -- $L
    PT_B200_HCONV=1 PT_B200_HCONV_EXP=$ex timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:umma_hconv --csv python tests/prof_one.py --layer $1 --pass $2 --iters 3 2>&1 | grep -E "gpu__time" | tail -1 | awk -F, '{print $NF}' | sed "s/^/exp $ex $1 $2: /"
  done
done
