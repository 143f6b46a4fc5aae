#!/bin/bash
for ex in 0 1 5; do
  PT_B200_ROWCONV_EXP=$ex timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:umma_rowconv --csv python tests/prof_one.py --layer L1 --pass fwd --iters 3 2>&1 | grep -E "gpu__time" | tail -1 | awk -F, '{print $NF}' | sed "s/^/exp $ex: /"
done
