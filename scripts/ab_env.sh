#!/bin/bash
# interleaved A/B of two env settings over workloads: ab_env.sh "ENV_A" "ENV_B" "wl1 wl2" reps
A=$1; B=$2; WLS=$3; REPS=${4:-2}
O=gpurun_out/ab_env; mkdir -p $O
for i in $(seq 1 $REPS); do for wl in $WLS; do for side in A B; do
  if [ $side = A ]; then cfg="$A"; else cfg="$B"; fi
  env $cfg timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-e2e > $O/${wl}_${side}_$i.json 2>> $O/err.txt
  python -c "
import json
d=json.load(open('$O/${wl}_${side}_$i.json'))
pl=d['roofline']['per_launch']
print('$side [$cfg] $wl $i', round(d['ms_per_step'],4), ' '.join(f\"{k.split('@')[1]}:{v['ms']:.3f}\" for k,v in pl.items() if 'wgrad' in k))
" >> $O/summary.txt 2>&1
done; done; done
