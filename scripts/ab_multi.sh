#!/bin/bash
# interleaved runs of several env settings (separated by ';') over workloads, all per-launch times
# usage: ab_multi.sh "ENV_A;ENV_B;..." "wl1 wl2" reps
IFS=';' read -ra CFGS <<< "$1"; WLS=$2; REPS=${3:-2}
O=gpurun_out/ab_multi; mkdir -p $O
for i in $(seq 1 $REPS); do for wl in $WLS; do for j in "${!CFGS[@]}"; do
  cfg="${CFGS[$j]}"
  env $cfg timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-e2e > $O/${wl}_${j}_$i.json 2>> $O/err.txt
  python -c "
import json
d=json.load(open('$O/${wl}_${j}_$i.json'))
pl=d['roofline']['per_launch']
print('$j [$cfg] $wl $i', round(d['ms_per_step'],4), ' '.join(f\"{k.split('@')[1]}:{v['ms']*1000:.0f}\" for k,v in pl.items()))
" >> $O/summary.txt 2>&1
done; done; done
