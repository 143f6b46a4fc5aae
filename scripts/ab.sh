#!/bin/bash
# interleaved A/B of an env switch: ab.sh VAR "wl1 wl2" reps
V=$1; WLS=$2; REPS=${3:-2}
O=gpurun_out/ab_$V; mkdir -p $O
for i in $(seq 1 $REPS); do for val in 1 0; do for wl in $WLS; do
  env $V=$val timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-e2e > $O/${wl}_${val}_$i.json 2>> $O/err.txt
done; done; done
python - <<PY
import json,glob,collections
r=collections.defaultdict(list)
for f in sorted(glob.glob("$O/*_*_*.json")):
    wl,val,i=f.split('/')[-1][:-5].rsplit('_',2)
    try: r[(wl,val)].append(round(json.load(open(f))['ms_per_step'],4))
    except Exception as e: r[(wl,val)].append(str(e)[:30])
for k in sorted(r): print(k, r[k])
PY
