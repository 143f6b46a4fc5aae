#!/bin/bash
O=gpurun_out/r2bh; mkdir -p $O; : > $O/sweep.txt
for rep in 1 2; do for oh in 24 6 12 48; do for wl in convnet vgga; do
  PT_B200_HWGRAD_UNIT_OH=$oh timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-e2e > $O/${wl}_${oh}_$rep.json 2>>$O/err.txt
done; done; done
python - <<PY
import json,collections
r=collections.defaultdict(list)
for wl in ("convnet","vgga"):
  for oh in (24,6,12,48):
    for rep in (1,2):
      d=json.loads(open("$O/%s_%d_%d.json"%(wl,oh,rep)).read().strip().splitlines()[-1])
      wg={k:round(v['ms']*1000,1) for k,v in d['roofline']['per_launch'].items() if 'wgrad' in k and k.split('@')[0]=='umma_wgrad'}
      r[(wl,oh)].append((round(d['ms_per_step'],4), wg))
for k in sorted(r): print(k, r[k])
PY
