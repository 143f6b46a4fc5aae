#!/bin/bash
O=gpurun_out/hconv_force; mkdir -p $O; : > $O/runs.txt
for rep in 1 2; do for v in rule force; do for wl in vgga alexnet overfeat convnet; do
  if [ $v = force ]; then E="PT_B200_HCONV=1"; else E="X=1"; fi
  env $E timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-e2e > $O/${wl}_${v}_$rep.json 2>>$O/err.txt
  echo ${wl}_${v}_$rep >> $O/runs.txt
done; done; done
python - <<PY
import json
for tag in open("$O/runs.txt").read().split():
    d=json.loads(open("$O/%s.json"%tag).read().strip().splitlines()[-1])
    pl=d['roofline']['per_launch']
    print(f"{tag:20s} step {d['ms_per_step']:.3f}", {k.split('@')[1]:round(v['ms']*1000,1) for k,v in pl.items() if k.startswith('umma_conv')})
PY
