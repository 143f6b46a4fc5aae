#!/bin/bash
O=gpurun_out/flat_ab; mkdir -p $O; : > $O/runs.txt
run() { local tag=$1; shift; env "$@" timeout 300 python bench.py --workload $WL --no-cpu-baseline --no-e2e > $O/${WL}_$tag.json 2>>$O/err.txt; echo "${WL}_$tag" >> $O/runs.txt; }
for rep in 1 2; do for WL in alexnet overfeat vgga convnet; do
  run rule_$rep
  run halves_$rep PT_B200_HCONV_FLAT=2
  run flat_$rep PT_B200_HCONV_FLAT=1
done; done
python - <<PY
import json
for tag in open("$O/runs.txt").read().split():
    d=json.loads(open("$O/%s.json"%tag).read().strip().splitlines()[-1])
    pl=d['roofline']['per_launch']
    print(f"{tag:18s} step {d['ms_per_step']:.3f}", {k.split('@')[1]:round(v['ms']*1000,1) for k,v in pl.items() if k.startswith('umma_conv')})
PY
