#!/bin/bash
O=gpurun_out/eff_check; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_engines.py tests/test_gpu_conv.py tests/test_gpu_fullsize.py tests/test_gpu_workloads.py -m gpu -q -x > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
grep -E "passed|failed" $O/tests.txt | tail -1
for rep in 1 2; do for wl in overfeat vgga alexnet convnet; do
  timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-e2e > $O/${wl}_$rep.json 2>>$O/err.txt
done; done
python - <<PY
import json
for wl in ("overfeat","vgga","alexnet","convnet"):
    for rep in (1,2):
        d=json.loads(open("$O/%s_%d.json"%(wl,rep)).read().strip().splitlines()[-1])
        pl=d['roofline']['per_launch']
        print(wl, rep, round(d['ms_per_step'],4), {k.split('@')[1]:round(v['ms']*1000,1) for k,v in pl.items() if 'dgrad' in k and k.startswith('umma_conv')})
PY
