#!/bin/bash
O=gpurun_out/flat_check; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_engines.py tests/test_gpu_conv.py tests/test_gpu_fullsize.py tests/test_gpu_workloads.py tests/test_gpu_graphs.py -m gpu -q -x > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
tail -2 $O/tests.txt
for rep in 1 2; do for v in 0 2; do for wl in convnet alexnet vgga overfeat; do
  PT_B200_HCONV_FLAT=$v timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-e2e > $O/${wl}_${v}_$rep.json 2>>$O/err.txt
done; done; done
python - <<PY
import json,collections
r=collections.defaultdict(list)
for wl in ("convnet","alexnet","vgga","overfeat"):
    for v in (0,2):
        for rep in (1,2):
            d=json.loads(open("$O/%s_%d_%d.json"%(wl,v,rep)).read().strip().splitlines()[-1])
            r[(wl,v)].append(round(d['ms_per_step'],4))
for k in sorted(r): print(k, r[k])
PY
