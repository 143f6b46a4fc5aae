#!/bin/bash
O=gpurun_out/r2be; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_workloads.py tests/test_gpu_ops.py -m gpu -q -x > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
tail -2 $O/tests.txt
for i in 1 2; do for wl in alexnet convnet overfeat; do timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-e2e > $O/${wl}_$i.json 2>>$O/err.txt; done; done
python - <<PY
import json
for wl in ("alexnet","convnet","overfeat"):
    print(wl, [round(json.loads(open("$O/%s_%d.json"%(wl,i)).read().strip().splitlines()[-1])['ms_per_step'],4) for i in (1,2)])
d=json.loads(open("$O/alexnet_1.json").read().strip().splitlines()[-1])
print({k:(round(v['ms']*1000,1),int(v['gbs'])) for k,v in d['layout_per_pass'].items()})
PY
