#!/bin/bash
O=gpurun_out/r2bi; mkdir -p $O
for n in 2 4 8; do timeout 600 python bench.py --workload convnet --no-cpu-baseline --e2e-steps $n > $O/e2e_$n.json 2>>$O/err.txt; done
python - <<PY
import json
for n in (2,4,8):
    d=json.loads(open("$O/e2e_%d.json"%n).read().strip().splitlines()[-1])
    e=d['e2e']; print(n, round(e['value'],1), 'ms/step', round(2741.9/e['value']*1000,2))
PY
