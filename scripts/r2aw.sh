#!/bin/bash
O=gpurun_out/r2aw; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_engines.py tests/test_gpu_fullsize.py tests/test_gpu_workloads.py tests/test_gpu_conv.py tests/test_gpu_graphs.py -m gpu -q -x > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
tail -3 $O/tests.txt
for i in 1 2 3; do timeout 300 python bench.py --workload vgga --no-cpu-baseline --no-e2e > $O/vgga_$i.json 2>>$O/err.txt; done
python - <<PY
import json
for i in (1,2,3):
    d=json.loads(open("$O/vgga_%d.json"%i).read().strip().splitlines()[-1])
    print(d['ms_per_step'], d['roofline']['per_launch']['umma_wgrad@c1.bwd'])
PY
