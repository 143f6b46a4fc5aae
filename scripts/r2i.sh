#!/bin/bash
O=gpurun_out/r2i; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_3xtf32.py tests/test_gpu_plan_cache.py -q -rf > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for wl in convnet alexnet; do
  timeout 120 python tests/host_probe.py $wl >> $O/host_probe.jsonl 2>>$O/host.err
  PT_B200_NO_TMAP_CACHE=1 timeout 120 python tests/host_probe.py $wl >> $O/host_probe.jsonl 2>>$O/host.err
done
