#!/bin/bash
O=gpurun_out/r2aj; mkdir -p $O
for m in dgrad wgrad both; do CUDA_LAUNCH_BLOCKING=1 timeout 60 python tests/scbwd_debug.py $m > $O/$m.txt 2>&1; echo "rc=$?" >> $O/$m.txt; done
CUDA_LAUNCH_BLOCKING=1 timeout 60 python tests/scbwd_debug.py both big > $O/bothbig.txt 2>&1; echo "rc=$?" >> $O/bothbig.txt
timeout 900 python -m pytest tests/test_gpu_engines.py tests/test_gpu_fullsize.py tests/test_gpu_workloads.py tests/test_gpu_conv.py tests/test_gpu_dp.py -q -rf -x -k "default or scbwd or vgga or cfg1 or spec" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
timeout 300 python tests/scbwd_probe.py > $O/probe.jsonl 2>&1
bash scripts/ab.sh PT_B200_SCBWD "vgga" 2 > $O/ab.txt 2>&1
