#!/bin/bash
O=gpurun_out/r2j; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_engines.py -q -rf -k "default or scbwd" > $O/engines.txt 2>&1; echo "rc=$?" >> $O/engines.txt
timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_workloads.py -q -rf -k "vgga-c1" > $O/full.txt 2>&1; echo "rc=$?" >> $O/full.txt
timeout 300 python tests/scbwd_probe.py > $O/probe.jsonl 2>&1
