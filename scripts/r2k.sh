#!/bin/bash
O=gpurun_out/r2t; mkdir -p $O
for m in dgrad wgrad both; do CUDA_LAUNCH_BLOCKING=1 timeout 60 python tests/scbwd_debug.py $m > $O/$m.txt 2>&1; echo "rc=$?" >> $O/$m.txt; done
CUDA_LAUNCH_BLOCKING=1 timeout 60 python tests/scbwd_debug.py both big > $O/bothbig.txt 2>&1; echo "rc=$?" >> $O/bothbig.txt
for e in 0 1; do PT_B200_SCBWD_EXP=$e timeout 120 python tests/scbwd_probe.py run > $O/probe_$e.json 2>&1; done
