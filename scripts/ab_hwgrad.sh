#!/bin/bash
# hwgrad schedule A/B: parity of the wgrad engines, then interleaved convnet bench lines
O=gpurun_out/ab_hw; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_engines.py tests/test_gpu_workloads.py tests/test_gpu_fullsize.py -q -x -m gpu > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for i in 1 2; do
for cfg in "PT_B200_HWGRAD_VBETA=0 PT_B200_HWGRAD_TBUF=1" "PT_B200_HWGRAD_VBETA=0 PT_B200_HWGRAD_TBUF=2" "PT_B200_HWGRAD_VBETA=1" "PT_B200_HWGRAD_VBETA=1.2" "PT_B200_HWGRAD_VBETA=1 PT_B200_HWGRAD_OVH=24"; do
  tag=$(echo $cfg | tr ' =' '_-')
  env $cfg timeout 300 python bench.py --workload convnet --no-cpu-baseline --no-e2e > $O/b_${tag}_$i.json 2>> $O/err.txt
  python -c "
import json
d=json.load(open('$O/b_${tag}_$i.json'))
pl=d['roofline']['per_launch']
print('[$cfg] $i', round(d['ms_per_step'],4), 'L2w', round(pl['umma_wgrad@L2.wgrad']['ms'],4), 'L3w', round(pl['umma_wgrad@L3.wgrad']['ms'],4), 'reduce', d['kernels'].get('layout'))
" >> $O/summary.txt 2>&1
done; done
