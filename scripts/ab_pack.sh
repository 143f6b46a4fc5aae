#!/bin/bash
# staged weight pack: GPU suite, then interleaved A/B at batch 128 and at 8 emulated ranks
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_pack.txt 2>&1; echo rc=$? >> gpurun_out/gpu_tests_pack.txt
bash scripts/ab_multi.sh "PT_B200_PACK_STAGED=0;PT_B200_PACK_STAGED=1" "alexnet convnet vgga" 2
O=gpurun_out/ab_multi
for i in 1 2; do for v in 0 1; do
  PT_B200_PACK_STAGED=$v timeout 300 python bench.py --workload alexnet --emulate-ranks 8 --no-cpu-baseline --no-e2e --no-alexnet 2>>$O/err.txt | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('emu8 alexnet PACK_STAGED=$v $i', round(d['ms_per_step'],4), {k:round(v['ms']/d['steps'],4) for k,v in d['kernels'].items()})" >> $O/summary.txt
done; done
