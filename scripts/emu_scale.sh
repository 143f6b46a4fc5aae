#!/bin/bash
# Per-GPU compute of the strong-scaling curve on one B200: rank 0's shard of a G-rank job
# (bench.py --emulate-ranks G; no collective). Writes one JSON line per (workload, G).
O=gpurun_out/emu; mkdir -p $O; : > $O/emulated_scaling.jsonl
for wl in alexnet vgga convnet overfeat; do for G in 1 2 4 8; do
  timeout 300 python bench.py --workload $wl --emulate-ranks $G --no-cpu-baseline --no-e2e --no-alexnet \
     2>>$O/err.txt | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(json.dumps({'workload':'$wl','ranks':$G,'per_rank_batch':d.get('emulated_ranks',{}).get('per_rank_batch',d['config'].get('per_gpu_batch')),
 'ms_per_step':d['ms_per_step'],'value':d['value'],'unit':d['unit'],'clocks':d['clocks']}))" >> $O/emulated_scaling.jsonl
done; done
cat $O/emulated_scaling.jsonl
