#!/bin/bash
# quick A/B: probe parity, then convnet bench lines for the given env settings
OUT=gpurun_out/${TAG:-q}; mkdir -p $OUT
[ -n "$NOPROBE" ] || timeout 300 python tests/gpu_probe.py > $OUT/probe.log 2>&1; echo "probe rc=$?" >> $OUT/probe.log
grep -E "ERROR|rc=|': [0-9.]+e-0[12]|': [0-9]\.[0-9]" $OUT/probe.log | head
for envs in "$@"; do
  for wl in ${WLS:-convnet}; do
    env $envs timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-e2e $BARGS > $OUT/b.json 2>$OUT/b.err
    python -c "
import json
d=json.load(open('$OUT/b.json'))
print('[$envs] $wl', round(d['value']), 'GFLOP/s', round(d['ms_per_step'],3), 'ms')
print('   ', ' '.join(f\"{k.split('@')[1]}:{v['ms']:.3f}/{v['tflops']:.0f}\" for k,v in d['roofline']['per_launch'].items()))
print('    layout', ' '.join(f\"{k}:{v['ms']:.3f}/{v['launches']}/{(v['gbs'] or 0):.0f}\" for k,v in d.get('layout_per_pass',{}).items()))
print('    kernels', {k:(round(v['ms']/d['steps'],3)) for k,v in d['kernels'].items()})
" || tail -5 $OUT/b.err
  done
done
