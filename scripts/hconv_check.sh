#!/bin/bash
OUT=gpurun_out/${1:-hc}; mkdir -p $OUT
for d in 0 1; do
  PT_B200_HCONV=1 PT_B200_HCONV_DESC=$d timeout 300 python tests/gpu_probe.py > $OUT/probe_desc$d.log 2>&1
  echo "desc $d rc=$?" >> $OUT/probe_desc$d.log
done
cat $OUT/probe_desc*.log
BEST=0
if grep -q "fwd': [0-9.e-]*[1-9]e-0[1-2]\|ERROR\|nan" $OUT/probe_desc0.log; then BEST=1; fi
echo "using desc $BEST"
export PT_B200_HCONV_DESC=$BEST
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -15 $OUT/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > $OUT/bench_convnet.json 2>$OUT/bench.err
for wl in vgga alexnet overfeat; do timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-e2e > $OUT/bench_$wl.json 2>>$OUT/bench.err; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/${1:-hc}/bench_*.json".replace("${1:-hc}", __import__('os').environ.get('T','hc')))):
    pass
PY
for f in $OUT/bench_*.json; do python -c "
import json,sys
d=json.load(open('$f'))
print('$f', round(d['value']), 'GFLOP/s', round(d['ms_per_step'],3), 'ms', d['roofline']['kernel'], round(d['roofline']['frac'],3))
for k,v in d['roofline']['per_launch'].items(): print('   ',k, round(v['ms'],3), round(v['tflops'],1))
"; done
