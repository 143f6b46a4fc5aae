#!/bin/bash
# Round-2 final evidence: GPU tests + smoke, bench lines (convnet with cpu_baseline + e2e, other
# workloads), the reference arm, launch list, ncu --set full of the top launches (incl. the
# weight gradients rescheduled this session), the emulated strong-scaling curve.
TAG=${1:-r2h}
O=gpurun_out/ev_$TAG; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/gpu_tests.txt 2>&1; echo "rc=$?" >> $O/gpu_tests.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench_convnet.json 2> $O/bench_convnet.err
for wl in alexnet vgga overfeat; do timeout 300 python bench.py --workload $wl --no-cpu-baseline > $O/bench_$wl.json 2>> $O/bench.err; done
timeout 600 python bench.py --impl reference > $O/bench_reference_convnet.json 2>> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
   python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
KEEP="convnet_L2_dgrad convnet_L2_wgrad" bash scripts/ncu_top.sh ev_$TAG "L2:dgrad:umma_hconv" "L2:wgrad:umma_hwgrad" "L2:fwd:umma_hconv" \
   "L3:wgrad:umma_hwgrad" "c2:wgrad:umma_wgrad:alexnet" "c4:wgrad:umma_wgrad:vgga" "L1:fwd:umma_rowconv" > $O/ncu_top.log 2>&1
bash scripts/emu_scale.sh > /dev/null 2>&1; cp gpurun_out/emu/emulated_scaling.jsonl $O/ 2>/dev/null
