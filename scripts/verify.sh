O=gpurun_out/verify; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf -x > $O/gpu_tests.txt 2>&1; echo "rc=$?" >> $O/gpu_tests.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
for wl in convnet alexnet vgga overfeat; do timeout 300 python bench.py --workload $wl --no-cpu-baseline > $O/bench_$wl.json 2>> $O/bench.err; done
