OUT=gpurun_out/hot1; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:umma_hconv -s 1 -c 1 -o $OUT/a python tests/prof_one.py --workload alexnet --layer c1 --pass fwd --iters 2 > $OUT/a.log 2>&1
ncu -i $OUT/a.ncu-rep --page source --csv --print-source sass > $OUT/a_src.csv 2>/dev/null
rm -f $OUT/a.ncu-rep
