#!/bin/bash
# source-level (SASS) warp-stall profile of one kernel launch: hot_src.sh NAME KREGEX WORKLOAD LAYER PASS
N=$1; K=$2; WL=$3; L=$4; P=$5
OUT=gpurun_out/hot; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o $OUT/$N python tests/prof_one.py --workload $WL --layer $L --pass $P --iters 2 > $OUT/$N.log 2>&1
ncu -i $OUT/$N.ncu-rep --page source --csv --print-source sass > $OUT/${N}_src.csv 2>/dev/null
ncu -i $OUT/$N.ncu-rep --page raw --csv > $OUT/${N}_raw.csv 2>/dev/null
rm -f $OUT/$N.ncu-rep
