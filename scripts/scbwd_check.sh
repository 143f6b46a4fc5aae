#!/bin/bash
O=gpurun_out/scbwd_check; mkdir -p $O
SPECS='[[2,3,20,20,32,3,3,1,1,1,1],[1,1,20,40,48,5,5,2,2,1,1],[3,2,18,36,32,3,5,1,2,1,1],[2,3,224,224,64,3,3,1,1,1,1],[2,3,38,44,64,3,3,1,1,1,1]]'
timeout 300 python tests/engine_check.py "$SPECS" > $O/check.txt 2>&1; echo "rc=$?" >> $O/check.txt
for i in 1 2 3; do timeout 120 python tests/scbwd_tl.py 2>&1 | grep 'rep 2'; done > $O/t.txt
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -k vgga > $O/full.txt 2>&1; echo "rc=$?" >> $O/full.txt
cat $O/t.txt; tail -2 $O/full.txt
