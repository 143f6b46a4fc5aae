#!/bin/bash
O=gpurun_out/r2ar; mkdir -p $O
timeout 120 compute-sanitizer --tool memcheck python tests/gfold_probe.py 3 3 40 40 96 11 11 0 0 1 > $O/san1.txt 2>&1; echo "rc=$?" >> $O/san1.txt
timeout 120 python tests/gfold_probe.py 2 3 40 40 96 11 11 0 0 2 > $O/p2.txt 2>&1; echo "rc=$?" >> $O/p2.txt
timeout 120 python tests/gfold_probe.py 3 3 40 40 96 11 11 0 0 2 > $O/p3.txt 2>&1; echo "rc=$?" >> $O/p3.txt
timeout 120 python tests/gfold_probe.py 128 3 128 128 96 11 11 0 0 3 > $O/pl1.txt 2>&1; echo "rc=$?" >> $O/pl1.txt
timeout 300 ncu --set full --import-source on --clock-control none -k regex:umma_gfold -c 1 -o $O/gfold_l1 python tests/gfold_probe.py 128 3 128 128 96 11 11 0 0 1 > $O/ncu.txt 2>&1
tail -3 $O/*.txt
