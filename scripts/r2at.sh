#!/bin/bash
O=gpurun_out/r2at; mkdir -p $O
for d in 15 143 128; do echo "dbg=$d $(PT_B200_GFOLD_DBG=$d timeout 60 python tests/gfold_probe.py 128 3 128 128 96 11 11 0 0 3 2>&1 | grep -E 'rep 2' | tr '\n' ' ')"; done > $O/t.txt
PT_B200_GFOLD_DBG=159 timeout 60 python tests/gfold_probe.py 128 3 128 128 96 11 11 0 0 2 > $O/tl15.txt 2>&1
cat $O/t.txt
