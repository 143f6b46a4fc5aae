#!/bin/bash
O=gpurun_out/r2bg; mkdir -p $O
SPECS='[[2,3,40,40,96,11,11,0,0,1,1],[2,3,128,128,96,11,11,0,0,1,1],[2,1,30,33,16,5,5,2,2,1,1],[1,4,21,72,128,7,7,3,3,1,1],[2,2,17,20,40,3,5,0,2,1,1],[1,4,30,40,32,11,11,1,1,1,1],[2,3,37,44,64,3,3,1,1,1,1]]'
PT_B200_SCBWD=0 timeout 300 python tests/engine_check.py "$SPECS" > $O/check.txt 2>&1; echo "rc=$?" >> $O/check.txt
tail -c 300 $O/check.txt
timeout 900 bash scripts/ab.sh PT_B200_SWGRAD_XE "convnet" 3 > $O/ab.txt 2>&1
cat $O/ab.txt
python - <<PY
import json
for v in "01":
    d=json.loads(open("gpurun_out/ab_PT_B200_SWGRAD_XE/convnet_%s_1.json"%v).read().strip().splitlines()[-1])
    print(v, d['roofline']['per_launch']['umma_wgrad@L1.wgrad'], d['layout_per_pass'].get('L1.wgrad'))
PY
