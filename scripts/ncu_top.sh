#!/bin/bash
# ncu --set full captures of the hot kernels, one pass per capture (1 GPU). Each report is
# exported to <name>_raw.csv on the box; the .ncu-rep is kept only for names in $KEEP
# (gpurun copies back at most 64 MiB).
# usage: gpurun --timeout 1800 -- KEEP="convnet_L2_dgrad" bash scripts/ncu_top.sh TAG "layer:pass:kregex[:workload]" ...
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
for spec in "$@"; do
  IFS=: read layer pass kre wl <<< "$spec"
  wl=${wl:-convnet}
  name=${wl}_${layer}_${pass}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kre -s 1 -c 1 \
     -o $OUT/$name python tests/prof_one.py --workload $wl --layer $layer --pass $pass --iters 2 \
     > $OUT/$name.log 2>&1
  echo "$spec rc=$?"
  if [ -f $OUT/$name.ncu-rep ]; then
    ncu -i $OUT/$name.ncu-rep --page raw --csv > $OUT/${name}_raw.csv 2>/dev/null
    case " $KEEP " in *" $name "*) ;; *) rm -f $OUT/$name.ncu-rep ;; esac
  fi
done
