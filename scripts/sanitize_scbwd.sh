#!/bin/bash
# focused sanitizer pass incl. the fused small-C backward (scbwd) geometries
mkdir -p gpurun_out/san_r2d
G='[[2,3,20,20,32,3,3,1,1,1,1],[1,1,20,40,48,5,5,2,2,1,1],[3,2,18,36,32,3,5,1,2,1,1]]'
for tool in memcheck synccheck racecheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tests/engine_check.py "$G" > gpurun_out/san_r2d/$tool.txt 2>&1
  echo "$tool scbwd rc=$? $(grep -c 'Error' gpurun_out/san_r2d/$tool.txt) $(grep 'ERROR SUMMARY' gpurun_out/san_r2d/$tool.txt | tail -1)"
done | tee gpurun_out/san_r2d/summary.txt
