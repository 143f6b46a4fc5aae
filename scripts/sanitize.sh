#!/bin/bash
# compute-sanitizer memcheck / synccheck / racecheck over one small geometry per engine
# (tests/engine_check.py: exact + real-valued runs, finput + combined backward + separate
# passes). Output: gpurun_out/sanitize_<tool>_<cfg>.txt
G='[[2,3,20,20,32,3,3,1,1,1,1],[1,1,20,40,48,5,5,2,2,1,1],[2,3,20,20,32,5,5,2,2,1,1],[1,3,35,35,64,11,11,2,2,4,4],[2,64,12,12,64,3,3,1,1,1,1],[1,32,14,14,64,9,9,0,0,1,1],[1,32,9,9,32,3,3,1,1,2,2],[2,3,18,18,16,3,3,1,1,1,1]]'
run() {  # tool cfg env...
  local tool=$1 cfg=$2; shift 2
  env "$@" timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python tests/engine_check.py "$G" > gpurun_out/sanitize_${tool}_${cfg}.txt 2>&1
  echo "$tool $cfg rc=$?" | tee -a gpurun_out/sanitize_summary.txt
}
: > gpurun_out/sanitize_summary.txt
for tool in memcheck synccheck; do
  run $tool default
  run $tool hankel PT_B200_HCONV=1
  run $tool im2col PT_B200_HCONV=0
  run $tool hwgrad PT_B200_HWGRAD=2
  run $tool nos2d PT_B200_NO_S2D=1 PT_B200_NO_ROWCONV=1
done
run racecheck default
run initcheck default
