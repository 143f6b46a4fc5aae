#!/bin/bash
# Sanitizer pass over the rescheduled weight gradients + a randomised parity sweep with new seeds.
G='[[2,3,20,20,32,3,3,1,1,1,1],[1,32,14,14,64,9,9,0,0,1,1],[2,32,20,20,64,9,9,0,0,1,1],[2,64,12,12,64,3,3,1,1,1,1],[3,128,13,13,192,3,3,1,1,1,1],[2,64,27,27,96,5,5,2,2,1,1]]'
O=gpurun_out/final; mkdir -p $O; : > $O/sanitize_summary.txt
run() {  # tool cfg env...
  local tool=$1 cfg=$2; shift 2
  env "$@" timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python tests/engine_check.py "$G" > $O/sanitize_${tool}_${cfg}.txt 2>&1
  echo "$tool $cfg rc=$?" >> $O/sanitize_summary.txt
}
run memcheck default
run synccheck default
run memcheck hwgrad PT_B200_HWGRAD=2
run synccheck hwgrad PT_B200_HWGRAD=2
timeout 1200 python tests/stress_tc.py 200 21 > $O/stress_default.txt 2>&1; echo "rc=$?" >> $O/stress_default.txt
timeout 900 python tests/stress_tc.py 120 22 wide > $O/stress_wide.txt 2>&1; echo "rc=$?" >> $O/stress_wide.txt
