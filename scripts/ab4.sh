O=gpurun_out/ab4; mkdir -p $O
PT_B200_SWGRAD_MINST=2 timeout 600 python -m pytest tests/test_gpu_workloads.py -q -x -m gpu -k "L1" > $O/tests_minst2.txt 2>&1; echo rc=$? >> $O/tests_minst2.txt
bash scripts/ab_env.sh "PT_B200_SWGRAD_MINST=3" "PT_B200_SWGRAD_MINST=2" "convnet" 3
mv gpurun_out/ab_env gpurun_out/ab4/minst
bash scripts/ab_env.sh "PT_B200_WGRAD_OVH=2" "PT_B200_WGRAD_OVH=6" "alexnet vgga" 2
mv gpurun_out/ab_env gpurun_out/ab4/ovh
