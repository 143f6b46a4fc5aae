#!/bin/bash
python -m pytest tests/test_gpu_winograd.py tests/test_gpu_model.py -q -rf > gpurun_out/r2e_wino_model.txt 2>&1
python tests/wino_probe.py > gpurun_out/r2e_wino_probe.jsonl 2> gpurun_out/r2e_wino_probe.err
python -m paper_1606_04884_b200.bench_cli apply --reps 20 --out gpurun_out/r2e_bw.csv
python -m paper_1606_04884_b200.bench_cli model --name vgg-a --batch 64 --backward --out gpurun_out/r2e_vgga_layers.csv --summary gpurun_out/r2e_vgga_summary.csv
python -m paper_1606_04884_b200.bench_cli model --name alexnet --batch 128 --backward --out gpurun_out/r2e_alex_layers.csv --summary gpurun_out/r2e_alex_summary.csv
python -m pytest tests -m gpu -q -rf -x --deselect tests/test_gpu_winograd.py --deselect tests/test_gpu_model.py > gpurun_out/r2e_all.txt 2>&1
