"""Timing probe (GPU box, not collected by pytest): the Winograd entry vs the default
implicit-GEMM engines on every 3x3 stride-1 bench layer, forward and gradInput, CUDA
events over 20 repetitions after warm-up. Prints one JSON object per layer.

  python tests/wino_probe.py > profiles/r2/winograd_vs_implicit.jsonl
"""
import json
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__)))]
import torch  # noqa: E402

import paper_1606_04884_b200 as pt  # noqa: E402
from bench import WORKLOADS  # noqa: E402


def t_ms(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for wl in ("convnet", "alexnet", "overfeat", "vgga"):
    for l in WORKLOADS[wl]:
        name, N, C, H, W, K, kH, kW, pH, pW, sH, sW = l
        if (kH, kW, sH, sW) != (3, 3, 1, 1):
            continue
        g = pt.ConvGeometry(N, C, H, W, K, kH, kW, pH, pW, sH, sW)
        x = pt.fill_uniform(torch.empty(g.input_shape(), device="cuda"), 1)
        w = pt.fill_uniform(torch.empty(g.weight_shape(), device="cuda"), 2, -0.05, 0.05)
        b = pt.fill_uniform(torch.empty((K,), device="cuda"), 3)
        gy = pt.fill_uniform(torch.empty(g.output_shape(), device="cuda"), 4)
        y, gx = torch.empty(g.output_shape(), device="cuda"), torch.empty(g.input_shape(), device="cuda")
        flops = g.flops()
        r = {"layer": f"{wl}/{name}", "geometry": str(g)}
        r["implicit_fwd_ms"] = t_ms(lambda: pt.conv_forward(g, x, w, b, y))
        r["winograd_fwd_ms"] = t_ms(lambda: pt.conv_winograd_2x2_3x3(g, x, w, b, y))
        r["implicit_dgrad_ms"] = t_ms(lambda: pt.conv_backward_input(g, gy, w, gx))
        if pt.winograd_supported(g, 1):
            r["winograd_dgrad_ms"] = t_ms(lambda: pt.conv_backward_input_winograd(g, gy, w, gx))
        for k in list(r):
            if k.endswith("_ms"):
                r[k.replace("_ms", "_tflops")] = flops / (r[k] * 1e-3) / 1e12
        print(json.dumps(r), flush=True)
