"""Timing probe (GPU box, not collected by pytest): the small-C stride-1 bench layers'
backward — combined (conv_backward), gradInput only, gradWeight only — with the fused
one-read kernel (default) and with the separate engines (PT_B200_SCBWD=0, subprocess).
CUDA events over 20 reps after warm-up."""
import json
import os
import subprocess
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__)))]


def t_ms(torch, fn, reps=20):
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


if len(sys.argv) > 1 and sys.argv[1] == "run":
    import torch
    import paper_1606_04884_b200 as pt
    from bench import WORKLOADS
    out = {}
    for wl, name in (("vgga", "c1"), ("cfg1", "cfg1"), ("convnet", "L1")):
        l = [x for x in WORKLOADS[wl] if x[0] == name][0]
        G = pt.ConvGeometry(*l[1:])
        t = lambda s: pt.fill_uniform(torch.empty(s, device="cuda"), 3)  # noqa: E731
        x, w, gy = t(G.input_shape()), t(G.weight_shape()), t(G.output_shape())
        gx, gw, gb = torch.empty(G.input_shape(), device="cuda"), torch.empty(G.weight_shape(), device="cuda"), \
            torch.empty((G.outChannels,), device="cuda")
        r = {"bwd_ms": t_ms(torch, lambda: pt.conv_backward(G, x, gy, w, gx, gw, gb)),
             "dgrad_ms": t_ms(torch, lambda: pt.conv_backward_input(G, gy, w, gx)),
             "wgrad_ms": t_ms(torch, lambda: pt.conv_backward_weight(G, x, gy, gw, gb))}
        r["gy_GBs_bwd"] = gy.numel() * 4 / r["bwd_ms"] / 1e6
        out[f"{wl}/{name}"] = r
    print(json.dumps(out))
else:
    for env in ({}, {"PT_B200_SCBWD": "0"}):
        r = subprocess.run([sys.executable, __file__, "run"], env={**os.environ, **env}, capture_output=True,
                           text=True)
        print(json.dumps({"env": env, "result": r.stdout.strip() or r.stderr[-2000:]}))
