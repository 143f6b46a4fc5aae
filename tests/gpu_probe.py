"""Quick GPU probe (run under gpurun with an outer timeout): one geometry per tcgen05
variant, printing relative errors vs the oracle as it goes so a hang is localised."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1606_04884_b200 as pt  # noqa: E402
import pyoracle as po  # noqa: E402
from helpers import conv_inputs  # noqa: E402


def rel(a, r):
    return float(np.linalg.norm(a.astype(np.float64) - r) / max(np.linalg.norm(r), 1e-30))


def run(g, math, passes=("fwd", "dgrad", "wgrad")):
    x, w, b, gy = conv_inputs(g, 5)
    G = pt.ConvGeometry(g.N, g.C, g.H, g.W, g.K, g.kH, g.kW, g.padH, g.padW, g.strideH, g.strideW)
    out = {}
    if "fwd" in passes:
        y = pt.conv_forward(G, torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(),
                            torch.from_numpy(b).cuda(), math=math)
        torch.cuda.synchronize()
        out["fwd"] = rel(y.cpu().numpy(), po.conv_direct(g, x, w, b, f64=True))
    if "dgrad" in passes:
        gx = pt.conv_backward_input(G, torch.from_numpy(gy).cuda(), torch.from_numpy(w).cuda(),
                                    math=math)
        torch.cuda.synchronize()
        out["dgrad"] = rel(gx.cpu().numpy(), po.conv_backward_input(g, gy, w))
    if "wgrad" in passes:
        gw, gb = pt.conv_backward_weight(G, torch.from_numpy(x).cuda(),
                                         torch.from_numpy(gy).cuda(), math=math)
        torch.cuda.synchronize()
        rgw, rgb = po.conv_backward_weight(g, x, gy)
        out["wgrad"] = rel(gw.cpu().numpy(), rgw)
        out["gbias"] = rel(gb.cpu().numpy(), rgb)
    return out


if __name__ == "__main__":
    cases = [
        ("fp32 small", po.geom(2, 8, 10, 10, 16, 3, 3, 1, 1, 1, 1), "fp32"),
        ("tf32 cb32 fwd", po.geom(1, 32, 8, 8, 64, 3, 3, 1, 1, 1, 1), "tf32"),
        ("tf32 cb4 fwd", po.geom(1, 3, 16, 16, 64, 3, 3, 1, 1, 1, 1), "tf32"),
        ("tf32 cb32 multi-tile", po.geom(2, 64, 20, 20, 96, 5, 5, 2, 2, 1, 1), "tf32"),
        ("tf32 L5-like", po.geom(2, 384, 13, 13, 384, 3, 3, 0, 0, 1, 1), "tf32"),
        ("tf32 L1-like", po.geom(1, 3, 40, 40, 96, 11, 11, 0, 0, 1, 1), "tf32"),
        ("tf32 L2-like hconv", po.geom(2, 64, 20, 20, 128, 9, 9, 0, 0, 1, 1), "tf32"),
        ("tf32 p2 C96", po.geom(2, 96, 17, 19, 80, 5, 5, 2, 2, 1, 1), "tf32"),
        ("tf32 stride4", po.geom(2, 3, 63, 63, 64, 11, 11, 2, 2, 4, 4), "tf32"),
    ]
    for name, g, math in cases:
        print(name, "...", flush=True)
        try:
            print("   ", run(g, math), flush=True)
        except Exception as e:  # keep going
            print("    ERROR", type(e).__name__, e, flush=True)
