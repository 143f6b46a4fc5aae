"""Randomised channel-rich geometries through the default tensor-core engines vs the oracle
(fwd / dgrad / wgrad / gradBias), TF32 tolerance. Stress companion of test_gpu_conv.py:
  python tests/stress_tc.py [count] [seed] [wide]
"""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"),
                os.path.dirname(os.path.abspath(__file__))]
import numpy as np  # noqa: E402

import pyoracle as po  # noqa: E402


def tc_random_geometries(n, seed, wide=False):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        if wide:  # odd channel counts, small K, strides up to 4, rectangular kernels below
            C = int(rng.choice([1, 2, 3, 4, 5, 8, 12, 24, 40, 72]))
            K = int(rng.choice([4, 8, 16, 24, 40, 56, 72, 136]))
        else:
            C = int(rng.choice([3, 16, 32, 48, 64, 96, 128, 160]))
            K = int(rng.choice([16, 32, 48, 64, 96, 128, 192, 256, 320]))
        k = int(rng.choice([1, 3, 5, 7, 9, 11]))
        s = int(rng.choice([1, 1, 2, 3, 4] if wide else [1, 1, 1, 2]))
        p = int(rng.integers(0, k // 2 + 1))
        H, W = int(rng.integers(k, 48)), int(rng.integers(k, 72))
        N = int(rng.integers(1, 4))
        kw = int(rng.choice([1, 3, 5, 7])) if wide and rng.random() < 0.3 else k
        sw = int(rng.choice([1, 2])) if wide and rng.random() < 0.3 else s
        g = po.geom(N, C, H, W, K, k, kw, p, min(p, kw // 2), s, sw)
        if po.oracle().or_validate(g) == 0:
            out.append(g)
    return out


def run(n=40, seed=7, wide=False):
    import torch
    import paper_1606_04884_b200 as pt
    from helpers import conv_inputs
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    rel = lambda a, r: float(np.linalg.norm(a.astype(np.float64) - r) / max(np.linalg.norm(r), 1e-30))  # noqa: E731
    worst = 0.0
    bad = []
    for i, g in enumerate(tc_random_geometries(n, seed, wide)):
        x, w, b, gy = conv_inputs(g, 3)
        G = pt.ConvGeometry(g.N, g.C, g.H, g.W, g.K, g.kH, g.kW, g.padH, g.padW, g.strideH, g.strideW)
        # every other geometry keeps Torch's finput (the forward's relaid x) for the backward
        fb = pt.finput_bytes(G) if i % 2 else 0
        fin = torch.empty(fb, dtype=torch.uint8, device="cuda") if fb else None
        y = pt.conv_forward(G, d(x), d(w), d(b), finput=fin)
        gx, gw, gb = pt.conv_backward(G, d(x), d(gy), d(w), finput=fin)
        torch.cuda.synchronize()
        rgw, rgb = po.conv_backward_weight(g, x, gy)
        e = [rel(y.cpu().numpy(), po.conv_direct(g, x, w, b, f64=True)),
             rel(gx.cpu().numpy(), po.conv_backward_input(g, gy, w)),
             rel(gw.cpu().numpy(), rgw), rel(gb.cpu().numpy(), rgb)]
        worst = max(worst, max(e))
        if max(e) >= 5e-3:
            bad.append((g, e))
    return worst, bad


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 7
    wide = len(sys.argv) > 3 and sys.argv[3] == "wide"
    worst, bad = run(n, seed, wide)
    print(f"{n} geometries, worst normwise error {worst:.3e}, failures {len(bad)}")
    for g, e in bad:
        print("FAIL", (g.N, g.C, g.H, g.W, g.K, g.kH, g.kW, g.padH, g.padW, g.strideH, g.strideW), e)
    sys.exit(1 if bad else 0)
