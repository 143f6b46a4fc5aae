"""Randomised channel-rich geometries through the default tensor-core engines vs the oracle
(fwd / dgrad / wgrad / gradBias): bitwise on TF32-exact inputs, elementwise TF32 bounds on
real-valued ones (tests/engine_check.py). Stress companion of test_gpu_conv.py:
  python tests/stress_tc.py [count] [seed] [wide|smallc]
smallc: stride-1 layers with C*kH*kW <= 32 and K <= 64 (the fused small-C backward).
"""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"),
                os.path.dirname(os.path.abspath(__file__))]
import numpy as np  # noqa: E402

import pyoracle as po  # noqa: E402


def smallc_geometries(n, seed):
    """Fused small-C backward candidates: W, oW multiples of 4 (TMA row strides), odd
    heights, K padded 32 / 64, rectangular filters, pads 0..k-1."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        C = int(rng.integers(1, 5))
        kh, kw = int(rng.choice([1, 2, 3, 5])), int(rng.choice([1, 3, 5]))
        if C * kh * kw > 32:
            continue
        K = int(rng.choice([4, 16, 24, 32, 40, 48, 64]))
        ph, pw = int(rng.integers(0, kh)), int(rng.integers(0, kw))
        W = 4 * int(rng.integers(2, 20))
        if (W + 2 * pw - kw + 1) % 4:
            continue
        H, N = int(rng.integers(kh, 40)), int(rng.integers(1, 4))
        g = po.geom(N, C, H, W, K, kh, kw, ph, pw, 1, 1)
        if po.oracle().or_validate(g) == 0:
            out.append(g)
    return out


def tc_random_geometries(n, seed, wide=False):
    if wide == "smallc":
        return smallc_geometries(n, seed)
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
    """Each geometry through engine_check: TF32-exact integer inputs bitwise vs the oracle,
    real-valued inputs within the elementwise TF32 bounds (finput + combined backward for
    every geometry, the separate passes for every other one)."""
    from engine_check import check_geometry
    worst = 0.0
    bad = []
    for i, g in enumerate(tc_random_geometries(n, seed, wide)):
        fails, rels = check_geometry(g, seed=3 + i, separate=bool(i % 2))
        worst = max([worst] + list(rels.values()))
        if fails:
            bad.append((g, fails))
    return worst, bad


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 7
    wide = sys.argv[3] if len(sys.argv) > 3 and sys.argv[3] in ("wide", "smallc") else False
    worst, bad = run(n, seed, wide)
    print(f"{n} geometries, worst normwise error {worst:.3e}, failures {len(bad)}")
    for g, e in bad:
        print("FAIL", (g.N, g.C, g.H, g.W, g.K, g.kH, g.kW, g.padH, g.padW, g.strideH, g.strideW), e[:3])
    sys.exit(1 if bad else 0)
