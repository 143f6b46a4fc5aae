"""Shared parity helpers: seeded inputs, the stated tolerances, geometry sets.

Tolerances:
  * unfold / fold / identity-weight paths .................. bitwise
  * FP32-FFMA mode: |d| <= 1e-4*|ref| + atol elementwise, atol = L*2^-23*max|a|*max|b|
    (L = reduction length: worst-case FP32 accumulation bound), and ||d||/||ref|| <= 1e-4
  * TF32 mode: ||d||_2/||ref||_2 <= 5e-3 and max|d| <= 1e-2*max|ref|
    (operands rounded to 10-bit mantissa: 2^-11 relative each, sqrt(L)-growth random walk)
  * reductions: <= 1e-5 relative
"""
from __future__ import annotations

import numpy as np

import pyoracle as po

EPS32 = 2.0 ** -23


def seeded(shape, seed, lo=-1.0, hi=1.0):
    return po.uniform(shape, seed, lo, hi)


def conv_inputs(g, seed=0x5EED):
    """x ~ U(-1,1), w ~ U(-1,1)/sqrt(CRS), b ~ U(-0.1,0.1), gy ~ U(-1,1)."""
    oh, ow = po.out_hw(g)
    crs = g.C * g.kH * g.kW
    s = 1.0 / np.sqrt(crs)
    x = seeded((g.N, g.C, g.H, g.W), seed + 1)
    w = seeded((g.K, g.C, g.kH, g.kW), seed + 2, -s, s)
    b = seeded((g.K,), seed + 3, -0.1, 0.1)
    gy = seeded((g.N, g.K, oh, ow), seed + 4)
    return x, w, b, gy


def check_fp32(out, ref, L, amax, bmax, what=""):
    out = np.asarray(out, np.float64)
    ref = np.asarray(ref, np.float64)
    atol = 4.0 * L * EPS32 * amax * bmax + 1e-30
    d = np.abs(out - ref)
    bad = d > 1e-4 * np.abs(ref) + atol
    assert not bad.any(), (f"{what}: {bad.sum()} elements outside FP32 tolerance, "
                           f"max|d|={d.max():.3e} atol={atol:.3e}")
    nrm = np.linalg.norm(ref)
    if nrm > 0:
        assert np.linalg.norm(out - ref) / nrm <= 1e-4, f"{what}: normwise FP32 error too large"


def check_tf32(out, ref, what=""):
    out = np.asarray(out, np.float64)
    ref = np.asarray(ref, np.float64)
    nrm = np.linalg.norm(ref)
    rel = np.linalg.norm(out - ref) / nrm if nrm > 0 else np.linalg.norm(out)
    assert rel <= 5e-3, f"{what}: TF32 normwise error {rel:.3e} > 5e-3"
    mx = np.abs(ref).max() if ref.size else 0.0
    d = np.abs(out - ref).max() if ref.size else 0.0
    assert d <= 1e-2 * mx + 1e-30, f"{what}: TF32 max error {d:.3e} > 1e-2*max|ref| ({mx:.3e})"
    return rel


def spec_random_geometries(n=50, seed=1234):
    """N<=4, C,K<=8, H,W<=16, k in {1,3,5}, stride in {1,2}, pad in {0,1,2}."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        N, C, K = rng.integers(1, 5), rng.integers(1, 9), rng.integers(1, 9)
        H, W = rng.integers(1, 17), rng.integers(1, 17)
        k = int(rng.choice([1, 3, 5]))
        s = int(rng.choice([1, 2]))
        p = int(rng.choice([0, 1, 2]))
        g = po.geom(int(N), int(C), int(H), int(W), int(K), k, k, p, p, s, s)
        if po.oracle().or_validate(g) == 0:
            out.append(g)
    return out


def gstr(g):
    return (f"N{g.N}C{g.C}H{g.H}W{g.W}K{g.K}k{g.kH}x{g.kW}p{g.padH}x{g.padW}"
            f"s{g.strideH}x{g.strideW}")


# Channel-aligned shapes exercising the tcgen05 tile variants (bn 64/96/128/192/256,
# SW128 + small-C layouts, ragged last M tile, multi-image tiles, strided fprop).
TC_GEOMS = [
    po.geom(2, 64, 20, 20, 96, 5, 5, 2, 2, 1, 1),
    po.geom(2, 128, 13, 13, 384, 3, 3, 0, 0, 1, 1),      # L5-like
    po.geom(1, 3, 40, 40, 96, 11, 11, 0, 0, 1, 1),       # L1-like (C=3 small-C path)
    po.geom(3, 32, 24, 24, 128, 9, 9, 0, 0, 1, 1),       # L3-like
    po.geom(2, 128, 16, 16, 128, 7, 7, 0, 0, 1, 1),      # L4-like
    po.geom(2, 3, 63, 63, 64, 11, 11, 2, 2, 4, 4),       # AlexNet c1-like (stride 4)
    po.geom(2, 64, 27, 27, 192, 5, 5, 2, 2, 1, 1),       # AlexNet c2-like
    po.geom(1, 256, 14, 14, 512, 3, 3, 1, 1, 1, 1),      # VGG-like, 2 N-tiles of 256
    po.geom(4, 3, 32, 32, 64, 3, 3, 1, 1, 1, 1),         # cfg1 at batch 4
    po.geom(2, 96, 9, 11, 80, 3, 5, 1, 2, 1, 1),         # rectangular, bn=80
]

# BASELINE.json configs (convnet-benchmarks L1-L5 pad 0, cfg1)
CFG1 = po.geom(16, 3, 32, 32, 64, 3, 3, 1, 1, 1, 1)
LAYERS = {
    "L1": po.geom(128, 3, 128, 128, 96, 11, 11, 0, 0, 1, 1),
    "L2": po.geom(128, 64, 64, 64, 128, 9, 9, 0, 0, 1, 1),
    "L3": po.geom(128, 128, 32, 32, 128, 9, 9, 0, 0, 1, 1),
    "L4": po.geom(128, 128, 16, 16, 128, 7, 7, 0, 0, 1, 1),
    "L5": po.geom(128, 384, 13, 13, 384, 3, 3, 0, 0, 1, 1),
}


def with_batch(g, n):
    return po.geom(n, g.C, g.H, g.W, g.K, g.kH, g.kW, g.padH, g.padW, g.strideH, g.strideW)
