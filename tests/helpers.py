"""Shared parity helpers: seeded inputs, the stated tolerances, geometry sets.

Tolerances:
  * unfold / fold / identity-weight paths .................. bitwise
  * FP32-FFMA mode: |d| <= 1e-4*|ref| + atol elementwise, atol = L*2^-23*max|a|*max|b|
    (L = reduction length: worst-case FP32 accumulation bound), and ||d||/||ref|| <= 1e-4
  * TF32 mode, elementwise: |d_i| <= (2^-10 + 2*L*2^-23) * A_i, A_i = the same pass computed
    on |operands| (sum of |a_j*b_j| feeding element i, oracle-computed; tf32_bounds): each
    operand is rounded to a 10-bit mantissa (rna: 2^-11 relative each, 2^-10 per product),
    plus worst-case FP32 accumulation over L terms in any order, device and oracle. Normwise
    ||d||_2/||ref||_2 <= 1e-3 (observed 2.5-4e-4: two independent 2^-11 roundings per
    product random-walk to ~2^-11*sqrt(2/3) relative; round 1 allowed 5e-3).
    Without bounds (legacy callers): max|d| <= 3e-3*max|ref|.
  * TF32-EXACT inputs (exact_inputs): integer x, gy in [-8, 8], weights in {-1, 0, 1},
    integer bias: every operand is exact in TF32, every product and partial sum is an
    integer below 2^24, so any summation order gives the exact result -> the device result
    must equal the oracle BITWISE (proves the index mapping of every tcgen05 engine).
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


TF32_NORMWISE = 1e-3


def check_tf32(out, ref, what="", tol=None):
    """TF32 parity: elementwise against `tol` (tf32_bounds) when given, else 3e-3*max|ref|;
    normwise <= TF32_NORMWISE."""
    out = np.asarray(out, np.float64)
    ref = np.asarray(ref, np.float64)
    assert out.shape == ref.shape, f"{what}: shape {out.shape} != {ref.shape}"
    if not ref.size:
        return 0.0
    assert np.isfinite(out).all(), f"{what}: non-finite values in the device result"
    nrm = np.linalg.norm(ref)
    rel = np.linalg.norm(out - ref) / nrm if nrm > 0 else np.linalg.norm(out)
    assert rel <= TF32_NORMWISE, f"{what}: TF32 normwise error {rel:.3e} > {TF32_NORMWISE}"
    d = np.abs(out - ref)
    lim = (np.asarray(tol, np.float64) if tol is not None else 3e-3 * np.abs(ref).max()) + 1e-30
    bad = d > lim
    if bad.any():
        i = np.unravel_index(np.argmax(d - lim), d.shape)
        raise AssertionError(f"{what}: {int(bad.sum())} of {d.size} elements outside the TF32 "
                             f"bound; worst at {tuple(int(v) for v in i)}: out={out[i]:.6e} "
                             f"ref={ref[i]:.6e} bound={float(np.broadcast_to(lim, d.shape)[i]):.3e}")
    return rel


def check_exact(out, ref, what=""):
    """Bitwise equality (TF32-exact inputs, unfold/fold, batched == per-image)."""
    out = np.asarray(out, np.float32)
    ref = np.asarray(ref, np.float32)
    assert out.shape == ref.shape, f"{what}: shape {out.shape} != {ref.shape}"
    bad = out.view(np.uint32) != ref.view(np.uint32)
    if bad.any():
        i = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {int(bad.sum())} of {out.size} elements differ; first at "
                             f"{tuple(int(v) for v in i)}: out={out[tuple(i)]!r} "
                             f"ref={ref[tuple(i)]!r}")


def exact_inputs(g, seed=0x1E7):
    """TF32-exact operands: x, gy integers in [-8, 8], w in {-1, 0, 1}, b integers in
    [-4, 4] (float32). Every product/partial sum is an integer < 2^24 at slice sizes."""
    rng = np.random.default_rng(seed)
    oh, ow = po.out_hw(g)
    x = rng.integers(-8, 9, (g.N, g.C, g.H, g.W)).astype(np.float32)
    w = rng.integers(-1, 2, (g.K, g.C, g.kH, g.kW)).astype(np.float32)
    b = rng.integers(-4, 5, (g.K,)).astype(np.float32)
    gy = rng.integers(-8, 9, (g.N, g.K, oh, ow)).astype(np.float32)
    return x, w, b, gy


def tf32_bounds(g, x, w, b, gy, passes=("fwd", "dgrad", "wgrad")):
    """Elementwise TF32 tolerances (see module docstring) for fwd, dgrad, wgrad, gradBias,
    from the oracle run on absolute values (the FP32 oracle's own error is < 1e-6 relative
    of these bounds)."""
    oh, ow = po.out_hw(g)
    ab_ = lambda a: None if a is None else np.abs(a)  # noqa: E731
    ax, aw, agy, ab = ab_(x), ab_(w), ab_(gy), ab_(b)
    u = 2.0 ** -10
    e = EPS32
    L_f, L_d, L_w = g.C * g.kH * g.kW, g.K * g.kH * g.kW, g.N * oh * ow
    # 2*L*eps: worst-case accumulation of the device (any order, RN or truncating) plus
    # that of the FP32 oracle it is compared with
    out = {}
    if "fwd" in passes:
        out["fwd"] = (u + 2 * (L_f + 1) * e) * po.conv_forward(g, ax, aw, ab).astype(np.float64)
    if "dgrad" in passes:
        out["dgrad"] = (u + 2 * L_d * e) * po.conv_backward_input(g, agy, aw).astype(np.float64)
    if "wgrad" in passes:
        a_gw, a_gb = po.conv_backward_weight(g, ax, agy)
        out["wgrad"] = (u + 2 * L_w * e) * a_gw.astype(np.float64)
        out["gradBias"] = 2 * L_w * e * a_gb.astype(np.float64)
    return out


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
