"""GPU parity: the sm_100a conv passes through the C ABI vs the CPU oracle.

Every device computation below runs in libpt_b200.so (called via ctypes on torch
device memory). The oracle (oracle/liboracle.so) is only the checker.
"""
import numpy as np
import pytest

import pyoracle as po
from engine_check import check_geometry
from helpers import (CFG1, EPS32, TC_GEOMS, check_fp32, check_tf32, conv_inputs, gstr,
                     spec_random_geometries, tf32_bounds)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _pt():
    import paper_1606_04884_b200 as pt
    return pt


def _g(g):
    pt = _pt()
    return pt.ConvGeometry(g.N, g.C, g.H, g.W, g.K, g.kH, g.kW, g.padH, g.padW, g.strideH,
                           g.strideW)


def _d(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _h(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def run_all(g, math, seed=0x5EED):
    pt = _pt()
    x, w, b, gy = conv_inputs(g, seed)
    G = _g(g)
    y = pt.conv_forward(G, _d(x), _d(w), _d(b), math=math)
    gx = pt.conv_backward_input(G, _d(gy), _d(w), math=math)
    gw, gb = pt.conv_backward_weight(G, _d(x), _d(gy), math=math)
    return (x, w, b, gy), (_h(y), _h(gx), _h(gw), _h(gb))


def oracle_all(g, x, w, b, gy):
    y = po.conv_direct(g, x, w, b, f64=True)
    gx = po.conv_backward_input(g, gy, w)
    gw, gb = po.conv_backward_weight(g, x, gy)
    return y, gx, gw, gb


def check_all_tf32(g, inputs, outs, refs=None):
    """fwd / dgrad / wgrad / gradBias against the oracle with elementwise TF32 bounds."""
    x, w, b, gy = inputs
    refs = refs or oracle_all(g, x, w, b, gy)
    tol = tf32_bounds(g, x, w, b, gy)
    for o, r, k in zip(outs, refs, ("fwd", "dgrad", "wgrad", "gradBias")):
        check_tf32(o, r, f"{gstr(g)} {k}", tol[k])


@pytest.mark.parametrize("math", ["fp32", "tf32"])
@pytest.mark.parametrize("g", spec_random_geometries(50), ids=gstr)
def test_spec_random_geometries(g, math):
    """SPEC.md:436 oracle-equivalence sweep (50 random desk-scale geometries)."""
    (x, w, b, gy), (y, gx, gw, gb) = run_all(g, math)
    ry, rgx, rgw, rgb = oracle_all(g, x, w, b, gy)
    oh, ow = po.out_hw(g)
    crs = g.C * g.kH * g.kW
    if math == "fp32":
        check_fp32(y, ry, crs, 1.0, np.abs(w).max(), "fwd")
        check_fp32(gx, rgx, g.K * g.kH * g.kW, 1.0, np.abs(w).max(), "dgrad")
        check_fp32(gw, rgw, g.N * oh * ow, 1.0, 1.0, "wgrad")
    else:
        check_all_tf32(g, (x, w, b, gy), (y, gx, gw, gb), (ry, rgx, rgw, rgb))
    np.testing.assert_allclose(gb, rgb, rtol=1e-5, atol=1e-5 * g.N * oh * ow)


@pytest.mark.parametrize("g", TC_GEOMS, ids=gstr)
def test_tensor_core_tiles(g):
    """tcgen05 tile variants (SW128 / small-C, bn 64..256, ragged tiles) in TF32 mode."""
    (x, w, b, gy), (y, gx, gw, gb) = run_all(g, "tf32", seed=77)
    check_all_tf32(g, (x, w, b, gy), (y, gx, gw, gb))


@pytest.mark.parametrize("g", TC_GEOMS, ids=gstr)
def test_tensor_core_tiles_exact(g):
    """TF32-exact integer inputs: bitwise equal to the oracle through the default engines
    (finput + combined backward and the separate passes)."""
    fails, _ = check_geometry(g, seed=79, exact=True, real=False)
    assert not fails, "\n".join(fails[:4])


@pytest.mark.parametrize("g", TC_GEOMS[:4], ids=gstr)
def test_fp32_mode_tight(g):
    (x, w, b, gy), (y, gx, gw, gb) = run_all(g, "fp32", seed=78)
    ry, rgx, rgw, rgb = oracle_all(g, x, w, b, gy)
    oh, ow = po.out_hw(g)
    check_fp32(y, ry, g.C * g.kH * g.kW, 1.0, np.abs(w).max(), "fwd")
    check_fp32(gx, rgx, g.K * g.kH * g.kW, 1.0, np.abs(w).max(), "dgrad")
    check_fp32(gw, rgw, g.N * oh * ow, 1.0, 1.0, "wgrad")


@pytest.mark.parametrize("math", ["fp32", "tf32"])
def test_cfg1_full(math):
    """BASELINE configs[0]: batch 16, 3->64, 3x3 pad 1, 32x32 — full size vs oracle."""
    (x, w, b, gy), (y, gx, gw, gb) = run_all(CFG1, math)
    ry, rgx, rgw, rgb = oracle_all(CFG1, x, w, b, gy)
    if math == "tf32":
        check_all_tf32(CFG1, (x, w, b, gy), (y, gx, gw, gb), (ry, rgx, rgw, rgb))
    else:
        check_fp32(y, ry, 27, 1.0, np.abs(w).max(), "fwd")
        check_fp32(gx, rgx, 64 * 9, 1.0, np.abs(w).max(), "dgrad")
        check_fp32(gw, rgw, 16 * 1024, 1.0, 1.0, "wgrad")
    np.testing.assert_allclose(gb, rgb, rtol=1e-5, atol=1e-3)


@pytest.mark.parametrize("math", ["fp32", "tf32"])
@pytest.mark.parametrize("g", TC_GEOMS[:6] + [CFG1], ids=gstr)
def test_fused_backward_matches_separate_passes(g, math):
    """pt_b200_conv_bwd (shared gy transform, fused gradBias) == the separate ABI passes,
    and Torch accumulate/scale semantics (gw += scale*dW) hold."""
    pt = _pt()
    x, w, b, gy = conv_inputs(g, 31)
    G = _g(g)
    gx, gw, gb = pt.conv_backward(G, _d(x), _d(gy), _d(w), math=math)
    sgx = pt.conv_backward_input(G, _d(gy), _d(w), math=math)
    sgw, sgb = pt.conv_backward_weight(G, _d(x), _d(gy), math=math)
    np.testing.assert_array_equal(_h(gx), _h(sgx))
    np.testing.assert_allclose(_h(gw), _h(sgw), rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(_h(gb), _h(sgb), rtol=1e-5, atol=1e-5)
    # accumulate: start from gw0, add 0.5 * dW
    gw0 = po.uniform((g.K, g.C, g.kH, g.kW), 5)
    gb0 = po.uniform((g.K,), 6)
    _, agw, agb = pt.conv_backward(G, _d(x), _d(gy), _d(w), gw=_d(gw0), gb=_d(gb0), scale=0.5,
                                   accumulate=True, need_input_grad=False, math=math)
    rgw, rgb = po.conv_backward_weight(g, x, gy)
    oh, ow = po.out_hw(g)
    if math == "fp32":
        check_fp32(_h(agw), gw0 + 0.5 * rgw, g.N * oh * ow, 1.0, 1.0, "acc wgrad")
    else:
        tol = tf32_bounds(g, x, w, b, gy)["wgrad"]
        check_tf32(_h(agw), gw0 + 0.5 * rgw, "acc wgrad", 0.5 * tol + 2 * EPS32 * np.abs(gw0))
    np.testing.assert_allclose(_h(agb), gb0 + 0.5 * rgb, rtol=1e-5, atol=1e-4)


# Small-C layers with fewer than 32 (or a non-multiple of 32) output channels: the combined
# backward's shared gy copy is padded to 32 channels, which a small-K dgrad plan must not
# read as its own 8/16-channel layout (found by tests/stress_tc.py).
SMALLK_COMBINED = [
    po.geom(3, 3, 32, 10, 16, 7, 7, 3, 3, 1, 1),
    po.geom(1, 3, 32, 21, 16, 11, 11, 2, 2, 1, 1),
    po.geom(1, 3, 18, 50, 16, 7, 7, 3, 3, 1, 1),
    po.geom(2, 3, 20, 24, 8, 5, 5, 2, 2, 1, 1),
    po.geom(2, 3, 20, 24, 48, 7, 7, 3, 3, 1, 1),
    po.geom(2, 4, 16, 30, 24, 3, 3, 1, 1, 1, 1),
    po.geom(2, 3, 35, 35, 16, 11, 11, 2, 2, 4, 4),
    po.geom(2, 16, 20, 20, 16, 5, 5, 2, 2, 1, 1),
]


@pytest.mark.parametrize("math", ["fp32", "tf32"])
@pytest.mark.parametrize("g", SMALLK_COMBINED, ids=gstr)
def test_combined_backward_small_k(g, math):
    pt = _pt()
    x, w, b, gy = conv_inputs(g, 41)
    G = _g(g)
    nb = pt.finput_bytes(G, math)
    fin = torch.empty(max(nb, 1), dtype=torch.uint8, device="cuda") if nb else None
    pt.conv_forward(G, _d(x), _d(w), _d(b), math=math, finput=fin)
    gx, gw, gb = pt.conv_backward(G, _d(x), _d(gy), _d(w), math=math, finput=fin)
    sgx = pt.conv_backward_input(G, _d(gy), _d(w), math=math)
    np.testing.assert_array_equal(_h(gx), _h(sgx))
    rgx = po.conv_backward_input(g, gy, w)
    rgw, rgb = po.conv_backward_weight(g, x, gy)
    oh, ow = po.out_hw(g)
    if math == "fp32":
        check_fp32(_h(gx), rgx, g.K * g.kH * g.kW, 1.0, np.abs(w).max(), "dgrad")
        check_fp32(_h(gw), rgw, g.N * oh * ow, 1.0, 1.0, "wgrad")
    else:
        tol = tf32_bounds(g, x, w, b, gy)
        check_tf32(_h(gx), rgx, "dgrad", tol["dgrad"])
        check_tf32(_h(gw), rgw, "wgrad", tol["wgrad"])
    np.testing.assert_allclose(_h(gb), rgb, rtol=1e-5, atol=1e-5 * g.N * oh * ow)


FINPUT_GEOMS = [g for g in TC_GEOMS] + [
    po.geom(2, 64, 20, 20, 128, 9, 9, 0, 0, 1, 1),   # Hankel fwd, pad 0
    po.geom(2, 96, 17, 19, 80, 5, 5, 2, 2, 1, 1),    # Hankel fwd copy carries a 2-pixel border
    po.geom(2, 32, 30, 30, 64, 3, 3, 1, 1, 1, 1),    # tap-paired Hankel (<= 64 out channels)
]


@pytest.mark.parametrize("g", FINPUT_GEOMS, ids=gstr)
def test_finput_reuse_bitwise(g):
    """Torch's finput: the forward's channels-last copy of x reused by accGradParameters
    gives bitwise the same y / gradInput / gradWeight / gradBias as re-laying x out."""
    pt = _pt()
    x, w, b, gy = conv_inputs(g, 77)
    G = _g(g)
    nb = pt.finput_bytes(G)
    fin = torch.empty(max(nb, 1), dtype=torch.uint8, device="cuda")
    y0 = pt.conv_forward(G, _d(x), _d(w), _d(b))
    y1 = pt.conv_forward(G, _d(x), _d(w), _d(b), finput=fin)
    gx0, gw0, gb0 = pt.conv_backward(G, _d(x), _d(gy), _d(w))
    gx1, gw1, gb1 = pt.conv_backward(G, _d(x), _d(gy), _d(w), finput=fin)
    for a, c, what in ((y0, y1, "y"), (gx0, gx1, "gx"), (gw0, gw1, "gw"), (gb0, gb1, "gb")):
        np.testing.assert_array_equal(_h(a), _h(c), err_msg=f"{gstr(g)} {what} (finput {nb} B)")


# Geometries aimed at the Hankel engine's edge cases: odd output heights (unequal image
# halves), asymmetric kernels/pads, padded rows near the 256-pixel TMA box limit, tap
# pairing with odd kW, multi-chunk stages, rows that need NR vs NR-1 boxes.
HANKEL_EDGE = [
    po.geom(2, 32, 13, 37, 48, 5, 7, 2, 3, 1, 1),
    po.geom(1, 64, 9, 250, 64, 3, 3, 1, 1, 1, 1),
    po.geom(3, 96, 11, 30, 160, 3, 5, 0, 2, 1, 1),
    po.geom(2, 128, 17, 17, 64, 9, 9, 4, 4, 1, 1),
    po.geom(1, 32, 40, 61, 32, 11, 11, 5, 5, 1, 1),
]

@pytest.mark.parametrize("g", HANKEL_EDGE, ids=gstr)
def test_hankel_edge_default_engines(g):
    """The same edge geometries through whatever engines the default plan picks."""
    x, w, b, gy = conv_inputs(g, 92)
    pt = _pt()
    G = _g(g)
    y = pt.conv_forward(G, _d(x), _d(w), _d(b))
    gx, gw, gb = pt.conv_backward(G, _d(x), _d(gy), _d(w))
    check_all_tf32(g, (x, w, b, gy), (_h(y), _h(gx), _h(gw), _h(gb)))


@pytest.mark.parametrize("g", HANKEL_EDGE, ids=gstr)
def test_hankel_edge_exact(g):
    fails, _ = check_geometry(g, seed=93, exact=True, real=False)
    assert not fails, "\n".join(fails[:4])


# small-C stride-1 layers: the planes-of-taps weight gradient (umma_swgrad.cu) — odd
# output extents, padding, C = 1..4, K not a multiple of 32, two N halves (npad = 512)
SMALLC_GEOMS = [
    po.geom(2, 3, 37, 45, 64, 3, 3, 1, 1, 1, 1),       # VGG conv1-like, odd oH / oW
    po.geom(2, 1, 30, 33, 16, 5, 5, 2, 2, 1, 1),       # C = 1
    po.geom(1, 4, 21, 70, 128, 7, 7, 3, 3, 1, 1),      # C = 4, K = 128 (all TMEM lanes)
    po.geom(2, 3, 40, 40, 96, 11, 11, 0, 0, 1, 1),     # L1-like: 363 columns, two N halves
    po.geom(1, 2, 17, 17, 40, 3, 5, 0, 2, 1, 1),       # rectangular filter, Kp = 64
    po.geom(1, 4, 30, 40, 32, 11, 11, 1, 1, 1, 1),     # 484 columns: two halves of 256
    po.geom(3, 3, 12, 12, 8, 1, 1, 0, 0, 1, 1),        # 1x1
]


@pytest.mark.parametrize("g", SMALLC_GEOMS, ids=gstr)
def test_small_c_weight_gradient(g):
    pt = _pt()
    x, w, b, gy = conv_inputs(g, 123)
    G = _g(g)
    gw, gb = pt.conv_backward_weight(G, _d(x), _d(gy), math="tf32")
    rgw, rgb = po.conv_backward_weight(g, x, gy)
    tol = tf32_bounds(g, x, w, b, gy)
    check_tf32(_h(gw), rgw, "wgrad", tol["wgrad"])
    np.testing.assert_allclose(_h(gb), rgb, rtol=1e-5, atol=1e-4)
    # fused backward with Torch's accumulate / scale: gw = gw0 + 0.5 * dW
    gw0 = po.uniform((g.K, g.C, g.kH, g.kW), 9)
    gb0 = po.uniform((g.K,), 10)
    gx, agw, agb = pt.conv_backward(G, _d(x), _d(gy), _d(w), gw=_d(gw0), gb=_d(gb0), scale=0.5,
                                    accumulate=True, math="tf32")
    check_tf32(_h(agw), gw0 + 0.5 * rgw, "acc wgrad", 0.5 * tol["wgrad"] + 2 * EPS32 * np.abs(gw0))
    check_tf32(_h(gx), po.conv_backward_input(g, gy, w), "dgrad", tol["dgrad"])


# Hankel tap-quad weight gradient (umma_hwgrad.cu) forced on: odd chunk counts (C = 96 ->
# 3 chunks), K = 320 (two n-tiles), kW = 3 / 5 / 11 (1-3 quads, dropped tap slots), padding,
# rows split into several 128-column segments, non-square outputs
HWGRAD_EDGE = [
    po.geom(2, 96, 15, 21, 320, 9, 9, 4, 4, 1, 1),
    po.geom(1, 64, 9, 140, 64, 3, 5, 1, 2, 1, 1),
    po.geom(2, 32, 20, 18, 128, 11, 11, 5, 5, 1, 1),
    po.geom(3, 64, 12, 12, 96, 3, 3, 1, 1, 1, 1),
    po.geom(1, 128, 7, 9, 256, 7, 7, 3, 3, 1, 1),
]


# default-engine parity for shapes that select the newer paths: two position tiles per
# weight stage (short reduction), tap-quad wgrad at <= 64 channels, flat tiling with
# border filter-row skipping (large padding)
DEFAULT_PATHS = [
    po.geom(2, 64, 30, 30, 128, 3, 3, 1, 1, 1, 1),     # VGG conv2-like: RUNS = 2 fwd, quad wgrad
    po.geom(3, 64, 18, 21, 64, 3, 3, 1, 1, 1, 1),      # 64 -> 64, odd sizes
    po.geom(2, 64, 24, 24, 128, 9, 9, 0, 0, 1, 1),     # L2-like: flat dgrad (8-row zero border)
    po.geom(2, 32, 17, 23, 48, 7, 7, 3, 3, 1, 1),      # padded 7x7
]


@pytest.mark.parametrize("g", DEFAULT_PATHS, ids=gstr)
def test_default_engine_paths(g):
    (x, w, b, gy), (y, gx, gw, gb) = run_all(g, "tf32", seed=57)
    check_all_tf32(g, (x, w, b, gy), (y, gx, gw, gb))


@pytest.mark.parametrize("wide", [False, True])
def test_randomised_geometries(wide):
    """64 random channel-rich (or odd-channel / strided / rectangular: wide) geometries
    (tests/stress_tc.py) through the default engines: bitwise on TF32-exact inputs,
    elementwise TF32 bounds on real-valued ones."""
    import stress_tc
    worst, bad = stress_tc.run(64, 11 + wide, wide)
    assert not bad, f"worst {worst:.3e}: {bad[:3]}"
