"""GPU: the Winograd F(2x2,3x3) registry entry and the tcgen05 TF32 GEMM
under it and under pt_b200_gemm's TF32 mode.

  * SPEC examples: one 4x4 tile / one channel, the delta kernel (output == input), a desk-
    scale VGG-style layer, all vs conv_direct within 1e-3 relative;
  * TF32-exact integer inputs: transforms with 1/2 factors keep every value a multiple of
    1/4 below 2^22, so forward and gradInput equal the oracle BITWISE on the bench's 3x3
    stride-1 layers (AlexNet c3-c5, Overfeat c3-c5, VGG-A c1-c8, convnet L5) at batch 2;
  * unsupported geometries (5x5, stride 2, gradInput with pad > 2) are ValidationErrors;
  * pt_b200_gemm TF32: all four transpose combinations, alpha / beta, off-tile sizes
    (129 x 129 x 129, "side of 128m+1"), batch of one, vs the oracle's naive GEMM.
"""
import numpy as np
import pytest

import pyoracle as po
from bench import WORKLOADS
from helpers import check_exact, check_tf32, conv_inputs, exact_inputs, gstr, tf32_bounds, with_batch

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _pt():
    import paper_1606_04884_b200 as pt
    return pt


def _G(g):
    return _pt().ConvGeometry(g.N, g.C, g.H, g.W, g.K, g.kH, g.kW, g.padH, g.padW, g.strideH, g.strideW)


def _d(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _h(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _rel(a, r):
    return float(np.linalg.norm(a.astype(np.float64) - r) / max(np.linalg.norm(r), 1e-30))


def test_spec_single_tile_one_channel():
    g = po.geom(1, 1, 4, 4, 1, 3, 3, 0, 0, 1, 1)
    x, w, b, _ = conv_inputs(g, 5)
    y = _pt().conv_winograd_2x2_3x3(_G(g), _d(x), _d(w), _d(b))
    assert _rel(_h(y), po.conv_direct(g, x, w, b, f64=True)) <= 1e-3


def test_spec_delta_kernel_is_identity():
    g = po.geom(2, 4, 9, 11, 4, 3, 3, 1, 1, 1, 1)
    x = po.uniform((2, 4, 9, 11), 3)
    w = np.zeros((4, 4, 3, 3), np.float32)
    for c in range(4):
        w[c, c, 1, 1] = 1.0
    y = _pt().conv_winograd_2x2_3x3(_G(g), _d(x), _d(w))
    # the center tap passes x through the transforms; TF32 rounds the transformed values
    # (sums of up to 4 inputs) to 10 mantissa bits
    np.testing.assert_allclose(_h(y), x, rtol=0, atol=2.0 ** -8 * np.abs(x).max())


@pytest.mark.parametrize("g", [po.geom(1, 4, 16, 16, 4, 3, 3, 1, 1, 1, 1),
                               po.geom(3, 35, 13, 17, 40, 3, 3, 0, 0, 1, 1),
                               po.geom(2, 64, 15, 14, 96, 3, 3, 2, 2, 1, 1),
                               po.geom(1, 130, 9, 9, 300, 3, 3, 1, 0, 1, 1)], ids=gstr)
def test_winograd_fwd_dgrad_vs_oracle(g):
    """VGG-style desk-scale layer within 1e-3 relative; plus odd sizes, C and K
    off the 32 / 256 tiles, asymmetric padding."""
    pt = _pt()
    x, w, b, gy = conv_inputs(g, 9)
    y = _h(pt.conv_winograd_2x2_3x3(_G(g), _d(x), _d(w), _d(b)))
    gx = _h(pt.conv_backward_input_winograd(_G(g), _d(gy), _d(w)))
    tol = tf32_bounds(g, x, w, b, gy, passes=("fwd", "dgrad"))
    assert _rel(y, po.conv_direct(g, x, w, b, f64=True)) <= 1e-3
    assert _rel(gx, po.conv_backward_input(g, gy, w)) <= 1e-3
    # transform-domain rounding: each V / U entry sums up to 4 (9) operands, so the
    # elementwise bound is 4x the direct-conv one
    check_tf32(y, po.conv_forward(g, x, w, b), "winograd fwd", 4 * tol["fwd"])
    check_tf32(gx, po.conv_backward_input(g, gy, w), "winograd dgrad", 4 * tol["dgrad"])


WINO_LAYERS = [(wl, l) for wl in ("convnet", "alexnet", "overfeat", "vgga") for l in WORKLOADS[wl]
               if l[6] == 3 and l[7] == 3 and l[10] == 1 and l[11] == 1]


@pytest.mark.parametrize("wl,l", WINO_LAYERS, ids=[f"{a}-{b[0]}" for a, b in WINO_LAYERS])
def test_winograd_bench_layers_exact(wl, l):
    pt = _pt()
    g = with_batch(po.geom(*l[1:]), 2)
    x, w, b, gy = exact_inputs(g, 0xA11)
    y = _h(pt.conv_winograd_2x2_3x3(_G(g), _d(x), _d(w), _d(b)))
    check_exact(y, po.conv_forward(g, x, w, b), f"{wl}/{l[0]} winograd fwd")
    gx = _h(pt.conv_backward_input_winograd(_G(g), _d(gy), _d(w)))
    check_exact(gx, po.conv_backward_input(g, gy, w), f"{wl}/{l[0]} winograd dgrad")


@pytest.mark.parametrize("g,op", [(po.geom(1, 8, 9, 9, 8, 5, 5, 2, 2, 1, 1), 0),
                                  (po.geom(1, 8, 9, 9, 8, 3, 3, 1, 1, 2, 2), 0),
                                  (po.geom(1, 8, 9, 9, 8, 3, 3, 3, 3, 1, 1), 1)])
def test_winograd_rejects_unsupported(g, op):
    pt = _pt()
    x, w, b, gy = conv_inputs(g, 1)
    with pytest.raises(pt.ValidationError, match="unsupported geometry"):
        if op == 0:
            pt.conv_winograd_2x2_3x3(_G(g), _d(x), _d(w), _d(b))
        else:
            pt.conv_backward_input_winograd(_G(g), _d(gy), _d(w))


GEMMS = [(64, 48, 40), (129, 129, 129), (300, 257, 96), (1, 1, 1), (8, 520, 33)]


@pytest.mark.parametrize("tA", [False, True])
@pytest.mark.parametrize("tB", [False, True])
@pytest.mark.parametrize("mnk", GEMMS)
def test_gemm_tf32_tensor_cores(mnk, tA, tB):
    """pt_b200_gemm honours math: TF32 runs the tcgen05 GEMM (leading dims padded to
    multiples of 4 for TMA), FP32 the FFMA kernel; both vs the oracle's naive GEMM."""
    pt = _pt()
    M, N, K = mnk
    pad = lambda r, c: (r, (c + 3) // 4 * 4)  # noqa: E731
    rng = np.random.default_rng(M * 7 + N)
    A_full = rng.uniform(-1, 1, pad(*((K, M) if tA else (M, K)))).astype(np.float32)
    B_full = rng.uniform(-1, 1, pad(*((N, K) if tB else (K, N)))).astype(np.float32)
    C0 = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    A = A_full[:, :(M if tA else K)]
    B = B_full[:, :(K if tB else N)]
    opA = A.T if tA else A
    opB = B.T if tB else B
    ref = 0.75 * opA.astype(np.float64) @ opB.astype(np.float64) + (-0.5) * C0
    dA, dB = _d(A_full), _d(B_full)
    # views over the padded storage: leading dims are the padded row lengths
    import ctypes as C
    from paper_1606_04884_b200 import _lib as L
    for math in ("tf32", "fp32"):
        dC = _d(C0)
        L.check(L.lib().pt_b200_gemm(int(tA), int(tB), M, N, K, C.c_float(0.75), dA.data_ptr(),
                                     A_full.shape[1], dB.data_ptr(), B_full.shape[1], C.c_float(-0.5),
                                     dC.data_ptr(), N, L.PT_MATH_TF32 if math == "tf32" else L.PT_MATH_FP32,
                                     torch.cuda.current_stream().cuda_stream))
        out = _h(dC)
        absb = 0.75 * np.abs(opA).astype(np.float64) @ np.abs(opB) + 0.5 * np.abs(C0)
        lim = (2.0 ** -10 + 2 * K * 2.0 ** -23) * absb if math == "tf32" else 4 * K * 2.0 ** -23 * absb
        assert (np.abs(out - ref) <= lim + 1e-30).all(), (math, np.abs(out - ref).max())


def test_gemm_tf32_rejects_unaligned_leading_dim():
    pt = _pt()
    a = torch.zeros((5, 5), device="cuda")
    c = torch.zeros((5, 5), device="cuda")
    with pytest.raises(pt.ValidationError, match="TF32"):
        pt.gemm(a, a, c, math="tf32")
    pt.gemm(a, a, c, math="fp32")
