"""GPU: every layer of BASELINE.json's full-size configs as bench.py times them
(convnet-benchmarks L1-L5, AlexNet c1-c5, Overfeat-fast c1-c5 at batch 128, VGG-A c1-c8
at batch 64), real-valued inputs — checks the oracle can afford at these sizes (the
TF32-exact full-batch checks of the same layers are in test_gpu_workloads.py):

  * batched == per-image, BITWISE: fwd / dgrad of an image do not depend
    on which images share its tile (accumulation order is per output element);
  * spot parity: images 0 and N-1 of the full-batch device result vs the oracle;
  * wgrad / gradBias are sums over the batch: full-batch == sum of 4 quarter-batch
    device results (TF32 tolerance), and one quarter vs the oracle;
  * linearity in the weights of the forward pass.
"""
import numpy as np
import pytest

import pyoracle as po
from bench import WORKLOADS
from helpers import check_tf32, tf32_bounds, with_batch

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FULL = {f"{wl}-{l[0]}": po.geom(*l[1:]) for wl in ("convnet", "alexnet", "overfeat", "vgga")
        for l in WORKLOADS[wl]}


def _pt():
    import paper_1606_04884_b200 as pt
    return pt


def _G(g):
    return _pt().ConvGeometry(g.N, g.C, g.H, g.W, g.K, g.kH, g.kW, g.padH, g.padW, g.strideH,
                              g.strideW)


def _dev_inputs(g, seed):
    pt = _pt()
    G = _G(g)
    s = 1.0 / np.sqrt(g.C * g.kH * g.kW)
    x = pt.fill_uniform(torch.empty(G.input_shape(), device="cuda"), seed + 1)
    w = pt.fill_uniform(torch.empty(G.weight_shape(), device="cuda"), seed + 2, -s, s)
    b = pt.fill_uniform(torch.empty((g.K,), device="cuda"), seed + 3, -0.1, 0.1)
    gy = pt.fill_uniform(torch.empty(G.output_shape(), device="cuda"), seed + 4)
    return G, x, w, b, gy


@pytest.mark.parametrize("name", list(FULL))
def test_fullsize_fwd_dgrad_batched_equals_per_image(name):
    pt = _pt()
    g = FULL[name]
    G, x, w, b, gy = _dev_inputs(g, 0x5EED)
    y = pt.conv_forward(G, x, w, b)
    gx, gw, gb = pt.conv_backward(G, x, gy, w)
    G1 = _G(with_batch(g, 1))
    for n in (0, g.N - 1):
        y1 = pt.conv_forward(G1, x[n:n + 1].contiguous(), w, b)
        gx1 = pt.conv_backward_input(G1, gy[n:n + 1].contiguous(), w)
        torch.cuda.synchronize()
        assert torch.equal(y[n:n + 1], y1), f"{name}: fwd image {n} differs from per-image run"
        assert torch.equal(gx[n:n + 1], gx1), f"{name}: dgrad image {n} differs"
        g1 = with_batch(g, 1)
        xn = x[n:n + 1].cpu().numpy()
        gyn = gy[n:n + 1].cpu().numpy()
        wn, bn = w.cpu().numpy(), b.cpu().numpy()
        tol = tf32_bounds(g1, xn, wn, bn, gyn)
        check_tf32(y1.cpu().numpy(), po.conv_forward(g1, xn, wn, bn), f"{name} fwd[{n}]", tol["fwd"])
        check_tf32(gx1.cpu().numpy(), po.conv_backward_input(g1, gyn, wn), f"{name} dgrad[{n}]",
                   tol["dgrad"])


@pytest.mark.parametrize("name", list(FULL))
def test_fullsize_wgrad_is_sum_over_batch(name):
    pt = _pt()
    g = FULL[name]
    G, x, w, b, gy = _dev_inputs(g, 0xBEEF)
    _, gw, gb = pt.conv_backward(G, x, gy, w, need_input_grad=False)
    q = g.N // 4
    Gq = _G(with_batch(g, q))
    acc_w = torch.zeros_like(gw)
    acc_b = torch.zeros_like(gb)
    for i in range(4):
        pt.conv_backward_weight(Gq, x[i * q:(i + 1) * q].contiguous(),
                                gy[i * q:(i + 1) * q].contiguous(), acc_w, acc_b, accumulate=True)
        if i == 0:
            gw0 = acc_w.clone()
            gb0 = acc_b.clone()
    # both sides are TF32 results of the same sum split differently: twice the bound
    h = lambda t: t.cpu().numpy()  # noqa: E731
    hx, hgy = h(x), h(gy)
    tol = tf32_bounds(g, hx, None, None, hgy, passes=("wgrad",))
    check_tf32(h(gw), h(acc_w), f"{name} wgrad split", 2 * tol["wgrad"])
    np.testing.assert_allclose(gb.cpu().numpy(), acc_b.cpu().numpy(), rtol=1e-4, atol=1e-2)
    # one image of the first quarter against the oracle (cheap), via a 1-image device run
    g1 = with_batch(g, 1)
    gw1, gb1 = pt.conv_backward_weight(_G(g1), x[:1].contiguous(), gy[:1].contiguous())
    x1, gy1 = x[:1].cpu().numpy(), gy[:1].cpu().numpy()
    rgw, rgb = po.conv_backward_weight(g1, x1, gy1)
    tol1 = tf32_bounds(g1, x1, None, None, gy1, passes=("wgrad",))
    check_tf32(gw1.cpu().numpy(), rgw, f"{name} wgrad[0]", tol1["wgrad"])
    np.testing.assert_allclose(gb1.cpu().numpy(), rgb, rtol=1e-4, atol=1e-3)
    del gw0, gb0


@pytest.mark.parametrize("name", ["convnet-L2", "convnet-L5", "vgga-c6"])
def test_fullsize_forward_linear_in_weights(name):
    pt = _pt()
    g = FULL[name]
    G, x, w, b, _ = _dev_inputs(g, 7)
    w2 = pt.fill_uniform(torch.empty_like(w), 99, -0.01, 0.01)
    y1 = pt.conv_forward(G, x, w, None)
    y2 = pt.conv_forward(G, x, w2, None)
    y12 = pt.conv_forward(G, x, 2.0 * w - 3.0 * w2, None)
    check_tf32(y12.cpu().numpy(), (2.0 * y1 - 3.0 * y2).cpu().numpy(), f"{name} linearity")
