"""GPU parity of the standalone ops on the conv path, through the C ABI:
im2col / col2im (bitwise), SPEC gemm, pointwise apply (exact) and reduce (1e-5),
against the committed golden fixtures made from the reference itself and the oracle."""
import json
import os

import numpy as np
import pytest

import pyoracle as po
from helpers import gstr, spec_random_geometries

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _pt():
    import paper_1606_04884_b200 as pt
    return pt


def _G(g):
    return _pt().ConvGeometry(g.N, g.C, g.H, g.W, g.K, g.kH, g.kW, g.padH, g.padW, g.strideH,
                              g.strideW)


def _d(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _h(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def test_im2col_bitwise_vs_reference_golden():
    """Device unfold == the reference's own rendered OpenCL im2col kernel, bit for bit."""
    z = np.load(os.path.join(GOLD, "im2col_ref.npz"))
    for i, gk in enumerate(z["geoms"]):
        g = po.geom(*[int(v) for v in gk])
        col = _pt().im2col(_G(g), _d(z[f"img{i}"]))
        np.testing.assert_array_equal(_h(col), z[f"col{i}"])


@pytest.mark.parametrize("g", spec_random_geometries(20, seed=11), ids=gstr)
def test_im2col_col2im_bitwise_vs_oracle(g):
    pt = _pt()
    img = po.uniform((g.C, g.H, g.W), 3)
    np.testing.assert_array_equal(_h(pt.im2col(_G(g), _d(img))), po.im2col(g, img))
    oh, ow = po.out_hw(g)
    col = po.uniform((g.C * g.kH * g.kW, oh * ow), 4)
    np.testing.assert_array_equal(_h(pt.col2im(_G(g), _d(col))), po.col2im(g, col))


def test_im2col_batched_is_chunk_of_per_image():
    pt = _pt()
    g = po.geom(5, 3, 9, 8, 4, 3, 3, 1, 1, 2, 1)
    x = po.uniform((5, 3, 9, 8), 8)
    oh, ow = po.out_hw(g)
    col = _h(pt.im2col_batched(_G(g), _d(x), 1, 3))
    for t in range(3):
        np.testing.assert_array_equal(col[:, t * oh * ow:(t + 1) * oh * ow],
                                      po.im2col(g, x[1 + t]))
    with pytest.raises(pt.ValidationError):
        pt.im2col_batched(_G(g), _d(x), 4, 2)


@pytest.mark.parametrize("shape", [(17, 13, 9), (129, 129, 129), (1, 1, 1), (64, 300, 7), (5, 200, 33)])
@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_gemm_vs_oracle(shape, ta, tb):
    """SPEC.md:380-388 gemm on device, <= 1e-5 relative vs the naive oracle."""
    pt = _pt()
    M, K, N = shape
    A = po.uniform((K, M) if ta else (M, K), 1)
    B = po.uniform((N, K) if tb else (K, N), 2)
    c0 = po.uniform((M, N), 3)
    ref = po.gemm(A, B, c0.copy(), ta, tb, 1.25, -0.5)
    out = _h(pt.gemm(_d(A), _d(B), _d(c0), bool(ta), bool(tb), 1.25, -0.5))
    np.testing.assert_allclose(out, ref, rtol=1e-5, atol=2e-6 * K)


def _cases():
    with open(os.path.join(GOLD, "apply_reduce_ref.json")) as f:
        return json.load(f)


def _strided(storage: np.ndarray, sizes, strides, offset):
    t = _d(storage)
    return t.as_strided(sizes, strides, offset)


@pytest.mark.parametrize("case", [c for c in _cases() if c["kind"] == "apply"],
                         ids=lambda c: f"apply{c['id']}")
def test_apply_vs_reference_golden(case):
    """dispatch_apply on device == the reference backend, exactly, on strided/offset views."""
    from paper_1606_04884_b200.backend import dispatch_apply
    z = np.load(os.path.join(GOLD, "apply_reduce_ref.npz"))
    c = case["id"]
    stores = [_d(z[f"a{c}_in{t}"]) for t in range(case["arity"])]
    views = [s.as_strided(case["sizes"], case["strides"], case["offset"]) for s in stores]
    dispatch_apply(case["expr"], views, case["scalar"])
    np.testing.assert_array_equal(_h(stores[0]), z[f"a{c}_out"])


@pytest.mark.parametrize("case", [c for c in _cases() if c["kind"] == "reduce"],
                         ids=lambda c: f"reduce{c['id']}")
def test_reduce_vs_reference_golden(case):
    """Device tree reduce vs the reference's sequential fold: <= 1e-5 relative."""
    from paper_1606_04884_b200.backend import dispatch_reduce_all, dispatch_reduce_dim
    z = np.load(os.path.join(GOLD, "apply_reduce_ref.npz"))
    c = case["id"]
    v = _d(z[f"r{c}_in"]).as_strided(case["sizes"], case["strides"], case["offset"])
    ref_all = float(z[f"r{c}_all"][0])
    got = dispatch_reduce_all(case["op"], v)
    assert abs(got - ref_all) <= 1e-5 * max(1.0, abs(ref_all)) * max(1, v.numel())
    rd = _h(dispatch_reduce_dim(case["op"], v, case["dim"])).ravel()
    np.testing.assert_allclose(rd, z[f"r{c}_dim"], rtol=1e-5, atol=1e-5 * case["sizes"][case["dim"]])


def test_apply_fast_paths_and_bias_add():
    pt = _pt()
    from paper_1606_04884_b200.backend import dispatch_apply
    x = po.uniform((4, 6, 5, 7), 1)
    y = po.uniform((4, 6, 5, 7), 2)
    for expr, ref in (("x = s", np.full_like(x, 0.5)), ("x = x * s", x * np.float32(0.5)),
                      ("x = x + s", x + np.float32(0.5)), ("x = y", y), ("x = x + y", x + y)):
        tx = _d(x)
        ops = [tx, _d(y)] if "y" in expr else [tx]
        dispatch_apply(expr, ops, 0.5)
        np.testing.assert_array_equal(_h(tx), ref)
    b = po.uniform((6,), 3)
    ty = _d(x)
    pt.bias_add(ty, _d(b))
    np.testing.assert_array_equal(_h(ty), x + b[None, :, None, None])


def test_apply_validation_errors():
    pt = _pt()
    from paper_1606_04884_b200.backend import dispatch_apply
    x = _d(po.uniform((3, 4), 1))
    with pytest.raises(pt.ValidationError):
        dispatch_apply("x = y", [x])
    with pytest.raises(pt.ValidationError):
        dispatch_apply("x = x + y", [x, _d(po.uniform((4, 3), 2))])
    with pytest.raises(pt.ValidationError):
        dispatch_apply("x = x", [x, x, x, x])


def test_fill_uniform_matches_oracle_generator():
    pt = _pt()
    t = torch.empty(100003, device="cuda")
    pt.fill_uniform(t, 12345, -0.3, 0.7)
    np.testing.assert_array_equal(_h(t), po.uniform((100003,), 12345, -0.3, 0.7))
