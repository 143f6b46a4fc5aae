"""CPU: the oracle restatement pinned against the reference itself and the SPEC examples.

  * im2col: bitwise vs the reference's own rendered kernel (proj/templates/im2col.kt.tmpl)
  * apply / reduce: vs the reference's dispatch_apply / dispatch_reduce_* on
    reference_backend() (proj/src/backend.cpp:115-161) over strided / offset views
  * conv / gemm / col2im / backward: the SPEC.md:353-424 known answers and properties
    (the reference ships no conv code or tests: SURVEY.md §8c "parity unpinned" for GEMM)
"""
import numpy as np
import pytest

import pyoracle as po
from helpers import spec_random_geometries

ref_only = pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref not built")


# ---------------------------------------------------------------- reference-pinned
IM2COL_GEOMS = [
    po.geom(1, 3, 32, 32, 64, 3, 3, 1, 1, 1, 1),      # cfg1 (unrolled taps, pad guard)
    po.geom(1, 3, 20, 20, 8, 11, 11, 0, 0, 1, 1),     # L1-like: rolled loops (121 taps), no pad
    po.geom(1, 2, 9, 7, 4, 5, 3, 2, 1, 2, 3),         # rectangular, stride, asymmetric pad
    po.geom(1, 4, 15, 15, 4, 11, 11, 2, 2, 4, 4),     # AlexNet c1-like (stride 4, pad 2)
    po.geom(1, 1, 3, 3, 1, 3, 3, 1, 1, 1, 1),
]


@ref_only
@pytest.mark.parametrize("g", IM2COL_GEOMS)
def test_im2col_bitwise_vs_reference_kernel(g):
    from ref_kernels import ref_im2col
    img = po.uniform((g.C, g.H, g.W), 1000 + g.kH)
    np.testing.assert_array_equal(po.im2col(g, img), ref_im2col(g, img))


@ref_only
def test_reference_defect_d1_gen_im2col_throws():
    """the shipped gen_im2col_kernel throws at render time."""
    st, msg = po.ref_gen_im2col_kernel(po.geom(16, 3, 32, 32, 64, 3, 3, 1, 1, 1, 1))
    assert st == 2 and "non-boolean value 'unrolled'" in msg


def _view_from_ops(shape, ops):
    """sizes/strides/offset after narrow/select ops (proj/src/tensor.cpp:118-145)."""
    sizes = list(shape)
    strides = [int(np.prod(shape[d + 1:])) for d in range(len(shape))]
    off = 0
    for op in ops:
        if op[0] == "narrow":
            _, d, start, ln = op
            off += start * strides[d]
            sizes[d] = ln
        else:
            _, d, idx = op
            off += idx * strides[d]
            del sizes[d]
            del strides[d]
    return sizes, strides, off


def random_view(rng, max_rank=4):
    rank = int(rng.integers(1, max_rank + 1))
    shape = [int(rng.integers(1, 6)) for _ in range(rank)]
    ops = []
    cur = list(shape)
    for _ in range(int(rng.integers(0, 3))):
        d = int(rng.integers(0, len(cur)))
        if rng.random() < 0.5 or len(cur) == 1:
            start = int(rng.integers(0, cur[d]))
            ln = int(rng.integers(1, cur[d] - start + 1))
            ops.append(("narrow", d, start, ln))
            cur[d] = ln
        else:
            ops.append(("select", d, int(rng.integers(0, cur[d]))))
            del cur[d]
    return shape, ops


EXPRS = [("x = x + s", 1), ("x = s", 1), ("x = x * s", 1), ("x = y", 2), ("x = x + y", 2),
         ("x = max(x, y) * 2.5 - z / 4", 3), ("x = -x + abs(y)", 2), ("x = min(x, 0.5)", 1),
         ("x = x * y + z", 3), ("x = (x - s) / 3", 1)]


def compile_expr(text, arity):
    """Test-side RPN compiler for the reference grammar (expression.cpp:158-334)."""
    from paper_1606_04884_b200.expr import compile_expression
    return compile_expression(text, arity)


@ref_only
@pytest.mark.parametrize("seed", range(100))
def test_apply_oracle_vs_reference_backend(seed):
    """SPEC acceptance 8: apply on strided/offset views equals the reference, exactly."""
    rng = np.random.default_rng(seed)
    text, arity = EXPRS[seed % len(EXPRS)]
    shape, ops = random_view(rng)
    sizes, strides, off = _view_from_ops(shape, ops)
    bases, views, shapes, vops = [], [], [], []
    for t in range(arity):
        # operands share sizes: same view chain over same-shaped storages
        bases.append(po.uniform(shape, 100 * seed + t).ravel().copy())
        views.append((sizes, strides, off))
        shapes.append(shape)
        vops.append(ops)
    ref_bases = [b.copy() for b in bases]
    st, err = po.ref_apply(text, ref_bases, shapes, vops, 1.75)
    assert st == 0, err
    po.apply(compile_expr(text, arity), arity, bases, views, 1.75)
    np.testing.assert_array_equal(bases[0], ref_bases[0])


@ref_only
@pytest.mark.parametrize("seed", range(60))
def test_reduce_oracle_vs_reference_backend(seed):
    rng = np.random.default_rng(1000 + seed)
    shape, ops = random_view(rng)
    sizes, strides, off = _view_from_ops(shape, ops)
    base = po.uniform(shape, 7 + seed).ravel().copy()
    op = seed % 3
    st, rv, err = po.ref_reduce_all(op, base, shape, ops)
    assert st == 0, err
    assert po.reduce_all(op, base, sizes, strides, off) == rv  # same sequential order
    dim = int(rng.integers(0, len(sizes)))
    out_n = int(np.prod(sizes)) // sizes[dim]
    st, rd, err = po.ref_reduce_dim(op, base, shape, ops, dim, out_n)
    assert st == 0, err
    np.testing.assert_array_equal(po.reduce_dim(op, base, sizes, strides, off, dim).ravel(), rd)


@ref_only
@pytest.mark.parametrize("seed", range(40))
def test_geometry_validation_matches_reference(seed):
    """conv_geometry.hpp:53-63 — same accept/reject as the reference, incl. invalid ones."""
    rng = np.random.default_rng(seed)
    vals = [int(v) for v in rng.integers(-1, 7, size=11)]
    g = po.geom(*vals)
    st, _ = po.ref_geom_validate(g)
    assert (po.oracle().or_validate(g) == 0) == (st == 0)
    import paper_1606_04884_b200 as pt
    import ctypes as C
    gc = pt._lib.PtConvGeom(*vals)
    assert (pt.lib().pt_b200_conv_validate(C.byref(gc)) == 0) == (st == 0)


# ---------------------------------------------------------------- SPEC known answers
def test_conv_direct_ones_kat():
    """3x3 ones on 3x3 ones, pad 1 -> center 9, edges 6, corners 4."""
    g = po.geom(1, 1, 3, 3, 1, 3, 3, 1, 1, 1, 1)
    y = po.conv_direct(g, np.ones((1, 1, 3, 3), np.float32), np.ones((1, 1, 3, 3), np.float32))
    np.testing.assert_array_equal(y[0, 0], [[4, 6, 4], [6, 9, 6], [4, 6, 4]])


def test_identity_kernel_kat():
    """SPEC.md:359-360 and :368."""
    g = po.geom(2, 1, 4, 5, 1, 1, 1)
    x = po.uniform((2, 1, 4, 5), 3)
    np.testing.assert_array_equal(po.conv_direct(g, x, np.ones((1, 1, 1, 1), np.float32)), x)
    np.testing.assert_array_equal(po.im2col(po.geom(1, 1, 4, 5, 1, 1, 1), x[0]), x[0].reshape(1, 20))


def test_im2col_kats():
    """SPEC.md:369-370."""
    g = po.geom(1, 1, 2, 2, 1, 2, 2)
    img = np.array([[[1, 2], [3, 4]]], np.float32)
    np.testing.assert_array_equal(po.im2col(g, img), [[1], [2], [3], [4]])
    g = po.geom(1, 1, 3, 3, 1, 3, 3, 1, 1, 1, 1)
    col = po.im2col(g, po.uniform((1, 3, 3), 9, 1.0, 2.0))
    assert col.shape == (9, 9)
    assert (col[:, 0] == 0).sum() == 5


def test_col2im_kats():
    """SPEC.md:377-379."""
    g = po.geom(1, 1, 3, 3, 1, 3, 3, 1, 1, 1, 1)
    img = po.col2im(g, np.ones((9, 9), np.float32))
    assert img[0, 1, 1] == 9
    np.testing.assert_array_equal(po.col2im(g, np.zeros((9, 9), np.float32)), 0)
    g1 = po.geom(1, 2, 3, 4, 1, 1, 1)
    x = po.uniform((2, 3, 4), 4)
    np.testing.assert_array_equal(po.col2im(g1, po.im2col(g1, x)), x)


def test_gemm_kats_and_tiled_equals_naive():
    """SPEC.md:386-388 and acceptance 5 (25 shapes incl. off-tile 129x129)."""
    B = po.uniform((3, 5), 1)
    Cm = np.full((3, 5), 7.0, np.float32)
    np.testing.assert_array_equal(po.gemm(np.eye(3, dtype=np.float32), B, Cm.copy()), B)
    np.testing.assert_array_equal(po.gemm(np.eye(3, dtype=np.float32), B, Cm.copy(), alpha=0.0,
                                          beta=1.0), Cm)
    rng = np.random.default_rng(5)
    shapes = [(17, 13, 9), (129, 129, 129), (1, 1, 1), (64, 300, 7)]
    while len(shapes) < 25:
        shapes.append(tuple(int(v) for v in rng.integers(1, 140, size=3)))
    for i, (M, K, N) in enumerate(shapes):
        ta, tb = i % 2, (i // 2) % 2
        A = po.uniform((K, M) if ta else (M, K), 10 + i)
        Bm = po.uniform((N, K) if tb else (K, N), 50 + i)
        c0 = po.uniform((M, N), 90 + i)
        naive = po.gemm(A, Bm, c0.copy(), ta, tb, 1.5, 0.5)
        tiled = po.gemm(A, Bm, c0.copy(), ta, tb, 1.5, 0.5, blocked=True)
        np.testing.assert_allclose(tiled, naive, rtol=1e-5, atol=1e-5 * max(1, K))


@pytest.mark.parametrize("g", spec_random_geometries(50, seed=77))
def test_im2col_forward_equals_direct(g):
    """SPEC.md:392 / acceptance 1: <= 1e-4 relative vs conv_direct."""
    x = po.uniform((g.N, g.C, g.H, g.W), 1)
    w = po.uniform((g.K, g.C, g.kH, g.kW), 2)
    b = po.uniform((g.K,), 3)
    y = po.conv_forward(g, x, w, b)
    r = po.conv_direct(g, x, w, b, f64=True)
    assert np.linalg.norm(y - r) <= 1e-4 * max(np.linalg.norm(r), 1e-12)


@pytest.mark.parametrize("g", spec_random_geometries(10, seed=78))
def test_batched_equals_unbatched_bitwise(g):
    """SPEC.md:401, acceptance 2: chunk sizes {1, 2, N}."""
    x = po.uniform((g.N, g.C, g.H, g.W), 1)
    w = po.uniform((g.K, g.C, g.kH, g.kW), 2)
    y1 = po.conv_forward(g, x, w, None, chunk=1)
    for chunk in (2, g.N):
        np.testing.assert_array_equal(po.conv_forward(g, x, w, None, chunk=chunk), y1)


@pytest.mark.parametrize("i", range(20))
def test_im2col_col2im_adjoint(i):
    """SPEC.md:437, acceptance 4: <im2col(x), y> = <x, col2im(y)>."""
    g = spec_random_geometries(20, seed=79)[i]
    x = po.uniform((g.C, g.H, g.W), i)
    oh, ow = po.out_hw(g)
    y = po.uniform((g.C * g.kH * g.kW, oh * ow), 100 + i)
    a = float(np.dot(po.im2col(g, x).ravel().astype(np.float64), y.ravel()))
    b = float(np.dot(x.ravel().astype(np.float64), po.col2im(g, y).ravel()))
    assert abs(a - b) <= 1e-4 * max(abs(a), 1e-6)


FD_GEOMS = [po.geom(1, 2, 5, 5, 3, 3, 3, 1, 1, 1, 1), po.geom(1, 1, 4, 4, 2, 2, 2, 0, 0, 1, 1),
            po.geom(1, 2, 6, 5, 2, 3, 1, 1, 0, 2, 1), po.geom(2, 1, 5, 5, 1, 3, 3, 2, 2, 2, 2),
            po.geom(1, 3, 4, 4, 2, 1, 1, 0, 0, 1, 1)]


@pytest.mark.parametrize("g", FD_GEOMS)
def test_finite_difference_gradients(g):
    """SPEC.md:422, acceptance 3: |analytic - central difference| <= 1e-2 at step 1e-2."""
    x = po.uniform((g.N, g.C, g.H, g.W), 1)
    w = po.uniform((g.K, g.C, g.kH, g.kW), 2)
    oh, ow = po.out_hw(g)
    gy = po.uniform((g.N, g.K, oh, ow), 3)
    gx = po.conv_backward_input(g, gy, w)
    gw, gb = po.conv_backward_weight(g, x, gy)

    def loss(xx, ww, bb):
        return float(np.sum(po.conv_direct(g, xx, ww, bb, f64=True).astype(np.float64) * gy))

    b0 = np.zeros((g.K,), np.float32)
    h = 1e-2
    for arr, grad in ((x, gx), (w, gw)):
        for idx in list(np.ndindex(arr.shape))[:12]:
            p, m = arr.copy(), arr.copy()
            p[idx] += h
            m[idx] -= h
            if arr is x:
                fd = (loss(p, w, b0) - loss(m, w, b0)) / (2 * h)
            else:
                fd = (loss(x, p, b0) - loss(x, m, b0)) / (2 * h)
            assert abs(fd - grad[idx]) <= 1e-2
    for k in range(g.K):
        p, m = b0.copy(), b0.copy()
        p[k] += h
        m[k] -= h
        assert abs((loss(x, w, p) - loss(x, w, m)) / (2 * h) - gb[k]) <= 1e-2


def test_zero_grad_output_gives_zero_grads():
    """SPEC.md:423."""
    g = po.geom(2, 3, 6, 6, 4, 3, 3, 1, 1, 1, 1)
    x = po.uniform((2, 3, 6, 6), 1)
    w = po.uniform((4, 3, 3, 3), 2)
    gy = np.zeros((2, 4, 6, 6), np.float32)
    assert not po.conv_backward_input(g, gy, w).any()
    gw, gb = po.conv_backward_weight(g, x, gy)
    assert not gw.any() and not gb.any()


def test_1x1_grad_weight_closed_form():
    """gradWeight[k,c] = sum input[c] * gradOutput[k] over positions."""
    g = po.geom(2, 3, 4, 5, 2, 1, 1)
    x = po.uniform((2, 3, 4, 5), 1)
    gy = po.uniform((2, 2, 4, 5), 2)
    gw, _ = po.conv_backward_weight(g, x, gy)
    ref = np.einsum("nchw,nkhw->kc", x.astype(np.float64), gy.astype(np.float64))
    np.testing.assert_allclose(gw[:, :, 0, 0], ref, rtol=1e-5, atol=1e-5)


def test_fill_uniform_is_counter_based():
    a = po.uniform((1000,), 42)
    np.testing.assert_array_equal(a[500:], po.uniform((1000,), 42)[500:])
    assert -1.0 <= a.min() and a.max() < 1.0
