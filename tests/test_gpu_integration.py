"""GPU: the drop-in boundary, proven from the REFERENCE's side.

integration/_ref/libportten_refdev.so is the reference's own backend layer
(proj/src/backend.cpp, tensor.cpp, reference_backend.cpp, expression.cpp, ... compiled in
place with its device slot PORTTEN_HAVE_OPENCL enabled) whose slot function
opencl_probe_devices() is integration/b200_backend.cpp: a B200Backend deriving from the
reference's portten::Backend over the libpt_b200 C ABI. The tests call the reference's
select_backend("device"), dispatch_apply, dispatch_reduce_all / _dim, device_upload /
device_download (backend.cpp:78-181) through oracle/ref_shim.cpp, and compare with the same
calls on the reference's host interpreter (oracle/_ref): SPEC acceptance 10 ("criteria 1, 8
re-run on the device backend with identical tolerances").
"""
import numpy as np
import pytest

import pyoracle as po
from test_oracle import EXPRS, _view_from_ops, random_view

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (po.refdev_available() and po.ref_available()),
                                 reason="integration/_ref or oracle/_ref not built")]

# transcendental functions may differ by an ulp between the device and the host libm
EXPRS_FN = [("x = tanh(x) + exp(y) * log(abs(z) + 1)", 3), ("x = sqrt(abs(x)) - min(y, 0.25)", 2),
            ("x = -max(x, s) / 3", 1)]


def test_device_slot_filled_by_b200():
    st, info = po.ref_backend_info(po.refdev())
    assert st == 0, info
    sel, names = info.split(";", 1)
    assert sel.startswith("b200:") and sel.endswith(" device"), info
    assert names.split(";")[0] == "reference" and any(n.startswith("b200:") for n in names.split(";")), info


def _operands(rng, seed, arity):
    shape, ops = random_view(rng)
    bases = [po.uniform(shape, 100 * seed + t, 0.05, 2.0).ravel().copy() for t in range(arity)]
    return shape, ops, bases


@pytest.mark.parametrize("seed", range(60))
def test_reference_dispatch_apply_on_b200(seed):
    """dispatch_apply through the reference's backend layer onto the B200 plug-in equals the
    reference's host interpreter on strided / offset views (exactly for + - * / max min abs,
    SPEC acceptance 8)."""
    rng = np.random.default_rng(seed)
    exact = seed % 4 != 3
    text, arity = EXPRS[seed % len(EXPRS)] if exact else EXPRS_FN[seed % len(EXPRS_FN)]
    shape, ops, bases = _operands(rng, seed, arity)
    host = [b.copy() for b in bases]
    dev = [b.copy() for b in bases]
    st, err = po.ref_apply(text, host, [shape] * arity, [ops] * arity, 1.75)
    assert st == 0, err
    st, err = po.ref_apply(text, dev, [shape] * arity, [ops] * arity, 1.75, lib=po.refdev())
    assert st == 0, err
    if exact:
        np.testing.assert_array_equal(dev[0], host[0])
    else:
        np.testing.assert_allclose(dev[0], host[0], rtol=2e-6, atol=1e-7)
    for t in range(1, arity):  # inputs untouched
        np.testing.assert_array_equal(dev[t], bases[t])


@pytest.mark.parametrize("seed", range(30))
def test_reference_dispatch_reduce_on_b200(seed):
    rng = np.random.default_rng(500 + seed)
    shape, ops = random_view(rng)
    sizes, strides, off = _view_from_ops(shape, ops)
    base = po.uniform(shape, 9 + seed).ravel().copy()
    op = seed % 3
    st, hv, err = po.ref_reduce_all(op, base, shape, ops)
    assert st == 0, err
    st, dv, err = po.ref_reduce_all(op, base, shape, ops, lib=po.refdev())
    assert st == 0, err
    assert abs(dv - hv) <= 1e-5 * max(1.0, abs(hv)), (dv, hv)
    dim = int(rng.integers(0, len(sizes)))
    out_n = int(np.prod(sizes)) // sizes[dim]
    st, hd, err = po.ref_reduce_dim(op, base, shape, ops, dim, out_n)
    assert st == 0, err
    st, dd, err = po.ref_reduce_dim(op, base, shape, ops, dim, out_n, lib=po.refdev())
    assert st == 0, err
    np.testing.assert_allclose(dd, hd, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("seed", range(10))
def test_reference_upload_download_roundtrip_on_b200(seed):
    """device_upload / device_download through the plug-in: bitwise identity."""
    rng = np.random.default_rng(900 + seed)
    shape, ops = random_view(rng)
    sizes, _, _ = _view_from_ops(shape, ops)
    base = po.uniform(shape, 77 + seed).ravel().copy()
    n = int(np.prod(sizes))
    st, out, err = po.ref_roundtrip(base, shape, ops, n, lib=po.refdev())
    assert st == 0, err
    st, ref_out, err = po.ref_roundtrip(base, shape, ops, n)
    assert st == 0, err
    np.testing.assert_array_equal(out.view(np.uint32), ref_out.view(np.uint32))


@pytest.mark.parametrize("text,arity", [("x = w", 1), ("x = y", 1), ("x = (x", 1), ("x = x $ 2", 1)])
def test_reference_validation_errors_identical_on_b200(text, arity):
    """Bad expressions fail with the same error class and message on either backend."""
    shape = (2, 3)
    bases = [po.uniform(shape, 5).ravel().copy() for _ in range(arity)]
    h = po.ref_apply(text, [b.copy() for b in bases], [shape] * arity, [[]] * arity, 1.0)
    d = po.ref_apply(text, [b.copy() for b in bases], [shape] * arity, [[]] * arity, 1.0,
                     lib=po.refdev())
    assert h[0] == 2 and d == h, (h, d)
