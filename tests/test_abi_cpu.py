"""CPU: the C-ABI library loads and exports every symbol include/pt_b200.h declares;
host-side validation, error mapping and planning work without a GPU; the host
expression compiler matches the reference's grammar and error classes."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1606_04884_b200 as pt
from paper_1606_04884_b200 import _lib
from paper_1606_04884_b200.backend import BackendDescriptor, choose_launch
from paper_1606_04884_b200.expr import parse

import pyoracle as po

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "pt_b200.h")).read()
    return sorted(set(re.findall(r"\b(pt_b200_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = pt.lib()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), f"libpt_b200.so does not export {s}"
    assert set(syms) <= set(_lib.EXPORTED)


def test_abi_version_and_no_device_here():
    assert pt.lib().pt_b200_abi_version() == 1
    # no GPU in the CI container: count is 0, never an error
    assert pt.lib().pt_b200_device_count() >= 0


def test_validation_errors_map_to_reference_classes():
    g = _lib.PtConvGeom(1, 1, 3, 3, 1, 5, 5, 0, 0, 1, 1)  # kernel exceeds padded input
    st = pt.lib().pt_b200_conv_validate(C.byref(g))
    assert st == _lib.PT_EVALIDATION
    assert "kernel exceeds padded input" in pt.lib().pt_b200_last_error().decode()
    with pytest.raises(pt.ValidationError):
        _lib.check(st)
    # null tensors are validation errors, reported before any device work
    g = _lib.PtConvGeom(1, 1, 3, 3, 1, 3, 3, 1, 1, 1, 1)
    assert pt.lib().pt_b200_conv_fwd(C.byref(g), None, None, None, None, 0, None, 0, None) == 2
    assert pt.lib().pt_b200_conv_fwd(C.byref(g), 16, 16, None, 16, 7, None, 0, None) == 2


@pytest.mark.parametrize("op", [0, 1, 2, 3])
def test_workspace_query_is_host_only(op):
    for name, g in [("L1", (128, 3, 128, 128, 96, 11, 11, 0, 0, 1, 1)),
                    ("L5", (128, 384, 13, 13, 384, 3, 3, 0, 0, 1, 1)),
                    ("alex1", (128, 3, 224, 224, 64, 11, 11, 2, 2, 4, 4))]:
        gg = pt.ConvGeometry(*g)
        for m in ("tf32", "fp32"):
            n = pt.conv.workspace_bytes(gg, op, m)
            assert 0 <= n < 64 << 30, (name, op, m, n)


def test_geometry_mirror():
    g = pt.ConvGeometry(16, 3, 32, 32, 64, 3, 3, 1, 1, 1, 1)
    assert (g.outHeight(), g.outWidth(), g.patchSize(), g.outSpatial()) == (32, 32, 27, 1024)
    assert g.toString() == "N16 C3 H32 W32 K64 k3x3 p1x1 s1x1"
    g.validate()
    with pytest.raises(pt.ValidationError):
        pt.ConvGeometry(1, 1, 3, 3, 1, 3, 3, -1, 0).validate()


@pytest.mark.parametrize("n,maxwg", [(1, 256), (1000, 256), (257, 1024), (5, 64), (1 << 30, 1)])
def test_choose_launch_matches_reference(n, maxwg):
    lc = choose_launch(n, BackendDescriptor("b200:0", maxwg, 0))
    if po.ref_available():
        st, glob, wg, _ = po.ref_choose_launch(n, maxwg)
        assert st == 0 and (glob, wg) == (lc.globalSize, lc.workgroupSize)


EXPRS_OK = ["x = x + s", "x = s", "x=x*2", "x = max(x, y) * 2.5 - z / 4", "x = -(-x)",
            "x = tanh(exp(log(sqrt(abs(x)))))", "x = min(x, .5e1) + 1e-3", "x = ((x))",
            "x = x - y - z", "x = 2 * -y"]
EXPRS_BAD = [("y = x", 1), ("x + 1", 1), ("x = w", 1), ("x = y", 1), ("x = max(x)", 1),
             ("x = (x", 1), ("x = x +", 1), ("x = x $ 2", 1), ("x = 1.2.3", 1), ("x = x x", 1),
             ("x = foo(x)", 1), ("x = sqrt x", 1)]


@pytest.mark.parametrize("text", EXPRS_OK)
def test_expression_accepts_like_reference(text):
    prog = parse(text, 3)
    assert prog.code
    if po.ref_available():
        st, _ = po.ref_parse_expr(text, 3)
        assert st == 0


@pytest.mark.parametrize("text,arity", EXPRS_BAD)
def test_expression_rejects_like_reference(text, arity):
    with pytest.raises(pt.ValidationError) as ei:
        parse(text, arity)
    if po.ref_available():
        st, msg = po.ref_parse_expr(text, arity)
        assert st == 2
        assert str(ei.value) == msg


def test_expression_depth_limit():
    deep = "x = " + "(" * 10 + "+".join(["x"] * 40) + ")" * 10
    parse(deep, 1)  # left-assoc sums keep the stack shallow
    nested = "x = " + "+".join(["(x*" * 1 + "x)"] * 2)
    parse(nested, 1)
    very = "x = " + "".join(f"x*(" for _ in range(33)) + "x" + ")" * 33
    with pytest.raises(pt.ValidationError):
        parse(very, 1)


# ---- the library's expression compiler (csrc/exprc.cpp) against the reference's parser ----
_TOKS = ["x", "y", "z", "s", "1", "2.5", ".5e1", "1e-3", "+", "-", "*", "/", "(", ")", ",", "abs",
         "max", "min", "tanh", "exp", "log", "sqrt", "w", "foo", "$", "1.2.3", "=", "1e", "3.", "e5"]


def _gen(rng, d):
    if d <= 0:
        return str(rng.choice(["x", "y", "z", "s", "1", "2.5", ".5e1", "7e-2"]))
    r = rng.random()
    if r < 0.3:
        return _gen(rng, d - 1) + str(rng.choice([" + ", " - ", " * ", " / "])) + _gen(rng, d - 1)
    if r < 0.4:
        return "-" + _gen(rng, d - 1)
    if r < 0.5:
        return "(" + _gen(rng, d - 1) + ")"
    if r < 0.7:
        return str(rng.choice(["abs", "exp", "log", "sqrt", "tanh"])) + "(" + _gen(rng, d - 1) + ")"
    if r < 0.85:
        return str(rng.choice(["max", "min"])) + "(" + _gen(rng, d - 1) + ", " + _gen(rng, d - 1) + ")"
    return _gen(rng, d - 1)


@pytest.mark.skipif(not po.ref_available(), reason="reference not built (oracle/_ref)")
@pytest.mark.parametrize("seed", range(4))
def test_expression_compiler_fuzz_vs_reference(seed):
    """Token soup and well-formed expressions: accept/reject, the exact error message and
    the canonical kernel statement all equal the reference parser's (expression.cpp)."""
    rng = np.random.default_rng(seed)
    cases = []
    for _ in range(4000):
        head = str(rng.choice(["x = ", "x = ", "x = ", "y = ", "x ", "x = x ", "", "x=", "$"]))
        body = " ".join(str(rng.choice(_TOKS)) for _ in range(int(rng.integers(1, 12))))
        cases.append((head + body, int(rng.integers(1, 4))))
    cases += [("x = " + _gen(rng, int(rng.integers(0, 9))), 3) for _ in range(1500)]
    for text, arity in cases:
        st, msg = po.ref_parse_expr(text, arity)
        try:
            prog = parse(text, arity)
            got = (0, prog.statement)
        except pt.ValidationError as ex:
            got = (2, str(ex))
        assert got == (st, msg), f"{text!r} (arity {arity}): library {got} vs reference {(st, msg)}"


@pytest.mark.skipif(not po.ref_available(), reason="reference not built (oracle/_ref)")
def test_expression_bytecode_evaluates_like_reference():
    """The compiled bytecode, evaluated by the oracle's stack machine, equals the
    reference backend's dispatch_apply of the same text on the same data bitwise."""
    rng = np.random.default_rng(99)
    for i in range(300):
        text = "x = " + _gen(rng, int(rng.integers(1, 7)))
        shape = (3, 5)
        bases = [po.uniform(shape, 10 * i + t, 0.1, 2.0).ravel().copy() for t in range(3)]
        ref_bases = [b.copy() for b in bases]
        st, err = po.ref_apply(text, ref_bases, [shape] * 3, [[]] * 3, 0.75)
        assert st == 0, err
        view = ((3, 5), (5, 1), 0)
        po.apply(parse(text, 3).code, 3, bases, [view] * 3, 0.75)
        np.testing.assert_array_equal(bases[0].view(np.uint32), ref_bases[0].view(np.uint32),
                                      err_msg=text)


@pytest.mark.skipif(not po.refdev_available(), reason="integration/_ref not built")
def test_reference_device_slot_loads_without_gpu():
    """The reference's backend layer with the B200 plug-in in its device slot loads on a
    host without a GPU: the plug-in probes zero devices (not an error), so the reference's
    own select_backend("device") raises its own BackendError (backend.cpp:93-96)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by tests/test_gpu_integration.py")
    st, msg = po.ref_backend_info(po.refdev())
    assert st == 3 and msg.startswith("no device backend available"), (st, msg)
