"""Python loader for the TEST-ONLY oracle libraries.

  liboracle.so            — the C restatement (oracle/oracle.c)
  _ref/libportten_ref.so  — the reference's own proj/src compiled in place (ref_shim.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs import this module, and only as the checker or the timed CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libportten_ref.so")


class Geom(C.Structure):
    _fields_ = [(n, C.c_int64) for n in
                ("N", "C", "H", "W", "K", "kH", "kW", "padH", "padW", "strideH", "strideW")]


class View(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("sizes", C.c_int64 * 8), ("strides", C.c_int64 * 8),
                ("offset", C.c_int64)]


_F = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_o = None
_r = None


def oracle():
    global _o
    if _o is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"{ORACLE_SO} not built (make -C oracle)")
        o = C.CDLL(ORACLE_SO)
        G = C.POINTER(Geom)
        o.or_out_h.restype = o.or_out_w.restype = C.c_int64
        o.or_out_h.argtypes = o.or_out_w.argtypes = [G]
        o.or_validate.argtypes = [G]
        o.or_fill_uniform.argtypes = [_F, C.c_int64, C.c_uint64, C.c_float, C.c_float]
        o.or_conv_direct.argtypes = [G, _F, _F, C.c_void_p, _F]
        o.or_conv_direct_f64.argtypes = [G, _F, _F, C.c_void_p, _F]
        o.or_im2col.argtypes = [G, _F, _F]
        o.or_col2im.argtypes = [G, _F, _F]
        gemm_args = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_float, _F, C.c_int64,
                     _F, C.c_int64, C.c_float, _F, C.c_int64]
        o.or_gemm_naive.argtypes = gemm_args
        o.or_gemm_blocked.argtypes = gemm_args + [C.c_int]
        o.or_conv_forward.argtypes = [G, _F, _F, C.c_void_p, _F, C.c_int64, C.c_int]
        o.or_conv_backward_input.argtypes = [G, _F, _F, _F, C.c_int]
        o.or_conv_backward_weight.argtypes = [G, _F, _F, _F, C.c_void_p, C.c_float, C.c_int,
                                              C.c_int]
        o.or_reduce_all.restype = C.c_float
        o.or_reduce_all.argtypes = [C.c_int, C.c_void_p, C.POINTER(View)]
        o.or_reduce_dim.argtypes = [C.c_int, C.c_void_p, C.POINTER(View), C.c_int, _F]
        o.or_apply.argtypes = [C.POINTER(C.c_int32), C.c_int32, C.c_int, C.POINTER(C.c_void_p),
                               C.POINTER(View), C.c_float]
        o.or_version.restype = C.c_char_p
        _o = o
    return _o


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _r
    if _r is None:
        if not ref_available():
            raise RuntimeError(f"{REF_SO} not built (needs /root/reference; make -C oracle ref)")
        _r = C.CDLL(REF_SO)
    return _r


REFDEV_SO = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "integration",
                         "_ref", "libportten_refdev.so")
_rd = None


def refdev_available() -> bool:
    return os.path.exists(REFDEV_SO)


def refdev():
    """The reference's backend layer with the B200 plug-in in its device slot
    (integration/Makefile): the same ref_* entry points, run on select_backend("device")."""
    global _rd
    if _rd is None:
        if not refdev_available():
            raise RuntimeError(f"{REFDEV_SO} not built (needs /root/reference; make -C integration)")
        _rd = C.CDLL(REFDEV_SO)
    return _rd


def ref_backend_info(lib=None):
    buf = C.create_string_buffer(1024)
    st = (lib or ref()).ref_backend_info(buf, len(buf))
    return st, buf.value.decode()


def ref_roundtrip(base, base_shape, view_ops, out_elems, lib=None):
    ops = _ops_array([(0, o[1], o[2], o[3]) if o[0] == "narrow" else (1, o[1], o[2], 0)
                      for o in view_ops])
    sizes = (C.c_int64 * 8)(*base_shape)
    out = np.empty(out_elems, np.float32)
    err = C.create_string_buffer(1024)
    st = (lib or ref()).ref_roundtrip(base.ctypes.data_as(C.POINTER(C.c_float)), sizes,
                                      len(base_shape), ops, len(view_ops),
                                      out.ctypes.data_as(C.POINTER(C.c_float)), out_elems, err,
                                      len(err))
    return st, out, err.value.decode()


def geom(N, C_, H, W, K, kH, kW, padH=0, padW=0, strideH=1, strideW=1) -> Geom:
    return Geom(N, C_, H, W, K, kH, kW, padH, padW, strideH, strideW)


def out_hw(g: Geom):
    o = oracle()
    return o.or_out_h(C.byref(g)), o.or_out_w(C.byref(g))


def uniform(shape, seed, lo=-1.0, hi=1.0) -> np.ndarray:
    a = np.empty(int(np.prod(shape)), dtype=np.float32)
    oracle().or_fill_uniform(a, a.size, seed & (2**64 - 1), lo, hi)
    return a.reshape(shape)


def _bias_ptr(b):
    return None if b is None else np.ascontiguousarray(b, np.float32).ctypes.data


def conv_direct(g, x, w, b=None, f64=False):
    oh, ow = out_hw(g)
    y = np.empty((g.N, g.K, oh, ow), np.float32)
    bb = None if b is None else np.ascontiguousarray(b, np.float32)
    fn = oracle().or_conv_direct_f64 if f64 else oracle().or_conv_direct
    fn(C.byref(g), np.ascontiguousarray(x, np.float32), np.ascontiguousarray(w, np.float32),
       None if bb is None else bb.ctypes.data, y)
    return y


def conv_forward(g, x, w, b=None, chunk=1, threads=0):
    oh, ow = out_hw(g)
    y = np.empty((g.N, g.K, oh, ow), np.float32)
    bb = None if b is None else np.ascontiguousarray(b, np.float32)
    oracle().or_conv_forward(C.byref(g), np.ascontiguousarray(x, np.float32),
                             np.ascontiguousarray(w, np.float32),
                             None if bb is None else bb.ctypes.data, y, chunk, threads)
    return y


def conv_backward_input(g, gy, w, threads=0):
    gx = np.empty((g.N, g.C, g.H, g.W), np.float32)
    oracle().or_conv_backward_input(C.byref(g), np.ascontiguousarray(gy, np.float32),
                                    np.ascontiguousarray(w, np.float32), gx, threads)
    return gx


def conv_backward_weight(g, x, gy, scale=1.0, gw=None, gb=None, accumulate=False, threads=0,
                         with_bias=True):
    gw = np.zeros((g.K, g.C, g.kH, g.kW), np.float32) if gw is None else gw
    if with_bias and gb is None:
        gb = np.zeros((g.K,), np.float32)
    oracle().or_conv_backward_weight(C.byref(g), np.ascontiguousarray(x, np.float32),
                                     np.ascontiguousarray(gy, np.float32), gw,
                                     None if gb is None else gb.ctypes.data, scale,
                                     int(accumulate), threads)
    return gw, gb


def im2col(g, img):
    oh, ow = out_hw(g)
    col = np.empty((g.C * g.kH * g.kW, oh * ow), np.float32)
    oracle().or_im2col(C.byref(g), np.ascontiguousarray(img, np.float32), col)
    return col


def col2im(g, col):
    img = np.empty((g.C, g.H, g.W), np.float32)
    oracle().or_col2im(C.byref(g), np.ascontiguousarray(col, np.float32), img)
    return img


def gemm(A, B, Cm, transA=False, transB=False, alpha=1.0, beta=0.0, blocked=False, threads=0):
    M, K = (A.shape[1], A.shape[0]) if transA else A.shape
    N = B.shape[0] if transB else B.shape[1]
    args = (int(transA), int(transB), M, N, K, alpha, np.ascontiguousarray(A, np.float32),
            A.shape[1], np.ascontiguousarray(B, np.float32), B.shape[1], beta, Cm, Cm.shape[1])
    if blocked:
        oracle().or_gemm_blocked(*args, threads)
    else:
        oracle().or_gemm_naive(*args)
    return Cm


def make_view(sizes, strides, offset) -> View:
    v = View()
    v.ndim = len(sizes)
    for d, (s, st) in enumerate(zip(sizes, strides)):
        v.sizes[d] = s
        v.strides[d] = st
    v.offset = offset
    return v


def reduce_all(op, base: np.ndarray, sizes, strides, offset) -> float:
    v = make_view(sizes, strides, offset)
    return float(oracle().or_reduce_all(op, base.ctypes.data, C.byref(v)))


def reduce_dim(op, base: np.ndarray, sizes, strides, offset, dim) -> np.ndarray:
    v = make_view(sizes, strides, offset)
    out_sizes = list(sizes)
    out_sizes[dim] = 1
    out = np.empty(int(np.prod(out_sizes)), np.float32)
    oracle().or_reduce_dim(op, base.ctypes.data, C.byref(v), dim, out)
    return out.reshape(out_sizes)


def apply(code, arity, bases, views, scalar):
    """bases: list of float32 numpy storages (modified in place); views: (sizes, strides, off)."""
    arr = (C.c_int32 * len(code))(*code)
    ptrs = (C.c_void_p * 3)(*[b.ctypes.data for b in bases] + [None] * (3 - len(bases)))
    vs = (View * 3)(*[make_view(*v) for v in views] + [View()] * (3 - len(views)))
    oracle().or_apply(arr, len(code), arity, ptrs, vs, scalar)


# ---- the reference itself (oracle/_ref) ----

def ref_render_im2col(g) -> str:
    buf = C.create_string_buffer(1 << 22)
    st = ref().ref_render_im2col(C.byref(g), buf, len(buf))
    if st != 0:
        raise RuntimeError(buf.value.decode())
    return buf.value.decode()


def ref_gen_im2col_kernel(g):
    buf = C.create_string_buffer(1 << 22)
    st = ref().ref_gen_im2col_kernel(C.byref(g), buf, len(buf))
    return st, buf.value.decode()


def ref_parse_expr(text: str, arity: int):
    buf = C.create_string_buffer(4096)
    st = ref().ref_parse_expr(text.encode(), arity, buf, len(buf))
    return st, buf.value.decode()


def _ops_array(ops):
    arr = (C.c_int64 * 64)()
    for i, (kind, dim, a, b) in enumerate(ops):
        arr[4 * i:4 * i + 4] = [kind, dim, a, b]
    return arr


def ref_apply(expr: str, bases, base_shapes, view_ops, scalar: float, lib=None):
    """bases: float32 arrays (contiguous, modified in place), view_ops per operand:
    list of ("narrow", dim, start, len) / ("select", dim, idx)."""
    arity = len(bases)
    data = (C.POINTER(C.c_float) * arity)(*[b.ctypes.data_as(C.POINTER(C.c_float)) for b in bases])
    sizes = (C.c_int64 * (8 * arity))()
    ndim = (C.c_int32 * arity)()
    ops = (C.c_int64 * (64 * arity))()
    nops = (C.c_int32 * arity)()
    for t in range(arity):
        ndim[t] = len(base_shapes[t])
        for d, s in enumerate(base_shapes[t]):
            sizes[8 * t + d] = s
        for i, op in enumerate(view_ops[t]):
            enc = (0, op[1], op[2], op[3]) if op[0] == "narrow" else (1, op[1], op[2], 0)
            ops[64 * t + 4 * i:64 * t + 4 * i + 4] = list(enc)
        nops[t] = len(view_ops[t])
    err = C.create_string_buffer(1024)
    st = (lib or ref()).ref_apply(expr.encode(), arity, data, sizes, ndim, ops, nops, C.c_float(scalar),
                         err, len(err))
    return st, err.value.decode()


def ref_reduce_all(op, base, base_shape, view_ops, lib=None):
    ops = _ops_array([(0, o[1], o[2], o[3]) if o[0] == "narrow" else (1, o[1], o[2], 0)
                      for o in view_ops])
    sizes = (C.c_int64 * 8)(*base_shape)
    out = C.c_float()
    err = C.create_string_buffer(1024)
    st = (lib or ref()).ref_reduce_all(op, base.ctypes.data_as(C.POINTER(C.c_float)), sizes,
                              len(base_shape), ops, len(view_ops), C.byref(out), err, len(err))
    return st, out.value, err.value.decode()


def ref_reduce_dim(op, base, base_shape, view_ops, dim, out_elems, lib=None):
    ops = _ops_array([(0, o[1], o[2], o[3]) if o[0] == "narrow" else (1, o[1], o[2], 0)
                      for o in view_ops])
    sizes = (C.c_int64 * 8)(*base_shape)
    out = np.empty(out_elems, np.float32)
    err = C.create_string_buffer(1024)
    st = (lib or ref()).ref_reduce_dim(op, base.ctypes.data_as(C.POINTER(C.c_float)), sizes,
                              len(base_shape), ops, len(view_ops), dim,
                              out.ctypes.data_as(C.POINTER(C.c_float)), out_elems, err, len(err))
    return st, out, err.value.decode()


def ref_choose_launch(n, maxwg):
    g, w = C.c_int64(), C.c_int()
    err = C.create_string_buffer(512)
    st = ref().ref_choose_launch(C.c_int64(n), maxwg, C.byref(g), C.byref(w), err, len(err))
    return st, g.value, w.value, err.value.decode()


def ref_geom_validate(g):
    err = C.create_string_buffer(512)
    st = ref().ref_geom_validate(C.byref(g), err, len(err))
    return st, err.value.decode()


# ---- the model-stack layers (SPEC.md:470 pool-max / relu; Torch nn.ReLU /
# nn.SpatialMaxPooling semantics, floor output rule), numpy restatement, TEST-ONLY ----
def relu_fwd(x):
    return np.maximum(x, np.float32(0)).astype(np.float32)


def relu_bwd(y, gy):
    return np.where(y > 0, gy, np.float32(0)).astype(np.float32)


def maxpool_fwd(x, kH, kW, sH, sW, pH=0, pW=0):
    """Returns (y, argmax): argmax = h*W + w of the first maximum in row-major window order
    (padding never selected)."""
    N, Cc, H, W = x.shape
    oH, oW = (H + 2 * pH - kH) // sH + 1, (W + 2 * pW - kW) // sW + 1
    y = np.full((N, Cc, oH, oW), -np.inf, np.float32)
    arg = np.full((N, Cc, oH, oW), -1, np.int32)
    for r in range(kH):
        for s in range(kW):
            hs = np.arange(oH) * sH - pH + r
            ws = np.arange(oW) * sW - pW + s
            vh, vw = (hs >= 0) & (hs < H), (ws >= 0) & (ws < W)
            v = np.full((N, Cc, oH, oW), -np.inf, np.float32)
            v[:, :, vh[:, None] & vw[None, :]] = x[:, :, hs[vh]][:, :, :, ws[vw]].reshape(N, Cc, -1)
            idx = (hs[:, None] * W + ws[None, :]).astype(np.int32)
            take = (v > y) | ((arg < 0) & (vh[:, None] & vw[None, :]))
            y = np.where(take, v, y)
            arg = np.where(take, idx[None, None], arg)
    return y, arg


def maxpool_bwd(gy, arg, in_shape):
    N, Cc, H, W = in_shape
    gx = np.zeros((N * Cc, H * W), np.float64)
    g2, a2 = gy.reshape(N * Cc, -1), arg.reshape(N * Cc, -1)
    for p in range(N * Cc):
        np.add.at(gx[p], a2[p], g2[p])
    return gx.reshape(in_shape).astype(np.float32)
