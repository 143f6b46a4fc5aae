"""Device convolution ops over the C ABI — the SPEC convolution module's op names
 on device-resident torch tensors.

torch is plumbing here (device memory, streams); every computation is a
libpt_b200.so kernel. Tensors are float32 CUDA tensors: NCHW activations,
KCRS weights. Results are written into caller-provided tensors or freshly
allocated ones ("destination tensors freshly allocated").
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Tuple

import torch

from . import _lib
from ._lib import PT_MATH_3XTF32, PT_MATH_FP32, PT_MATH_TF32, ValidationError, check, lib

MATH = {"tf32": PT_MATH_TF32, "fp32": PT_MATH_FP32, "3xtf32": PT_MATH_3XTF32}


@dataclass(frozen=True)
class ConvGeometry:
    """Mirror of conv::ConvGeometry (proj/include/portten/conv_geometry.hpp:28-75)."""
    batch: int = 1
    inChannels: int = 1
    inHeight: int = 1
    inWidth: int = 1
    outChannels: int = 1
    kernelH: int = 1
    kernelW: int = 1
    padH: int = 0
    padW: int = 0
    strideH: int = 1
    strideW: int = 1

    def outHeight(self) -> int:  # conv_geometry.hpp:41-43 (floor rule)
        return (self.inHeight + 2 * self.padH - self.kernelH) // self.strideH + 1

    def outWidth(self) -> int:  # conv_geometry.hpp:44-46
        return (self.inWidth + 2 * self.padW - self.kernelW) // self.strideW + 1

    def patchSize(self) -> int:  # conv_geometry.hpp:49
        return self.inChannels * self.kernelH * self.kernelW

    def outSpatial(self) -> int:  # conv_geometry.hpp:51
        return self.outHeight() * self.outWidth()

    def validate(self) -> None:  # conv_geometry.hpp:53-63
        if not (self.batch >= 1 and self.inChannels >= 1 and self.inHeight >= 1 and
                self.inWidth >= 1 and self.outChannels >= 1 and self.kernelH >= 1 and
                self.kernelW >= 1 and self.strideH >= 1 and self.strideW >= 1):
            raise ValidationError("conv geometry: counts, dims, kernel and stride must be >= 1")
        if self.padH < 0 or self.padW < 0:
            raise ValidationError("conv geometry: padding must be >= 0")
        if (self.kernelH > self.inHeight + 2 * self.padH or
                self.kernelW > self.inWidth + 2 * self.padW):
            raise ValidationError(f"conv geometry: kernel exceeds padded input ({self})")
        if self.outHeight() < 1 or self.outWidth() < 1:
            raise ValidationError(f"conv geometry: empty output ({self})")

    def toString(self) -> str:  # conv_geometry.hpp:65-72
        return (f"N{self.batch} C{self.inChannels} H{self.inHeight} W{self.inWidth} "
                f"K{self.outChannels} k{self.kernelH}x{self.kernelW} p{self.padH}x{self.padW} "
                f"s{self.strideH}x{self.strideW}")

    __str__ = toString

    def c(self) -> _lib.PtConvGeom:
        return _lib.PtConvGeom(self.batch, self.inChannels, self.inHeight, self.inWidth,
                               self.outChannels, self.kernelH, self.kernelW, self.padH,
                               self.padW, self.strideH, self.strideW)

    # shapes
    def input_shape(self):
        return (self.batch, self.inChannels, self.inHeight, self.inWidth)

    def weight_shape(self):
        return (self.outChannels, self.inChannels, self.kernelH, self.kernelW)

    def output_shape(self):
        return (self.batch, self.outChannels, self.outHeight(), self.outWidth())

    def flops(self) -> int:
        """2*N*K*CRS*oH*oW for one pass (fprop, dgrad or wgrad)."""
        return 2 * self.batch * self.outChannels * self.patchSize() * self.outSpatial()

    def with_batch(self, n: int) -> "ConvGeometry":
        return ConvGeometry(n, self.inChannels, self.inHeight, self.inWidth, self.outChannels,
                            self.kernelH, self.kernelW, self.padH, self.padW, self.strideH,
                            self.strideW)


def _math(math) -> int:
    if isinstance(math, int):
        return math
    try:
        return MATH[math]
    except KeyError:
        raise ValidationError(f"unknown math mode {math!r} (tf32|fp32|3xtf32)") from None


def _dev(t: torch.Tensor, shape, what: str) -> int:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValidationError(f"{what}: expected a CUDA tensor")
    if t.device.index != torch.cuda.current_device():
        # the workspace, the stream and the library's device are the current device's
        raise ValidationError(f"{what}: on {t.device}, but the current device is "
                              f"cuda:{torch.cuda.current_device()}")
    if t.dtype != torch.float32:
        raise ValidationError(f"{what}: expected float32, got {t.dtype}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValidationError(f"{what}: shape {tuple(t.shape)} != expected {tuple(shape)}")
    if not t.is_contiguous():
        raise ValidationError(f"{what}: must be contiguous")
    return t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


class _Workspace:
    """Grow-only scratch per (device, stream); conv passes on one stream are ordered."""

    def __init__(self):
        self._bufs = {}

    def get(self, nbytes: int) -> Tuple[int, int]:
        if nbytes <= 0:
            return 0, 0
        key = (torch.cuda.current_device(), _stream())
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device="cuda")
            self._bufs[key] = buf
        return buf.data_ptr(), buf.numel()


WORKSPACE = _Workspace()


def workspace_bytes(g: ConvGeometry, op: int, math="tf32") -> int:
    gc = g.c()
    n = lib().pt_b200_conv_workspace_bytes(C.byref(gc), op, _math(math))
    if n == C.c_size_t(-1).value:
        check(lib().pt_b200_conv_validate(C.byref(gc)))
        raise ValidationError(lib().pt_b200_last_error().decode())
    return n


def finput_bytes(g: ConvGeometry, math="tf32") -> int:
    """Bytes of Torch's `finput` buffer for this geometry: the forward pass's channels-last
    copy of x that accGradParameters reuses (0 = no shared layout, the buffer is ignored)."""
    gc = g.c()
    return int(lib().pt_b200_conv_finput_bytes(C.byref(gc), _math(math)))


def conv_forward(g: ConvGeometry, x, w, b=None, y=None, math="tf32", finput=None):
    """updateOutput == conv_im2col_forward: y = W * im2col(x) + b.
    finput (uint8 device tensor of finput_bytes(g)): keep the relaid input for backward."""
    gc, m = g.c(), _math(math)
    check(lib().pt_b200_conv_validate(C.byref(gc)))
    if y is None:
        y = torch.empty(g.output_shape(), dtype=torch.float32, device=x.device)
    px = _dev(x, g.input_shape(), "input")
    pw = _dev(w, g.weight_shape(), "weight")
    pb = _dev(b, (g.outChannels,), "bias") if b is not None else None
    py = _dev(y, g.output_shape(), "output")
    ws, wsn = WORKSPACE.get(workspace_bytes(g, _lib.PT_CONV_FWD, m))
    if finput is not None:
        check(lib().pt_b200_conv_fwd_finput(C.byref(gc), px, pw, pb, py, m, ws or None, wsn,
                                            _finput(g, finput, m), _stream()))
    else:
        check(lib().pt_b200_conv_fwd(C.byref(gc), px, pw, pb, py, m, ws or None, wsn, _stream()))
    return y


def _finput(g: ConvGeometry, buf, m):
    need = int(lib().pt_b200_conv_finput_bytes(C.byref(g.c()), m))
    if need == 0:
        return None
    if not (buf.is_cuda and buf.is_contiguous() and buf.numel() * buf.element_size() >= need):
        raise ValidationError(f"finput: need a contiguous device buffer of {need} bytes")
    return buf.data_ptr()


def conv_im2col_batched(g: ConvGeometry, x, w, b=None, batchChunk: int = 1, y=None, math="tf32"):
    """SPEC.md:398-406. The implicit GEMM lowers the whole batch lazily on chip, so every
    batchChunk gives the same (bitwise) result as conv_forward; the chunk is validated."""
    if not (1 <= batchChunk <= g.batch):
        raise ValidationError(f"invalid batchChunk {batchChunk} for batch {g.batch}")
    return conv_forward(g, x, w, b, y, math)


def conv_backward_input(g: ConvGeometry, gy, w, gx=None, math="tf32"):
    """updateGradInput == conv_backward_input."""
    gc, m = g.c(), _math(math)
    check(lib().pt_b200_conv_validate(C.byref(gc)))
    if gx is None:
        gx = torch.empty(g.input_shape(), dtype=torch.float32, device=gy.device)
    pgy = _dev(gy, g.output_shape(), "gradOutput")
    pw = _dev(w, g.weight_shape(), "weight")
    pgx = _dev(gx, g.input_shape(), "gradInput")
    ws, wsn = WORKSPACE.get(workspace_bytes(g, _lib.PT_CONV_BWD_DATA, m))
    check(lib().pt_b200_conv_bwd_data(C.byref(gc), pgy, pw, pgx, m, ws or None, wsn, _stream()))
    return gx


def conv_backward_weight(g: ConvGeometry, x, gy, gw=None, gb=None, scale: float = 1.0,
                         accumulate: bool = False, with_bias: bool = True, math="tf32"):
    """accGradParameters == conv_backward_weight + gradBias.
    accumulate=False returns fresh gradients (SPEC); True is Torch's gw += scale*dW."""
    gc, m = g.c(), _math(math)
    check(lib().pt_b200_conv_validate(C.byref(gc)))
    if gw is None:
        gw = torch.zeros(g.weight_shape(), dtype=torch.float32, device=x.device)
    if gb is None and with_bias:
        gb = torch.zeros((g.outChannels,), dtype=torch.float32, device=x.device)
    px = _dev(x, g.input_shape(), "input")
    pgy = _dev(gy, g.output_shape(), "gradOutput")
    pgw = _dev(gw, g.weight_shape(), "gradWeight")
    pgb = _dev(gb, (g.outChannels,), "gradBias") if gb is not None else None
    ws, wsn = WORKSPACE.get(workspace_bytes(g, _lib.PT_CONV_BWD_FILTER, m))
    check(lib().pt_b200_conv_bwd_filter(C.byref(gc), px, pgy, pgw, pgb, float(scale),
                                        int(bool(accumulate)), m, ws or None, wsn, _stream()))
    return gw, gb


def conv_backward(g: ConvGeometry, x, gy, w, gx=None, gw=None, gb=None, scale: float = 1.0,
                  accumulate: bool = False, need_input_grad: bool = True, with_bias: bool = True,
                  math="tf32", finput=None):
    """Torch backward() = updateGradInput + accGradParameters in one C-ABI call
    (pt_b200_conv_bwd): one NHWC transform of gy, gradBias fused into it, feeds both
    tensor-core passes. Returns (gx, gw, gb); gx is None when need_input_grad=False."""
    gc, m = g.c(), _math(math)
    check(lib().pt_b200_conv_validate(C.byref(gc)))
    if gx is None and need_input_grad:
        gx = torch.empty(g.input_shape(), dtype=torch.float32, device=gy.device)
    if gw is None:
        gw = torch.zeros(g.weight_shape(), dtype=torch.float32, device=gy.device)
    if gb is None and with_bias:
        gb = torch.zeros((g.outChannels,), dtype=torch.float32, device=gy.device)
    ws, wsn = WORKSPACE.get(workspace_bytes(g, _lib.PT_CONV_BWD, m))
    args = (C.byref(gc), _dev(x, g.input_shape(), "input"), _dev(gy, g.output_shape(), "gradOutput"),
            _dev(w, g.weight_shape(), "weight"),
            _dev(gx, g.input_shape(), "gradInput") if gx is not None else None,
            _dev(gw, g.weight_shape(), "gradWeight"),
            _dev(gb, (g.outChannels,), "gradBias") if gb is not None else None,
            float(scale), int(bool(accumulate)), m, ws or None, wsn)
    if finput is not None:
        check(lib().pt_b200_conv_bwd_finput(*args, _finput(g, finput, m), _stream()))
    else:
        check(lib().pt_b200_conv_bwd(*args, _stream()))
    return gx, gw, gb


def im2col(g: ConvGeometry, img):
    """One image C x H x W -> (C*kH*kW) x (oH*oW), bit-exact with im2col.kt.tmpl:9-21."""
    gc = g.c()
    col = torch.empty((g.patchSize(), g.outSpatial()), dtype=torch.float32, device=img.device)
    check(lib().pt_b200_im2col(C.byref(gc), _dev(img, (g.inChannels, g.inHeight, g.inWidth),
                                                 "image"), col.data_ptr(), _stream()))
    return col


def im2col_batched(g: ConvGeometry, x, n0: int, count: int):
    gc = g.c()
    col = torch.empty((g.patchSize(), count * g.outSpatial()), dtype=torch.float32,
                      device=x.device)
    check(lib().pt_b200_im2col_batched(C.byref(gc), _dev(x, g.input_shape(), "input"), n0, count,
                                       col.data_ptr(), _stream()))
    return col


def col2im(g: ConvGeometry, col):
    """Scatter-add inverse of im2col for one image."""
    gc = g.c()
    img = torch.empty((g.inChannels, g.inHeight, g.inWidth), dtype=torch.float32,
                      device=col.device)
    check(lib().pt_b200_col2im(C.byref(gc), _dev(col, (g.patchSize(), g.outSpatial()), "columns"),
                               img.data_ptr(), _stream()))
    return img


def gemm(A, B, Cm, transA=False, transB=False, alpha=1.0, beta=0.0, math="fp32"):
    """SPEC gemm: Cm <- alpha*op(A)*op(B) + beta*Cm (row-major, 2-D)."""
    M, K = (A.shape[1], A.shape[0]) if transA else (A.shape[0], A.shape[1])
    K2, N = (B.shape[1], B.shape[0]) if transB else (B.shape[0], B.shape[1])
    if K != K2 or tuple(Cm.shape) != (M, N):
        raise ValidationError("gemm: dimension mismatch")
    check(lib().pt_b200_gemm(int(transA), int(transB), M, N, K, float(alpha), _dev(A, None, "A"),
                             A.shape[1], _dev(B, None, "B"), B.shape[1], float(beta),
                             _dev(Cm, None, "C"), Cm.shape[1], _math(math), _stream()))
    return Cm


def bias_add(y, b):
    """y[n,k,:,:] += b[k] — the conv-path apply of SURVEY.md §3(B) as one launch."""
    N, K = y.shape[0], y.shape[1]
    hw = y.numel() // (N * K)
    check(lib().pt_b200_bias_add(_dev(y, None, "y"), _dev(b, (K,), "bias"), N, K, hw, _stream()))
    return y


def fill_uniform(t, seed: int, lo: float = -1.0, hi: float = 1.0):
    """Counter-based synthetic fill, identical to oracle or_fill_uniform."""
    check(lib().pt_b200_fill_uniform(_dev(t, None, "tensor"), t.numel(), seed & (2**64 - 1),
                                     lo, hi, _stream()))
    return t


def launch_count() -> int:
    return int(lib().pt_b200_launch_count())


def plan_cache_stats():
    """(hits, encodes) of the library's TMA-descriptor cache since process start."""
    h, e = C.c_int64(0), C.c_int64(0)
    lib().pt_b200_plan_cache_stats(C.byref(h), C.byref(e))
    return int(h.value), int(e.value)


def device_count() -> int:
    return int(lib().pt_b200_device_count())


# ---- Winograd F(2x2,3x3) registry entry ----
def winograd_supported(g: ConvGeometry, op: int = _lib.PT_CONV_FWD) -> bool:
    """3x3 stride-1 geometries (gradInput: padding <= 2)."""
    gc = g.c()
    return lib().pt_b200_winograd_workspace_bytes(C.byref(gc), op) != C.c_size_t(-1).value


def _wino_ws(g: ConvGeometry, op: int):
    gc = g.c()
    n = lib().pt_b200_winograd_workspace_bytes(C.byref(gc), op)
    if n == C.c_size_t(-1).value:
        raise ValidationError(lib().pt_b200_last_error().decode())
    return WORKSPACE.get(n)


def conv_winograd_2x2_3x3(g: ConvGeometry, x, w, b=None, y=None):
    """conv_winograd_2x2_3x3: weight / input transforms, 16 tensor-core
    GEMMs with the channel sums in the transform domain, output transform + bias. Equals
    conv_direct within 1e-3 relative (SPEC); ValidationError for unsupported geometries."""
    gc = g.c()
    check(lib().pt_b200_conv_validate(C.byref(gc)))
    ws, wsn = _wino_ws(g, _lib.PT_CONV_FWD)
    if y is None:
        y = torch.empty(g.output_shape(), dtype=torch.float32, device=x.device)
    pb = _dev(b, (g.outChannels,), "bias") if b is not None else None
    check(lib().pt_b200_conv_fwd_winograd(C.byref(gc), _dev(x, g.input_shape(), "input"),
                                          _dev(w, g.weight_shape(), "weight"), pb,
                                          _dev(y, g.output_shape(), "output"), ws or None, wsn,
                                          _stream()))
    return y


def conv_backward_input_winograd(g: ConvGeometry, gy, w, gx=None):
    """updateGradInput through the Winograd entry (rotated, channel-swapped filter)."""
    gc = g.c()
    check(lib().pt_b200_conv_validate(C.byref(gc)))
    ws, wsn = _wino_ws(g, _lib.PT_CONV_BWD_DATA)
    if gx is None:
        gx = torch.empty(g.input_shape(), dtype=torch.float32, device=gy.device)
    check(lib().pt_b200_conv_bwd_data_winograd(C.byref(gc), _dev(gy, g.output_shape(), "gradOutput"),
                                               _dev(w, g.weight_shape(), "weight"),
                                               _dev(gx, g.input_shape(), "gradInput"), ws or None,
                                               wsn, _stream()))
    return gx
