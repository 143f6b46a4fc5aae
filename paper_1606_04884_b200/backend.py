"""Device pointwise apply / reduce on the conv path — Python mirror of the reference's
dispatch_apply / dispatch_reduce_all / dispatch_reduce_dim (proj/src/backend.cpp:115-161)
for the B200 backend. Operands are CUDA tensors, possibly strided views with storage
offsets (tensor.hpp:56-120); the work runs in libpt_b200.so (pt_b200_apply /
pt_b200_reduce_*). choose_launch mirrors proj/src/backend.cpp:25-33.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import torch

from . import _lib
from ._lib import ValidationError, check, lib
from .expr import parse

SUM, MAX, MIN = _lib.PT_REDUCE_SUM, _lib.PT_REDUCE_MAX, _lib.PT_REDUCE_MIN


@dataclass
class BackendDescriptor:
    """proj/include/portten/backend.hpp:35-40."""
    name: str
    maxWorkgroupSize: int
    localMemBytes: int
    isDevice: bool = True


@dataclass
class LaunchConfig:
    globalSize: int
    workgroupSize: int


def choose_launch(n: int, d: BackendDescriptor) -> LaunchConfig:
    """workgroupSize = min(256, device max); globalSize = n rounded up (backend.cpp:25-33)."""
    if n < 1:
        raise ValidationError("choose_launch requires at least one work item")
    if d.maxWorkgroupSize < 1:
        raise ValidationError("backend reports no workgroup capacity")
    wg = min(256, d.maxWorkgroupSize)
    return LaunchConfig((n + wg - 1) // wg * wg, wg)


def descriptor(device: int = 0) -> BackendDescriptor:
    dd = _lib.PtDeviceDesc()
    check(lib().pt_b200_device_info(device, C.byref(dd)))
    return BackendDescriptor(dd.name.decode(), dd.maxWorkgroupSize, dd.localMemBytes, True)


def _view(t: torch.Tensor) -> _lib.PtView:
    if not t.is_cuda or t.dtype != torch.float32:
        raise ValidationError("apply/reduce operands must be float32 CUDA tensors")
    if t.dim() < 1 or t.dim() > 8:
        raise ValidationError("apply/reduce operands must have rank 1..8")
    v = _lib.PtView()
    v.ndim = t.dim()
    for d in range(t.dim()):
        v.sizes[d] = t.shape[d]
        v.strides[d] = t.stride(d)
    v.offset = 0
    return v


def dispatch_apply(expression: str, operands: Sequence[torch.Tensor], scalar: float = 0.0):
    """x = f(x, y, z, s) elementwise over 1..3 same-shaped views; operands[0] is written."""
    if not 1 <= len(operands) <= 3:
        raise ValidationError(f"apply takes 1..3 operands, got {len(operands)}")
    for t in operands:
        if tuple(t.shape) != tuple(operands[0].shape):
            raise ValidationError(f"apply operands must share sizes: {list(operands[0].shape)} vs "
                                  f"{list(t.shape)}")
    prog = parse(expression, len(operands))
    code = (C.c_int32 * len(prog.code))(*prog.code)
    bases = (C.c_void_p * 3)(*([t.data_ptr() for t in operands] + [None] * (3 - len(operands))))
    views = (_lib.PtView * 3)(*([_view(t) for t in operands] +
                                [_lib.PtView()] * (3 - len(operands))))
    check(lib().pt_b200_apply(code, len(prog.code), len(operands), bases, views, float(scalar),
                              torch.cuda.current_stream().cuda_stream))
    return operands[0]


def dispatch_reduce_all(op: int, t: torch.Tensor) -> float:
    out = torch.empty((), dtype=torch.float32, device=t.device)
    v = _view(t)
    check(lib().pt_b200_reduce_all(op, t.data_ptr(), C.byref(v), out.data_ptr(),
                                   torch.cuda.current_stream().cuda_stream))
    return float(out.item())


def dispatch_reduce_dim(op: int, t: torch.Tensor, dim: int) -> torch.Tensor:
    """Keeps the reduced dimension with size 1 (backend.hpp:106-107)."""
    if not 0 <= dim < t.dim():
        raise ValidationError(f"reduce dim {dim} out of range for rank {t.dim()}")
    shape = list(t.shape)
    shape[dim] = 1
    out = torch.empty(shape, dtype=torch.float32, device=t.device)
    v = _view(t)
    check(lib().pt_b200_reduce_dim(op, t.data_ptr(), C.byref(v), dim, out.data_ptr(),
                                   torch.cuda.current_stream().cuda_stream))
    return out
