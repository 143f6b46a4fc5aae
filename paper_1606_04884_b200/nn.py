"""Torch7-style SpatialConvolutionMM layer over the B200 kernels.

Mirrors nn.SpatialConvolutionMM (the cltorch/clnn layer the paper benchmarks,
SURVEY.md §0 naming bridge): constructor argument order
(nInputPlane, nOutputPlane, kW, kH, dW, dH, padW, padH), updateOutput,
updateGradInput, accGradParameters(input, gradOutput, scale) accumulating into
gradWeight/gradBias, zeroGradParameters, forward/backward.

Inputs may be CUDA tensors (device-resident path) or CPU tensors (the
reference's host-storage Tensor, SURVEY.md §1 process boundary): CPU inputs are
uploaded, computed on the GPU and the result downloaded — there is no CPU
compute path.
"""
from __future__ import annotations

import torch

from . import conv as _conv
from ._lib import ValidationError


class SpatialConvolutionMM:
    def __init__(self, nInputPlane, nOutputPlane, kW, kH, dW=1, dH=1, padW=0, padH=None,
                 math="tf32", device="cuda"):
        self.nInputPlane, self.nOutputPlane = int(nInputPlane), int(nOutputPlane)
        self.kW, self.kH, self.dW, self.dH = int(kW), int(kH), int(dW), int(dH)
        self.padW = int(padW)
        self.padH = int(padW if padH is None else padH)
        self.math = math
        self.device = torch.device(device)
        self.weight = torch.empty(nOutputPlane, nInputPlane, kH, kW, device=self.device)
        self.bias = torch.empty(nOutputPlane, device=self.device)
        self.gradWeight = torch.zeros_like(self.weight)
        self.gradBias = torch.zeros_like(self.bias)
        self.output = None
        self.gradInput = None
        # Torch's finput: updateOutput's relaid input, reused by accGradParameters while the
        # input is unchanged (same storage, same version counter)
        self.finput = None
        self._finput_key = None
        self.reset()

    def reset(self, stdv=None, seed=0x5EED):
        """Uniform(-stdv, stdv), stdv = 1/sqrt(kW*kH*nInputPlane) (Torch's reset)."""
        if stdv is None:
            stdv = 1.0 / (self.kW * self.kH * self.nInputPlane) ** 0.5
        _conv.fill_uniform(self.weight, seed, -stdv, stdv)
        _conv.fill_uniform(self.bias, seed + 1, -stdv, stdv)
        return self

    def geometry(self, x) -> _conv.ConvGeometry:
        if x.dim() != 4 or x.shape[1] != self.nInputPlane:
            raise ValidationError(f"SpatialConvolutionMM: expected N x {self.nInputPlane} x H x W "
                                  f"input, got {tuple(x.shape)}")
        g = _conv.ConvGeometry(x.shape[0], self.nInputPlane, x.shape[2], x.shape[3],
                               self.nOutputPlane, self.kH, self.kW, self.padH, self.padW,
                               self.dH, self.dW)
        g.validate()
        return g

    def _on_device(self, t):
        host = not t.is_cuda
        return (t.to(self.device, non_blocking=True).contiguous() if host else t.contiguous()), host

    def updateOutput(self, input):
        x, host = self._on_device(input)
        g = self.geometry(x)
        need = _conv.finput_bytes(g, self.math)
        if need:
            if self.finput is None or self.finput.numel() < need:
                self.finput = torch.empty(need, dtype=torch.uint8, device=self.device)
            y = _conv.conv_forward(g, x, self.weight, self.bias, math=self.math, finput=self.finput)
            self._finput_key = (x.data_ptr(), x._version, tuple(x.shape))
        else:
            y = _conv.conv_forward(g, x, self.weight, self.bias, math=self.math)
            self._finput_key = None
        self.output = y.cpu() if host else y
        return self.output

    def _saved_finput(self, x):
        key = (x.data_ptr(), x._version, tuple(x.shape))
        return self.finput if self._finput_key is not None and key == self._finput_key else None

    def updateGradInput(self, input, gradOutput):
        x, host = self._on_device(input)
        gy, _ = self._on_device(gradOutput)
        g = self.geometry(x)
        gx = _conv.conv_backward_input(g, gy, self.weight, math=self.math)
        self.gradInput = gx.cpu() if host else gx
        return self.gradInput

    def accGradParameters(self, input, gradOutput, scale=1.0):
        x, _ = self._on_device(input)
        gy, _ = self._on_device(gradOutput)
        g = self.geometry(x)
        _conv.conv_backward_weight(g, x, gy, self.gradWeight, self.gradBias, scale=scale,
                                   accumulate=True, math=self.math)

    def zeroGradParameters(self):
        self.gradWeight.zero_()
        self.gradBias.zero_()

    def forward(self, input):
        return self.updateOutput(input)

    def backward(self, input, gradOutput, scale=1.0):
        """updateGradInput + accGradParameters as one fused C-ABI call (pt_b200_conv_bwd)."""
        x, host = self._on_device(input)
        gy, _ = self._on_device(gradOutput)
        g = self.geometry(x)
        gx, _, _ = _conv.conv_backward(g, x, gy, self.weight, gw=self.gradWeight, gb=self.gradBias,
                                       scale=scale, accumulate=True, math=self.math,
                                       finput=self._saved_finput(x))
        self.gradInput = gx.cpu() if host else gx
        return self.gradInput

    def parameters(self):
        return [self.weight, self.bias], [self.gradWeight, self.gradBias]

    def __repr__(self):
        return (f"SpatialConvolutionMM({self.nInputPlane} -> {self.nOutputPlane}, "
                f"{self.kW}x{self.kH}, {self.dW},{self.dH}, {self.padW},{self.padH})")
