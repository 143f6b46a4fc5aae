"""portten-b200: sm_100a SpatialConvolutionMM (cltorch hot path) behind the reference's
operator API. See DESIGN.md. The compute lives in lib/libpt_b200.so (C ABI,
include/pt_b200.h); this package is the Python host mirror used by tests and bench.
"""
from ._lib import (BackendError, LibraryMissing, ValidationError, PT_MATH_FP32,  # noqa: F401
                   PT_MATH_TF32, PT_MATH_3XTF32, lib)
from .conv import (ConvGeometry, conv_backward, conv_backward_input,  # noqa: F401
                   conv_backward_weight,
                   conv_forward, conv_im2col_batched, col2im, im2col, im2col_batched, gemm,
                   bias_add, fill_uniform, launch_count, plan_cache_stats, device_count, finput_bytes,
                   conv_winograd_2x2_3x3, conv_backward_input_winograd, winograd_supported)
from .nn import SpatialConvolutionMM  # noqa: F401

__all__ = [
    "ConvGeometry", "SpatialConvolutionMM", "conv_forward", "conv_backward_input",
    "conv_backward_weight", "conv_im2col_batched", "im2col", "im2col_batched", "col2im", "gemm",
    "bias_add", "fill_uniform", "finput_bytes", "conv_winograd_2x2_3x3",
    "conv_backward_input_winograd", "winograd_supported", "ValidationError", "BackendError", "LibraryMissing", "lib",
]
