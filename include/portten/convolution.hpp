// Convolution module — the SPEC op set and the pluggable registry
// (ConvImplEntry, SPEC.md:342-346 / :425-433) over the B200 kernels, plus the
// Torch-facing SpatialConvolutionMM layer (updateOutput / updateGradInput /
// accGradParameters) the paper benchmarks.
//
// Built-in registry entries (highest priority that supports the geometry wins):
//   "implicitgemm-sm100a"      priority 100  tcgen05 TF32 implicit GEMM (all geometries)
//   "implicitgemm-fp32-sm100a" priority  50  CUDA-core FFMA implicit GEMM (tight mode)
// The reference's "direct"/"im2col"/"winograd" entries are host algorithms: they live in
// the oracle (oracle/) as the checker, not in this library.
#pragma once

#include <functional>
#include <string>
#include <vector>

#include "portten/backend.hpp"
#include "portten/conv_geometry.hpp"
#include "portten/tensor.hpp"

namespace portten::conv {

// TF32 tensor cores / FP32 CUDA-core FFMA / FP32-accurate 3xTF32 split on the tensor cores
enum class Math { TF32 = PT_MATH_TF32, FP32 = PT_MATH_FP32, TF32x3 = PT_MATH_3XTF32 };

// ---- device-resident ops (NCHW activations, KCRS weights) ----
DeviceTensor conv_forward(const ConvGeometry& g, const DeviceTensor& x, const DeviceTensor& w,
                          const DeviceTensor* b, Math math = Math::TF32, void* stream = nullptr);
DeviceTensor conv_backward_input(const ConvGeometry& g, const DeviceTensor& gy,
                                 const DeviceTensor& w, Math math = Math::TF32,
                                 void* stream = nullptr);
/// gw (+)= scale * dW ; gb (+)= scale * db (accumulate=false: overwrite, SPEC fresh grads).
void conv_backward_weight(const ConvGeometry& g, const DeviceTensor& x, const DeviceTensor& gy,
                          DeviceTensor& gw, DeviceTensor* gb, float scale = 1.0f,
                          bool accumulate = false, Math math = Math::TF32, void* stream = nullptr);

// ---- host-Tensor SPEC ops (upload -> device -> download; freshly allocated results) ----
Tensor conv_im2col_forward(const Tensor& input, const Tensor& weight, const Tensor* bias,
                           const ConvGeometry& g, Math math = Math::TF32);
/// lowering batchChunk images per GEMM is what the implicit GEMM does
/// on chip for the whole batch; results are bitwise equal for every valid chunk.
Tensor conv_im2col_batched(const Tensor& input, const Tensor& weight, const Tensor* bias,
                           const ConvGeometry& g, std::int64_t batchChunk, Math math = Math::TF32);
Tensor conv_backward_input(const Tensor& gradOutput, const Tensor& weight, const ConvGeometry& g,
                           Math math = Math::TF32);
/// Returns gradWeight; gradBias written to *gradBias when non-null.
Tensor conv_backward_weight(const Tensor& input, const Tensor& gradOutput, const ConvGeometry& g,
                            Tensor* gradBias, Math math = Math::TF32);
/// Winograd F(2x2,3x3), 3x3 stride-1 geometries only (ValidationError
/// "unsupported geometry" otherwise); the gradInput variant needs padding <= 2.
Tensor conv_winograd_2x2_3x3(const Tensor& input, const Tensor& weight, const Tensor* bias,
                             const ConvGeometry& g);
Tensor conv_backward_input_winograd(const Tensor& gradOutput, const Tensor& weight, const ConvGeometry& g);
Tensor im2col(const Tensor& image, const ConvGeometry& g);   // one C x H x W image
Tensor col2im(const Tensor& columns, const ConvGeometry& g);
/// SPEC gemm: C <- alpha*op(A)*op(B) + beta*C on 2-D row-major host tensors.
void gemm(bool transA, bool transB, float alpha, const Tensor& A, const Tensor& B, float beta,
          Tensor& C);

// ---- pluggable registry ----
struct ConvImplEntry {
    std::string name;
    std::function<bool(const ConvGeometry&, const BackendDescriptor&)> supports;
    std::function<Tensor(const Tensor& input, const Tensor& weight, const Tensor* bias,
                         const ConvGeometry& g)>
        run;
    int priority = 0;
    // B200 extension: the backward passes of the same implementation.
    std::function<Tensor(const Tensor& gradOutput, const Tensor& weight, const ConvGeometry& g)>
        backward_input;
    std::function<Tensor(const Tensor& input, const Tensor& gradOutput, const ConvGeometry& g,
                         Tensor* gradBias)>
        backward_weight;
};

void conv_registry_register(ConvImplEntry entry);  // ValidationError on duplicate name
const ConvImplEntry& conv_registry_select(const ConvGeometry& g, const BackendDescriptor& d);
std::vector<std::string> conv_registry_names();

// ---- Torch nn.SpatialConvolutionMM over device tensors ----
class SpatialConvolutionMM {
public:
    SpatialConvolutionMM(int nInputPlane, int nOutputPlane, int kW, int kH, int dW = 1, int dH = 1,
                         int padW = 0, int padH = -1, Math math = Math::TF32);
    void reset(float stdv = -1.0f, std::uint64_t seed = 0x5EED);
    ConvGeometry geometry(const DeviceTensor& input) const;
    const DeviceTensor& updateOutput(const DeviceTensor& input);
    const DeviceTensor& updateGradInput(const DeviceTensor& input, const DeviceTensor& gradOutput);
    void accGradParameters(const DeviceTensor& input, const DeviceTensor& gradOutput,
                           float scale = 1.0f);
    /// updateGradInput + accGradParameters in one fused pass (pt_b200_conv_bwd).
    const DeviceTensor& backward(const DeviceTensor& input, const DeviceTensor& gradOutput,
                                 float scale = 1.0f);
    void zeroGradParameters();

    DeviceTensor weight, bias, gradWeight, gradBias, output, gradInput;
    /// Torch's finput: updateOutput's relaid (channels-last) input, reused by backward()
    /// while the same input tensor is passed (pt_b200_conv_finput_bytes may be 0).
    DeviceTensor finput;
    int nInputPlane, nOutputPlane, kW, kH, dW, dH, padW, padH;
    Math math;

private:
    const float* finputFor_ = nullptr;
};

}  // namespace portten::conv
