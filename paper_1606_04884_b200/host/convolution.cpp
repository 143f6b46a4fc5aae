// convolution.cpp — SPEC convolution ops, registry and SpatialConvolutionMM over the
// libpt_b200 C ABI (include/portten/convolution.hpp).
#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>

#include "portten/convolution.hpp"

namespace portten::conv {

namespace {

// Grow-only device scratch per (device, stream): the conv passes on one stream are ordered,
// so one buffer per stream is never in use by two passes at once, while calls on different
// streams (or devices) get different buffers. A buffer is replaced only after its stream has
// drained, since queued work may still read the old one.
struct Scratch {
    std::shared_ptr<void> buf;
    std::size_t bytes = 0;
};

void* scratch(void* stream, std::size_t need) {
    if (need == 0) return nullptr;
    static std::mutex mu;
    static std::map<std::pair<int, void*>, Scratch> pool;
    int dev = 0;
    throw_if_error(pt_b200_get_device(&dev));
    std::lock_guard<std::mutex> lk(mu);
    Scratch& s = pool[{dev, stream}];
    if (need > s.bytes) {
        if (s.buf) throw_if_error(pt_b200_stream_sync(stream));
        s.buf.reset();
        void* p = nullptr;
        throw_if_error(pt_b200_malloc(&p, need));
        s.buf = std::shared_ptr<void>(p, [](void* q) { pt_b200_free(q); });
        s.bytes = need;
    }
    return s.buf.get();
}

std::size_t ws_bytes(const ConvGeometry& g, int op, Math m) {
    const pt_conv_geom a = g.abi();
    const std::size_t n = pt_b200_conv_workspace_bytes(&a, op, static_cast<int>(m));
    if (n == static_cast<std::size_t>(-1)) throw_if_error(pt_b200_conv_validate(&a));
    return n;
}

void require_shape(const std::vector<std::int64_t>& got, std::vector<std::int64_t> want, const char* what) {
    PORTTEN_CHECK(got == want, std::string(what) + ": shape mismatch with the conv geometry");
}

std::vector<std::int64_t> in_shape(const ConvGeometry& g) {
    return {g.batch, g.inChannels, g.inHeight, g.inWidth};
}
std::vector<std::int64_t> w_shape(const ConvGeometry& g) {
    return {g.outChannels, g.inChannels, g.kernelH, g.kernelW};
}
std::vector<std::int64_t> out_shape(const ConvGeometry& g) {
    return {g.batch, g.outChannels, g.outHeight(), g.outWidth()};
}

}  // namespace

DeviceTensor conv_forward(const ConvGeometry& g, const DeviceTensor& x, const DeviceTensor& w,
                          const DeviceTensor* b, Math math, void* stream) {
    g.validate();
    require_shape(x.sizes(), in_shape(g), "input");
    require_shape(w.sizes(), w_shape(g), "weight");
    PORTTEN_CHECK(x.isContiguous() && w.isContiguous(), "conv operands must be contiguous");
    if (b) require_shape(b->sizes(), {g.outChannels}, "bias");
    DeviceTensor y = DeviceTensor::empty(out_shape(g));
    const pt_conv_geom a = g.abi();
    const std::size_t n = ws_bytes(g, PT_CONV_FWD, math);
    throw_if_error(pt_b200_conv_fwd(&a, x.data(), w.data(), b ? b->data() : nullptr, y.data(),
                                    static_cast<int>(math), scratch(stream, n), n, stream));
    return y;
}

DeviceTensor conv_backward_input(const ConvGeometry& g, const DeviceTensor& gy, const DeviceTensor& w,
                                 Math math, void* stream) {
    g.validate();
    require_shape(gy.sizes(), out_shape(g), "gradOutput");
    require_shape(w.sizes(), w_shape(g), "weight");
    DeviceTensor gx = DeviceTensor::empty(in_shape(g));
    const pt_conv_geom a = g.abi();
    const std::size_t n = ws_bytes(g, PT_CONV_BWD_DATA, math);
    throw_if_error(pt_b200_conv_bwd_data(&a, gy.data(), w.data(), gx.data(), static_cast<int>(math),
                                         scratch(stream, n), n, stream));
    return gx;
}

void conv_backward_weight(const ConvGeometry& g, const DeviceTensor& x, const DeviceTensor& gy,
                          DeviceTensor& gw, DeviceTensor* gb, float scale, bool accumulate, Math math,
                          void* stream) {
    g.validate();
    require_shape(x.sizes(), in_shape(g), "input");
    require_shape(gy.sizes(), out_shape(g), "gradOutput");
    if (!gw.defined()) gw = DeviceTensor::empty(w_shape(g));
    require_shape(gw.sizes(), w_shape(g), "gradWeight");
    if (gb && !gb->defined()) *gb = DeviceTensor::empty({g.outChannels});
    const pt_conv_geom a = g.abi();
    const std::size_t n = ws_bytes(g, PT_CONV_BWD_FILTER, math);
    throw_if_error(pt_b200_conv_bwd_filter(&a, x.data(), gy.data(), gw.data(), gb ? gb->data() : nullptr,
                                           scale, accumulate ? 1 : 0, static_cast<int>(math),
                                           scratch(stream, n), n, stream));
}

// ---- host-Tensor SPEC ops ----
Tensor conv_im2col_forward(const Tensor& input, const Tensor& weight, const Tensor* bias,
                           const ConvGeometry& g, Math math) {
    g.validate();
    require_shape(input.sizes(), in_shape(g), "input");
    require_shape(weight.sizes(), w_shape(g), "weight");
    DeviceTensor x = DeviceTensor::upload(input), w = DeviceTensor::upload(weight), b;
    if (bias) {
        require_shape(bias->sizes(), {g.outChannels}, "bias");
        b = DeviceTensor::upload(*bias);
    }
    return conv_forward(g, x, w, bias ? &b : nullptr, math).download();
}

Tensor conv_im2col_batched(const Tensor& input, const Tensor& weight, const Tensor* bias,
                           const ConvGeometry& g, std::int64_t batchChunk, Math math) {
    PORTTEN_CHECK(batchChunk >= 1 && batchChunk <= g.batch,
                  "invalid batchChunk " + std::to_string(batchChunk));
    return conv_im2col_forward(input, weight, bias, g, math);
}

Tensor conv_backward_input(const Tensor& gradOutput, const Tensor& weight, const ConvGeometry& g,
                           Math math) {
    g.validate();
    require_shape(gradOutput.sizes(), out_shape(g), "gradOutput");
    require_shape(weight.sizes(), w_shape(g), "weight");
    return conv_backward_input(g, DeviceTensor::upload(gradOutput), DeviceTensor::upload(weight), math)
        .download();
}

Tensor conv_backward_weight(const Tensor& input, const Tensor& gradOutput, const ConvGeometry& g,
                            Tensor* gradBias, Math math) {
    g.validate();
    require_shape(input.sizes(), in_shape(g), "input");
    require_shape(gradOutput.sizes(), out_shape(g), "gradOutput");
    DeviceTensor gw, gb;
    conv_backward_weight(g, DeviceTensor::upload(input), DeviceTensor::upload(gradOutput), gw,
                         gradBias ? &gb : nullptr, 1.0f, false, math);
    if (gradBias) *gradBias = gb.download();
    return gw.download();
}

Tensor conv_winograd_2x2_3x3(const Tensor& input, const Tensor& weight, const Tensor* bias,
                             const ConvGeometry& g) {
    g.validate();
    require_shape(input.sizes(), in_shape(g), "input");
    require_shape(weight.sizes(), w_shape(g), "weight");
    const pt_conv_geom a = g.abi();
    const std::size_t n = pt_b200_winograd_workspace_bytes(&a, PT_CONV_FWD);
    if (n == static_cast<std::size_t>(-1)) throw ValidationError(pt_b200_last_error());
    DeviceTensor x = DeviceTensor::upload(input), w = DeviceTensor::upload(weight), b;
    if (bias) {
        require_shape(bias->sizes(), {g.outChannels}, "bias");
        b = DeviceTensor::upload(*bias);
    }
    DeviceTensor y = DeviceTensor::empty(out_shape(g));
    throw_if_error(pt_b200_conv_fwd_winograd(&a, x.data(), w.data(), bias ? b.data() : nullptr, y.data(),
                                             scratch(nullptr, n), n, nullptr));
    return y.download();
}

Tensor conv_backward_input_winograd(const Tensor& gradOutput, const Tensor& weight, const ConvGeometry& g) {
    g.validate();
    require_shape(gradOutput.sizes(), out_shape(g), "gradOutput");
    require_shape(weight.sizes(), w_shape(g), "weight");
    const pt_conv_geom a = g.abi();
    const std::size_t n = pt_b200_winograd_workspace_bytes(&a, PT_CONV_BWD_DATA);
    if (n == static_cast<std::size_t>(-1)) throw ValidationError(pt_b200_last_error());
    DeviceTensor gy = DeviceTensor::upload(gradOutput), w = DeviceTensor::upload(weight);
    DeviceTensor gx = DeviceTensor::empty(in_shape(g));
    throw_if_error(pt_b200_conv_bwd_data_winograd(&a, gy.data(), w.data(), gx.data(), scratch(nullptr, n), n,
                                                  nullptr));
    return gx.download();
}

Tensor im2col(const Tensor& image, const ConvGeometry& g) {
    g.validate();
    require_shape(image.sizes(), {g.inChannels, g.inHeight, g.inWidth}, "image");
    DeviceTensor img = DeviceTensor::upload(image);
    DeviceTensor col = DeviceTensor::empty({g.patchSize(), g.outSpatial()});
    const pt_conv_geom a = g.abi();
    throw_if_error(pt_b200_im2col(&a, img.data(), col.data(), nullptr));
    return col.download();
}

Tensor col2im(const Tensor& columns, const ConvGeometry& g) {
    g.validate();
    require_shape(columns.sizes(), {g.patchSize(), g.outSpatial()}, "columns");
    DeviceTensor col = DeviceTensor::upload(columns);
    DeviceTensor img = DeviceTensor::empty({g.inChannels, g.inHeight, g.inWidth});
    const pt_conv_geom a = g.abi();
    throw_if_error(pt_b200_col2im(&a, col.data(), img.data(), nullptr));
    return img.download();
}

void gemm(bool transA, bool transB, float alpha, const Tensor& A, const Tensor& B, float beta,
          Tensor& C) {
    PORTTEN_CHECK(A.dim() == 2 && B.dim() == 2 && C.dim() == 2, "gemm: operands must be 2-D");
    const std::int64_t M = transA ? A.size(1) : A.size(0), K = transA ? A.size(0) : A.size(1);
    const std::int64_t K2 = transB ? B.size(1) : B.size(0), N = transB ? B.size(0) : B.size(1);
    PORTTEN_CHECK(K == K2 && C.size(0) == M && C.size(1) == N, "gemm: dimension mismatch");
    DeviceTensor a = DeviceTensor::upload(A), b = DeviceTensor::upload(B), c = DeviceTensor::upload(C);
    throw_if_error(pt_b200_gemm(transA, transB, M, N, K, alpha, a.data(), A.size(1), b.data(), B.size(1),
                                beta, c.data(), N, PT_MATH_FP32, nullptr));
    Tensor out = c.download();
    C.copyFrom(out);
}

// ---- registry ----
namespace {
std::mutex g_reg_mu;
std::vector<ConvImplEntry>& registry() {
    static std::vector<ConvImplEntry> r = [] {
        std::vector<ConvImplEntry> v;
        auto mk = [](std::string name, int prio, Math m) {
            ConvImplEntry e;
            e.name = std::move(name);
            e.priority = prio;
            e.supports = [](const ConvGeometry& g, const BackendDescriptor& d) {
                const pt_conv_geom a = g.abi();
                return d.isDevice && pt_b200_conv_validate(&a) == PT_OK;
            };
            e.run = [m](const Tensor& x, const Tensor& w, const Tensor* b, const ConvGeometry& g) {
                return conv_im2col_forward(x, w, b, g, m);
            };
            e.backward_input = [m](const Tensor& gy, const Tensor& w, const ConvGeometry& g) {
                return conv_backward_input(gy, w, g, m);
            };
            e.backward_weight = [m](const Tensor& x, const Tensor& gy, const ConvGeometry& g, Tensor* gb) {
                return conv_backward_weight(x, gy, g, gb, m);
            };
            return e;
        };
        v.push_back(mk("implicitgemm-sm100a", 100, Math::TF32));
        v.push_back(mk("implicitgemm-3xtf32-sm100a", 60, Math::TF32x3));
        v.push_back(mk("implicitgemm-fp32-sm100a", 50, Math::FP32));
        // Winograd F(2x2,3x3): 3x3 stride-1 only; registered BELOW the
        // implicit GEMM because it measures slower on B200 — selected by
        // name, or by a caller re-registering it at a higher priority
        ConvImplEntry w;
        w.name = "winograd-sm100a";
        w.priority = 30;
        w.supports = [](const ConvGeometry& g, const BackendDescriptor& d) {
            const pt_conv_geom a = g.abi();
            return d.isDevice && pt_b200_conv_validate(&a) == PT_OK &&
                   pt_b200_winograd_workspace_bytes(&a, PT_CONV_FWD) != static_cast<std::size_t>(-1);
        };
        w.run = [](const Tensor& x, const Tensor& wt, const Tensor* b, const ConvGeometry& g) {
            return conv_winograd_2x2_3x3(x, wt, b, g);
        };
        w.backward_input = [](const Tensor& gy, const Tensor& wt, const ConvGeometry& g) {
            const pt_conv_geom a = g.abi();
            if (pt_b200_winograd_workspace_bytes(&a, PT_CONV_BWD_DATA) != static_cast<std::size_t>(-1))
                return conv_backward_input_winograd(gy, wt, g);
            return conv_backward_input(gy, wt, g, Math::TF32);
        };
        w.backward_weight = [](const Tensor& x, const Tensor& gy, const ConvGeometry& g, Tensor* gb) {
            return conv_backward_weight(x, gy, g, gb, Math::TF32);
        };
        v.push_back(std::move(w));
        return v;
    }();
    return r;
}
}  // namespace

void conv_registry_register(ConvImplEntry entry) {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    for (const auto& e : registry())
        PORTTEN_CHECK(e.name != entry.name, "conv registry: duplicate implementation name '" + entry.name + "'");
    registry().push_back(std::move(entry));
}

const ConvImplEntry& conv_registry_select(const ConvGeometry& g, const BackendDescriptor& d) {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    const ConvImplEntry* best = nullptr;
    for (const auto& e : registry())
        if (e.supports && e.supports(g, d) && (!best || e.priority > best->priority)) best = &e;
    if (!best) throw ValidationError("conv registry: no implementation supports " + g.toString());
    return *best;
}

std::vector<std::string> conv_registry_names() {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    std::vector<std::string> n;
    for (const auto& e : registry()) n.push_back(e.name);
    return n;
}

// ---- SpatialConvolutionMM ----
SpatialConvolutionMM::SpatialConvolutionMM(int nIn, int nOut, int kW_, int kH_, int dW_, int dH_,
                                           int padW_, int padH_, Math m)
    : nInputPlane(nIn), nOutputPlane(nOut), kW(kW_), kH(kH_), dW(dW_), dH(dH_), padW(padW_),
      padH(padH_ < 0 ? padW_ : padH_), math(m) {
    weight = DeviceTensor::empty({nOut, nIn, kH, kW});
    bias = DeviceTensor::empty({nOut});
    gradWeight = DeviceTensor::empty({nOut, nIn, kH, kW});
    gradBias = DeviceTensor::empty({nOut});
    reset();
    zeroGradParameters();
}

void SpatialConvolutionMM::reset(float stdv, std::uint64_t seed) {
    if (stdv < 0) stdv = 1.0f / std::sqrt(static_cast<float>(kW * kH * nInputPlane));
    throw_if_error(pt_b200_fill_uniform(weight.data(), weight.numel(), seed, -stdv, stdv, nullptr));
    throw_if_error(pt_b200_fill_uniform(bias.data(), bias.numel(), seed + 1, -stdv, stdv, nullptr));
}

ConvGeometry SpatialConvolutionMM::geometry(const DeviceTensor& x) const {
    PORTTEN_CHECK(x.dim() == 4 && x.sizes()[1] == nInputPlane,
                  "SpatialConvolutionMM: expected N x " + std::to_string(nInputPlane) + " x H x W input");
    ConvGeometry g{x.sizes()[0], nInputPlane, x.sizes()[2], x.sizes()[3], nOutputPlane, kH, kW,
                   padH, padW, dH, dW};
    g.validate();
    return g;
}

const DeviceTensor& SpatialConvolutionMM::updateOutput(const DeviceTensor& input) {
    const ConvGeometry g = geometry(input);
    const pt_conv_geom a = g.abi();
    const std::size_t fb = pt_b200_conv_finput_bytes(&a, static_cast<int>(math));
    finputFor_ = nullptr;
    if (fb == 0) {
        output = conv_forward(g, input, weight, &bias, math);
        return output;
    }
    // Torch's finput: keep the forward's relaid input for accGradParameters
    const std::int64_t fe = static_cast<std::int64_t>((fb + 3) / 4);
    if (finput.numel() < fe) finput = DeviceTensor::empty({fe});
    PORTTEN_CHECK(input.isContiguous() && weight.isContiguous(), "conv operands must be contiguous");
    output = DeviceTensor::empty({g.batch, g.outChannels, g.outHeight(), g.outWidth()});
    const std::size_t n = ws_bytes(g, PT_CONV_FWD, math);
    throw_if_error(pt_b200_conv_fwd_finput(&a, input.data(), weight.data(), bias.data(), output.data(),
                                           static_cast<int>(math), scratch(nullptr, n), n, finput.data(),
                                           nullptr));
    finputFor_ = input.data();
    return output;
}

const DeviceTensor& SpatialConvolutionMM::updateGradInput(const DeviceTensor& input,
                                                          const DeviceTensor& gradOutput) {
    gradInput = conv_backward_input(geometry(input), gradOutput, weight, math);
    return gradInput;
}

void SpatialConvolutionMM::accGradParameters(const DeviceTensor& input, const DeviceTensor& gradOutput,
                                             float scale) {
    conv_backward_weight(geometry(input), input, gradOutput, gradWeight, &gradBias, scale, true, math);
}

const DeviceTensor& SpatialConvolutionMM::backward(const DeviceTensor& input, const DeviceTensor& gradOutput,
                                                   float scale) {
    const ConvGeometry g = geometry(input);
    gradInput = DeviceTensor::empty({g.batch, g.inChannels, g.inHeight, g.inWidth});
    const pt_conv_geom a = g.abi();
    const std::size_t n = ws_bytes(g, PT_CONV_BWD, math);
    // the saved finput stands for `input` only if it is the tensor updateOutput saw
    const float* fin = finputFor_ == input.data() ? finput.data() : nullptr;
    throw_if_error(pt_b200_conv_bwd_finput(&a, input.data(), gradOutput.data(), weight.data(),
                                           gradInput.data(), gradWeight.data(), gradBias.data(), scale, 1,
                                           static_cast<int>(math), scratch(nullptr, n), n, fin, nullptr));
    return gradInput;
}

void SpatialConvolutionMM::zeroGradParameters() {
    throw_if_error(pt_b200_fill_uniform(gradWeight.data(), gradWeight.numel(), 0, 0.0f, 0.0f, nullptr));
    throw_if_error(pt_b200_fill_uniform(gradBias.data(), gradBias.numel(), 0, 0.0f, 0.0f, nullptr));
}

}  // namespace portten::conv
