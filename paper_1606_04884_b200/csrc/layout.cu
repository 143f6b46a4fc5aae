// layout.cu — HBM-bound layout passes around the tensor-core convolution:
//   * NCHW -> NHWC (channels-innermost, the layout TMA im2col mode gathers from),
//     zero-padding channels and rounding to TF32 in the same pass;
//   * weight packing (KCRS -> implicit-GEMM B operand, optionally flipped for dgrad);
//   * gradBias, a per-channel reduction of gradOutput (the reference's
//     reduce over gy.select(1,k), proj/src/reference_backend.cpp:115-127).
#include <cstdlib>

#include "kernels.cuh"

namespace ptb {

namespace {

__device__ __forceinline__ float to_tf32(float v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
}

// Tile transpose through smem: a block owns 32 channels x kStripPx pixels of one
// image, moved as 32x32 tiles (reads coalesced along pixels, writes coalesced along
// channels). With `part` set it also emits the block's per-channel sums of the
// UNROUNDED source (the gradBias partials, fixed order -> deterministic):
// part[c * (N * strips) + n * strips + strip] (channel-major: the final reduce reads each
// channel's partials contiguously). grid = (strips, ceil(Cp/32), N), block = 32x8.
constexpr int kStripPx = 128;

// PAD: destinations are zero-bordered (pixel index remapped); TWO: write d1 as well.
template <bool PAD, bool TWO>
__global__ void nchw_to_nhwc_kernel(const float* __restrict__ src, NhwcDst d0, NhwcDst d1,
                                    int64_t C, int64_t HW, int64_t Cp, int round_tf32,
                                    float* __restrict__ part) {
    // the whole 32-channel x 128-pixel strip is loaded before the first barrier: 16
    // independent loads per thread keep enough bytes in flight to run at HBM rate
    // (one 32x32 tile per barrier capped this pass at ~3.3 TB/s)
    __shared__ float tile[32][kStripPx + 1];
    const int64_t n = blockIdx.z;
    const int64_t c0 = (int64_t)blockIdx.y * 32;
    const float* s = src + n * C * HW;
    float* o0 = d0.p + n * d0.img * Cp;
    float* o1 = TWO ? d1.p + n * d1.img * Cp : nullptr;
    const int64_t p0 = (int64_t)blockIdx.x * kStripPx;
    float rowsum[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t c = c0 + threadIdx.y + 8 * i;
        const float* sc = s + c * HW + p0;
#pragma unroll
        for (int t = 0; t < kStripPx / 32; ++t) {
            const int64_t p = p0 + threadIdx.x + 32 * t;
            const float v = (c < C && p < HW) ? __ldg(sc + threadIdx.x + 32 * t) : 0.f;
            tile[threadIdx.y + 8 * i][threadIdx.x + 32 * t] = v;
            rowsum[i] += v;
        }
    }
    __syncthreads();
    const int64_t c = c0 + threadIdx.x;
    // zero-bordered destinations: (h, w) of this thread's pixel advanced incrementally
    // (a division per element made the padded pass ALU-bound)
    const int Wd = (int)(PAD ? d0.W : d1.W);
    int ph_ = (int)((p0 + threadIdx.y) / Wd), pw_ = (int)((p0 + threadIdx.y) - (int64_t)ph_ * Wd);
#pragma unroll 4
    for (int k = 0; k < kStripPx / 8; ++k) {
        const int pl = threadIdx.y + 8 * k;
        const int64_t p = p0 + pl;
        if (p < HW && c < Cp) {
            float v = tile[threadIdx.x][pl];
            if (round_tf32) v = to_tf32(v);
            if constexpr (PAD) {
                o0[((ph_ + d0.ph) * d0.Wp + pw_ + d0.pw) * Cp + c] = v;
                if constexpr (TWO) o1[((ph_ + d1.ph) * d1.Wp + pw_ + d1.pw) * Cp + c] = v;
            } else {
                o0[p * Cp + c] = v;
                if constexpr (TWO) o1[((ph_ + d1.ph) * d1.Wp + pw_ + d1.pw) * Cp + c] = v;
            }
        }
        if constexpr (PAD || TWO) {
            pw_ += 8;
            while (pw_ >= Wd) {
                pw_ -= Wd;
                ++ph_;
            }
        }
    }
    if (part) {
        // reduce each channel row's 32 lanes (warp = fixed threadIdx.y -> fixed channels)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float v = rowsum[i];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            const int64_t c = c0 + threadIdx.y + 8 * i;
            if (threadIdx.x == 0 && c < C) part[c * (gridDim.z * gridDim.x) + n * gridDim.x + blockIdx.x] = v;
        }
    }
}

// Zero the spatial border of a padded NHWC image stack dst[n][Hp][Wp][Cp]: only the
// border pixels are visited (top/bottom rows, then the left/right columns of the
// interior rows), float4 stores.
__global__ void zero_border_kernel(float4* __restrict__ dst, int64_t N, int Hp, int Wp, int ph, int pw,
                                   int H, int cp4) {
    const int64_t per_img = 2ll * ph * Wp + 2ll * H * pw;  // border pixels per image
    const int64_t total = N * per_img * cp4;
    const int W = Wp - 2 * pw;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t bp = e / cp4;
        const int c4 = (int)(e - bp * cp4);
        const int64_t n = bp / per_img;
        int64_t b = bp - n * per_img;
        int h, w;
        if (b < 2ll * ph * Wp) {
            const int r = (int)(b / Wp);
            w = (int)(b - (int64_t)r * Wp);
            h = r < ph ? r : H + r;  // rows [0, ph) and [ph + H, Hp)
        } else {
            b -= 2ll * ph * Wp;
            const int r = (int)(b / (2 * pw)), k = (int)(b - (int64_t)r * 2 * pw);
            h = ph + r;
            w = k < pw ? k : W + k;
        }
        dst[((n * Hp + h) * Wp + w) * cp4 + c4] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

// gb[k] = (acc ? gb[k] : 0) + scale * sum_r part[k * rows + r], r over N*strips (each
// thread's strided share in order, then a fixed tree: deterministic).
__global__ void bias_from_partials_kernel(const float* __restrict__ part, int64_t rows, int64_t K,
                                          float* __restrict__ gb, float scale, int accumulate) {
    const int64_t k = blockIdx.x;
    float acc = 0.f;
    const float* pk = part + k * rows;
    for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) acc += __ldg(pk + r);
    __shared__ float red[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        acc = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (threadIdx.x == 0) gb[k] = (accumulate ? gb[k] : 0.f) + scale * acc;
    }
}

// Small-channel variant (Cp <= 8): one thread per pixel writes its Cp-vector.
__global__ void nchw_to_nhwc_small_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                          int64_t N, int64_t C, int64_t HW, int64_t Cp,
                                          int round_tf32) {
    const int64_t total = N * HW;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t n = i / HW, p = i - n * HW;
        const float* s = src + n * C * HW + p;
        float* d = dst + i * Cp;
        for (int64_t c = 0; c < Cp; ++c) {
            float v = c < C ? __ldg(s + c * HW) : 0.f;
            d[c] = round_tf32 ? to_tf32(v) : v;
        }
    }
}

// 32-bit index math throughout (a 64-bit division per element made these packs of a few
// MB take 10-13 us); the caller guarantees total < 2^31.
__global__ void pack_weights_kernel(const float* __restrict__ w, float* __restrict__ dst,
                                    int K, int C, int kH, int kW, int mode,
                                    int layout, int n_pad, int cin_p, int slots_p,
                                    int total, int round_tf32) {
    const int taps = mode == kPackGcol ? 1 : kH * kW;
    const int n_real = mode == kPackFprop ? K : (mode == kPackDgradFlip ? C : C * kH * kW);
    const int cin_real = mode == kPackFprop ? C : K;
    const int chunks = cin_p / 4;
    const int kdim_p = total / n_pad;  // layout 32: row stride (>= taps*cin_p)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        int row, tap, ch;
        if (layout == 32) {
            row = i / kdim_p;
            const int kd = i - row * kdim_p;
            tap = kd / cin_p;
            ch = kd - tap * cin_p;
        } else {
            const int e = i & 3;
            const int q = i >> 2;
            row = q % n_pad;
            const int slot = q / n_pad;
            tap = slot / chunks;
            ch = (slot - tap * chunks) * 4 + e;
        }
        float v = 0.f;
        if (row < n_real && ch < cin_real && tap < taps) {
            const int r = tap / kW, s = tap - r * kW;
            if (mode == kPackFprop) {
                v = __ldg(w + ((row * C + ch) * kH + r) * kW + s);
            } else if (mode == kPackDgradFlip) {  // B[c][(r',s')][k] = W[k][c][kH-1-r'][kW-1-s']
                v = __ldg(w + ((ch * C + row) * kH + (kH - 1 - r)) * kW + (kW - 1 - s));
            } else {  // B[(c,r,s)][k] = W[k][(c,r,s)]
                v = __ldg(w + ch * C * kH * kW + row);
            }
        }
        dst[i] = round_tf32 ? to_tf32(v) : v;
    }
}

// Stage 1: block (k, split) sums its contiguous share of the N*HW run of channel k.
__global__ void bias_grad_partial_kernel(const float* __restrict__ gy, float* __restrict__ part,
                                         int64_t N, int64_t K, int64_t HW, int splits) {
    const int64_t k = blockIdx.x;
    const int split = blockIdx.y;
    const int64_t total = N * HW;
    const int64_t per = (total + splits - 1) / splits;
    const int64_t lo = split * per, hi = lo + per < total ? lo + per : total;
    float acc = 0.f;
    // walk the images overlapping [lo, hi); consecutive threads read consecutive p
    for (int64_t n = lo / HW; n * HW < hi; ++n) {
        const int64_t p0 = lo > n * HW ? lo - n * HW : 0;
        const int64_t p1 = hi - n * HW < HW ? hi - n * HW : HW;
        const float* src = gy + (n * K + k) * HW;
        for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) acc += __ldg(src + p);
    }
    __shared__ float red[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        acc = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (threadIdx.x == 0) part[k * splits + split] = acc;
    }
}

__global__ void bias_grad_final_kernel(const float* __restrict__ part, float* __restrict__ gb,
                                       int64_t K, int splits, float scale, int accumulate) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= K) return;
    float s = 0.f;
    for (int i = 0; i < splits; ++i) s += part[k * splits + i];
    gb[k] = (accumulate ? gb[k] : 0.f) + scale * s;
}

int bias_splits(int64_t N, int64_t K, int64_t HW) {
    const int64_t per_split = 1 << 16;  // >= 64K elements per block
    int64_t s = (N * HW + per_split - 1) / per_split;
    const int64_t want = (4 * (int64_t)sm_count() + K - 1) / K;
    if (s > want) s = want;
    if (s < 1) s = 1;
    if (s > 1024) s = 1024;
    return (int)s;
}

}  // namespace

void nchw_to_nhwc(const float* src, float* dst, int64_t N, int64_t C, int64_t HW, int64_t Cp,
                  bool round_tf32, cudaStream_t st) {
    if (Cp <= 8) {
        const int64_t total = N * HW;
        const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 8 * (int64_t)sm_count());
        nchw_to_nhwc_small_kernel<<<blocks, 256, 0, st>>>(src, dst, N, C, HW, Cp, round_tf32);
        after_launch("nchw_to_nhwc_small");
        return;
    }
    PTB_REQUIRE(N <= 65535, "nchw_to_nhwc: batch too large");
    dim3 grid((unsigned)ceil_div(HW, kStripPx), (unsigned)ceil_div(Cp, 32), (unsigned)N);
    nchw_to_nhwc_kernel<false, false><<<grid, dim3(32, 8), 0, st>>>(src, NhwcDst::dense(dst, HW), NhwcDst{},
                                                                     C, HW, Cp, round_tf32, nullptr);
    after_launch("nchw_to_nhwc");
}

void nchw_to_nhwc_padded(const float* src, const NhwcDst& d0, const NhwcDst& d1, int64_t N,
                         int64_t C, int64_t H, int64_t W, int64_t Cp, float* gb, float scale,
                         int accumulate, float* part, cudaStream_t st) {
    PTB_REQUIRE(N <= 65535 && Cp >= C && Cp % 4 == 0, "nchw_to_nhwc_padded: bad shape");
    const int64_t HW = H * W;
    for (const NhwcDst* d : {&d0, &d1}) {
        if (!d->p || d->img == HW) continue;
        const int Hp = (int)(d->img / d->Wp);
        const int64_t total = N * (2 * d->ph * d->Wp + 2 * H * d->pw) * (Cp / 4);
        if (total == 0) continue;
        const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 8 * (int64_t)sm_count());
        zero_border_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<float4*>(d->p), N, Hp, (int)d->Wp,
                                                   (int)d->ph, (int)d->pw, (int)H, (int)(Cp / 4));
        after_launch("zero_border");
    }
    const int64_t strips = ceil_div(HW, kStripPx);
    dim3 grid((unsigned)strips, (unsigned)ceil_div(Cp, 32), (unsigned)N);
    float* pp = gb ? part : nullptr;
    const bool pad = d0.img != HW;
    if (d1.p) {
        if (pad) nchw_to_nhwc_kernel<true, true><<<grid, dim3(32, 8), 0, st>>>(src, d0, d1, C, HW, Cp, 1, pp);
        else nchw_to_nhwc_kernel<false, true><<<grid, dim3(32, 8), 0, st>>>(src, d0, d1, C, HW, Cp, 1, pp);
    } else {
        if (pad) nchw_to_nhwc_kernel<true, false><<<grid, dim3(32, 8), 0, st>>>(src, d0, d1, C, HW, Cp, 1, pp);
        else nchw_to_nhwc_kernel<false, false><<<grid, dim3(32, 8), 0, st>>>(src, d0, d1, C, HW, Cp, 1, pp);
    }
    after_launch("nchw_to_nhwc_padded");
    if (gb) {
        bias_from_partials_kernel<<<(unsigned)C, 1024, 0, st>>>(part, N * strips, C, gb, scale,
                                                               accumulate);
        after_launch("bias_from_partials");
    }
}

size_t nhwc_bias_partials_bytes(int64_t N, int64_t C, int64_t HW) {
    return sizeof(float) * (size_t)(N * ceil_div(HW, kStripPx) * C);
}

void nchw_to_nhwc_bias(const float* src, float* dst, int64_t N, int64_t C, int64_t HW, int64_t Cp,
                       float* gb, float scale, int accumulate, float* part, cudaStream_t st, bool defer_bias) {
    PTB_REQUIRE(N <= 65535 && Cp >= C, "nchw_to_nhwc_bias: bad shape");
    const int64_t strips = ceil_div(HW, kStripPx);
    dim3 grid((unsigned)strips, (unsigned)ceil_div(Cp, 32), (unsigned)N);
    nchw_to_nhwc_kernel<false, false><<<grid, dim3(32, 8), 0, st>>>(src, NhwcDst::dense(dst, HW), NhwcDst{},
                                                                     C, HW, Cp, 1, gb ? part : nullptr);
    after_launch("nchw_to_nhwc_bias");
    if (gb && !defer_bias) bias_from_nhwc_partials(part, N, C, HW, gb, scale, accumulate, st);
}

void bias_from_nhwc_partials(const float* part, int64_t N, int64_t C, int64_t HW, float* gb, float scale,
                             int accumulate, cudaStream_t st) {
    bias_from_partials_kernel<<<(unsigned)C, 1024, 0, st>>>(part, N * ceil_div(HW, kStripPx), C, gb, scale,
                                                           accumulate);
    after_launch("bias_from_partials");
}

void pack_weights(const float* w, float* dst, int64_t K, int64_t C, int64_t kH, int64_t kW,
                  int mode, int layout, int64_t n_pad, int64_t cin_p, int64_t slots_p,
                  int64_t total, bool round_tf32, cudaStream_t st) {
    PTB_REQUIRE(total < (1ll << 31) && K * C * kH * kW < (1ll << 31), "pack_weights: weights too large");
    const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 32 * (int64_t)sm_count());
    pack_weights_kernel<<<blocks, 256, 0, st>>>(w, dst, (int)K, (int)C, (int)kH, (int)kW, mode, layout,
                                                (int)n_pad, (int)cin_p, (int)slots_p, (int)total, round_tf32);
    after_launch("pack_weights");
}

// Tap-grouped packing for the Hankel engine's G-tap MMAs: rows of group (r, sg) are the
// (delta, n) stack of taps (r, sg*G + delta), so one CTA's G*bn/2 rows are contiguous:
// dst[((r*ng + sg)*G + delta)*bn + n][ch], zero for taps past kW / rows past n_real.
__global__ void pack_grouped_kernel(const float* __restrict__ w, float* __restrict__ dst, int K, int C,
                                    int kH, int kW, int dgrad, int G, int ng, int bn, int cin_p,
                                    int total) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int rowi = i / cin_p;
        const int ch = i - rowi * cin_p;
        const int gd = rowi / bn;  // ((r*ng + sg)*G + delta)
        const int n = rowi - gd * bn;
        const int rs = gd / G;
        const int delta = gd - rs * G;
        const int r = rs / ng, sg = rs - r * ng;
        const int s = sg * G + delta;
        float v = 0.f;
        if (s < kW) {
            if (!dgrad) {  // row n = k, channel ch = c
                if (n < K && ch < C) v = __ldg(w + ((n * C + ch) * kH + r) * kW + s);
            } else {  // row n = c, channel ch = k, flipped tap
                if (n < C && ch < K) v = __ldg(w + ((ch * C + n) * kH + (kH - 1 - r)) * kW + (kW - 1 - s));
            }
        }
        dst[i] = to_tf32(v);
    }
}

void pack_grouped(const float* w, float* dst, int64_t K, int64_t C, int64_t kH, int64_t kW, bool dgrad,
                  int G, int bn, int64_t cin_p, cudaStream_t st) {
    const int ng = (int)ceil_div(kW, G);
    const int64_t total = kH * ng * G * (int64_t)bn * cin_p;
    PTB_REQUIRE(total < (1ll << 31) && K * C * kH * kW < (1ll << 31), "pack_grouped: weights too large");
    const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 32 * (int64_t)sm_count());
    pack_grouped_kernel<<<blocks, 256, 0, st>>>(w, dst, (int)K, (int)C, (int)kH, (int)kW, dgrad ? 1 : 0, G,
                                                ng, bn, (int)cin_p, (int)total);
    after_launch("pack_grouped");
}

size_t bias_grad_workspace(int64_t N, int64_t K, int64_t HW) {
    return sizeof(float) * (size_t)K * (size_t)bias_splits(N, K, HW);
}

void bias_grad(const float* gy, float* gb, int64_t N, int64_t K, int64_t HW, float scale,
               int accumulate, float* ws, size_t ws_bytes, cudaStream_t st) {
    const int splits = bias_splits(N, K, HW);
    PTB_REQUIRE(ws_bytes >= sizeof(float) * (size_t)K * splits, "bias_grad: workspace too small");
    PTB_REQUIRE(K <= 2147483647, "bias_grad: K too large");
    bias_grad_partial_kernel<<<dim3((unsigned)K, (unsigned)splits), 256, 0, st>>>(gy, ws, N, K, HW,
                                                                                 splits);
    after_launch("bias_grad_partial");
    bias_grad_final_kernel<<<(unsigned)ceil_div(K, 128), 128, 0, st>>>(ws, gb, K, splits, scale,
                                                                       accumulate);
    after_launch("bias_grad_final");
}

}  // namespace ptb
