// s2d.cu — space-to-depth re-indexing of a strided small-channel convolution.
//
// A stride-s convolution with few input channels (AlexNet / Overfeat conv1: C = 3,
// 11x11, stride 4) maps badly onto the tensor cores: 3 useful channels per 32-channel
// (or 4-channel) operand slot and one tiny gather per tap. Splitting the padded input
// into s x s phases turns it into a STRIDE-1 convolution over C*s*s channels with a
// ceil(k/s) x ceil(k/s) filter (taps beyond k are zero):
//
//   x'[n][(c,a,b)][I][J] = x[n][c][s*I + a - pH][s*J + b - pW]          (0 outside)
//   W'[k][(c,a,b)][p][q] = W[k][c][s*p + a][s*q + b]                      (0 if >= k)
//   y[n][k][i][j]        = sum_{(c,a,b),p,q} x'[n][(c,a,b)][i+p][j+q] W'[k][(c,a,b)][p][q]
//
// which is exactly SPEC.md:353-361's conv_direct sum regrouped (every (r, s) tap of the
// original appears once as (p, a) / (q, b)). The backward passes follow: gx is the
// depth-to-space gather of gx' (each input pixel is one x' element), gW the gather of
// gW'. Output y and gradBias are untouched.
#include "kernels.cuh"

namespace ptb {

namespace {

// One block per (n, c, a, I): the padded input row s*I + a - pH is read once, coalesced,
// and scattered into the s phase planes b of x' (thread t = padded column: plane t % s,
// column t / s). Reading each phase plane's row separately would stride the loads by s.
template <int S>
__global__ void s2d_input_kernel(const float* __restrict__ x, float* __restrict__ xs, int rows, int C,
                                 int H, int W, int pH, int pW, int Hs, int Ws) {
    const int row = blockIdx.x;  // (n, c, a, I)
    const int I = row % Hs;
    const int a = (row / Hs) % S;
    const int c = (row / (Hs * S)) % C;
    const int n = row / (Hs * S * C);
    const int h = S * I + a - pH;
    const bool hin = h >= 0 && h < H;
    const float* src = x + (((int64_t)n * C + c) * H + (hin ? h : 0)) * W;
    const int64_t plane = (int64_t)Hs * Ws;
    float* dst = xs + (((int64_t)n * C * S * S + (int64_t)(c * S + a) * S) * Hs + I) * Ws;
    for (int t = threadIdx.x; t < Ws * S; t += blockDim.x) {
        const int w = t - pW;
        const float v = (hin && w >= 0 && w < W) ? __ldg(src + w) : 0.f;
        dst[(t % S) * plane + t / S] = v;
    }
}

__device__ __forceinline__ float to_tf32_s2d(float v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
}

// x' straight into the tensor-core engines' NHWC layout, channels zero-padded to Cp and
// rounded to TF32 (what s2d_input + nchw_to_nhwc produce, in one HBM pass). One block per
// (n, I): the C*S input rows s*I + a - pH are staged in smem (coalesced), then the Ws x Cp
// output row is written as float4 channel quads (Cp % 4 == 0; S = 4 or 8: a quad is
// four b phases of one (c, a); S = 2: two (c, a) pairs).
template <int S>
__global__ void s2d_input_nhwc_kernel(const float* __restrict__ x, float4* __restrict__ xh, int C, int H,
                                      int W, int pH, int pW, int Hs, int Ws, int Cp, int vec_load) {
    extern __shared__ float tile[];  // [C*S][Ws*S]
    const int I = blockIdx.x % Hs;
    const int n = blockIdx.x / Hs;
    const int Wt = Ws * S;
    const int tid = threadIdx.y * blockDim.x + threadIdx.x, nthr = blockDim.x * blockDim.y;
    // padded columns t < pW or t >= pW + W read as zero
    const int lo = pW < Wt ? pW : Wt, hi = pW + W < Wt ? pW + W : Wt;
    for (int e = tid; e < C * S * (Wt - (hi - lo)); e += nthr) {
        const int nb = Wt - (hi - lo), ca = e / nb, k = e - ca * nb;
        tile[ca * Wt + (k < lo ? k : k + (hi - lo))] = 0.f;
    }
    if (vec_load && W / 4 <= (int)blockDim.x) {
        // one (c, a) row per threadIdx.y, one float4 per lane: no index division, all of a
        // thread's loads issued before the first store
        const int nq = W / 4, q = (int)threadIdx.x;
#pragma unroll 4
        for (int ca = threadIdx.y; ca < C * S; ca += blockDim.y) {
            const int c = ca / S, a = ca - c * S;
            const int h = S * I + a - pH;
            if (q >= nq) continue;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (h >= 0 && h < H) v = __ldg(reinterpret_cast<const float4*>(x + (((int64_t)n * C + c) * H + h) * W) + q);
            float* t = tile + ca * Wt + pW + 4 * q;
            const int room = Wt - (pW + 4 * q);
            if (room >= 4) {
                t[0] = v.x; t[1] = v.y; t[2] = v.z; t[3] = v.w;
            } else {
                if (room > 0) t[0] = v.x;
                if (room > 1) t[1] = v.y;
                if (room > 2) t[2] = v.z;
            }
        }
    } else if (vec_load) {  // W % 4 == 0 and x 16-byte aligned: float4 loads, several in flight
        const int nq = W / 4;
#pragma unroll 4
        for (int e = tid; e < C * S * nq; e += nthr) {
            const int ca = e / nq, q = e - ca * nq;
            const int c = ca / S, a = ca - c * S;
            const int h = S * I + a - pH;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (h >= 0 && h < H) v = __ldg(reinterpret_cast<const float4*>(x + (((int64_t)n * C + c) * H + h) * W) + q);
            float* t = tile + ca * Wt + pW + 4 * q;
            const int room = Wt - (pW + 4 * q);
            if (room >= 4) {
                t[0] = v.x; t[1] = v.y; t[2] = v.z; t[3] = v.w;
            } else {
                if (room > 0) t[0] = v.x;
                if (room > 1) t[1] = v.y;
                if (room > 2) t[2] = v.z;
            }
        }
    } else {  // one (c, a) row per threadIdx.y, threads sweep the columns
        for (int ca = threadIdx.y; ca < C * S; ca += blockDim.y) {
            const int c = ca / S, a = ca - c * S;
            const int h = S * I + a - pH;
            if (h < 0 || h >= H) {
                for (int t = lo + threadIdx.x; t < hi; t += blockDim.x) tile[ca * Wt + t] = 0.f;
                continue;
            }
            const float* src = x + (((int64_t)n * C + c) * H + h) * W - pW;
#pragma unroll 4
            for (int t = lo + threadIdx.x; t < hi; t += blockDim.x) tile[ca * Wt + t] = __ldg(src + t);
        }
    }
    __syncthreads();
    const int Cs = C * S * S, q4 = Cp / 4;
    float4* dst = xh + ((int64_t)n * Hs + I) * Ws * q4;
    if (nthr % q4 == 0) {
        // each thread always writes the same four channels: their tile offsets are decoded
        // once (the per-element decode made this pass issue-bound: 49 M instructions for
        // 127 MB, 2.3 TB/s)
        const int ch0 = (tid % q4) * 4;
        int off[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int ch = ch0 + u;
            off[u] = ch < Cs ? (ch / S) * Wt + (ch % S) : -1;
        }
        const int jstep = nthr / q4;
#pragma unroll 4
        for (int J = tid / q4; J < Ws; J += jstep) {
            float v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = off[u] >= 0 ? to_tf32_s2d(tile[off[u] + J * S]) : 0.f;
            dst[(int64_t)J * q4 + (tid % q4)] = make_float4(v[0], v[1], v[2], v[3]);
        }
        return;
    }
    for (int e = tid; e < Ws * q4; e += nthr) {
        const int J = e / q4, ch0 = (e - J * q4) * 4;
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int ch = ch0 + u;
            const int ca = ch / S, b = ch - ca * S;
            v[u] = ch < Cs ? to_tf32_s2d(tile[ca * Wt + J * S + b]) : 0.f;
        }
        dst[e] = make_float4(v[0], v[1], v[2], v[3]);
    }
}

__global__ void s2d_weight_kernel(const float* __restrict__ w, float* __restrict__ ws, int64_t K, int C,
                                  int kH, int kW, int s, int kHs, int kWs) {
    const int Cs = C * s * s;
    const int64_t total = K * Cs * (int64_t)kHs * kWs;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int q = (int)(e % kWs);
        const int p = (int)((e / kWs) % kHs);
        const int cs = (int)((e / ((int64_t)kWs * kHs)) % Cs);
        const int64_t k = e / ((int64_t)kWs * kHs * Cs);
        const int c = cs / (s * s), a = (cs / s) % s, b = cs % s;
        const int r = s * p + a, t = s * q + b;
        ws[e] = (r < kH && t < kW) ? __ldg(w + ((k * C + c) * kH + r) * (int64_t)kW + t) : 0.f;
    }
}

// gx[n][c][h][w] = gx'[n][(c, (h+pH)%S, (w+pW)%S)][(h+pH)/S][(w+pW)/S]; one gx row per
// (blockIdx.x, threadIdx.y), threads sweep w (compile-time S: no runtime divisions).
template <int S>
__global__ void d2s_grad_kernel(const float* __restrict__ gxs, float* __restrict__ gx, int rows, int C,
                                int H, int W, int pH, int pW, int Hs, int Ws) {
    const int row = blockIdx.x * blockDim.y + threadIdx.y;  // (n, c, h)
    if (row >= rows) return;
    const int h = row % H;
    const int c = (row / H) % C;
    const int n = row / (H * C);
    const int hh = h + pH, I = hh / S;
    float* dst = gx + (int64_t)row * W;
    // pixels past the last output's receptive field get no gradient
    const float* src = gxs + (((int64_t)n * C * S * S + (c * S + hh % S) * S) * Hs + I) * (int64_t)Ws;
    const int64_t plane = (int64_t)Hs * Ws;
    for (int w = threadIdx.x; w < W; w += blockDim.x) {
        const int ww = w + pW, J = ww / S;
        dst[w] = (I < Hs && J < Ws) ? __ldg(src + (ww % S) * plane + J) : 0.f;
    }
}

// Four consecutive w per thread (four independent phase-plane loads in flight, one float4
// store): the one-element-per-thread form above ran latency-bound at ~1.6 TB/s.
template <int S>
__global__ void d2s_grad4_kernel(const float* __restrict__ gxs, float4* __restrict__ gx4, int rows, int C, int H,
                                 int W, int pH, int pW, int Hs, int Ws) {
    const int row = blockIdx.x * blockDim.y + threadIdx.y;  // (n, c, h)
    if (row >= rows) return;
    const int h = row % H;
    const int c = (row / H) % C;
    const int n = row / (H * C);
    const int hh = h + pH, I = hh / S;
    const int64_t plane = (int64_t)Hs * Ws;
    const float* src = gxs + (((int64_t)n * C * S * S + (c * S + hh % S) * S) * Hs + I) * (int64_t)Ws;
    float4* dst = gx4 + (int64_t)row * (W / 4);
    for (int w4 = threadIdx.x; w4 < W / 4; w4 += blockDim.x) {
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int ww = 4 * w4 + u + pW, J = ww / S;
            v[u] = (I < Hs && J < Ws) ? __ldg(src + (ww % S) * plane + J) : 0.f;
        }
        dst[w4] = make_float4(v[0], v[1], v[2], v[3]);
    }
}

// gw[k][c][r][t] = (acc ? gw : 0) + scale * gW'[k][(c, r%s, t%s)][r/s][t/s]
__global__ void d2s_weight_grad_kernel(const float* __restrict__ gws, float* __restrict__ gw, int64_t K,
                                       int C, int kH, int kW, int s, int kHs, int kWs, float scale,
                                       int accumulate) {
    const int64_t total = K * C * (int64_t)kH * kW;
    const int Cs = C * s * s;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int t = (int)(e % kW);
        const int r = (int)((e / kW) % kH);
        const int c = (int)((e / ((int64_t)kW * kH)) % C);
        const int64_t k = e / ((int64_t)kW * kH * C);
        const int cs = (c * s + r % s) * s + t % s;
        const float v = __ldg(gws + ((k * Cs + cs) * kHs + r / s) * (int64_t)kWs + t / s);
        gw[e] = (accumulate ? gw[e] : 0.f) + scale * v;
    }
}

unsigned blocks_for(int64_t total) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 16 * (int64_t)sm_count()));
}

}  // namespace

bool s2d_applies(const Geo& g) {
    const int64_t s = g.sH;
    if (!(s == 2 || s == 3 || s == 4 || s == 8) || g.sW != s || g.C * s * s > 64 || g.kH < s || g.kW < s) return false;
    if (g.N * g.C * g.H >= (1ll << 31)) return false;  // 32-bit row indices
    const Geo e = s2d_geo(g);
    // the regrouped filter may not inflate the contraction by more than 1.5x
    return e.CRS * 2 <= g.CRS * 3 && e.N * e.C * e.H * e.W < (1ll << 31);
}

Geo s2d_geo(const Geo& g) {
    const int64_t s = g.sH;
    const int64_t kHs = (g.kH + s - 1) / s, kWs = (g.kW + s - 1) / s;
    pt_conv_geom e{g.N, g.C * s * s, g.oH + kHs - 1, g.oW + kWs - 1, g.K, kHs, kWs, 0, 0, 1, 1};
    return Geo(e);
}

void s2d_input(const Geo& g, const float* x, float* xs, cudaStream_t st) {
    const Geo e = s2d_geo(g);
    ProfScope prof("layout", st, 0.0, 4.0 * (g.N * g.C * g.HW + e.N * e.C * e.HW));
    const int rows = (int)(g.N * g.C * g.sH * e.H);  // (n, c, a, I)
    const int tb = (int)std::min<int64_t>(256, align_up((size_t)(e.W * g.sH), 32));
#define PTB_S2D_IN(S_)                                                                             \
    s2d_input_kernel<S_><<<(unsigned)rows, tb, 0, st>>>(x, xs, rows, (int)g.C, (int)g.H, (int)g.W, \
                                                        (int)g.pH, (int)g.pW, (int)e.H, (int)e.W)
    if (g.sH == 2) PTB_S2D_IN(2);
    else if (g.sH == 3) PTB_S2D_IN(3);
    else if (g.sH == 4) PTB_S2D_IN(4);
    else PTB_S2D_IN(8);
#undef PTB_S2D_IN
    after_launch("s2d_input");
}

bool s2d_nhwc_ok(const Geo& g, int64_t Cp) {
    const Geo e = s2d_geo(g);
    return Cp % 4 == 0 && Cp >= e.C && (size_t)(g.C * g.sH * e.W * g.sH) * 4 <= 48 * 1024 &&
           g.N * e.H < (1ll << 31);
}

void s2d_input_nhwc(const Geo& g, const float* x, float* xh, int64_t Cp, cudaStream_t st) {
    const Geo e = s2d_geo(g);
    PTB_REQUIRE(s2d_nhwc_ok(g, Cp), "s2d_input_nhwc: unsupported geometry");
    ProfScope prof("layout", st, 0.0, 4.0 * (g.N * g.C * g.HW + e.N * e.HW * Cp));
    const size_t smem = (size_t)(g.C * g.sH * e.W * g.sH) * 4;
    const dim3 blk(64, 4);
#define PTB_S2D_NHWC(S_)                                                                                  \
    s2d_input_nhwc_kernel<S_><<<(unsigned)(g.N * e.H), blk, smem, st>>>(                                    \
        x, reinterpret_cast<float4*>(xh), (int)g.C, (int)g.H, (int)g.W, (int)g.pH, (int)g.pW, (int)e.H, \
        (int)e.W, (int)Cp, vec)
    const int vec = (g.W % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) ? 1 : 0;
    if (g.sH == 2) PTB_S2D_NHWC(2);
    else if (g.sH == 3) PTB_S2D_NHWC(3);
    else if (g.sH == 4) PTB_S2D_NHWC(4);
    else PTB_S2D_NHWC(8);
#undef PTB_S2D_NHWC
    after_launch("s2d_input_nhwc");
}

void s2d_weight(const Geo& g, const float* w, float* ws, cudaStream_t st) {
    const Geo e = s2d_geo(g);
    s2d_weight_kernel<<<blocks_for(e.K * e.CRS), 256, 0, st>>>(w, ws, g.K, (int)g.C, (int)g.kH, (int)g.kW,
                                                               (int)g.sH, (int)e.kH, (int)e.kW);
    after_launch("s2d_weight");
}

void d2s_grad(const Geo& g, const float* gxs, float* gx, cudaStream_t st) {
    const Geo e = s2d_geo(g);
    ProfScope prof("layout", st, 0.0, 4.0 * (g.N * g.C * g.HW * 2));
    const int rows = (int)(g.N * g.C * g.H);
    if (g.W % 4 == 0 && (reinterpret_cast<uintptr_t>(gx) & 15) == 0) {
        const int tx = g.W / 4 >= 64 ? 64 : 32;
        const dim3 blk(tx, 256 / tx);
#define PTB_D2S4(S_)                                                                                    \
    d2s_grad4_kernel<S_><<<(unsigned)ceil_div(rows, (int)blk.y), blk, 0, st>>>(                       \
        gxs, reinterpret_cast<float4*>(gx), rows, (int)g.C, (int)g.H, (int)g.W, (int)g.pH, (int)g.pW,   \
        (int)e.H, (int)e.W)
        if (g.sH == 2) PTB_D2S4(2);
        else if (g.sH == 3) PTB_D2S4(3);
        else if (g.sH == 4) PTB_D2S4(4);
        else PTB_D2S4(8);
#undef PTB_D2S4
        after_launch("d2s_grad4");
        return;
    }
#define PTB_D2S(S_)                                                                                    \
    d2s_grad_kernel<S_><<<(unsigned)ceil_div(rows, 2), dim3(128, 2), 0, st>>>(                         \
        gxs, gx, rows, (int)g.C, (int)g.H, (int)g.W, (int)g.pH, (int)g.pW, (int)e.H, (int)e.W)
    if (g.sH == 2) PTB_D2S(2);
    else if (g.sH == 3) PTB_D2S(3);
    else if (g.sH == 4) PTB_D2S(4);
    else PTB_D2S(8);
#undef PTB_D2S
    after_launch("d2s_grad");
}

void d2s_weight_grad(const Geo& g, const float* gws, float* gw, float scale, int accumulate,
                     cudaStream_t st) {
    const Geo e = s2d_geo(g);
    d2s_weight_grad_kernel<<<blocks_for(g.K * g.CRS), 256, 0, st>>>(gws, gw, g.K, (int)g.C, (int)g.kH,
                                                                    (int)g.kW, (int)g.sH, (int)e.kH,
                                                                    (int)e.kW, scale, accumulate);
    after_launch("d2s_weight_grad");
}

}  // namespace ptb
