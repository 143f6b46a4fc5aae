// umma_rowwgrad.cu — weight gradient for small-channel, stride-1 layers (C <= 4: the
// first layer of L1 / VGG-A; accGradParameters).
//
// With C = 3 the im2col-TMA wgrad kernel would pad every 32-channel box from 3 real
// channels (10.7x wasted MMA work). Instead the horizontal taps are folded into the
// channel dimension once, in HBM:
//   Xe[n][h][j][e],  e = s*C + c  (Ce = kW*C rounded up to 32),
//   Xe[n][h][j][s*C + c] = x[n][c][h][j*sW + s - pW]   (0 outside the image)
// so the layer becomes a (kH x 1) convolution over Xe with Ce channels, width oW and
// the same output grid:  gW'[k][e][r] = sum_{n,i,j} gy[n][k][i][j] * Xe[n][i*sH+r-pH][j][e],
// computed by the tcgen05 CTA-pair wgrad kernel (umma_wgrad.cu) with no channel waste
// beyond Ce; a remap kernel writes gW[k][c][r][s] = gW'[k][s*C + c][r] with scale /
// accumulate. (The tensor cores cannot take the un-expanded Hankel row as an MN-major
// tf32 operand: that layout needs the 32-byte-atom swizzle.)
#include <cuda.h>

#include <cstdlib>

#include "kernels.cuh"

namespace ptb {

namespace {

// One block per image row (n, h): the C input rows are staged (zero-padded, TF32-rounded)
// in shared memory, then the oW x Ce expanded row is written with consecutive threads
// storing consecutive float4s (fully coalesced).
__global__ void expand_rows_kernel(const float* __restrict__ x, float4* __restrict__ xe, int64_t rows,
                                   int C, int H, int W, int oW, int kW, int pW, int sW, int Ce) {
    extern __shared__ float srow[];  // [C][Wpad], Wpad = (oW-1)*sW + kW
    const int Wpad = (oW - 1) * sW + kW;
    for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
        const int64_t n = row / H;
        const int h = (int)(row - n * H);
        const float* xr = x + (n * C * H + h) * (int64_t)W;
        __syncthreads();
        for (int t = threadIdx.x; t < C * Wpad; t += blockDim.x) {
            const int c = t / Wpad, u = t - c * Wpad, w = u - pW;
            float f = (w >= 0 && w < W) ? __ldg(xr + (int64_t)c * H * W + w) : 0.f;
            uint32_t r;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(f));
            srow[t] = __uint_as_float(r);
        }
        __syncthreads();
        float4* dst = xe + row * (int64_t)oW * (Ce / 4);
        const int q4 = Ce / 4;
        if (blockDim.x % q4 == 0) {
            // each thread always writes the same 4 expanded channels: decode them once
            const int e0 = (threadIdx.x % q4) * 4;
            int off[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int e = e0 + q, s = e / C, c = e - s * C;
                off[q] = s < kW ? c * Wpad + s : -1;
            }
            const int jstep = blockDim.x / q4;
            for (int j = threadIdx.x / q4; j < oW; j += jstep) {
                float v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) v[q] = off[q] >= 0 ? srow[off[q] + j * sW] : 0.f;
                dst[(int64_t)j * q4 + (threadIdx.x % q4)] = make_float4(v[0], v[1], v[2], v[3]);
            }
            continue;
        }
        for (int t = threadIdx.x; t < oW * q4; t += blockDim.x) {
            const int j = t / q4, e0 = (t - j * q4) * 4;
            float v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int e = e0 + q, s = e / C, c = e - s * C;
                v[q] = s < kW ? srow[c * Wpad + j * sW + s] : 0.f;
            }
            dst[t] = make_float4(v[0], v[1], v[2], v[3]);
        }
    }
}

// gw[k][c][r][s] = (acc ? gw : 0) + scale * gwe[k][s*C + c][r]
__global__ void remap_rows_kernel(const float* __restrict__ gwe, float* __restrict__ gw, int64_t K,
                                  int C, int kH, int kW, int Ce, float scale, int accumulate) {
    const int64_t total = K * C * kH * kW;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(i % kW), r = (int)((i / kW) % kH), c = (int)((i / ((int64_t)kW * kH)) % C);
        const int64_t k = i / ((int64_t)kW * kH * C);
        const float v = gwe[(k * Ce + (s * C + c)) * kH + r];
        gw[i] = (accumulate ? gw[i] : 0.f) + scale * v;
    }
}

// W[k][c][r][s] -> W'[k][r*C + c][0][s]: the filter of the (1 x kW) column-expanded conv.
__global__ void expand_filter_v_kernel(const float* __restrict__ w, float* __restrict__ we, int64_t K, int C,
                                       int kH, int kW) {
    const int64_t total = K * C * kH * kW;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(i % kW), r = (int)((i / kW) % kH), c = (int)((i / ((int64_t)kW * kH)) % C);
        const int64_t k = i / ((int64_t)kW * kH * C);
        we[((k * kH + r) * C + c) * kW + s] = w[i];
    }
}

// gx[n][c][h][w] = sum_{r=0..kH-1} gxe[n][r*C + c][h + pH - r][w + pW]   (r in fixed order)
// gxe: [N][kH*C][oH][Wp]. One gx row per (blockIdx.x, threadIdx.y); each thread owns four
// consecutive w, so every tap issues four independent loads (kH as small as 3 would
// otherwise leave too few bytes in flight to cover HBM latency).
__global__ void fold_cols_kernel(const float* __restrict__ gxe, float* __restrict__ gx, int rows, int C,
                                 int H, int W, int oH, int Wp, int kH, int pH, int pW, int vec_store) {
    const int row = blockIdx.x * blockDim.y + threadIdx.y;  // (n, c, h)
    if (row >= rows) return;
    const int h = row % H;
    const int c = (row / H) % C;
    const int n = row / (H * C);
    const int64_t plane = (int64_t)oH * Wp;
    const float* src = gxe + ((int64_t)n * kH * C + c) * plane + pW;
    float* dst = gx + (int64_t)row * W;
    const int r0 = max(0, h + pH - oH + 1), r1 = min(kH, h + pH + 1);  // taps with a valid row
    // aligned rows (pW % 4 == 0, Wp % 4 == 0): one float4 load per tap
    const bool vec_load = vec_store && ((pW | Wp) & 3) == 0;
    for (int w0 = threadIdx.x * 4; w0 < W; w0 += blockDim.x * 4) {
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        const bool full = w0 + 4 <= W;
        if (full && vec_load) {
#pragma unroll 4
            for (int r = r0; r < r1; ++r) {
                const float4 t = __ldg(reinterpret_cast<const float4*>(
                    src + (int64_t)r * C * plane + (int64_t)(h + pH - r) * Wp + w0));
                acc[0] += t.x;
                acc[1] += t.y;
                acc[2] += t.z;
                acc[3] += t.w;
            }
        } else {
#pragma unroll 4
            for (int r = r0; r < r1; ++r) {
                const float* p = src + (int64_t)r * C * plane + (int64_t)(h + pH - r) * Wp + w0;
                if (full) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) acc[u] += __ldg(p + u);
                } else {
                    for (int u = 0; u < W - w0; ++u) acc[u] += __ldg(p + u);
                }
            }
        }
        if (full && vec_store) {
            *reinterpret_cast<float4*>(dst + w0) = make_float4(acc[0], acc[1], acc[2], acc[3]);
        } else {
            for (int u = 0; u < 4 && w0 + u < W; ++u) dst[w0 + u] = acc[u];
        }
    }
}

// W[k][c][r][s] -> W''[k][s*C + c][r][0]: the filter of the (kH x 1) row-expanded conv.
__global__ void expand_filter_kernel(const float* __restrict__ w, float* __restrict__ we, int64_t K, int C,
                                     int kH, int kW) {
    const int64_t total = K * C * kH * kW;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(i % kW), r = (int)((i / kW) % kH), c = (int)((i / ((int64_t)kW * kH)) % C);
        const int64_t k = i / ((int64_t)kW * kH * C);
        we[((k * kW * C) + s * C + c) * kH + r] = w[i];
    }
}

// gx[n][c][h][w] = sum_{s=0..kW-1} gxe[n][s*C + c][h][(w + pW - s)/sW]  (taps in fixed order)
// One block-iteration per output row (n, c, h); threads sweep w (coalesced reads per tap).
__global__ void fold_rows_kernel(const float* __restrict__ gxe, float* __restrict__ gx, int64_t N, int C,
                                 int H, int W, int oW, int kW, int pW, int sW) {
    const int64_t rows = N * C * (int64_t)H;
    const int64_t plane = (int64_t)H * oW;
    for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
        const int h = (int)(row % H);
        const int64_t nc = row / H;
        const int c = (int)(nc % C);
        const int64_t n = nc / C;
        const float* src = gxe + ((n * kW * C + c) * H + h) * (int64_t)oW;
        float* dst = gx + row * W;
        for (int w = threadIdx.x; w < W; w += blockDim.x) {
            float acc = 0.f;
            if (sW == 1) {
                // stride 1: tap s reads column w + pW - s; independent predicated loads
#pragma unroll 4
                for (int s = 0; s < kW; ++s) {
                    const int j = w + pW - s;
                    if (j >= 0 && j < oW) acc += __ldg(src + (int64_t)s * C * plane + j);
                }
            } else {
                for (int s = 0; s < kW; ++s) {
                    const int wn = w + pW - s;
                    if (wn < 0) break;
                    const int j = wn / sW;
                    if (j * sW != wn || j >= oW) continue;
                    acc += __ldg(src + (int64_t)s * C * plane + j);
                }
            }
            dst[w] = acc;
        }
    }
}

// Two expansions of a small-C stride-1 layer for its input gradient:
//  * horizontal (row): x'[(s,c)][h][j] = x[c][h][j+s-pW], a (kH x 1) conv, fold over s;
//  * vertical (col): x'[(r,c)][i][w] = xpad[c][i+r][w], a (1 x kW) conv, fold over r.
// The vertical form's (1 x kW) transposed conv is a Hankel pixel-run job (kW taps share
// one run, tap-paired for <= 64 output rows), reading gy dense with the kW-1 border as
// TMA out-of-bounds fill; the horizontal form (kH x 1) has no horizontal taps to share.
bool dgrad_vertical(const Geo& g) {
    static const int v = [] {
        const char* e = std::getenv("PT_B200_ROWDGRAD");
        return e ? std::atoi(e) : 1;  // 1 = vertical, 0 = horizontal
    }();
    return v != 0 && g.kW >= 3;
}
Geo dgrad_rows_geo(const Geo& g) {
    if (dgrad_vertical(g)) {
        pt_conv_geom e{g.N, g.kH * g.C, g.oH, g.W + 2 * g.pW, g.K, 1, g.kW, 0, 0, 1, 1};
        return Geo(e);
    }
    pt_conv_geom e{g.N, g.kW * g.C, g.H, g.oW, g.K, g.kH, 1, g.pH, 0, g.sH, 1};
    return Geo(e);
}

Geo expanded_geo(const Geo& g, int64_t Ce) {
    pt_conv_geom e{g.N, Ce, g.H, g.oW, g.K, g.kH, 1, g.pH, 0, g.sH, 1};
    return Geo(e);
}

int64_t ce_of(const Geo& g) { return (g.kW * g.C + 31) / 32 * 32; }

}  // namespace

// ---- small-C dgrad: tensor-core tconv of the row-expanded layer + 1-D fold over s ----
bool rowdgrad_ok(const Geo& g, UmmaPlan* plan) {
    if (!(g.C <= 4 && g.sH == 1 && g.sW == 1 && g.kW * g.C <= 256 && g.kH * g.C <= 256)) return false;
    if (g.N * g.kH * g.C * g.H >= (1ll << 31) || g.N * g.C * g.H >= (1ll << 31)) return false;
    const UmmaPlan pl = umma_plan(dgrad_rows_geo(g), true);
    if (plan) *plan = pl;
    return pl.ok && pl.mode == UmmaPlan::kDgradTconv;
}

size_t rowdgrad_workspace(const Geo& g) {
    UmmaPlan pl;
    if (!rowdgrad_ok(g, &pl)) return 0;
    const Geo e = dgrad_rows_geo(g);
    return align_up((size_t)(g.K * g.CRS) * 4, 256) + align_up((size_t)(e.N * e.C * e.H * e.W) * 4, 256) +
           align_up(pl.ws_bytes, 256);
}

size_t rowdgrad_act_offset(const Geo& g) {
    const Geo e = dgrad_rows_geo(g);
    return align_up((size_t)(g.K * g.CRS) * 4, 256) + align_up((size_t)(e.N * e.C * e.H * e.W) * 4, 256);
}

void rowdgrad(const Geo& g, const float* gy, const float* w, float* gx, void* ws, cudaStream_t st,
              const float* gyh_pre, bool pre_padded) {
    UmmaPlan pl;
    PTB_REQUIRE(rowdgrad_ok(g, &pl), "rowdgrad: unsupported geometry");
    const Geo e = dgrad_rows_geo(g);
    char* base = reinterpret_cast<char*>(ws);
    float* we = reinterpret_cast<float*>(base);
    float* gxe = reinterpret_cast<float*>(base + align_up((size_t)(g.K * g.CRS) * 4, 256));
    char* dws = reinterpret_cast<char*>(gxe) + align_up((size_t)(e.N * e.C * e.H * e.W) * 4, 256);
    const int64_t nw = g.K * g.CRS;
    const unsigned wb = (unsigned)std::min<int64_t>(ceil_div(nw, 256), 4 * (int64_t)sm_count());
    const bool vert = dgrad_vertical(g);
    if (vert) expand_filter_v_kernel<<<wb, 256, 0, st>>>(w, we, g.K, (int)g.C, (int)g.kH, (int)g.kW);
    else expand_filter_kernel<<<wb, 256, 0, st>>>(w, we, g.K, (int)g.C, (int)g.kH, (int)g.kW);
    after_launch("expand_filter");
    umma_conv_bwd_data(e, pl, gy, we, gxe, dws, st, gyh_pre, 2.0 * g.M * g.K * g.CRS);
    const int64_t total = g.N * g.C * g.HW;
    ProfScope prof("layout", st, 0.0, 4.0 * (e.N * e.C * e.H * e.W + total));
    if (vert) {
        const int rows = (int)(g.N * g.C * g.H);
        const int tx = g.W >= 512 ? 128 : g.W >= 256 ? 64 : 32;  // 4 columns per thread
        fold_cols_kernel<<<(unsigned)ceil_div(rows, 256 / tx), dim3(tx, 256 / tx), 0, st>>>(
            gxe, gx, rows, (int)g.C, (int)g.H, (int)g.W, (int)g.oH, (int)e.W, (int)g.kH, (int)g.pH, (int)g.pW,
            (g.W % 4 == 0 && (reinterpret_cast<uintptr_t>(gx) & 15) == 0) ? 1 : 0);
        after_launch("fold_cols");
        return;
    }
    const int64_t rows = g.N * g.C * g.H;
    fold_rows_kernel<<<(unsigned)std::min<int64_t>(rows, 128 * (int64_t)sm_count()), 128, 0, st>>>(
        gxe, gx, g.N, (int)g.C, (int)g.H, (int)g.W, (int)g.oW, (int)g.kW, (int)g.pW, (int)g.sW);
    after_launch("fold_rows");
}

bool rowwgrad_ok(const Geo& g) {
    // worthwhile when C is tiny; the expanded layer must fit the CTA-pair wgrad kernel
    if (!(g.C <= 4 && g.sW <= 8 && g.kW * g.C <= 256)) return false;
    if (g.C * ((g.oW - 1) * g.sW + g.kW) * 4 > 48 * 1024) return false;  // expand_rows staging
    return umma_wgrad_ok(expanded_geo(g, ce_of(g)));
}

size_t rowwgrad_workspace(const Geo& g) {
    if (swgrad_ok(g)) return swgrad_workspace(g);
    const int64_t Ce = ce_of(g);
    const Geo e = expanded_geo(g, Ce);
    return align_up((size_t)(g.N * g.H * g.oW * Ce) * 4, 256) + align_up((size_t)(g.K * Ce * g.kH) * 4, 256) +
           align_up(umma_wgrad_workspace(e), 256);
}

void rowwgrad(const Geo& g, const float* x, const float* gyh, float* gw, float scale, int accumulate,
              void* ws, cudaStream_t st) {
    if (swgrad_ok(g)) {  // planes of horizontal taps, one B box per row group (umma_swgrad.cu)
        swgrad(g, x, gyh, gw, scale, accumulate, ws, st);
        return;
    }
    const int64_t Ce = ce_of(g);
    const Geo e = expanded_geo(g, Ce);
    char* base = reinterpret_cast<char*>(ws);
    float* xe = reinterpret_cast<float*>(base);
    float* gwe = reinterpret_cast<float*>(base + align_up((size_t)(g.N * g.H * g.oW * Ce) * 4, 256));
    char* kws = reinterpret_cast<char*>(gwe) + align_up((size_t)(g.K * Ce * g.kH) * 4, 256);
    {
        const int64_t total = g.N * g.H * g.oW * Ce;
        ProfScope prof("layout", st, 0.0, 4.0 * (g.N * g.C * g.HW + total));
        const int64_t rows = g.N * g.H;
        const size_t smem = sizeof(float) * (size_t)(g.C * ((g.oW - 1) * g.sW + g.kW));
        PTB_REQUIRE(smem <= 48 * 1024, "expand_rows: input row too wide");
        expand_rows_kernel<<<(unsigned)std::min<int64_t>(rows, 64 * (int64_t)sm_count()), 256, smem, st>>>(
            x, reinterpret_cast<float4*>(xe), rows, (int)g.C, (int)g.H, (int)g.W, (int)g.oW, (int)g.kW,
            (int)g.pW, (int)g.sW, (int)Ce);
        after_launch("expand_rows");
    }
    // the expanded layer: Xe is already NHWC with Ce channels, gy NHWC is shared
    umma_conv_bwd_filter(e, nullptr, nullptr, gwe, 1.0f, 0, kws, st, gyh, xe, 2.0 * g.M * g.K * g.CRS);
    const int64_t n = g.K * g.CRS;
    remap_rows_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 8 * (int64_t)sm_count()), 256, 0, st>>>(
        gwe, gw, g.K, (int)g.C, (int)g.kH, (int)g.kW, (int)Ce, scale, accumulate);
    after_launch("remap_rows");
}

}  // namespace ptb
