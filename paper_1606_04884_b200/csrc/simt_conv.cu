// simt_conv.cu — FP32-FFMA implicit-GEMM convolution (PT_MATH_FP32), the tight-
// tolerance mode of the north_star, and the CUDA-core fallback for geometries the
// tcgen05 path does not take. Works directly on the reference's NCHW / KCRS
// layouts: nothing is unfolded in HBM; each CTA gathers its
// im2col tile into shared memory on the fly.
//
//   fprop : D[k][m]    = sum_q W[k][q]          * im2col(x)[q][m]        q=(c,r,s), m=(n,i,j)
//   dgrad : D[c][m_in] = sum_t W[k][c][r][s]    * gy[n][k][(h+pH-r)/sH][(w+pW-s)/sW]   t=(k,r,s)
//   wgrad : D[k][q]    = sum_m gy[n][k][i][j]   * im2col(x)[q][m]        split over m, fixed-order reduce
#include "common.cuh"
#include "kernels.cuh"

namespace ptb {

namespace {

constexpr int kThreads = 256;

// Generic CUDA-core GEMM tile: rows x cols output per CTA, BK reduction slice per
// step, register double-buffered global->smem staging. P supplies gathers.
template <class P, int BM, int BN, int BK>
__global__ void __launch_bounds__(kThreads) simt_gemm_kernel(P p) {
    constexpr int TM = BM / 16, TN = BN / 16;  // 16x16 thread grid
    constexpr int A_PER = BM * BK / kThreads, B_PER = BK * BN / kThreads;
    static_assert(A_PER >= 1 && B_PER >= 1, "tile too small");
    __shared__ __align__(16) float As[2][BK][BM + 4];
    __shared__ __align__(16) float Bs[2][BK][BN + 4];

    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    const int64_t row0 = (int64_t)blockIdx.y * BM;
    const int64_t col0 = (int64_t)blockIdx.x * BN;
    const int64_t tb = p.t_begin(blockIdx.z), te = p.t_end(blockIdx.z);

    typename P::ColCtx cctx[B_PER];
#pragma unroll
    for (int i = 0; i < B_PER; ++i) {
        const int idx = tid + i * kThreads;
        cctx[i] = p.col_ctx(col0 + idx % BN);
    }
    typename P::RowCtx rctx[A_PER];
#pragma unroll
    for (int i = 0; i < A_PER; ++i) {
        const int idx = tid + i * kThreads;
        rctx[i] = p.row_ctx(row0 + idx / BK);
    }

    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

    float ra[A_PER], rb[B_PER];
    auto load = [&](int64_t t0) {
#pragma unroll
        for (int i = 0; i < A_PER; ++i) {
            const int idx = tid + i * kThreads;
            const int64_t t = t0 + idx % BK;
            ra[i] = (t < te) ? p.a(rctx[i], row0 + idx / BK, t) : 0.f;
        }
#pragma unroll
        for (int i = 0; i < B_PER; ++i) {
            const int idx = tid + i * kThreads;
            const int64_t t = t0 + idx / BN;
            rb[i] = (t < te) ? p.b(cctx[i], t, col0 + idx % BN) : 0.f;
        }
    };
    auto stash = [&](int buf) {
#pragma unroll
        for (int i = 0; i < A_PER; ++i) {
            const int idx = tid + i * kThreads;
            As[buf][idx % BK][idx / BK] = ra[i];
        }
#pragma unroll
        for (int i = 0; i < B_PER; ++i) {
            const int idx = tid + i * kThreads;
            Bs[buf][idx / BN][idx % BN] = rb[i];
        }
    };

    int buf = 0;
    if (tb < te) {
        load(tb);
        stash(0);
    }
    __syncthreads();
    for (int64_t t0 = tb; t0 < te; t0 += BK) {
        const bool more = t0 + BK < te;
        if (more) load(t0 + BK);
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float av[TM], bv[TN];
#pragma unroll
            for (int i = 0; i < TM; i += 4) {
                const float4 v = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4 + i * 16]);
                av[i] = v.x; av[i + 1] = v.y; av[i + 2] = v.z; av[i + 3] = v.w;
            }
#pragma unroll
            for (int j = 0; j < TN; j += 4) {
                const float4 v = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4 + j * 16]);
                bv[j] = v.x; bv[j + 1] = v.y; bv[j + 2] = v.z; bv[j + 3] = v.w;
            }
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        if (more) {
            stash(buf ^ 1);
            __syncthreads();
            buf ^= 1;
        }
    }

#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int64_t row = row0 + ty * 4 + (i / 4) * 64 + (i % 4);
        if (row >= p.rows) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int64_t col = col0 + tx * 4 + (j / 4) * 64 + (j % 4);
            if (col < p.cols) p.store(row, col, acc[i][j], blockIdx.z);
        }
    }
}

// ---- problem definitions -------------------------------------------------

struct FpropP {
    const float *x, *w, *bias;
    float* y;
    int C, H, W, K, kH, kW, pH, pW, sH, sW, oH, oW;
    int64_t rows, cols, crs;
    struct RowCtx { int64_t wrow; };
    struct ColCtx { int64_t xbase; int h0, w0; bool ok; };
    __device__ int64_t t_begin(int) const { return 0; }
    __device__ int64_t t_end(int) const { return crs; }
    __device__ RowCtx row_ctx(int64_t k) const { return {k * crs}; }
    __device__ ColCtx col_ctx(int64_t m) const {
        ColCtx c{0, 0, 0, m < cols};
        if (!c.ok) return c;
        const int64_t ohw = (int64_t)oH * oW;
        const int64_t n = m / ohw;
        const int p = (int)(m - n * ohw);
        const int i = p / oW, j = p - i * oW;
        c.xbase = n * C * (int64_t)H * W;
        c.h0 = i * sH - pH;
        c.w0 = j * sW - pW;
        return c;
    }
    __device__ float a(const RowCtx& r, int64_t k, int64_t q) const {
        return k < rows ? __ldg(w + r.wrow + q) : 0.f;
    }
    __device__ float b(const ColCtx& c, int64_t q, int64_t) const {
        if (!c.ok) return 0.f;
        const int khw = kH * kW;
        const int ci = (int)(q / khw);
        const int rs = (int)(q - (int64_t)ci * khw);
        const int r = rs / kW, s = rs - r * kW;
        const int h = c.h0 + r, ww = c.w0 + s;
        if (h < 0 || h >= H || ww < 0 || ww >= W) return 0.f;
        return __ldg(x + c.xbase + ((int64_t)ci * H + h) * W + ww);
    }
    __device__ void store(int64_t k, int64_t m, float v, int) const {
        const int64_t ohw = (int64_t)oH * oW;
        const int64_t n = m / ohw, pix = m - n * ohw;
        y[(n * K + k) * ohw + pix] = v + (bias ? __ldg(bias + k) : 0.f);
    }
};

struct DgradP {
    const float *gy, *w;
    float* gx;
    int C, H, W, K, kH, kW, pH, pW, sH, sW, oH, oW;
    int64_t rows, cols, tlen;  // rows=C, cols=N*H*W, tlen=K*kH*kW
    struct RowCtx { int c; };
    struct ColCtx { int64_t gybase; int h, w; bool ok; };
    __device__ int64_t t_begin(int) const { return 0; }
    __device__ int64_t t_end(int) const { return tlen; }
    __device__ RowCtx row_ctx(int64_t c) const { return {(int)c}; }
    __device__ ColCtx col_ctx(int64_t m) const {
        ColCtx cc{0, 0, 0, m < cols};
        if (!cc.ok) return cc;
        const int64_t hw = (int64_t)H * W;
        const int64_t n = m / hw;
        const int p = (int)(m - n * hw);
        cc.h = p / W;
        cc.w = p - cc.h * W;
        cc.gybase = n * K * (int64_t)oH * oW;
        return cc;
    }
    __device__ float a(const RowCtx& r, int64_t c, int64_t t) const {
        if (c >= rows) return 0.f;
        const int khw = kH * kW;
        const int k = (int)(t / khw);
        const int rs = (int)(t - (int64_t)k * khw);
        return __ldg(w + ((int64_t)k * C + r.c) * khw + rs);
    }
    __device__ float b(const ColCtx& cc, int64_t t, int64_t) const {
        if (!cc.ok) return 0.f;
        const int khw = kH * kW;
        const int k = (int)(t / khw);
        const int rs = (int)(t - (int64_t)k * khw);
        const int r = rs / kW, s = rs - r * kW;
        const int hn = cc.h + pH - r, wn = cc.w + pW - s;
        if (hn < 0 || wn < 0) return 0.f;
        const int oh = hn / sH, ow = wn / sW;
        if (oh * sH != hn || ow * sW != wn || oh >= oH || ow >= oW) return 0.f;
        return __ldg(gy + cc.gybase + ((int64_t)k * oH + oh) * oW + ow);
    }
    __device__ void store(int64_t c, int64_t m, float v, int) const {
        const int64_t hw = (int64_t)H * W;
        const int64_t n = m / hw, pix = m - n * hw;
        gx[(n * C + c) * hw + pix] = v;
    }
};

struct WgradP {
    const float *x, *gy;
    float* part;  // [splits][K][CRS]
    int C, H, W, K, kH, kW, pH, pW, sH, sW, oH, oW;
    int64_t rows, cols, M, chunk;  // rows=K, cols=CRS, reduction over M pixels in chunks
    struct RowCtx { int64_t k; };
    struct ColCtx { int64_t coff; int r, s; bool ok; };
    __device__ int64_t t_begin(int z) const { return (int64_t)z * chunk; }
    __device__ int64_t t_end(int z) const {
        const int64_t e = (int64_t)(z + 1) * chunk;
        return e < M ? e : M;
    }
    __device__ RowCtx row_ctx(int64_t k) const { return {k}; }
    __device__ ColCtx col_ctx(int64_t q) const {
        ColCtx cc{0, 0, 0, q < cols};
        if (!cc.ok) return cc;
        const int khw = kH * kW;
        const int c = (int)(q / khw);
        const int rs = (int)(q - (int64_t)c * khw);
        cc.r = rs / kW;
        cc.s = rs - cc.r * kW;
        cc.coff = (int64_t)c * H * W;
        return cc;
    }
    __device__ float a(const RowCtx& r, int64_t k, int64_t m) const {
        if (k >= rows) return 0.f;
        const int64_t ohw = (int64_t)oH * oW;
        const int64_t n = m / ohw, p = m - n * ohw;
        return __ldg(gy + (n * K + k) * ohw + p);
    }
    __device__ float b(const ColCtx& cc, int64_t m, int64_t) const {
        if (!cc.ok) return 0.f;
        const int64_t ohw = (int64_t)oH * oW;
        const int64_t n = m / ohw;
        const int p = (int)(m - n * ohw);
        const int i = p / oW, j = p - i * oW;
        const int h = i * sH - pH + cc.r, ww = j * sW - pW + cc.s;
        if (h < 0 || h >= H || ww < 0 || ww >= W) return 0.f;
        return __ldg(x + n * C * (int64_t)H * W + cc.coff + (int64_t)h * W + ww);
    }
    __device__ void store(int64_t k, int64_t q, float v, int z) const {
        part[((int64_t)z * rows + k) * cols + q] = v;
    }
};

// gw[i] = (acc ? gw[i] : 0) + scale * sum_z part[z][i] — fixed z order (deterministic).
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int splits, int64_t n,
                                     float* __restrict__ out, float scale, int accumulate) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float s = 0.f;
        for (int z = 0; z < splits; ++z) s += part[(int64_t)z * n + i];
        out[i] = (accumulate ? out[i] : 0.f) + scale * s;
    }
}

template <class P, int BM, int BN, int BK>
void launch_gemm(const P& p, int splits, cudaStream_t st, const char* what) {
    dim3 grid((unsigned)ceil_div(p.cols, BN), (unsigned)ceil_div(p.rows, BM), (unsigned)splits);
    PTB_REQUIRE(grid.y <= 65535 && grid.z <= 65535, "simt conv: grid too large");
    simt_gemm_kernel<P, BM, BN, BK><<<grid, kThreads, 0, st>>>(p);
    after_launch(what);
}

}  // namespace

void simt_conv_fwd(const Geo& g, const float* x, const float* w, const float* b, float* y,
                   cudaStream_t st) {
    FpropP p{x, w, b, y, (int)g.C, (int)g.H, (int)g.W, (int)g.K, (int)g.kH, (int)g.kW,
             (int)g.pH, (int)g.pW, (int)g.sH, (int)g.sW, (int)g.oH, (int)g.oW,
             g.K, g.M, g.CRS};
    ProfScope prof("simt_conv", st, 2.0 * g.M * g.K * g.CRS, 0.0);
    launch_gemm<FpropP, 64, 128, 8>(p, 1, st, "simt_fprop");
}

void simt_conv_bwd_data(const Geo& g, const float* gy, const float* w, float* gx,
                        cudaStream_t st) {
    DgradP p{gy, w, gx, (int)g.C, (int)g.H, (int)g.W, (int)g.K, (int)g.kH, (int)g.kW,
             (int)g.pH, (int)g.pW, (int)g.sH, (int)g.sW, (int)g.oH, (int)g.oW,
             g.C, g.N * g.HW, g.K * g.kH * g.kW};
    ProfScope prof("simt_conv", st, 2.0 * g.M * g.K * g.CRS, 0.0);
    launch_gemm<DgradP, 64, 128, 8>(p, 1, st, "simt_dgrad");
}

int simt_wgrad_splits(const Geo& g) {
    const int64_t tiles = ceil_div(g.K, 64) * ceil_div(g.CRS, 128);
    const int64_t want = (4 * (int64_t)sm_count() + tiles - 1) / tiles;  // ~4 waves
    const int64_t by_len = ceil_div(g.M, 256);                              // >=256 pixels/split
    int64_t s = want < by_len ? want : by_len;
    if (s < 1) s = 1;
    if (s > 512) s = 512;
    return (int)s;
}

size_t simt_wgrad_workspace(const Geo& g) {
    return sizeof(float) * (size_t)simt_wgrad_splits(g) * (size_t)(g.K * g.CRS);
}

void simt_conv_bwd_filter(const Geo& g, const float* x, const float* gy, float* gw, float scale,
                          int accumulate, float* ws, cudaStream_t st) {
    const int splits = simt_wgrad_splits(g);
    const int64_t chunk = ceil_div(ceil_div(g.M, splits), 16) * 16;
    WgradP p{x, gy, ws, (int)g.C, (int)g.H, (int)g.W, (int)g.K, (int)g.kH, (int)g.kW,
             (int)g.pH, (int)g.pW, (int)g.sH, (int)g.sW, (int)g.oH, (int)g.oW,
             g.K, g.CRS, g.M, chunk};
    const int used = (int)ceil_div(g.M, chunk);
    {
        ProfScope prof("simt_conv", st, 2.0 * g.M * g.K * g.CRS, 0.0);
        launch_gemm<WgradP, 64, 128, 16>(p, used, st, "simt_wgrad");
    }
    const int64_t n = g.K * g.CRS;
    splitk_reduce_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 4096), 256, 0, st>>>(
        ws, used, n, gw, scale, accumulate);
    after_launch("splitk_reduce");
}

// ---- SPEC gemm (row-major, op(A) M x K, op(B) K x N) ----------------------
namespace {
struct GemmP {
    const float *A, *B;
    float* Cm;
    int transA, transB;
    int64_t lda, ldb, ldc, rows, cols, K;
    float alpha, beta;
    struct RowCtx { int dummy; };
    struct ColCtx { int dummy; };
    __device__ int64_t t_begin(int) const { return 0; }
    __device__ int64_t t_end(int) const { return K; }
    __device__ RowCtx row_ctx(int64_t) const { return {0}; }
    __device__ ColCtx col_ctx(int64_t) const { return {0}; }
    __device__ float a(const RowCtx&, int64_t i, int64_t k) const {
        if (i >= rows) return 0.f;
        return transA ? A[k * lda + i] : A[i * lda + k];
    }
    __device__ float b(const ColCtx&, int64_t k, int64_t j) const {
        if (j >= cols) return 0.f;
        return transB ? B[j * ldb + k] : B[k * ldb + j];
    }
    __device__ void store(int64_t i, int64_t j, float v, int) const {
        float* c = Cm + i * ldc + j;
        *c = (beta == 0.f ? 0.f : beta * *c) + alpha * v;
    }
};
}  // namespace

void simt_gemm(int transA, int transB, int64_t M, int64_t N, int64_t K, float alpha,
               const float* A, int64_t lda, const float* B, int64_t ldb, float beta, float* C,
               int64_t ldc, cudaStream_t st) {
    GemmP p{A, B, C, transA, transB, lda, ldb, ldc, M, N, K, alpha, beta};
    launch_gemm<GemmP, 64, 128, 8>(p, 1, st, "simt_gemm");
}

}  // namespace ptb
