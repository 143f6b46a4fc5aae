// winograd.cu — the Winograd F(2x2,3x3) registry entry (conv_winograd_2x2_3x3):
// 3x3 stride-1 convolution as 16 transform-domain GEMMs on the tensor cores.
//
//   U = G g G^T  (4x4 per (out, in) channel pair)      weight transform
//   V = B^T d B  (4x4 per (tile, in channel)), d = the 4x4 input patch of a 2x2 output tile
//   M_xi[out][tile] = sum_in U_xi[out][in] * V_xi[tile][in]     xi = 0..15 (umma_gemm.cu)
//   Y = A^T M A  (2x2 outputs per tile) + bias                 output transform
//
// with the standard Lavin-Gray F(2,3) matrices (B^T rows {1,0,-1,0},{0,1,1,0},{0,-1,1,0},
// {0,1,0,-1}; G rows {1,0,0},{1/2,1/2,1/2},{1/2,-1/2,1/2},{0,0,1}; A^T rows {1,1,1,0},
// {0,1,-1,-1}); edge tiles read zero padding; channel sums happen in the transform domain
// (SPEC.md:450). updateGradInput uses the same pipeline: for stride 1, gradInput is the 3x3
// correlation of gradOutput padded by 2-p with the 180-degree-rotated filter whose in/out
// channels are swapped (applied in the weight transform), so p <= 2.
//
// Layouts (HBM, workspace): U [16][out][in_p], V [16][tiles][in_p] (both K-major for the
// GEMM, in_p = in rounded up to 4 floats so every row is 16-byte aligned for TMA), M
// [16][out][tiles] (the GEMM's n-major store: a warp writes 32 consecutive tiles). The
// transforms are HBM-bound streaming kernels; the input transform stages a 32-tile x
// 16-channel block in shared memory so both its NCHW reads (along tiles) and its V writes
// (along channels) are coalesced.
#include "kernels.cuh"

namespace ptb {

namespace {

constexpr int kTT = 32;  // tiles per input-transform block
constexpr int kTC = 16;  // channels per input-transform block

struct WinoShape {
    int64_t N, Cin, Hin, Win, Cout;
    int pH, pW;
    int64_t Ho, Wo, tH, tW, T, cin_p;
};

WinoShape wino_shape(int64_t N, int64_t Cin, int64_t Hin, int64_t Win, int64_t Cout, int pH, int pW) {
    WinoShape s;
    s.N = N;
    s.Cin = Cin;
    s.Hin = Hin;
    s.Win = Win;
    s.Cout = Cout;
    s.pH = pH;
    s.pW = pW;
    s.Ho = Hin + 2 * pH - 2;
    s.Wo = Win + 2 * pW - 2;
    s.tH = (s.Ho + 1) / 2;
    s.tW = (s.Wo + 1) / 2;
    s.T = N * s.tH * s.tW;
    s.cin_p = (Cin + 3) / 4 * 4;
    return s;
}

// g (3x3, row-major) -> U = G g G^T (4x4, row-major)
__device__ __forceinline__ void wino_g(const float g[9], float u[16]) {
    float h[4][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float a = g[c], b = g[3 + c], d = g[6 + c];
        h[0][c] = a;
        h[1][c] = 0.5f * (a + b + d);
        h[2][c] = 0.5f * (a - b + d);
        h[3][c] = d;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        u[4 * i + 0] = h[i][0];
        u[4 * i + 1] = 0.5f * (h[i][0] + h[i][1] + h[i][2]);
        u[4 * i + 2] = 0.5f * (h[i][0] - h[i][1] + h[i][2]);
        u[4 * i + 3] = h[i][2];
    }
}

// U[xi][r][q] (row stride qp) for r < R (GEMM out channels), q < Q (reduction channels).
// fwd: g = w[r][q]; dgrad (flip): g = rot180(w[q][r]) (w is [Q=K][R=C][3][3] there).
__global__ void wino_weight_kernel(const float* __restrict__ w, float* __restrict__ U, int64_t R,
                                   int64_t Q, int64_t qp, int flip) {
    const int64_t total = R * Q;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = i % Q, r = i / Q;
        float g[9];
        const float* src = flip ? w + (q * R + r) * 9 : w + (r * Q + q) * 9;
#pragma unroll
        for (int e = 0; e < 9; ++e) g[e] = __ldg(src + (flip ? 8 - e : e));
        float u[16];
        wino_g(g, u);
#pragma unroll
        for (int xi = 0; xi < 16; ++xi) U[((int64_t)xi * R + r) * qp + q] = u[xi];
    }
}

// V[xi][t][c] for a block of kTT tiles x kTC channels (threadIdx.x: tile, .y: channel).
__global__ void __launch_bounds__(kTT * kTC) wino_input_kernel(const float* __restrict__ x,
                                                               float* __restrict__ V, const WinoShape s) {
    __shared__ float sv[16][kTT][kTC + 1];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t t = blockIdx.x * (int64_t)kTT + tx;
    const int64_t c = blockIdx.y * (int64_t)kTC + ty;
    if (t < s.T && c < s.Cin) {
        const int64_t tw = t % s.tW, th = (t / s.tW) % s.tH, n = t / (s.tW * s.tH);
        const float* xp = x + (n * s.Cin + c) * s.Hin * s.Win;
        const int64_t h0 = 2 * th - s.pH, w0 = 2 * tw - s.pW;
        float d[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t h = h0 + i;
            const bool hv = h >= 0 && h < s.Hin;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t ww = w0 + j;
                d[i][j] = (hv && ww >= 0 && ww < s.Win) ? __ldg(xp + h * s.Win + ww) : 0.f;
            }
        }
        float u[4][4];  // B^T d
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            u[0][j] = d[0][j] - d[2][j];
            u[1][j] = d[1][j] + d[2][j];
            u[2][j] = d[2][j] - d[1][j];
            u[3][j] = d[1][j] - d[3][j];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {  // (B^T d) B
            sv[4 * i + 0][tx][ty] = u[i][0] - u[i][2];
            sv[4 * i + 1][tx][ty] = u[i][1] + u[i][2];
            sv[4 * i + 2][tx][ty] = u[i][2] - u[i][1];
            sv[4 * i + 3][tx][ty] = u[i][1] - u[i][3];
        }
    }
    __syncthreads();
    // write-out with channels along the fast thread index: 16 consecutive floats per tile row
    const int lin = ty * kTT + tx;
    const int wc = lin % kTC, wt = lin / kTC;  // 32 x 16 threads -> tiles 0..31, channels 0..15
    const int64_t ot = blockIdx.x * (int64_t)kTT + wt, oc = blockIdx.y * (int64_t)kTC + wc;
    if (ot < s.T && oc < s.Cin) {
#pragma unroll
        for (int xi = 0; xi < 16; ++xi) V[((int64_t)xi * s.T + ot) * s.cin_p + oc] = sv[xi][wt][wc];
    }
}

// y[n][k][2th+i][2tw+j] = (A^T M A)[i][j] + b[k]; thread per (k, tile), tiles fastest
__global__ void wino_output_kernel(const float* __restrict__ M, const float* __restrict__ bias,
                                   float* __restrict__ y, const WinoShape s) {
    const int64_t total = s.Cout * s.T;
    const int64_t plane = s.Cout * s.T;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = i % s.T, k = i / s.T;
        float m[16];
#pragma unroll
        for (int xi = 0; xi < 16; ++xi) m[xi] = __ldcs(M + xi * plane + k * s.T + t);
        float a[2][4];  // A^T m
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            a[0][j] = m[j] + m[4 + j] + m[8 + j];
            a[1][j] = m[4 + j] - m[8 + j] - m[12 + j];
        }
        const float b = bias ? __ldg(bias + k) : 0.f;
        const int64_t tw = t % s.tW, th = (t / s.tW) % s.tH, n = t / (s.tW * s.tH);
        float* yp = y + (n * s.Cout + k) * s.Ho * s.Wo;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int64_t h = 2 * th + r;
            if (h >= s.Ho) continue;
            const float y0 = a[r][0] + a[r][1] + a[r][2] + b;
            const float y1 = a[r][1] - a[r][2] - a[r][3] + b;
            const int64_t w0 = 2 * tw;
            yp[h * s.Wo + w0] = y0;
            if (w0 + 1 < s.Wo) yp[h * s.Wo + w0 + 1] = y1;
        }
    }
}

struct WinoWs {
    float *U, *V, *M;
};

size_t wino_bytes(const WinoShape& s, WinoWs* out, void* ws) {
    const size_t u = align_up(sizeof(float) * 16 * s.Cout * s.cin_p, 256);
    const size_t v = align_up(sizeof(float) * 16 * s.T * s.cin_p, 256);
    const size_t m = align_up(sizeof(float) * 16 * s.Cout * s.T, 256);
    if (out) {
        uint8_t* p = static_cast<uint8_t*>(ws);
        out->U = reinterpret_cast<float*>(p);
        out->V = reinterpret_cast<float*>(p + u);
        out->M = reinterpret_cast<float*>(p + u + v);
    }
    return u + v + m;
}

WinoShape shape_for(const Geo& g, int op) {
    return op == PT_CONV_FWD ? wino_shape(g.N, g.C, g.H, g.W, g.K, (int)g.pH, (int)g.pW)
                             : wino_shape(g.N, g.K, g.oH, g.oW, g.C, (int)(2 - g.pH), (int)(2 - g.pW));
}

int grid_of(int64_t n) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 8 * (int64_t)sm_count()));
}

void run_wino(const WinoShape& s, const float* in, const float* w, int flip, const float* bias,
              float* out, void* ws, double flops, cudaStream_t st) {
    WinoWs b;
    wino_bytes(s, &b, ws);
    {
        ProfScope ps("layout", st, 0.0, 4.0 * (9.0 + 16.0) * s.Cout * s.Cin);
        wino_weight_kernel<<<grid_of(s.Cout * s.Cin), 256, 0, st>>>(w, b.U, s.Cout, s.Cin, s.cin_p, flip);
        after_launch("wino_weight");
    }
    {
        ProfScope ps("layout", st, 0.0, 4.0 * (s.N * s.Cin * s.Hin * s.Win + 16.0 * s.T * s.Cin));
        const dim3 grid((unsigned)ceil_div(s.T, kTT), (unsigned)ceil_div(s.Cin, kTC));
        PTB_REQUIRE(grid.y < 65536, "winograd: too many channels");
        wino_input_kernel<<<grid, dim3(kTT, kTC), 0, st>>>(in, b.V, s);
        after_launch("wino_input");
    }
    UmmaGemm gm{};
    gm.a = b.V;
    gm.b = b.U;
    gm.d = b.M;
    gm.M = s.T;
    gm.N = s.Cout;
    gm.K = s.Cin;
    gm.batch = 16;
    gm.lda = s.cin_p;
    gm.ldb = s.cin_p;
    gm.ldd = s.T;
    gm.batch_a = s.T * s.cin_p;
    gm.batch_b = s.Cout * s.cin_p;
    gm.batch_d = s.Cout * s.T;
    gm.alpha = 1.f;
    gm.beta = 0.f;
    (void)flops;
    umma_gemm(gm, st);
    {
        ProfScope ps("layout", st, 0.0, 4.0 * (16.0 * s.Cout * s.T + s.N * s.Cout * s.Ho * s.Wo));
        wino_output_kernel<<<grid_of(s.Cout * s.T), 256, 0, st>>>(b.M, bias, out, s);
        after_launch("wino_output");
    }
}

}  // namespace

bool winograd_applies(const Geo& g, int op) {
    if (g.kH != 3 || g.kW != 3 || g.sH != 1 || g.sW != 1) return false;
    if (op == PT_CONV_BWD_DATA) return g.pH <= 2 && g.pW <= 2;
    return op == PT_CONV_FWD;
}

size_t winograd_workspace(const Geo& g, int op) {
    if (!winograd_applies(g, op)) return 0;
    return wino_bytes(shape_for(g, op), nullptr, nullptr);
}

void winograd_fwd(const Geo& g, const float* x, const float* w, const float* b, float* y, void* ws,
                  cudaStream_t st) {
    PTB_REQUIRE(winograd_applies(g, PT_CONV_FWD), "winograd: supports 3x3 stride-1 geometries only");
    PassScope pass("fwd");
    run_wino(shape_for(g, PT_CONV_FWD), x, w, 0, b, y, ws, 2.0 * g.N * g.K * g.CRS * g.oHW, st);
}

void winograd_bwd_data(const Geo& g, const float* gy, const float* w, float* gx, void* ws, cudaStream_t st) {
    PTB_REQUIRE(winograd_applies(g, PT_CONV_BWD_DATA),
                "winograd: gradInput supports 3x3 stride-1 geometries with padding <= 2 only");
    PassScope pass("dgrad");
    run_wino(shape_for(g, PT_CONV_BWD_DATA), gy, w, 1, nullptr, gx, ws, 2.0 * g.N * g.K * g.CRS * g.oHW, st);
}

}  // namespace ptb
