// umma_swgrad.cu — tcgen05 (kind::tf32) weight gradient of small-channel stride-1 layers
// (C <= 4: convnet L1, VGG-A conv1; accGradParameters).
//
//   gW[k][c][r][s] = sum_{n,i,j} gy[n][k][i][j] * x[n][c][i+r-pH][j+s-pW]
//
// GEMM with M = output channel k (<= 128, one CTA's 128 TMEM lanes), N = filter column
// (r, s, c) (<= 512: up to two MMAs of N <= 256) and K = output pixels. The horizontal taps
// are folded into "planes" once in HBM,
//   Xe[n][h][p][j] = x[n][c][h][j+s-pW],   p = s*C + c  (P = kW*C planes, rows padded to Wx),
// so for output row i the B operand row (r, p) is Xe row i+r-pH of plane p: a TMA box
// {32 px, P planes, R+kH-1 rows} lands as [row][plane][32 px], i.e. the K-major B rows
// (r, p) at a uniform 128-byte pitch for output row i, and the rows for output row i+1
// start P rows further on. One box therefore carries the whole kH*kW*C-column B operand
// of R output rows x 32 columns (each input row is fetched once per row group, not once
// per filter row as the im2col engines do). A = gy in NHWC (shared with the dgrad and the
// fused gradBias), MN-major: {32 ch, 32 px, R rows, 1, Kp/32} -> [ch block][row][px][32].
//
// Compared with running the (kH x 1) row-expanded layer through umma_wgrad.cu (32-channel
// operand granularity: C*kW = 33 -> 64 expanded channels, 3 m-tiles for 704 columns) this
// wastes only the M padding (K = 96 of 128 lanes) and N rounding (363 of 384 columns).
//
// Work split: the (n, row group, 32-column block) items are divided evenly over one CTA
// per SM; each CTA accumulates its share in TMEM for the whole run and drains it once to
// a partial slab; a fixed-order reduce kernel sums the slabs (deterministic) and applies
// scale / accumulate. Warp 0: TMA producer, warp 1: TMEM owner + MMA issuer, warps 2..5:
// epilogue.
#include <cuda.h>

#include <cstdlib>

#include "kernels.cuh"
#include "tmap.cuh"
#include "umma.cuh"

namespace ptb {

namespace {

using namespace umma;

constexpr int kThreadsS = 192;
constexpr int kSmemLimitS = 232448;

struct SWParams {
    CUtensorMap tmap_gy;  // gy NHWC, 5-D {32, oW, oH, N, Kp/32}, box {32, 32, R, 1, Kp/32}, SW128_32B
    CUtensorMap tmap_xe;  // Xe [N][H][P][Wx], 4-D {Wx, P, H, N}, box {32, P, R+kH-1, 1}, SW128
    int oH, oW, pH;
    int P;            // planes (kW*C)
    int nh, nhalf;    // N split into nh MMAs of nhalf columns
    int items, jbs, rgs;  // work items = N * rgs * jbs
    int per_cta, rem;     // CTA b takes per_cta (+1 for b < rem) consecutive items
    int stages;
    uint32_t stage_a, stage_b, tx, a_lbo, tmem_cols;
    int K;            // output channels (TMEM lanes written)
    int npad;         // nh * nhalf (partial slab row length)
    uint32_t pad;     // bytes after the ring the MMA may read (operand rows past the loaded boxes)
    float* part;      // [gridDim.x][K][npad]
};

template <int kRowsS>  // output rows per pipeline stage (2, 4 or 8: more rows amortise the per-stage cost)
__global__ void __launch_bounds__(kThreadsS, 1) umma_swgrad_kernel(const __grid_constant__ SWParams p) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((((raw + 1023u) & ~1023u)) - raw);
    const int S = p.stages;
    const uint32_t stage_bytes = p.stage_a + p.stage_b;
    // stage = [A][B]; the MMA may read past a stage (M lanes >= K, N columns past kH*P):
    // those rows only feed discarded accumulator rows / columns, and a pad follows the ring
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * stage_bytes + p.pad);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tfull + 1);

    const uint32_t warp = warp_id_uniform(), lane = lane_id();
    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.tmap_gy);
        tma_prefetch(&p.tmap_xe);
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(tfull, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_holder, p.tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    // this CTA's contiguous share of the work items
    // (32-bit: a 64-bit division is a call, after which the MMA loop's descriptors land in
    // vector registers and every MMA pays an R2UR + elect)
    const int b = (int)blockIdx.x;
    const int lo = b * p.per_cta + (b < p.rem ? b : p.rem);
    const int hi = lo + p.per_cta + (b < p.rem ? 1 : 0);

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int it = lo; it < hi; ++it) {
                const int jb = it % p.jbs;
                const int rg = (it / p.jbs) % p.rgs;
                const int n = it / (p.jbs * p.rgs);
                mbar_wait(&empty[stage], phase ^ 1);
                uint8_t* a = smem + (size_t)stage * stage_bytes;
                mbar_arrive_expect_tx(&full[stage], p.tx);
                tma_load_5d(a, &p.tmap_gy, &full[stage], 0, jb * 32, rg * kRowsS, n, 0);
                tma_load_4d(a + p.stage_a, &p.tmap_xe, &full[stage], jb * 32, 0, rg * kRowsS - p.pH, n);
                if (++stage == S) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        const uint32_t idesc = idesc_tf32(128, p.nhalf, 1, 0);
        constexpr uint32_t kHiA = desc_hi(512, kSwizzle128B_Base32B), kHiB = desc_hi(1024, kSwizzle128B);
        int stage = 0;
        uint32_t phase = 0;
        uint32_t accum = 0;
        for (int it = lo; it < hi; ++it) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t a_addr = smem_u32(smem + (size_t)stage * stage_bytes);
            const uint32_t alo = desc_lo(a_addr, p.a_lbo), blo = desc_lo(a_addr + p.stage_a, 16);
#pragma unroll
            for (int t = 0; t < kRowsS; ++t) {
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    // A: pixel rows (t, 8*ks ..) of the MN-major gy tile (128 B per pixel row);
                    // B: output row t's (r, p) rows start t*P rows in, K step = 32 bytes
                    const uint64_t ad = desc_make(alo + (uint32_t)(t * 32 + ks * 8) * 8u, kHiA);
                    const uint32_t bl = blo + (uint32_t)(t * p.P) * 8u + (uint32_t)ks * 2u;
                    for (int h = 0; h < p.nh; ++h) {
                        mma_tf32_warp(tmem_base + (uint32_t)(h * p.nhalf), ad,
                                      desc_make(bl + (uint32_t)(h * p.nhalf) * 8u, kHiB), idesc, accum);
                    }
                    accum = 1;
                }
            }
            mma_commit_warp(&empty[stage]);
            if (++stage == S) {
                stage = 0;
                phase ^= 1;
            }
        }
        mma_commit_warp(tfull);
    } else {
        // ===== epilogue: TMEM lane k, columns (r, p) -> part[cta][k][col] =====
        const uint32_t q = warp & 3;
        const int k = (int)(q * 32 + lane);
        mbar_wait(tfull, 0);
        tc_fence_after();
        float* dst = p.part + ((int64_t)blockIdx.x * p.K + k) * p.npad;
        const uint32_t taddr = tmem_base + ((q * 32u) << 16);
        for (int c0 = 0; c0 < p.npad; c0 += 16) {
            uint32_t v[16];
            tmem_ld_32x32b_x16(taddr + c0, v);
            tmem_ld_wait();
            if (k < p.K) {
                float4* d4 = reinterpret_cast<float4*>(dst + c0);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    d4[j] = make_float4(lo < hi ? __uint_as_float(v[4 * j]) : 0.f,
                                        lo < hi ? __uint_as_float(v[4 * j + 1]) : 0.f,
                                        lo < hi ? __uint_as_float(v[4 * j + 2]) : 0.f,
                                        lo < hi ? __uint_as_float(v[4 * j + 3]) : 0.f);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem_base, p.tmem_cols);
#endif
}

// Xe[n][h][s*C + c][j] = tf32(x[n][c][h][j + s - pW]) (0 outside the image or j >= oW).
// One block per input row (n, h): the C rows are staged in smem, the P x Wx slab is
// written as float4 (Wx % 4 == 0), consecutive threads -> consecutive addresses.
__global__ void expand_planes_kernel(const float* __restrict__ x, float4* __restrict__ xe, int64_t rows,
                                     int C, int H, int W, int oW, int kW, int pW, int Wx) {
    extern __shared__ float srow[];  // [C][W]
    const int P = kW * C, q4 = Wx / 4;
    for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
        const int64_t n = row / H;
        const int h = (int)(row - n * H);
        const float* xr = x + (n * C * H + h) * (int64_t)W;
        __syncthreads();
        for (int t = threadIdx.y * blockDim.x + threadIdx.x; t < C * W; t += blockDim.x * blockDim.y) {
            const int c = t / W, w = t - c * W;
            uint32_t r;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(__ldg(xr + (int64_t)c * H * W + w)));
            srow[t] = __uint_as_float(r);
        }
        __syncthreads();
        float4* dst = xe + row * (int64_t)P * q4;
        // thread -> (plane, float4 column) with the plane decoded once per plane sweep
        for (int pl = threadIdx.y; pl < P; pl += blockDim.y) {
            const int s = pl / C, c = pl - s * C;
            const float* sr = srow + c * W + s - pW;
            for (int j4 = threadIdx.x; j4 < q4; j4 += blockDim.x) {
                const int j0 = j4 * 4;
                float v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int j = j0 + u, w = j + s - pW;
                    v[u] = (j < oW && w >= 0 && w < W) ? sr[j] : 0.f;
                }
                dst[pl * q4 + j4] = make_float4(v[0], v[1], v[2], v[3]);
            }
        }
    }
}

// gw[k][c][r][s] = (acc ? gw : 0) + scale * sum_cta part[cta][k][r*P + s*C + c]. Four
// threads per partial column (k, col) each sum a quarter of the slabs in order, then the
// quarters are added in order (fixed tree: deterministic); consecutive threads read
// consecutive columns. (One thread per column over ~148 slabs was latency-bound: 24 us.)
__global__ void swgrad_reduce_kernel(const float* __restrict__ part, float* __restrict__ gw, int K, int C,
                                     int kH, int kW, int npad, int ctas, float scale, int accumulate) {
    __shared__ float red[4][64];
    const int P = kW * C;
    const int total = K * npad;
    const int64_t slab = (int64_t)K * npad;
    const int qtr = threadIdx.x >> 6, li = threadIdx.x & 63;
    const int per = (ctas + 3) / 4, b0 = qtr * per, b1 = min(ctas, b0 + per);
    for (int base = blockIdx.x * 64; base < total; base += gridDim.x * 64) {
        const int i = base + li;
        float acc = 0.f;
        if (i < total) {
            const float* src = part + i;
#pragma unroll 8
            for (int b = b0; b < b1; ++b) acc += __ldg(src + b * slab);
        }
        red[qtr][li] = acc;
        __syncthreads();
        if (qtr == 0 && i < total) {
            const float sum = ((red[0][li] + red[1][li]) + red[2][li]) + red[3][li];
            const int k = i / npad, col = i - k * npad;
            const int r = col / P, pl = col - r * P;
            if (r < kH) {
                const int s = pl / C, c = pl - s * C;
                const int64_t o = (((int64_t)k * C + c) * kH + r) * kW + s;
                gw[o] = (accumulate ? gw[o] : 0.f) + scale * sum;
            }
        }
        __syncthreads();
    }
}

struct SWPlan {
    int P, Ntot, nh, nhalf, npad, Kp, Wx, jbs, rgs, items, ctas, stages, R;
    uint32_t stage_a, stage_b, tmem_cols, pad;
    int64_t xe_elems, part_elems;
};

// least ring depth for more rows per stage (each stage re-fetches the kH - 1 halo rows of
// the tap planes, so fewer rows per stage cost L2->SM bytes)
int swgrad_min_stages() {
    static const int v = [] {
        const char* e = std::getenv("PT_B200_SWGRAD_MINST");
        return e ? std::max(2, std::atoi(e)) : 3;
    }();
    return v;
}

SWPlan swplan(const Geo& g) {
    SWPlan w;
    w.P = (int)(g.kW * g.C);
    w.Ntot = (int)g.kH * w.P;
    w.nh = (int)ceil_div(w.Ntot, 256);
    w.nhalf = (int)(ceil_div(ceil_div(w.Ntot, w.nh), 16) * 16);
    w.npad = w.nh * w.nhalf;
    w.Kp = (int)((g.K + 31) / 32 * 32);
    w.Wx = (int)((g.oW + 3) / 4 * 4);
    w.jbs = (int)ceil_div(g.oW, 32);
    // rows per stage: the most (2, 4, 8) that still leave a 3-deep ring (VGG conv1: 8 MMAs
    // per 2-row stage left the tensor pipe waiting on the per-stage round trip)
    for (int R : {8, 4, 2}) {
        w.R = R;
        w.rgs = (int)ceil_div(g.oH, R);
        const int64_t items = g.N * w.rgs * w.jbs;
        w.items = items < (1ll << 31) ? (int)items : -1;
        w.ctas = (int)std::min<int64_t>(items, sm_count());
        w.stage_a = (uint32_t)align_up((size_t)(w.Kp / 32) * R * 32 * 128, 1024);
        w.stage_b = (uint32_t)align_up((size_t)(R + g.kH - 1) * w.P * 128, 1024);
        // overrun past the last stage: B rows up to npad from output row R-1's start, A lanes
        // past Kp (4 x 32-channel atoms of M = 128) beyond the stage's own B region
        const int64_t b_over = ((int64_t)(R - 1) * w.P + w.npad - (R + g.kH - 1) * w.P) * 128;
        const int64_t a_over = (int64_t)(4 - w.Kp / 32) * R * 32 * 128 - w.stage_b;
        w.pad = (uint32_t)align_up((size_t)std::max<int64_t>(1024, std::max(b_over, a_over)), 1024);
        const int budget = kSmemLimitS - 1024 - (int)w.pad - 256;
        w.stages = std::min(8, budget / (int)(w.stage_a + w.stage_b));
        if (R == 2 || (w.stages >= swgrad_min_stages() && R <= g.oH && R + g.kH - 1 <= 256)) break;
    }
    uint32_t cols = 32;
    while ((int)cols < w.npad) cols <<= 1;
    w.tmem_cols = cols;
    w.xe_elems = g.N * g.H * w.P * (int64_t)w.Wx;
    w.part_elems = (int64_t)w.ctas * g.K * w.npad;
    return w;
}

bool swgrad_env() {
    static const bool on = [] {
        const char* e = std::getenv("PT_B200_SWGRAD");
        return e ? std::atoi(e) != 0 : true;
    }();
    return on;
}

}  // namespace

bool swgrad_ok(const Geo& g) {
    if (!swgrad_env()) return false;
    if (!(g.C <= 4 && g.sH == 1 && g.sW == 1 && g.K <= 128 && g.pH <= 64 && g.pW <= 64)) return false;
    const SWPlan w = swplan(g);
    if (w.items < 1 || w.npad > 512 || w.P > 256 || w.R + g.kH - 1 > 256) return false;
    if (w.pad > 65536) return false;
    if (g.N * g.H * w.P >= (1ll << 31) || g.M >= (1ll << 31)) return false;
    return w.stages >= 2 && sm_count() >= 1;
}

size_t swgrad_workspace(const Geo& g) {
    const SWPlan w = swplan(g);
    return align_up((size_t)w.xe_elems * 4, 256) + align_up((size_t)w.part_elems * 4, 256);
}

void swgrad(const Geo& g, const float* x, const float* gyh, float* gw, float scale, int accumulate, void* ws,
            cudaStream_t st) {
    PTB_REQUIRE(swgrad_ok(g), "swgrad: unsupported geometry");
    const SWPlan w = swplan(g);
    float* xe = reinterpret_cast<float*>(ws);
    float* part = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + align_up((size_t)w.xe_elems * 4, 256));
    {
        ProfScope prof("layout", st, 0.0, 4.0 * (g.N * g.C * g.HW + w.xe_elems));
        const int64_t rows = g.N * g.H;
        const size_t smem = sizeof(float) * (size_t)(g.C * g.W);
        PTB_REQUIRE(smem <= 48 * 1024, "expand_planes: input row too wide");
        const int tx = w.Wx / 4 >= 32 ? 32 : 16;
        expand_planes_kernel<<<(unsigned)std::min<int64_t>(rows, 64 * (int64_t)sm_count()), dim3(tx, 256 / tx), smem,
                               st>>>(
            x, reinterpret_cast<float4*>(xe), rows, (int)g.C, (int)g.H, (int)g.W, (int)g.oW, (int)g.kW,
            (int)g.pW, w.Wx);
        after_launch("expand_planes");
    }
    SWParams p;
    memset(&p, 0, sizeof p);
    {
        const uint64_t dims[5] = {32, (uint64_t)g.oW, (uint64_t)g.oH, (uint64_t)g.N, (uint64_t)(w.Kp / 32)};
        const uint64_t strides[4] = {(uint64_t)w.Kp * 4, (uint64_t)(g.oW * w.Kp * 4),
                                     (uint64_t)(g.oHW * w.Kp * 4), 128};
        const uint32_t box[5] = {32, 32, (uint32_t)w.R, 1, (uint32_t)(w.Kp / 32)};
        tmap_tiled(&p.tmap_gy, gyh, 5, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    }
    {
        const uint64_t dims[4] = {(uint64_t)w.Wx, (uint64_t)w.P, (uint64_t)g.H, (uint64_t)g.N};
        const uint64_t strides[3] = {(uint64_t)w.Wx * 4, (uint64_t)(w.P * w.Wx * 4),
                                     (uint64_t)(g.H * w.P * w.Wx * 4)};
        const uint32_t box[4] = {32, (uint32_t)w.P, (uint32_t)(w.R + g.kH - 1), 1};
        tmap_tiled(&p.tmap_xe, xe, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    }
    p.oH = (int)g.oH;
    p.oW = (int)g.oW;
    p.pH = (int)g.pH;
    p.P = w.P;
    p.nh = w.nh;
    p.nhalf = w.nhalf;
    p.items = w.items;
    p.per_cta = w.items / w.ctas;
    p.rem = w.items % w.ctas;
    p.jbs = w.jbs;
    p.rgs = w.rgs;
    p.stages = w.stages;
    p.stage_a = w.stage_a;
    p.stage_b = w.stage_b;
    p.tx = (uint32_t)((w.Kp / 32) * w.R * 32 * 128 + (w.R + g.kH - 1) * w.P * 128);
    p.a_lbo = (uint32_t)(w.R * 32 * 128);
    p.tmem_cols = w.tmem_cols;
    p.K = (int)g.K;
    p.npad = w.npad;
    p.part = part;
    p.pad = w.pad;
    const size_t smem = 1024 + (size_t)w.stages * (w.stage_a + w.stage_b) + w.pad + (2 * w.stages + 2) * 8 + 16;
    once_per_device((const void*)umma_swgrad_kernel<2>, [&] {  // the smem limit is a per-device attribute
        for (auto fn : {umma_swgrad_kernel<2>, umma_swgrad_kernel<4>, umma_swgrad_kernel<8>})
            PTB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimitS));
    });
    {
        ProfScope prof("umma_wgrad", st, 2.0 * g.M * g.K * g.CRS, 0.0);
        if (w.R == 8) umma_swgrad_kernel<8><<<(unsigned)w.ctas, kThreadsS, smem, st>>>(p);
        else if (w.R == 4) umma_swgrad_kernel<4><<<(unsigned)w.ctas, kThreadsS, smem, st>>>(p);
        else umma_swgrad_kernel<2><<<(unsigned)w.ctas, kThreadsS, smem, st>>>(p);
        after_launch("umma_swgrad");
    }
    const int64_t n = g.K * w.npad;
    swgrad_reduce_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 64), 16 * (int64_t)sm_count()), 256, 0, st>>>(
        part, gw, (int)g.K, (int)g.C, (int)g.kH, (int)g.kW, w.npad, w.ctas, scale, accumulate);
    after_launch("swgrad_reduce");
}

}  // namespace ptb
