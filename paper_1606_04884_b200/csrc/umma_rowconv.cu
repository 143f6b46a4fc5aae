// umma_rowconv.cu — tcgen05 forward convolution for small-channel, stride-1 layers
// (C <= 4: the first layer of L1 / VGG-A).
//
// Input is stored once as zero-bordered NHWC with 4 channels, xp[n][Hp][Wa][4]
// (Hp = H + 2pH, Wa = W + 2pW rounded up to 32), so every tap read is in bounds. For
// output row i and filter row r, the im2col tile A[j][(s,c)] = xp[n][i+r][j+s][c] sits
// at byte offset (j + s)*16 + c*4 of ONE contiguous row segment: a Hankel matrix. The
// UMMA no-swizzle K-major canonical layout addresses element (row j, k = (s, c)) as
//   (j%8)*16 + (j/8)*SBO + c*4 + s*LBO
// so SBO = 128 B and LBO = 16 B reproduce it exactly: one 2.5 KB row load per
// (output row, r) feeds all kW taps, no im2col expansion anywhere (the reference
// materialises the (C*kH*kW) x (oH*oW) column matrix per image, im2col.kt.tmpl:9-21).
//
// CTA pair (cta_group::2): M = 256 = two 128-pixel output-row segments, N = output
// channels (each CTA holds half of the weight rows). The whole (half) filter stays
// resident in shared memory — loaded once per CTA — so a pipeline stage is just one
// input row segment (one TMA box of 512-byte rows); K walks (r, s-pair): one stage
// per filter row r, ceil(kW/2) MMAs (K = 8 = two taps x 4 channels) per stage.
#include <cuda.h>
#include <cstdlib>

#include "kernels.cuh"
#include "tmap.cuh"
#include "umma.cuh"

namespace ptb {

namespace {

using namespace umma;

constexpr int kThreadsR = 320;  // warps 2..9: epilogue (4 or 8 used, p.epi)
// A-ring depth: each stage is one ~2.5 KB row-segment TMA load feeding only kW/2 MMAs,
// so many loads must be in flight to cover L2 latency
static int kMaxStagesR = [] {
    const char* e = std::getenv("PT_B200_ROWCONV_STAGES");
    return e ? std::atoi(e) : 12;
}();
constexpr int kSmemLimit = 232448;

struct RowConvParams {
    int rps;              // padded input rows per pipeline stage
    uint32_t stage_bytes; // bytes one CTA's stage TMA delivers
    uint32_t row16;       // bytes between consecutive rows in a stage, >> 4
    int epi;  // epilogue warps: 4, or 8 (two per TMEM lane quarter, each half of the columns)
    CUtensorMap tmap_x;  // xp viewed (128 floats, Wa*4/128 chunks, N*Hp rows), box {128, seg_chunks, 1}
    CUtensorMap tmap_w;  // packed weights viewed (128 floats, w_chunks, 2 halves), box {128, w_chunks, 1}
    int oH, oW, Hp, kH, S2;  // S2 = kW rounded up to even
    int segs, seg_chunks;    // 128-pixel segments per output row; 512 B chunks per segment load
    int n_rows, Np;          // output channels, padded to 16
    int tiles, stages;
    uint32_t stage_a, w_bytes, tmem_cols;
    float* out;
    const float* bias;
};

__global__ void __launch_bounds__(kThreadsR, 1) umma_rowconv_kernel(const __grid_constant__ RowConvParams p) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((((raw + 1023u) & ~1023u)) - raw);
    const int S = p.stages;
    uint8_t* sW = smem;                                   // resident half filter
    uint8_t* sA = smem + align_up(p.w_bytes, 1024);       // row-segment ring
    uint64_t* full = reinterpret_cast<uint64_t*>(sA + (size_t)S * p.stage_a);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint64_t* wbar = tempty + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(wbar + 1);
    float* sbias = reinterpret_cast<float*>(tmem_holder + 4);  // [Np] bias staged once (epilogue)

    const uint32_t warp = warp_id_uniform(), lane = lane_id();
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.tmap_x);
        tma_prefetch(&p.tmap_w);
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 2 * p.epi);
        }
        mbar_init(wbar, 2);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc_cg2(tmem_holder, p.tmem_cols);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const int pairs = (p.tiles + 1) / 2;
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

    if (warp == 0) {
        if (lane == 0) {
            // the CTA's half of the filter, once (both halves complete on the leader's wbar)
            if (leader) mbar_arrive_expect_tx(wbar, 2 * p.w_bytes);
            else mbar_arrive_cluster(wbar, 0);
            tma_load_3d_cg2(sW, &p.tmap_w, wbar, 0, 0, (int)rank);
            int stage = 0;
            uint32_t phase = 0;
            for (int u = cid; u < pairs; u += ncl) {
                int t = 2 * u + (int)rank;
                if (t >= p.tiles) t = p.tiles - 1;  // duplicate work, never stored
                const int row = t / p.segs, seg = t - row * p.segs;  // row = n*oH + i
                const int n = row / p.oH, i = row - n * p.oH;
                const int prow = n * p.Hp + i;  // padded input row of filter row r = 0
                // one stage = RPS consecutive padded input rows (a single 3-D TMA box); the
                // peer's bytes complete on the leader's barrier, which only the leader arms
                for (int r = 0; r < p.kH; r += p.rps) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) mbar_arrive_expect_tx(&full[stage], 2u * p.stage_bytes);
                    tma_load_3d_cg2(sA + (size_t)stage * p.stage_a, &p.tmap_x, &full[stage], 0,
                                    seg * 2, prow + r);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {  // whole warp, converged; one elected lane issues
            const uint32_t idesc = idesc_tf32(256, p.Np, 0, 0);
            const uint32_t lbo_b = (uint32_t)(p.Np / 2) * 16u;  // next tap s: next [Np/2][4] block
            const uint32_t wbase = smem_u32(sW);
            mbar_wait(wbar, 0);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int u = cid; u < pairs; u += ncl, ++it) {
                const uint32_t acc = it & 1;
                mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + acc * p.Np;
                const uint32_t bstep = (2u * lbo_b) >> 4;
                const int npair = p.S2 / 2;
                constexpr uint32_t kHi = desc_hi(128, kSwizzleNone);
                for (int r0 = 0; r0 < p.kH; r0 += p.rps) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t abase = desc_lo(smem_u32(sA + (size_t)stage * p.stage_a), 16);
                    const int rn = p.kH - r0 < p.rps ? p.kH - r0 : p.rps;
                    for (int rr = 0; rr < rn; ++rr) {
                        const int r = r0 + rr;
                        // A: Hankel view of the row segment — rows (pixels) 16 B apart inside a
                        // core matrix, next 8 pixels at SBO=128, next tap s at LBO=16.
                        const uint32_t alo = abase + (uint32_t)rr * p.row16;
                        uint32_t blo = desc_lo(wbase + (uint32_t)(r * p.S2) * lbo_b, lbo_b);
                        for (int k = 0; k < npair; ++k, blo += bstep)
                            mma_tf32_cg2_warp(d, desc_make(alo + 2u * k, kHi), desc_make(blo, kHi), idesc,
                                              (r | k) != 0);
                    }
                    mma_commit_cg2_warp(&empty[stage]);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                mma_commit_cg2_warp(&tfull[acc]);
            }
        }
    } else if (warp < 2 + (uint32_t)p.epi) {
        const uint32_t q = warp & 3;
        const int half = (int)(warp - 2) >> 2;  // p.epi == 8: this warp's column half
        const int ncol = p.epi == 8 ? p.Np / 2 : p.Np, col0 = half * ncol;
        int it = 0;
        const int64_t ohw = (int64_t)p.oH * p.oW;
        if (p.bias) {
            for (int e = (int)((warp - 2) * 32 + lane); e < p.Np; e += 32 * p.epi)
                sbias[e] = e < p.n_rows ? __ldg(p.bias + e) : 0.f;
            if (p.epi == 8) asm volatile("bar.sync 1, 256;" ::: "memory");
            else asm volatile("bar.sync 1, 128;" ::: "memory");
        }
        for (int u = cid; u < pairs; u += ncl, ++it) {
            const uint32_t acc = it & 1;
            mbar_wait(&tfull[acc], (it >> 1) & 1);
            tc_fence_after();
            const int t = 2 * u + (int)rank;
            const int row = t / p.segs, seg = t - row * p.segs;
            const int n = row / p.oH, i = row - n * p.oH;
            const int j = seg * 128 + (int)(q * 32 + lane);
            const bool valid = t < p.tiles && j < p.oW;
            const int64_t base = (int64_t)n * p.n_rows * ohw + (int64_t)i * p.oW + j;
            const uint32_t taddr = tmem_base + ((q * 32u) << 16) + acc * p.Np + col0;
            store_tmem_columns_nchw(taddr, ncol, p.out + (valid ? base + (int64_t)col0 * ohw : 0), ohw, p.bias, col0,
                                    p.n_rows, valid, p.bias ? sbias : nullptr);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (leader) mbar_arrive(&tempty[acc]);
                else mbar_arrive_cluster(&tempty[acc], 0);
            }
        }
    }
    __syncwarp();
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (warp == 1) tmem_dealloc_cg2(tmem_base, p.tmem_cols);
#endif
}

// x NCHW -> zero-bordered NHWC with 4 channels: xp[n][Hp][Wa][4], TF32-rounded.
__global__ void pad_nhwc4_kernel(const float* __restrict__ x, float4* __restrict__ xp, int64_t N, int C,
                                 int H, int W, int pH, int pW, int Hp, int Wa) {
    // one block per padded row (n, hp): no 64-bit division per element (it made this
    // 58 MB pass take 21 us)
    const int64_t row = blockIdx.x;
    const int n = (int)(row / Hp), hp = (int)(row - (int64_t)n * Hp);
    const int h = hp - pH;
    const bool hin = h >= 0 && h < H;
    const float* src = x + ((int64_t)n * C * H + (hin ? h : 0)) * W;
    float4* dst = xp + row * Wa;
    for (int wa = threadIdx.x; wa < Wa; wa += blockDim.x) {
        const int w = wa - pW;
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (hin && w >= 0 && w < W) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                if (c < C) {
                    uint32_t r;
                    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(__ldg(src + (int64_t)c * H * W + w)));
                    v[c] = __uint_as_float(r);
                }
            }
        }
        dst[wa] = make_float4(v[0], v[1], v[2], v[3]);
    }
}

__global__ void pack_rowconv_w_kernel(const float* __restrict__ w, float* __restrict__ bw, int K, int C,
                                      int kH, int kW, int S2, int Np, int64_t w_half) {
    const int Nh = Np / 2;
    const int64_t total = 2 * w_half;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int half = (int)(e / w_half);
        const int64_t o = e - half * w_half;
        float v = 0.f;
        if (o < (int64_t)kH * S2 * Nh * 4) {
            const int c = (int)(o & 3);
            const int nn = (int)((o >> 2) % Nh);
            const int s = (int)((o / (4 * Nh)) % S2);
            const int r = (int)(o / (4 * Nh * S2));
            const int n = half * Nh + nn;
            if (n < K && c < C && s < kW) v = __ldg(w + (((int64_t)n * C + c) * kH + r) * kW + s);
        }
        uint32_t q;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(q) : "f"(v));
        bw[e] = __uint_as_float(q);
    }
}

struct RowPlan {
    int Hp, Wa, S2, Np, segs, seg_chunks, w_chunks;
    int64_t xp_elems, w_half;  // floats per weight half (chunk-padded)
};

RowPlan rplan(const Geo& g) {
    RowPlan r;
    r.Hp = (int)(g.H + 2 * g.pH);
    r.Wa = (int)((g.W + 2 * g.pW + 63) / 64 * 64);
    r.S2 = (int)((g.kW + 1) / 2 * 2);
    r.Np = (int)((g.K + 15) / 16 * 16);
    r.segs = (int)ceil_div(g.oW, 128);
    // 64 pixels (1 KB) per TMA chunk: the per-row request count, not bytes, paced the loads
    r.seg_chunks = (128 + r.S2 - 1 + 63) / 64;
    r.xp_elems = g.N * r.Hp * r.Wa * 4 + 256 * r.seg_chunks;  // slack for the last segment
    const int64_t wf = g.kH * r.S2 * (r.Np / 2) * 4;
    r.w_chunks = (int)ceil_div(wf, 128);
    r.w_half = (int64_t)r.w_chunks * 128;
    return r;
}

}  // namespace

void pad_nhwc4(const float* x, float* xp, const Geo& g, int Hp, int Wa, cudaStream_t st) {
    const int64_t total = g.N * Hp * Wa;
    (void)total;
    pad_nhwc4_kernel<<<(unsigned)(g.N * Hp), Wa >= 256 ? 256 : 128, 0, st>>>(
        x, reinterpret_cast<float4*>(xp), g.N, (int)g.C, (int)g.H, (int)g.W, (int)g.pH, (int)g.pW, Hp, Wa);
    after_launch("pad_nhwc4");
}

bool rowconv_ok(const Geo& g) {
    if (!(g.C <= 4 && g.sH == 1 && g.sW == 1 && g.K <= 256 && g.kW <= 64 && g.kH <= 64 &&
          g.N * (g.H + 2 * g.pH) < (1ll << 31) && sm_count() >= 2))
        return false;
    const RowPlan r = rplan(g);
    return r.w_chunks <= 256 && r.w_half * 4 <= 160 * 1024;  // resident half filter fits smem
}

size_t rowconv_workspace(const Geo& g) {
    const RowPlan r = rplan(g);
    return align_up(r.xp_elems * 4, 256) + align_up(2 * r.w_half * 4, 256);
}

void rowconv_fwd(const Geo& g, const float* x, const float* w, const float* b, float* y, void* ws,
                 cudaStream_t st) {
    const RowPlan rp = rplan(g);
    float* xp = reinterpret_cast<float*>(ws);
    float* bw = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + align_up(rp.xp_elems * 4, 256));
    Fork fk(st, 1);  // the filter pack beside the layout pass
    pack_rowconv_w_kernel<<<(unsigned)ceil_div(2 * rp.w_half, 256), 256, 0, fk.side>>>(
        w, bw, (int)g.K, (int)g.C, (int)g.kH, (int)g.kW, rp.S2, rp.Np, rp.w_half);
    after_launch("pack_rowconv_w");
    {
        ProfScope prof("layout", st, 0.0, 4.0 * (g.N * g.C * g.HW + g.N * rp.Hp * rp.Wa * 4));
        const int64_t total = g.N * rp.Hp * rp.Wa;
        (void)total;
        pad_nhwc4_kernel<<<(unsigned)(g.N * rp.Hp), rp.Wa >= 256 ? 256 : 128, 0, st>>>(
            x, reinterpret_cast<float4*>(xp), g.N, (int)g.C, (int)g.H, (int)g.W, (int)g.pH, (int)g.pW, rp.Hp, rp.Wa);
        after_launch("pad_nhwc4");
    }
    fk.join();

    RowConvParams p;
    memset(&p, 0, sizeof p);
    {
        const uint64_t dims[3] = {256, (uint64_t)rp.Wa * 4 / 256, (uint64_t)(g.N * rp.Hp)};
        const uint64_t strides[2] = {1024, (uint64_t)rp.Wa * 16};
        // one stage = rps padded rows of seg_chunks x 512 B
        p.rps = (int)g.kH;
        while (p.rps > 1 && (size_t)p.rps * rp.seg_chunks * 1024 * 3 >
                                (size_t)(kSmemLimit - 2048 - (int)align_up(rp.w_half * 4, 1024)))
            p.rps = (p.rps + 1) / 2;
        const uint32_t box[3] = {256, (uint32_t)rp.seg_chunks, (uint32_t)p.rps};
        tmap_tiled(&p.tmap_x, xp, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE);
        p.stage_bytes = (uint32_t)(p.rps * rp.seg_chunks * 1024);
        p.row16 = (uint32_t)(rp.seg_chunks * 1024) >> 4;
    }
    {
        const uint64_t dims[3] = {128, (uint64_t)rp.w_chunks, 2};
        const uint64_t strides[2] = {512, (uint64_t)rp.w_half * 4};
        const uint32_t box[3] = {128, (uint32_t)rp.w_chunks, 1};
        tmap_tiled(&p.tmap_w, bw, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE);
    }
    p.oH = (int)g.oH;
    p.oW = (int)g.oW;
    p.Hp = rp.Hp;
    p.kH = (int)g.kH;
    p.S2 = rp.S2;
    p.segs = rp.segs;
    p.seg_chunks = rp.seg_chunks;
    p.n_rows = (int)g.K;
    p.Np = rp.Np;
    // 8 epilogue warps, each half of the columns (VGG-A conv1, output-write bound: 0.210 ->
    // 0.181 ms; convnet L1 unchanged)
    static const int epi_env = [] {
        const char* e = std::getenv("PT_B200_ROWCONV_EPI");
        return e ? std::atoi(e) : 0;
    }();
    p.epi = epi_env == 4 || epi_env == 8 ? epi_env : (rp.Np % 32 == 0 ? 8 : 4);
    p.tiles = (int)(g.N * g.oH * rp.segs);
    p.stage_a = (uint32_t)align_up((size_t)p.stage_bytes, 1024);
    p.w_bytes = (uint32_t)(rp.w_half * 4);
    const int avail = kSmemLimit - 1024 - 512 - (int)align_up(p.w_bytes, 1024) - rp.Np * 4;
    int s = avail / (int)p.stage_a;
    p.stages = s > kMaxStagesR ? kMaxStagesR : s;
    uint32_t cols = 32;
    while ((int)cols < 2 * rp.Np) cols <<= 1;
    p.tmem_cols = cols;
    p.out = y;
    p.bias = b;
    const size_t smem = 1024 + align_up(p.w_bytes, 1024) + (size_t)p.stages * p.stage_a + (2 * p.stages + 5) * 8 +
                        16 + (size_t)rp.Np * 4;  // + the staged bias
    const int pairs = (p.tiles + 1) / 2;
    const int ncl = std::min(pairs, sm_count() / 2);
    once_per_device((const void*)umma_rowconv_kernel, [&] {  // the smem limit is a per-device attribute
        PTB_CUDA(cudaFuncSetAttribute(umma_rowconv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kSmemLimit));
    });
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * ncl);
    cfg.blockDim = dim3(64 + 32 * p.epi);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    ProfScope prof("umma_conv", st, 2.0 * g.M * g.K * g.CRS, 0.0);
    PTB_CUDA(cudaLaunchKernelEx(&cfg, umma_rowconv_kernel, p));
    after_launch("umma_rowconv");
}

}  // namespace ptb
