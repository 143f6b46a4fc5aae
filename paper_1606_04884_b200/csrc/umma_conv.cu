// umma_conv.cu — tcgen05 (kind::tf32) implicit-GEMM convolution for sm_100a.
//
// GEMM view (SPEC.md:389-397 without materialising the unfold):
//   D[m][n] = sum_kd A[m][kd] * B[n][kd]
//   m  = output pixel (n_img, i, j) flattened — 128 per CTA (TMEM lanes)
//   n  = output channel — BN per tile (TMEM columns, fp32 accumulators)
//   kd = (r, s, c) — filter tap x channel, 32 channels per TMA box
// A is gathered by TMA in im2col mode straight from an NHWC copy of the
// activation (hardware zero-fill implements the padding), B is the packed
// weight matrix loaded by tiled TMA. Both land 128B-swizzled (K-major) in smem;
// one elected thread issues tcgen05.mma into a double-buffered TMEM accumulator,
// four epilogue warps drain it (tcgen05.ld), add the bias and write NCHW
// directly (a warp stores 32 consecutive pixels of one channel per instruction).
//
// Two variants:
//  * CB=32, CTA pair (cta_group::2): M = 256 pixels per pair (128 per CTA), each CTA
//    loads its own pixels and half of the BN weight rows; 64-deep K per pipeline
//    stage (two im2col boxes), division-free (tap, chunk) walk in the producer.
//  * CB=4 (C % 32 != 0, e.g. C=3 first layers), single CTA: 16-byte channel boxes
//    (C padded to 4) in the no-swizzle core-matrix layout: 8 (tap,chunk) slots of
//    128 px x 4 ch per stage, one MMA (K=8) spanning two slots.
//
// dgrad reuses this kernel: stride 1 as a conv of gy with the flipped filter and
// pad' = k-1-pad; small-C / strided as gcol = W^T gy (a 1x1 conv) + col2im.
//
// Warp roles (192 threads, 1 CTA/SM, persistent over tiles):
//   warp 0      TMA producer (1 lane; both CTAs of a pair)
//   warp 1      TMEM allocator + MMA issuer (1 lane; pair leader only)
//   warps 2..5  epilogue (warp w owns TMEM lanes 32*(w%4) .. +31)
#include <cuda.h>

#include <cstdlib>

#include "kernels.cuh"
#include "tmap.cuh"
#include "umma.cuh"

namespace ptb {

namespace {

using namespace umma;

constexpr int kTileM = 128;
constexpr uint32_t kBoxA = kTileM * 32 * 4;  // 16 KB: 128 px x 32 fp32
constexpr int kThreadsU = 320;  // warps 2..9: epilogue, two per TMEM lane quarter
constexpr int kSmemLimit = 232448;  // 227 KB opt-in per block on sm_100

struct UConvParams {
    CUtensorMap tmap_a;
    CUtensorMap tmap_b;
    int M;             // GEMM rows = output pixels
    int oH, oW;        // output spatial dims of this conv
    int sH, sW, pH, pW;
    int kW;
    int slots;         // taps * chunks (real k-slots of 32 or 4 channels)
    int chunks;        // cin_p / cb
    int num_kb;        // pipeline stages per tile
    int n_rows;        // real output channels
    int bn, n_tiles, m_tiles;
    int stages;
    uint32_t stage_a, stage_b;  // bytes per CTA per stage
    uint32_t tmem_cols;
    float* out;
    const float* bias;
    int sbias_n;  // > 0: bias staged in smem (this many floats, zero past n_rows)
    int64_t out_hw;
};

// (tap, chunk) cursor walking the reduction order kd = (r, s, c-chunk) without divisions.
struct KCursor {
    int r, s, cc;
    __device__ void reset() { r = s = cc = 0; }
    __device__ void next(int chunks, int kW) {
        if (++cc == chunks) {
            cc = 0;
            if (++s == kW) {
                s = 0;
                ++r;
            }
        }
    }
};

// SPS: (tap, 32-channel chunk) slots per pipeline stage on the CTA-pair path (2).
// Four slots (K = 128 per stage) halve the barrier round trips per MMA and keep more
// bytes per request in flight; used when two such stages fit in shared memory.
template <int CB, int CG, int SPS = 2>
__global__ void __launch_bounds__(kThreadsU, 1) umma_conv_kernel(const __grid_constant__ UConvParams p) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
    static_assert(CG == 1 || CB == 32, "CTA pairs only on the SW128 path");
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((((raw + 1023u) & ~1023u)) - raw);
    const int S = p.stages;
    uint8_t* sA = smem;
    uint8_t* sB = smem + (size_t)S * p.stage_a;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + (size_t)S * p.stage_b);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
    float* sbias = reinterpret_cast<float*>(tmem_holder + 4);  // [sbias_n] staged bias (epilogue)

    const uint32_t warp = warp_id_uniform(), lane = lane_id();
    const uint32_t rank = CG == 2 ? cluster_rank() : 0;
    const bool leader = rank == 0;
    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.tmap_a);
        tma_prefetch(&p.tmap_b);
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);  // armed by the leader only; the peer's bytes land on it
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 8 * CG);
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        if constexpr (CG == 2) tmem_alloc_cg2(tmem_holder, p.tmem_cols);
        else tmem_alloc(tmem_holder, p.tmem_cols);
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync();
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const int num_tiles = p.m_tiles * p.n_tiles;
    const int ohw = p.oH * p.oW;
    const int cid = blockIdx.x / CG, ncl = gridDim.x / CG;
    constexpr int kTileMC = kTileM * CG;  // pixels per tile (per pair)

    if (warp == 0) {
        if (lane == 0) {
            // ===== TMA producer =====
            int stage = 0;
            uint32_t phase = 0;
            const uint32_t tx = CG * (p.stage_a + p.stage_b);
            for (int tile = cid; tile < num_tiles; tile += ncl) {
                const int mt = tile / p.n_tiles, nt = tile - mt * p.n_tiles;
                const int m0 = mt * kTileMC + (int)rank * kTileM;
                const int n0 = m0 / ohw;
                const int rem = m0 - n0 * ohw;
                const int i0 = rem / p.oW, j0 = rem - i0 * p.oW;
                const int wc = j0 * p.sW - p.pW, hc = i0 * p.sH - p.pH;
                const int brow = nt * p.bn + (int)rank * (p.bn / CG);
                KCursor kc;
                kc.reset();
                int slot = 0;
                for (int kb = 0; kb < p.num_kb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* a = sA + (size_t)stage * p.stage_a;
                    uint8_t* b = sB + (size_t)stage * p.stage_b;
                    if constexpr (CG == 2) {
                        if (leader) mbar_arrive_expect_tx(&full[stage], tx);
                        // the stage's SPS consecutive 32-wide k slots of B: one 3-D box
                        tma_load_3d_cg2(b, &p.tmap_b, &full[stage], 0, brow, slot);
#pragma unroll
                        for (int t = 0; t < SPS; ++t) {
                            // past the last k-slot: any valid tap (the weights there are 0 / OOB)
                            const bool live = slot < p.slots;
                            tma_load_im2col_4d_cg2(a + t * kBoxA, &p.tmap_a, &full[stage],
                                                   live ? kc.cc * 32 : 0, wc, hc, n0,
                                                   (uint16_t)(live ? kc.s : 0),
                                                   (uint16_t)(live ? kc.r : 0));
                            ++slot;
                            kc.next(p.chunks, p.kW);
                        }
                    } else if constexpr (CB == 32) {
                        mbar_arrive_expect_tx(&full[stage], tx);
                        tma_load_im2col_4d(a, &p.tmap_a, &full[stage], kc.cc * 32, wc, hc, n0,
                                           (uint16_t)kc.s, (uint16_t)kc.r);
                        tma_load_2d(b, &p.tmap_b, &full[stage], slot * 32, brow);
                        ++slot;
                        kc.next(p.chunks, p.kW);
                    } else {
                        mbar_arrive_expect_tx(&full[stage], tx);
#pragma unroll 1
                        for (int t = 0; t < 8; ++t) {
                            const bool live = slot < p.slots;
                            tma_load_im2col_4d(a + t * 2048, &p.tmap_a, &full[stage],
                                               live ? kc.cc * 4 : 0, wc, hc, n0,
                                               (uint16_t)(live ? kc.s : 0),
                                               (uint16_t)(live ? kc.r : 0));
                            ++slot;
                            kc.next(p.chunks, p.kW);
                        }
                        tma_load_3d(b, &p.tmap_b, &full[stage], 0, brow, kb * 8);
                    }
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {  // whole warp, converged; one elected lane issues
            // ===== MMA issuer =====
            const uint32_t idesc = idesc_tf32(kTileMC, p.bn, 0, 0);
            constexpr uint32_t kHiSW128 = desc_hi(1024, kSwizzle128B), kHiNone = desc_hi(128, kSwizzleNone);
            const uint32_t bhalf16 = (p.stage_b / SPS) >> 4;    // CG=2: next slot's box of B
            const uint32_t bstep4 = (uint32_t)(2 * p.bn * 16) >> 4;  // CB=4: next K=8 slab of B
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int tile = cid; tile < num_tiles; tile += ncl, ++it) {
                const uint32_t acc = it & 1, acc_phase = (it >> 1) & 1;
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + acc * p.bn;
                for (int kb = 0; kb < p.num_kb; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a = smem_u32(sA + (size_t)stage * p.stage_a);
                    const uint32_t b = smem_u32(sB + (size_t)stage * p.stage_b);
                    const uint32_t acc0 = kb != 0;
                    if constexpr (CG == 2) {
                        const uint32_t alo = desc_lo(a, 16), blo = desc_lo(b, 16);
#pragma unroll
                        for (int k = 0; k < 4 * SPS; ++k) {
                            const uint32_t ao = ((k >> 2) * kBoxA + (k & 3) * 32) >> 4;
                            const uint32_t bo = (k >> 2) * bhalf16 + (uint32_t)(k & 3) * 2u;
                            mma_tf32_cg2_warp(d, desc_make(alo + ao, kHiSW128), desc_make(blo + bo, kHiSW128),
                                         idesc, k ? 1u : acc0);
                        }
                        mma_commit_cg2_warp(&empty[stage]);
                    } else {
                        if constexpr (CB == 32) {
                            const uint32_t alo = desc_lo(a, 16), blo = desc_lo(b, 16);
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                mma_tf32_warp(d, desc_make(alo + 2 * k, kHiSW128), desc_make(blo + 2 * k, kHiSW128),
                                         idesc, k ? 1u : acc0);
                        } else {
                            const uint32_t alo = desc_lo(a, 2048), blo = desc_lo(b, p.bn * 16);
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                mma_tf32_warp(d, desc_make(alo + k * 256, kHiNone), desc_make(blo + k * bstep4, kHiNone),
                                         idesc, k ? 1u : acc0);
                        }
                        mma_commit_warp(&empty[stage]);
                    }
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if constexpr (CG == 2) mma_commit_cg2_warp(&tfull[acc]);
                else mma_commit_warp(&tfull[acc]);
            }
        }
    } else {
        // ===== epilogue: TMEM -> registers -> (+bias) -> NCHW =====
        const uint32_t q = warp & 3;            // TMEM lane quarter
        const int half = (int)(warp - 2) >> 2;  // this warp drains column chunks 2*k + half
        if (p.sbias_n > 0) {  // the bias once per CTA (an L2 round trip per chunk per tile otherwise)
            for (int e = (int)((warp - 2) * 32 + lane); e < p.sbias_n; e += 256)
                sbias[e] = e < p.n_rows ? __ldg(p.bias + e) : 0.f;
            asm volatile("bar.sync 3, 256;" ::: "memory");
        }
        int it = 0;
        for (int tile = cid; tile < num_tiles; tile += ncl, ++it) {
            const uint32_t acc = it & 1;
            mbar_wait(&tfull[acc], (it >> 1) & 1);
            tc_fence_after();
            const int mt = tile / p.n_tiles, nt = tile - mt * p.n_tiles;
            const int m = mt * kTileMC + (int)rank * kTileM + (int)(q * 32 + lane);
            const bool valid = m < p.M;
            int64_t base = 0;
            if (valid) {
                const int64_t n = m / p.out_hw, pix = m - n * p.out_hw;
                base = n * (int64_t)p.n_rows * p.out_hw + pix;
            }
            const int ch0 = nt * p.bn;
            const uint32_t taddr = tmem_base + ((q * 32u) << 16) + acc * p.bn;
            const int nv = ch0 + p.bn < p.n_rows ? ch0 + p.bn : p.n_rows;
            for (int c0 = half * 16; c0 < p.bn; c0 += 32)
                store_tmem_columns_nchw(taddr + c0, 16,
                                        p.out + (valid ? base + (int64_t)(ch0 + c0) * p.out_hw : 0), p.out_hw,
                                        p.bias, ch0 + c0, nv, valid, p.sbias_n > 0 ? sbias : nullptr);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (CG == 1 || leader) mbar_arrive(&tempty[acc]);
                else mbar_arrive_cluster(&tempty[acc], 0);
            }
        }
    }
    __syncwarp();
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync();
    else __syncthreads();
    tc_fence_after();
    if (warp == 1) {
        if constexpr (CG == 2) tmem_dealloc_cg2(tmem_base, p.tmem_cols);
        else tmem_dealloc(tmem_base, p.tmem_cols);
    }
#endif
}

// ---- host ----
uint32_t tmem_cols_for(int bn) {
    const int need = 2 * bn;
    uint32_t c = 32;
    while ((int)c < need) c <<= 1;
    return c;
}

template <int CB, int CG, int SPS = 2>
void launch_k(const UConvParams& p, int grid, size_t smem, cudaStream_t st) {
    once_per_device((const void*)umma_conv_kernel<CB, CG, SPS>, [&] {  // the smem limit is a per-device attribute
        PTB_CUDA(cudaFuncSetAttribute(umma_conv_kernel<CB, CG, SPS>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit));
    });
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreadsU);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    PTB_CUDA(cudaLaunchKernelEx(&cfg, umma_conv_kernel<CB, CG, SPS>, p));
}

void encode_weights(CUtensorMap* m, const float* wt, const UmmaPlan& pl, int sps) {
    if (pl.cb == 32 && pl.cg == 2) {
        // [k slot][bn/2 rows][32]: a stage's sps slots in one request (OOB slots read 0)
        const uint64_t kdim = (uint64_t)(ceil_div(pl.taps * pl.cin_p, 64) * 64);
        const uint64_t dims[3] = {32, (uint64_t)pl.n_pad, kdim / 32};
        const uint64_t strides[2] = {kdim * 4, 128};
        const uint32_t box[3] = {32, (uint32_t)(pl.bn / 2), (uint32_t)sps};
        tmap_tiled(m, wt, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    } else if (pl.cb == 32) {
        const uint64_t kdim = (uint64_t)(ceil_div(pl.taps * pl.cin_p, 64) * 64);
        const uint64_t dims[2] = {kdim, (uint64_t)pl.n_pad};
        const uint64_t strides[1] = {kdim * 4};
        const uint32_t box[2] = {32, (uint32_t)(pl.bn / pl.cg)};
        tmap_tiled(m, wt, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    } else {
        const uint64_t dims[3] = {4, (uint64_t)pl.n_pad, (uint64_t)pl.slots_p};
        const uint64_t strides[2] = {16, (uint64_t)pl.n_pad * 16};
        const uint32_t box[3] = {4, (uint32_t)pl.bn, 8};
        tmap_tiled(m, wt, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE);
    }
}

// act: NHWC [N][aH][aW][cin_p]; conv kH x kW, pad, stride -> output oH x oW, NCHW
// with pl.n_rows channels.
void run_umma(const UmmaPlan& pl, const float* act, const float* wt, int64_t N, int64_t aH,
              int64_t aW, int kH, int kW, int pH, int pW, int sH, int sW, int64_t oH, int64_t oW,
              float* out, const float* bias, double alg_flops, cudaStream_t st) {
    UConvParams p;
    memset(&p, 0, sizeof p);
    tmap_im2col(&p.tmap_a, act, N, aH, aW, pl.cin_p, kH, kW, pH, pW, sH, sW, pl.cb, kTileM,
                pl.cb == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE);
    const int64_t M = N * oH * oW;
    PTB_REQUIRE(M < (1ll << 31), "umma conv: too many output pixels");
    p.M = (int)M;
    p.oH = (int)oH;
    p.oW = (int)oW;
    p.sH = sH;
    p.sW = sW;
    p.pH = pH;
    p.pW = pW;
    p.kW = kW;
    p.chunks = (int)(pl.cin_p / pl.cb);
    p.slots = (int)(pl.taps * p.chunks);
    // two 32-deep k slots per stage on the CTA-pair path (four measured slower: convnet L3 fwd
    // 0.255 -> 0.299 ms, removed)
    const int sps = 2;
    const int slots_per_stage = pl.cb == 32 ? (pl.cg == 2 ? sps : 1) : 8;
    encode_weights(&p.tmap_b, wt, pl, sps);
    p.num_kb = (int)ceil_div(p.slots, slots_per_stage);
    p.n_rows = (int)pl.n_rows;
    p.bn = pl.bn;
    p.n_tiles = pl.n_tiles;
    p.m_tiles = (int)ceil_div(M, (int64_t)kTileM * pl.cg);
    p.stage_a = pl.cb == 32 ? kBoxA * slots_per_stage : kBoxA;  // CG=2: sps 32-deep boxes per stage
    p.stage_b = pl.cb == 32 ? (uint32_t)(pl.bn / pl.cg) * 128u * slots_per_stage : (uint32_t)pl.bn * 128u;
    p.sbias_n = (bias && pl.n_rows <= 4096) ? (int)((pl.n_rows + 15) / 16 * 16 + 16) : 0;
    int s = (kSmemLimit - 1024 - 256 - p.sbias_n * 4) / (int)(p.stage_a + p.stage_b);
    p.stages = s > 8 ? 8 : s;
    p.tmem_cols = tmem_cols_for(pl.bn);
    p.out = out;
    p.bias = bias;
    p.out_hw = oH * oW;
    const size_t smem =
        1024 + (size_t)p.stages * (p.stage_a + p.stage_b) + (2 * p.stages + 4) * 8 + 16 + (size_t)p.sbias_n * 4;
    const int num_tiles = p.m_tiles * p.n_tiles;
    const int clusters = std::min(num_tiles, sm_count() / pl.cg);
    ProfScope prof("umma_conv", st, alg_flops, 0.0);
    if (pl.cb == 4) launch_k<4, 1>(p, clusters, smem, st);
    else if (pl.cg == 2) launch_k<32, 2>(p, 2 * clusters, smem, st);
    else launch_k<32, 1>(p, clusters, smem, st);
    after_launch("umma_conv");
}

void plan_channels(UmmaPlan& pl, int64_t cin) {
    const int64_t c32 = (cin + 31) / 32 * 32;
    pl.cin_real = cin;
    if (cin % 32 == 0 || c32 * 3 <= cin * 4) {
        pl.cb = 32;
        pl.cin_p = c32;
    } else {
        pl.cb = 4;
        pl.cin_p = (cin + 3) / 4 * 4;
    }
}

void plan_rows(UmmaPlan& pl) {
    const int64_t nt = (pl.n_rows + 255) / 256;
    // CTA pairs split the BN weight rows: BN is a multiple of 16 so BN/2 is a multiple of 8
    pl.bn = (int)(((pl.n_rows + nt - 1) / nt + 15) / 16 * 16);
    pl.n_tiles = (int)ceil_div(pl.n_rows, pl.bn);
    pl.n_pad = (int64_t)pl.n_tiles * pl.bn;
    pl.slots_p = ceil_div(pl.taps * (pl.cin_p / 4), 8) * 8;
    pl.cg = (pl.cb == 32 && sm_count() >= 2) ? 2 : 1;
    // weights padded so the last (possibly half-empty) 2-slot stage reads zeros
    const int64_t kdim_p = ceil_div(pl.taps * pl.cin_p, 64) * 64;
    pl.kdim = kdim_p;
    pl.wt_elems = pl.cb == 32 ? pl.n_pad * kdim_p : pl.slots_p * pl.n_pad * 4;
}

// Wave quantisation of the im2col engine on small layers: with few 256-pixel tiles (13x13
// maps at batch 128: 85) a 256-row N tile leaves 85 units for 74 CTA pairs — two rounds,
// 57 % busy. N tiles of 128 rows (an N=128 MMA costs the same ~64 cycles as N=256 costs
// 128) give more units; pick the tiling with the fewest MMA cycles over whole rounds,
// rounds x max(64, bn/2). Tiling never changes a sum's order (each output channel's
// reduction is the same), so this may depend on N. PT_B200_CONV_REBALANCE=0: off.
void rebalance_rows(UmmaPlan& pl, int64_t M) {
    static const bool on = [] {
        const char* e = std::getenv("PT_B200_CONV_REBALANCE");
        return e ? std::atoi(e) != 0 : true;
    }();
    if (!on || pl.n_rows <= 128) return;
    const int64_t pairs = std::max(1, sm_count() / 2);
    const int64_t m_tiles = ceil_div(M, 256);
    auto cost = [&](int64_t bn, int64_t nt) {
        const int64_t rounds = ceil_div(m_tiles * nt, pairs);
        return rounds * std::max<int64_t>(64, bn / 2) * 2;  // x2: keep integers for odd bn/2
    };
    const int64_t nt0 = pl.n_tiles, bn0 = pl.bn;
    const int64_t nt1 = ceil_div(pl.n_rows, 128);
    const int64_t bn1 = (ceil_div(pl.n_rows, nt1) + 15) / 16 * 16;
    // only for a clear win: the extra N tile re-fetches the im2col A operand (L2->SM), which
    // ate a 8 % paper gain on VGG-A conv5/6 (measured slower)
    if (cost(bn1, nt1) * 100 < cost(bn0, nt0) * 85) {
        pl.bn = (int)bn1;
        pl.n_tiles = (int)ceil_div(pl.n_rows, bn1);
        pl.n_pad = (int64_t)pl.n_tiles * pl.bn;
        pl.wt_elems = pl.n_pad * pl.kdim;
    }
}

// Hankel engine choice: the pixel-run kernel wastes the border columns it computes
// (valid / computed positions); the im2col kernel wastes nothing but is L2->SM bound.
int hconv_env() {
    static const int v = [] {
        const char* e = std::getenv("PT_B200_HCONV");
        return e ? std::atoi(e) : -1;
    }();
    return v;
}

int hconv_pair_env() {
    static const int v = [] {
        const char* e = std::getenv("PT_B200_HCONV_PAIR");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}

int hconv_group_max() {
    static const int v = [] {
        const char* e = std::getenv("PT_B200_HCONV_GROUP_MAX");
        // groups of 3-4 taps win once each CTA's G*bn/2 weight rows are one TMA request
        // (tap-grouped packing): L1 dgrad G=4 0.51 -> 0.49 ms, L2 dgrad G=3 0.90 -> 0.83 ms
        const int g = e ? std::atoi(e) : 4;
        return g < 2 ? 2 : g > 4 ? 4 : g;
    }();
    return v;
}

int hconv_pair_max() {
    static const int v = [] {
        const char* e = std::getenv("PT_B200_HCONV_PAIR_MAX");
        return e ? std::atoi(e) : 64;  // measured: pairing at 128 rows (N=256) is slower
    }();
    return v;
}

void plan_hankel(UmmaPlan& pl, int64_t N, int64_t aH, int64_t aW, int64_t ph, int64_t pw, int64_t kW,
                 int64_t oH, int64_t oW) {
    if (pl.cb != 32 || pl.cg != 2 || kW < 3 || kW > 120 || hconv_env() == 0) return;
    // position rows carry the left border only (hconv_wrap, umma_hconv.cu)
    const int64_t Hp = aH + 2 * ph, Wp = aW + (hconv_wrap() ? 1 : 2) * pw;
    if (Wp > 256 || N * aH * aW >= (1ll << 31)) return;  // a padded row is one TMA box dimension
    // efficiency from the geometry alone (not N) so a batch and its per-image slices
    // always take the same engine (batched == per-image bitwise), for the tiling
    // run_hconv will use: 128-position CTA runs over whole images (flat), or over image halves
    // for one-row filters (the row-expanded small-C dgrad)
    const int64_t kH_ = pl.taps / kW;
    const int64_t R = (oH + 1) / 2;
    const double eff = kH_ > 1 ? (double)(oH * oW) / (double)(ceil_div(oH * Wp, 128) * 128)
                               : (double)(oH * oW) / (double)(2 * ceil_div(R * Wp, 128) * 128);
    // measured (convnet L2/L3/L5): the pixel-run kernel wins at >= 0.85 of positions valid,
    // ties near 0.8 and loses below, where the im2col kernel's zero waste pays for its
    // L2->SM traffic
    // With <= 64 output rows the Hankel kernel also pairs taps (N = 2*bn beats the N=64
    // MMA floor the im2col kernel sits at), which pays for more border waste: AlexNet conv2
    // dgrad (71% valid) 0.151 -> 0.122 ms.
    // Many output channels make the im2col kernel's L2->SM traffic cheaper per MAC (VGG-A
    // conv5/6, 87.5 % of positions valid on the flat tiling: im2col 9-15 % faster), so more
    // than 128 rows need 0.9 (Overfeat conv2 dgrad, 96 rows at 0.9: pixel runs 10 % faster)
    const bool will_pair = pl.n_rows <= hconv_pair_max() && hconv_pair_env() != 0;
    if (hconv_env() != 1 && eff < (will_pair ? 0.6 : pl.n_rows <= 128 ? 0.84 : 0.9)) return;
    pl.hankel = true;
    // pairing doubles N: for <= 64 rows it beats the N=64 MMA floor (L2 dgrad 1.27 ->
    // 0.92 ms). Allowed up to 128 rows (N=256) by PT_B200_HCONV_PAIR_MAX, but measured
    // slower there (L2 fwd 0.65 -> 0.75 ms)
    if (will_pair) {
        // tap grouping: G taps per MMA (N = G*bn), one N tile of all the rows. An N <= 128
        // MMA costs ~64 cycles whatever N is, so pick G minimising
        // ceil(kW / G) * max(64, G*bn/2) (L1 dgrad bn=40: G=4; L2 dgrad bn=64: G=3)
        const int bn8 = (int)((pl.n_rows + 7) / 8 * 8), bn16 = (int)((pl.n_rows + 15) / 16 * 16);
        int best_g = 2, best_bn = bn8;
        double best_cost = 1e30;
        // a short reduction per tap (filter rows x 32-channel chunks <= 9) leaves the tile
        // epilogue-paced, and the epilogue grows with G: pairs only (L1 dgrad 0.38 -> 0.32 ms,
        // VGG-A conv1 dgrad 0.246 -> 0.206, Overfeat conv1 dgrad 0.112 -> 0.093; L2 dgrad,
        // 36 per tap, keeps G = 3: 0.79 vs 0.87 ms with pairs)
        const int g_max = (pl.taps / kW) * (pl.cin_p / 32) <= 9 ? 2 : hconv_group_max();
        for (int G = 2; G <= g_max; ++G) {
            const int bn = (G % 2 == 1) ? bn16 : bn8;
            if (G * bn > 256 || (G * bn) % 16 != 0) continue;
            const double cost = (double)ceil_div(kW, G) * std::max(64.0, G * bn / 2.0);
            if (cost < best_cost - 1e-9) {
                best_cost = cost;
                best_g = G;
                best_bn = bn;
            }
        }
        pl.tap_group = best_g;
        pl.bn = best_bn;
        pl.n_tiles = 1;
        pl.n_pad = pl.bn;
        // tap-grouped packing (pack_grouped): [kH][ceil(kW/G)][G][bn][cin_p]
        pl.kdim = pl.cin_p;
        pl.wt_elems = (pl.taps / kW) * ceil_div(kW, best_g) * best_g * pl.bn * pl.cin_p;
    }
    pl.aH = aH;
    pl.aW = aW;
    pl.aph = ph;
    pl.apw = pw;
    pl.aHp = Hp;
    pl.aWp = Wp;
    pl.act_elems = N * aH * aW * pl.cin_p;  // dense: the border is TMA out-of-bounds fill
}

}  // namespace

UmmaPlan umma_plan(const Geo& g, bool dgrad) {
    UmmaPlan pl;
    if (g.N * g.oHW >= (1ll << 31) || g.N * g.HW >= (1ll << 31)) return pl;
    if (!dgrad) {
        // TMA im2col limits: rank-4 corners in [-128,127], filter offsets in [0,255],
        // traversal stride <= 8.
        if (g.pH > 128 || g.pW > 128 || g.kH > 256 || g.kW > 256) return pl;
        if (g.pH - (g.kH - 1) < -128 || g.pW - (g.kW - 1) < -128) return pl;
        if (g.sH > 8 || g.sW > 8 || g.K > 65536) return pl;
        pl.mode = UmmaPlan::kFprop;
        pl.n_rows = g.K;
        pl.taps = g.kH * g.kW;
        plan_channels(pl, g.C);
        plan_rows(pl);
        pl.act_elems = g.N * g.HW * pl.cin_p;
        if (g.sH == 1 && g.sW == 1) plan_hankel(pl, g.N, g.H, g.W, g.pH, g.pW, g.kW, g.oH, g.oW);
    } else {
        const bool tconv_ok = g.sH == 1 && g.sW == 1 && g.pH <= g.kH - 1 && g.pW <= g.kW - 1 &&
                              g.kH <= 129 && g.kW <= 129 && g.C <= 65536;
        const bool gcol_ok = g.CRS <= 1024 && g.K <= 65536;
        // a Hankel transposed conv (tap-paired for few output channels) beats gcol + col2im
        // even for small C: no CRS-wide column buffer round trip through HBM
        bool hankel_tconv = false;
        if (tconv_ok) {
            UmmaPlan t;
            t.mode = UmmaPlan::kDgradTconv;
            t.n_rows = g.C;
            t.taps = g.kH * g.kW;
            plan_channels(t, g.K);
            plan_rows(t);
            plan_hankel(t, g.N, g.oH, g.oW, g.kH - 1 - g.pH, g.kW - 1 - g.pW, g.kW, g.H, g.W);
            hankel_tconv = t.hankel;
        }
        if (gcol_ok && !hankel_tconv && (g.C < 16 || !tconv_ok)) {
            // gcol[n] = W^T(CRS x K) * gy[n] as a 1x1 conv over NHWC gy, then col2im
            pl.mode = UmmaPlan::kDgradGcol;
            pl.n_rows = g.CRS;
            pl.taps = 1;
            plan_channels(pl, g.K);
            plan_rows(pl);
            pl.act_elems = g.N * g.oHW * pl.cin_p;
            pl.extra_elems = g.N * g.CRS * g.oHW;
        } else if (tconv_ok) {
            // transposed conv as a stride-1 conv on gy with the flipped filter, pad' = k-1-pad
            pl.mode = UmmaPlan::kDgradTconv;
            pl.n_rows = g.C;
            pl.taps = g.kH * g.kW;
            plan_channels(pl, g.K);
            plan_rows(pl);
            pl.act_elems = g.N * g.oHW * pl.cin_p;
            plan_hankel(pl, g.N, g.oH, g.oW, g.kH - 1 - g.pH, g.kW - 1 - g.pW, g.kW, g.H, g.W);
        } else {
            return pl;
        }
    }
    if (pl.taps * pl.cin_p > (1ll << 31) / 4) return pl;
    if (!pl.hankel && pl.cb == 32 && pl.cg == 2) rebalance_rows(pl, dgrad ? g.N * g.HW : g.M);
    pl.ws_bytes = align_up(pl.act_elems * 4, 256) + align_up(pl.wt_elems * 4, 256) +
                  align_up(pl.extra_elems * 4, 256);
    pl.ok = true;
    return pl;
}

void umma_conv_fwd(const Geo& g, const UmmaPlan& pl, const float* x, const float* w,
                   const float* b, float* y, void* ws, cudaStream_t st, float* act_out, bool act_ready) {
    float* act = act_out ? act_out : reinterpret_cast<float*>(ws);
    float* wt = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + align_up(pl.act_elems * 4, 256));
    PTB_REQUIRE(!act_ready || act_out, "umma_conv_fwd: act_ready without act_out");
    Fork fk(st, 1);  // the weight pack (latency-bound, ~10 us) beside the layout pass
    if (pl.hankel && pl.tap_group > 1)
        pack_grouped(w, wt, g.K, g.C, g.kH, g.kW, false, pl.tap_group, pl.bn, pl.cin_p, fk.side);
    else
        pack_weights(w, wt, g.K, g.C, g.kH, g.kW, kPackFprop, pl.cb, pl.n_pad, pl.cin_p, pl.slots_p,
                     pl.wt_elems, true, fk.side);
    if (!act_ready) {
        ProfScope prof("layout", st, 0.0, 4.0 * (g.N * g.C * g.HW + g.N * g.HW * pl.cin_p));
        nchw_to_nhwc(x, act, g.N, g.C, g.HW, pl.cin_p, true, st);
    }
    fk.join();
    if (pl.hankel) {
        run_hconv(pl, act, wt, g.N, g.H, g.W, g.pH, g.pW, (int)g.kH, (int)g.kW, g.oH, g.oW, y, b,
                  2.0 * g.M * g.K * g.CRS, st);
        return;
    }
    run_umma(pl, act, wt, g.N, g.H, g.W, (int)g.kH, (int)g.kW, (int)g.pH, (int)g.pW, (int)g.sH,
             (int)g.sW, g.oH, g.oW, y, b, 2.0 * g.M * g.K * g.CRS, st);
}

void umma_conv_bwd_data(const Geo& g, const UmmaPlan& pl, const float* gy, const float* w,
                        float* gx, void* ws, cudaStream_t st, const float* gyh_pre, double alg_flops) {
    if (alg_flops < 0) alg_flops = 2.0 * g.M * g.K * g.CRS;
    float* act = reinterpret_cast<float*>(ws);
    float* wt = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + align_up(pl.act_elems * 4, 256));
    // a shared gy copy (the combined backward's NHWC transform, channels padded to 32) is only
    // this plan's operand when the plan reads 32-channel chunks of exactly that padding (a
    // small-K plan packs gy to 8/16 channels: relay it itself)
    if (gyh_pre && !(pl.cb == 32 && pl.cin_p == (g.K + 31) / 32 * 32)) gyh_pre = nullptr;
    if (gyh_pre) {
        act = const_cast<float*>(gyh_pre);
    } else {
        ProfScope prof("layout", st, 0.0, 4.0 * (g.N * g.K * g.oHW + g.N * g.oHW * pl.cin_p));
        nchw_to_nhwc(gy, act, g.N, g.K, g.oHW, pl.cin_p, true, st);
    }
    if (pl.hankel) {
        if (pl.tap_group > 1)
            pack_grouped(w, wt, g.K, g.C, g.kH, g.kW, true, pl.tap_group, pl.bn, pl.cin_p, st);
        else
            pack_weights(w, wt, g.K, g.C, g.kH, g.kW, kPackDgradFlip, pl.cb, pl.n_pad, pl.cin_p,
                         pl.slots_p, pl.wt_elems, true, st);
        run_hconv(pl, act, wt, g.N, g.oH, g.oW, pl.aph, pl.apw, (int)g.kH, (int)g.kW, g.H, g.W, gx,
                  nullptr, alg_flops, st);
        return;
    }
    if (pl.mode == UmmaPlan::kDgradTconv) {
        pack_weights(w, wt, g.K, g.C, g.kH, g.kW, kPackDgradFlip, pl.cb, pl.n_pad, pl.cin_p,
                     pl.slots_p, pl.wt_elems, true, st);
        run_umma(pl, act, wt, g.N, g.oH, g.oW, (int)g.kH, (int)g.kW, (int)(g.kH - 1 - g.pH),
                 (int)(g.kW - 1 - g.pW), 1, 1, g.H, g.W, gx, nullptr, alg_flops, st);
        return;
    }
    // kDgradGcol: gcol = W^T * gy (tensor cores), then the deterministic gather col2im
    float* gcol = reinterpret_cast<float*>(reinterpret_cast<char*>(wt) + align_up(pl.wt_elems * 4, 256));
    pack_weights(w, wt, g.K, g.C, g.kH, g.kW, kPackGcol, pl.cb, pl.n_pad, pl.cin_p, pl.slots_p,
                 pl.wt_elems, true, st);
    run_umma(pl, act, wt, g.N, g.oH, g.oW, 1, 1, 0, 0, 1, 1, g.oH, g.oW, gcol, nullptr, alg_flops, st);
    {
        ProfScope prof("layout", st, 0.0, 4.0 * (g.N * g.CRS * g.oHW + g.N * g.C * g.HW));
        col2im_batched_launch(g, gcol, gx, st);
    }
}

}  // namespace ptb
