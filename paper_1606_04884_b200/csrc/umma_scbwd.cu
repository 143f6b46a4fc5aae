// umma_scbwd.cu — fused backward of small-channel stride-1 layers (C*kH*kW <= 32, K <= 64:
// VGG-A conv1, the 3x3 cfg1 layer): updateGradInput + accGradParameters + gradBias
// from ONE read of gradOutput in its NCHW layout.
//
// These layers are HBM-bound on gy (VGG-A conv1: 822 MB of gy for 11 GFLOP per pass). The
// separate engines read it three times plus an NCHW->NHWC transform (read + write); here a
// CTA stages a gy tile {32 px, K channels, 4 rows} by TMA once and feeds both products:
//
//   dgrad (gradCol GEMM + fold):  D[p][n] = sum_k gy[k][p] * W[k][n],  n = (r, s, c)
//       A = the gy tile as MN-major (pixels contiguous; 128B swizzle, 32-byte atoms),
//       B = W^T resident in smem; the col2im fold gx[c][i+r-pH][j+s-pW] += D[(i,j)][n]
//       runs in the epilogue into a ring of gx rows in shared memory.
//   wgrad:  gW[k][n] += sum_p gy[k][p] * Xe[n][p],  Xe[(r,s,c)][(t,j)] = x[c][t+r-pH][j+s-pW]
//       A = a K-major copy of the gy tile (k rows, pixels along K), B = Xe built in smem
//       from a TMA'd x tile (x is 1/21 of gy for C = 3, K = 64).
//   gradBias: FP32 sums of the unrounded gy tile.
//
// Builder warps round the tile to TF32 (cvt.rna, in place for the dgrad operand), write the
// K-major copy, accumulate gradBias and build Xe — the tensor cores then read both operand
// layouts of the same bytes (MN-major tf32 needs the 32-byte-atom swizzle, K-major the
// 16-byte one, so one TMA box cannot serve both).
//
// Work unit = a BAND of B gx rows of one image: the CTA reads the band's B + kH - 1 gy rows
// (kH - 1 halo rows, re-read from L2 by the neighbouring band) and produces the band's gx
// rows completely, in a fixed order independent of how bands are spread over CTAs — so the
// input gradient of an image is bitwise the same in a batch and alone. Each gy
// row is OWNED by one band for wgrad / gradBias (halo rows are masked out of Xe and the bias).
// B + kH - 1 is a multiple of 4 (the dgrad MMA's M = 4 rows x 32 px).
//
// Warps: 0 TMA producer, 1 MMA issuer (+ TMEM owner), 2..5 rounding (+ gradBias), 6..9 wgrad
// operands (K-major copy, Xe), 10..13 epilogue (fold +
// gx band flush; at the end the wgrad accumulator drain). TMEM: two 32-column dgrad
// accumulators (double-buffered) and the wgrad accumulator (128/Kp row groups x 32 columns:
// one MMA covers 128/Kp gy rows with M = rows x Kp, B = their Xe blocks side by side; only
// the diagonal blocks are kept).
#include <cuda.h>

#include <cstdlib>
#include <utility>

#include "kernels.cuh"
#include "tmap.cuh"
#include "umma.cuh"

namespace ptb {

namespace {

using namespace umma;

constexpr int kThreadsB = 448;  // TMA, MMA, 4 rounding, 4 wgrad-operand, 4 epilogue warps
constexpr int kSmemLimitB = 232448;
constexpr int kRowsB = 4;  // gy rows per stage = the dgrad M block (4 x 32 px)

struct SCParams {
    CUtensorMap tmap_gy;  // gy NCHW as {oW, K, oH, N}, box {32, Kp, 4, 1}, SWIZZLE_128B_ATOM_32B
    CUtensorMap tmap_x;   // x NCHW as {W, H, N*C}, box {32, 4 + kH - 1, C}, SW128 (two boxes: 64 columns)
    const float* w;       // KCRS
    float* gx;            // NCHW
    float* part_w;        // [ctas * (128/Kp)][K][32]
    float* part_b;        // [K][ctas]
    int N, C, H, W, K, kH, kW, pH, pW, oH, oW;
    int ntaps;            // C*kH*kW (<= 32)
    int B, nb, rstages, jbs;
    int per_cta, rem;
    int stages;
    uint32_t sz_gyt, sz_gyk, sz_xe, sz_x, stage_bytes, wt_off, ring_off, sd_off, bar_off;
    uint32_t tx;          // TMA bytes per stage
    int dstages;          // derived-operand ring depth (K-major gy copy + Xe)
    uint32_t dstage_bytes, d_off;
    int do_dg, do_wg, do_bias;
    uint32_t xbox;        // bytes of one x box (1024-aligned)
    int xoff;             // x tile starts xoff (= pW rounded up to 4) columns left of the gy block
};

__device__ __forceinline__ uint32_t sw16(uint32_t o) { return o ^ (((o >> 7) & 7u) << 4); }  // SW128
__device__ __forceinline__ uint32_t sw32(uint32_t o) { return o ^ (((o >> 7) & 3u) << 5); }  // SW128, 32B atoms
__device__ __forceinline__ float rna(float v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void named_sync(uint32_t id, uint32_t n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// KP: padded output channels (32 or 64); F3: 1 = the 3x3, C = 3 layer (VGG-A conv1), whose
// fold loops are then compile-time (unrolled, loads scheduled together)
template <int KP, int F3>
__global__ void __launch_bounds__(kThreadsB, 1) umma_scbwd_kernel(const __grid_constant__ SCParams p) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
    constexpr int kPairs = 128 / KP;          // gy rows per wgrad MMA
    constexpr int kWgMmas = kRowsB / kPairs;  // wgrad MMAs per K step per stage
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((((raw + 1023u) & ~1023u)) - raw);
    const int S = p.stages;
    uint8_t* wt = smem + p.wt_off;                                   // W^T [KP/32][32 n][32 k]
    float* ring = reinterpret_cast<float*>(smem + p.ring_off);       // [C][B][W]
    // two rings: TMA stages {gy tile (the dgrad operand, rounded in place), x tile} and
    // derived stages {K-major gy copy, Xe} (the wgrad operands): a TMA stage is released as
    // soon as the dgrad MMA and the Xe build are done with it, so more gy bytes are in flight
    const int SD = p.dstages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.bar_off);
    uint64_t* ready = full + S;      // builders' pass over the gy tile (dgrad operand ready)
    uint64_t* empty = ready + S;     // dgrad MMA commit + the epilogue's Xe reads of the x tile
    uint64_t* dready = empty + S;    // [SD] K-major copy + Xe written
    uint64_t* dfree = dready + SD;   // [SD] wgrad MMAs done with them
    uint64_t* tfull = dfree + SD;    // [2]
    uint64_t* tempty = tfull + 2;    // [2]
    uint64_t* tdone = tempty + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tdone + 1);

    const uint32_t warp = warp_id_uniform(), lane = lane_id();
    const int b = (int)blockIdx.x;
    const int lo = b * p.per_cta + (b < p.rem ? b : p.rem);
    const int hi = lo + p.per_cta + (b < p.rem ? 1 : 0);
    const int nstage_unit = p.rstages * p.jbs;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.tmap_gy);
        if (p.do_wg) tma_prefetch(&p.tmap_x);
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&ready[i], 4);                // builder warps
            mbar_init(&empty[i], p.do_wg ? 9 : 1);  // dgrad MMA commit (+ 8 builder warps: tile reads)
        }
        for (int i = 0; i < SD; ++i) {
            mbar_init(&dready[i], 8);  // builder warps (K-major copy; Xe)
            mbar_init(&dfree[i], 1);   // wgrad MMA commit
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        mbar_init(tdone, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_holder, 256);
    if (warp >= 2 && warp < 6 && p.do_dg) {
        // W^T (TF32-rounded, zero past C*kH*kW and K), K-major SW128: [k / 32][n][k % 32]
        const int bt = (int)threadIdx.x - 64;
        for (int e = bt; e < KP * 32; e += 128) {
            const int n = e / KP, k = e - n * KP;
            float v = 0.f;
            if (n < p.ntaps && k < p.K) {
                const int r = n / (p.kW * p.C), sc = n - r * p.kW * p.C, s = sc / p.C, c = sc - s * p.C;
                v = rna(__ldg(p.w + (((int64_t)k * p.C + c) * p.kH + r) * p.kW + s));
            }
            const uint32_t o = (uint32_t)((k >> 5) * 4096 + n * 128 + (k & 31) * 4);
            *reinterpret_cast<float*>(wt + sw16(o)) = v;
        }
        fence_proxy_async();
    }
    if (warp >= 10) {
        const int et = (int)threadIdx.x - 320;
        const int ring_n = p.C * p.B * p.W;
        for (int e = et; e < ring_n; e += 128) ring[e] = 0.f;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;

    if (warp == 0) {
        // ===== TMA producer (+ L2 prefetch kPf stages ahead: the strided NCHW boxes have a long
        // DRAM latency and the smem ring holds only two stages) =====
        if (lane == 0) {
            constexpr int kPf = 6;
            const int total = (hi - lo) * nstage_unit;
            auto coords = [&](int it, int& n, int& i0, int& jb) {
                const int u = lo + it / nstage_unit, rem = it - (it / nstage_unit) * nstage_unit;
                n = u / p.nb;
                const int band = u - n * p.nb, rs = rem / p.jbs;
                jb = rem - rs * p.jbs;
                i0 = band * p.B + p.pH - p.kH + 1 + rs * kRowsB;
            };
            for (int it = 0; it < kPf && it < total; ++it) {
                int n, i0, jb;
                coords(it, n, i0, jb);
                tma_prefetch_4d(&p.tmap_gy, jb * 32, 0, i0, n);
            }
            int stage = 0;
            uint32_t phase = 0;
            for (int it = 0; it < total; ++it) {
                if (it + kPf < total) {
                    int n, i0, jb;
                    coords(it + kPf, n, i0, jb);
                    tma_prefetch_4d(&p.tmap_gy, jb * 32, 0, i0, n);
                }
                int n, i0, jb;
                coords(it, n, i0, jb);
                mbar_wait(&empty[stage], phase ^ 1);
                uint8_t* sb = smem + (size_t)stage * p.stage_bytes;
                mbar_arrive_expect_tx(&full[stage], p.tx);
                tma_load_4d(sb, &p.tmap_gy, &full[stage], jb * 32, 0, i0, n);
                if (p.do_wg) {
                    // the box's first column must be 16-byte aligned: start xoff >= pW columns
                    // early (xoff % 4 == 0), the Xe builder skips xoff - pW
                    uint8_t* xs = sb + p.sz_gyt;
                    tma_load_3d(xs, &p.tmap_x, &full[stage], jb * 32 - p.xoff, i0 - p.pH, n * p.C);
                    tma_load_3d(xs + p.xbox, &p.tmap_x, &full[stage], jb * 32 - p.xoff + 32, i0 - p.pH, n * p.C);
                }
                if (++stage == S) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer (whole warp converged; one elected lane issues) =====
        constexpr uint32_t kIdescDg = idesc_tf32(128, 32, 1, 0);
        constexpr uint32_t kIdescWg = idesc_tf32(128, kPairs * 32, 0, 0);
        constexpr uint32_t kHiMN = desc_hi(512, kSwizzle128B_Base32B), kHiK = desc_hi(1024, kSwizzle128B);
        const uint32_t wt_lo = desc_lo(smem_u32(wt), 16);
        int stage = 0, buf = 0, dstage = 0;
        uint32_t phase = 0, tphase = 0, dphase = 0, wacc = 0;
        const int total = (hi - lo) * nstage_unit;
        for (int it = 0; it < total; ++it) {
            mbar_wait(&ready[stage], phase);
            tc_fence_after();
            const uint32_t sb = smem_u32(smem + (size_t)stage * p.stage_bytes);
            if (p.do_dg) {
                mbar_wait(&tempty[buf], tphase ^ 1);
                tc_fence_after();
                const uint32_t alo = desc_lo(sb, (uint32_t)KP * 128u);
#pragma unroll
                for (int ks = 0; ks < KP / 8; ++ks) {
                    // A: k rows 8ks.. of the MN-major tile (1 KB per 8 rows); B: W^T chunk ks/4, +32 B
                    const uint64_t ad = desc_make(alo + (uint32_t)ks * 64u, kHiMN);
                    const uint64_t bd = desc_make(wt_lo + (uint32_t)(ks >> 2) * 256u + (uint32_t)(ks & 3) * 2u, kHiK);
                    mma_tf32_warp(tmem + (uint32_t)buf * 32u, ad, bd, kIdescDg, ks > 0 ? 1u : 0u);
                }
                mma_commit_warp(&tfull[buf]);
                if (++buf == 2) {
                    buf = 0;
                    tphase ^= 1;
                }
            }
            mma_commit_warp(&empty[stage]);  // the gy tile is free once the dgrad MMAs are done
            if (++stage == S) {
                stage = 0;
                phase ^= 1;
            }
            if (p.do_wg) {
                mbar_wait(&dready[dstage], dphase);
                tc_fence_after();
                const uint32_t db = smem_u32(smem + p.d_off + (size_t)dstage * p.dstage_bytes);
                const uint32_t klo = desc_lo(db, 16), xlo = desc_lo(db + p.sz_gyk, 16);
#pragma unroll
                for (int g = 0; g < kWgMmas; ++g) {
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) {
                        // A: rows (t, k) g*128.. of the K-major copy; B: Xe rows of the same gy rows
                        const uint64_t ad = desc_make(klo + (uint32_t)g * 1024u + (uint32_t)ks * 2u, kHiK);
                        const uint64_t bd =
                            desc_make(xlo + (uint32_t)(g * kPairs * 32) * 8u + (uint32_t)ks * 2u, kHiK);
                        mma_tf32_warp(tmem + 64u, ad, bd, kIdescWg, wacc);
                        wacc = 1;
                    }
                }
                mma_commit_warp(&dfree[dstage]);
                if (++dstage == SD) {
                    dstage = 0;
                    dphase ^= 1;
                }
            }
        }
        mma_commit_warp(tdone);
    } else if (warp < 6) {
        // ===== rounding warps: the gy tile to TF32 in place (the dgrad operand, and the
        // source of the wgrad operands), gradBias from the unrounded values =====
        const int wb = (int)warp - 2;
        constexpr int kKPerWarp = KP / 4, kJ = KP / 16;  // k values per warp; per thread
        float bsum[kJ];
#pragma unroll
        for (int j = 0; j < kJ; ++j) bsum[j] = 0.f;
        const int chunk = (int)(lane & 7), kq = (int)(lane >> 3);
        int stage = 0, dstage = 0;
        uint32_t phase = 0, dphase = 0;
        for (int u = lo; u < hi; ++u) {
            const int n = u / p.nb, band = u - n * p.nb;
            const int i_start = band * p.B + p.pH - p.kH + 1;
            const int own_lo = max(0, band * p.B + p.pH - p.kH + 1);
            const int own_hi = band == p.nb - 1 ? p.oH : (band + 1) * p.B + p.pH - p.kH + 1;
            for (int rs = 0; rs < p.rstages; ++rs) {
                const int i0 = i_start + rs * kRowsB;
                for (int jb = 0; jb < p.jbs; ++jb) {
                    mbar_wait(&full[stage], phase);
                    uint8_t* sb = smem + (size_t)stage * p.stage_bytes;
                    // rows (t, k), 8 lanes per 128-byte row; two rows at a time (loads first)
                    // one pass when the wgrad operands are wanted: the K-major copy is written
                    // from the same registers (the derived slot must be free first, so the dgrad
                    // operand waits for the previous stage's wgrad MMA); otherwise round only
                    uint8_t* gyk = nullptr;
                    if (p.do_wg) {
                        mbar_wait(&dfree[dstage], dphase ^ 1);
                        gyk = smem + p.d_off + (size_t)dstage * p.dstage_bytes;
                    }
#pragma unroll
                    for (int th = 0; th < kRowsB; th += 2) {
                        float4 rv[2][kJ];
#pragma unroll
                        for (int t = 0; t < 2; ++t)
#pragma unroll
                            for (int j = 0; j < kJ; ++j) {
                                const int k = wb * kKPerWarp + j * 4 + kq;
                                const uint32_t o = (uint32_t)(((th + t) * KP + k) * 128 + chunk * 16);
                                rv[t][j] = *reinterpret_cast<const float4*>(sb + sw32(o));
                            }
#pragma unroll
                        for (int t = 0; t < 2; ++t) {
                            const bool own = i0 + th + t >= own_lo && i0 + th + t < own_hi;
#pragma unroll
                            for (int j = 0; j < kJ; ++j) {
                                const int k = wb * kKPerWarp + j * 4 + kq;
                                const uint32_t o = (uint32_t)(((th + t) * KP + k) * 128 + chunk * 16);
                                float4 v = rv[t][j];
                                if (p.do_bias && own) bsum[j] += (v.x + v.y) + (v.z + v.w);
                                v.x = rna(v.x);
                                v.y = rna(v.y);
                                v.z = rna(v.z);
                                v.w = rna(v.w);
                                if (p.do_dg) *reinterpret_cast<float4*>(sb + sw32(o)) = v;
                                if (gyk) *reinterpret_cast<float4*>(gyk + sw16(o)) = v;
                            }
                        }
                    }
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        mbar_arrive(&ready[stage]);
                        if (gyk) {
                            mbar_arrive(&dready[dstage]);
                            mbar_arrive(&empty[stage]);
                        }
                    }
                    if (p.do_wg && ++dstage == SD) {
                        dstage = 0;
                        dphase ^= 1;
                    }
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
        if (p.do_bias) {
            // fixed-order reduce over the 8 lanes sharing k, then one write per k
#pragma unroll
            for (int j = 0; j < kJ; ++j) {
                float v = bsum[j];
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                const int k = wb * kKPerWarp + j * 4 + kq;
                if (chunk == 0 && k < p.K) p.part_b[(int64_t)k * gridDim.x + b] = v;
            }
        }
    } else if (warp < 10) {
        // ===== Xe warps: Xe[t][n][px] = tf32(x[c][t + r][px + s]) from the x tile (two SW128
        // boxes [c][row][32 px]), zero for gy rows this band does not own =====
        if (p.do_wg) {
            const int bt = (int)threadIdx.x - 192;
            const int kWC = p.kW * p.C;
            // Xe items of this thread (fixed per stage): 8 float4 per (t, n) row
            constexpr int kXeIt = (kRowsB * 32 * 8 + 127) / 128;
            int xs_row[kXeIt], xs_col[kXeIt], xs_dst[kXeIt], xs_t[kXeIt];
            const int x_rows = kRowsB + p.kH - 1;
#pragma unroll
            for (int it = 0; it < kXeIt; ++it) {
                const int e = bt + 128 * it;
                const int qq = e & 7, tn = e >> 3;
                const int t = tn / p.ntaps, nn = tn - t * p.ntaps;
                const int r = nn / kWC, sc = nn - r * kWC, ss = sc / p.C, c = sc - ss * p.C;
                xs_t[it] = e < kRowsB * p.ntaps * 8 ? t : -1;
                xs_row[it] = (c * x_rows + t + r) * 128;
                xs_col[it] = p.xoff - p.pW + qq * 4 + ss;
                xs_dst[it] = (int)sw16((uint32_t)((t * 32 + nn) * 128 + qq * 16));
            }
            int stage = 0, dstage = 0;
            uint32_t phase = 0, dphase = 0;
            for (int u = lo; u < hi; ++u) {
                const int n = u / p.nb, band = u - n * p.nb;
                const int i_start = band * p.B + p.pH - p.kH + 1;
                const int own_lo = max(0, band * p.B + p.pH - p.kH + 1);
                const int own_hi = band == p.nb - 1 ? p.oH : (band + 1) * p.B + p.pH - p.kH + 1;
                for (int rs = 0; rs < p.rstages; ++rs) {
                    const int i0 = i_start + rs * kRowsB;
                    for (int jb = 0; jb < p.jbs; ++jb) {
                        mbar_wait(&full[stage], phase);  // the x tile has landed
                        mbar_wait(&dfree[dstage], dphase ^ 1);
                        const uint8_t* sb = smem + (size_t)stage * p.stage_bytes;
                        uint8_t* gyk = smem + p.d_off + (size_t)dstage * p.dstage_bytes;
                        const uint8_t* xt8 = sb + p.sz_gyt;
                        uint8_t* xe = gyk + p.sz_gyk;
#pragma unroll
                        for (int it = 0; it < kXeIt; ++it) {
                            if (xs_t[it] < 0) continue;
                            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                            const int gi = i0 + xs_t[it];
                            if (gi >= own_lo && gi < own_hi) {
                                float e4[4];
#pragma unroll
                                for (int z = 0; z < 4; ++z) {
                                    const int col = xs_col[it] + z;
                                    const uint32_t o = (uint32_t)(xs_row[it] + (col & 31) * 4);
                                    e4[z] = rna(*reinterpret_cast<const float*>(xt8 + (col >> 5) * p.xbox + sw16(o)));
                                }
                                v = make_float4(e4[0], e4[1], e4[2], e4[3]);
                            }
                            *reinterpret_cast<float4*>(xe + xs_dst[it]) = v;
                        }
                        fence_proxy_async();
                        __syncwarp();
                        if (lane == 0) {
                            mbar_arrive(&dready[dstage]);
                            mbar_arrive(&empty[stage]);  // done with this stage's x tile
                        }
                        if (++dstage == SD) {
                            dstage = 0;
                            dphase ^= 1;
                        }
                        if (++stage == S) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            }
        }
    } else {
        // ===== epilogue: dgrad fold into the band's gx rows, band flush, wgrad drain =====
        const uint32_t q = warp & 3;  // TMEM lane quarter = gy row t of the stage
        const int et = (int)threadIdx.x - 320;
        int buf = 0;
        uint32_t tphase = 0;
        const int ring_rows = p.B;
        const int kH_ = F3 ? 3 : p.kH, kW_ = F3 ? 3 : p.kW, C_ = F3 ? 3 : p.C, nt_ = F3 ? 27 : p.ntaps;
        const int kWC = kW_ * C_;
        float* sD = reinterpret_cast<float*>(smem + p.sd_off);  // [4 rows][ntaps][32 px]
        // gather cells of one stage: (c, gx row hr, gx col ur) over (4 + kH - 1) x (32 + kW - 1)
        const int g_rows = kRowsB + kH_ - 1, g_cols = 32 + kW_ - 1;
        const int g_cells = C_ * g_rows * g_cols;
        if (p.do_dg) {
            for (int u = lo; u < hi; ++u) {
                const int n = u / p.nb, band = u - n * p.nb;
                const int i_start = band * p.B + p.pH - p.kH + 1;
                for (int rs = 0; rs < p.rstages; ++rs) {
                    for (int jb = 0; jb < p.jbs; ++jb) {
                        if (!p.do_dg) continue;
                        mbar_wait(&tfull[buf], tphase);
                        tc_fence_after();
                        {
                            // D row block of this warp's gy row -> sD[q][n][lane] (conflict-free)
                            uint32_t a[16], c2[16];
                            const uint32_t ta = tmem + ((q * 32u) << 16) + (uint32_t)buf * 32u;
                            tmem_ld_32x32b_x16(ta, a);
                            tmem_ld_32x32b_x16(ta + 16, c2);
                            tmem_ld_wait();
                            float* d = sD + (int)q * nt_ * 32 + (int)lane;
#pragma unroll
                            for (int z = 0; z < 16; ++z) {
                                if (z < nt_) d[z * 32] = __uint_as_float(a[z]);
                                if (16 + z < nt_) d[(16 + z) * 32] = __uint_as_float(c2[z]);
                            }
                        }
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[buf]);
                        if (++buf == 2) {
                            buf = 0;
                            tphase ^= 1;
                        }
                        named_sync(1, 128);
                        // fold: each gx cell this stage touches has ONE owner thread, which sums
                        // its taps in (r, s) order and updates the band ring once (fixed order)
                        {
                            const int i0 = i_start + rs * kRowsB;
                            for (int e = et; e < g_cells; e += 128) {
                                const int c = e / (g_rows * g_cols), rem = e - c * (g_rows * g_cols);
                                const int hr = rem / g_cols, ur = rem - hr * g_cols;
                                const int hb = i0 - p.pH + hr - band * p.B;   // ring row
                                const int uu = jb * 32 - p.pW + ur;           // gx column
                                if (hb < 0 || hb >= ring_rows || uu < 0 || uu >= p.W) continue;
                                float acc = 0.f;
#pragma unroll
                                for (int r = 0; r < (F3 ? 3 : p.kH); ++r) {
                                    const int t = hr - r;
                                    const float* dr = sD + (t * nt_ + r * kWC + c) * 32;
#pragma unroll
                                    for (int s2 = 0; s2 < (F3 ? 3 : p.kW); ++s2) {
                                        const int j = ur - s2;
                                        const float v = (t >= 0 && t < kRowsB && j >= 0 && j < 32)
                                                            ? dr[s2 * C_ * 32 + j] : 0.f;
                                        acc += v;
                                    }
                                }
                                ring[((int64_t)c * ring_rows + hb) * p.W + uu] += acc;
                            }
                        }
                        named_sync(1, 128);
                    }
                }
                if (!p.do_dg) continue;
                // band complete: flush its gx rows, clear the ring
                named_sync(1, 128);
                const int h0 = band * p.B;
                const int rows = min(p.B, p.H - h0);
                // (c, ring row) pairs over the 4 warps, lanes along the row; every ring row is
                // cleared (the last band's rows past H hold contributions to rows outside gx)
                for (int cr = (int)q; cr < C_ * ring_rows; cr += 4) {
                    const int c = cr / ring_rows, hb = cr - c * ring_rows;
                    float* rp = ring + ((int64_t)c * ring_rows + hb) * p.W;
                    float* gp = p.gx + (((int64_t)n * C_ + c) * p.H + h0 + hb) * p.W;
                    for (int uu = (int)lane; uu < p.W; uu += 32) {
                        if (hb < rows) __stcs(gp + uu, rp[uu]);
                        rp[uu] = 0.f;
                    }
                }
                named_sync(1, 128);
            }
        }
        if (p.do_wg) {
            mbar_wait(tdone, 0);
            tc_fence_after();
            // lane L = q*32 + lane holds gy-row group g = L / KP, channel k = L % KP; its
            // diagonal block is columns 64 + g*32 ..
            const int L = (int)(q * 32 + lane);
            const int g = L / KP, k = L - g * KP;
            const uint32_t ta = tmem + ((q * 32u) << 16) + 64u + (uint32_t)g * 32u;
            uint32_t a[16], c2[16];
            tmem_ld_32x32b_x16(ta, a);
            tmem_ld_32x32b_x16(ta + 16, c2);
            tmem_ld_wait();
            if (k < p.K) {
                float* dst = p.part_w + (((int64_t)b * kPairs + g) * p.K + k) * 32;
                const bool any = lo < hi;
#pragma unroll
                for (int z = 0; z < 16; ++z) {
                    dst[z] = any ? __uint_as_float(a[z]) : 0.f;
                    dst[16 + z] = any ? __uint_as_float(c2[z]) : 0.f;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, 256);
#endif
}

// gw[k][c][r][s] = (acc ? gw : 0) + scale * sum_piece part[piece][k][n], n = (r*kW + s)*C + c.
// Four threads per output each sum a quarter of the pieces in order, then a fixed tree.
__global__ void scbwd_wreduce_kernel(const float* __restrict__ part, float* __restrict__ gw, int K, int C, int kH,
                                     int kW, int pieces, float scale, int accumulate) {
    __shared__ float red[4][64];
    const int ntaps = C * kH * kW, total = K * ntaps;
    const int qtr = threadIdx.x >> 6, li = threadIdx.x & 63;
    const int per = (pieces + 3) / 4, b0 = qtr * per, b1 = min(pieces, b0 + per);
    for (int base = blockIdx.x * 64; base < total; base += gridDim.x * 64) {
        const int i = base + li;
        float acc = 0.f;
        int k = 0, nn = 0;
        if (i < total) {
            k = i / ntaps;
            nn = i - k * ntaps;
            const float* src = part + (int64_t)k * 32 + nn;
            for (int pc = b0; pc < b1; ++pc) acc += __ldg(src + (int64_t)pc * K * 32);
        }
        red[qtr][li] = acc;
        __syncthreads();
        if (qtr == 0 && i < total) {
            const float sum = ((red[0][li] + red[1][li]) + red[2][li]) + red[3][li];
            const int r = nn / (kW * C), sc = nn - r * kW * C, s = sc / C, c = sc - s * C;
            const int64_t o = (((int64_t)k * C + c) * kH + r) * kW + s;
            gw[o] = (accumulate ? gw[o] : 0.f) + scale * sum;
        }
        __syncthreads();
    }
}

// gb[k] = (acc ? gb[k] : 0) + scale * sum_cta part[k][cta] (fixed order)
__global__ void scbwd_breduce_kernel(const float* __restrict__ part, float* __restrict__ gb, int ctas, float scale,
                                     int accumulate) {
    const int k = blockIdx.x;
    float acc = 0.f;
    for (int c = threadIdx.x; c < ctas; c += 32) acc += __ldg(part + (int64_t)k * ctas + c);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) gb[k] = (accumulate ? gb[k] : 0.f) + scale * acc;
}

struct SCPlan {
    bool ok = false;
    int Kp, ntaps, B, nb, rstages, jbs, units, ctas, stages, dstages;
    uint32_t dstage_bytes, d_off;
    uint32_t xbox;
    uint32_t sz_gyt, sz_gyk, sz_xe, sz_x, stage_bytes, wt_off, ring_off, sd_off, bar_off;
    size_t smem;
};

SCPlan scplan(const Geo& g) {
    SCPlan pl;
    if (!(g.sH == 1 && g.sW == 1 && g.K <= 64 && g.C * g.kH * g.kW <= 32 && g.oW % 4 == 0 && g.W % 4 == 0))
        return pl;
    if (g.N * g.K * g.oHW >= (1ll << 31) || g.N * g.C * g.HW >= (1ll << 31) || g.N >= 65536) return pl;
    pl.Kp = g.K <= 32 ? 32 : 64;
    pl.ntaps = (int)(g.C * g.kH * g.kW);
    pl.jbs = (int)ceil_div(g.oW, 32);
    if ((g.pW + 3) / 4 * 4 - g.pW + 32 + g.kW - 1 > 64) return pl;  // the x tile is two 32-column boxes
    pl.xbox = (uint32_t)align_up((size_t)(kRowsB + g.kH - 1) * g.C * 128, 1024);
    pl.sz_gyt = (uint32_t)(kRowsB * pl.Kp * 128);
    pl.sz_gyk = pl.sz_gyt;
    pl.sz_xe = (uint32_t)(kRowsB * 32 * 128);
    pl.sz_x = 2 * pl.xbox;
    pl.stage_bytes = pl.sz_gyt + pl.sz_x;          // TMA ring stage
    pl.dstage_bytes = pl.sz_gyk + pl.sz_xe;        // derived ring stage
    const uint32_t wt_bytes = (uint32_t)(pl.Kp * 128);
    const uint32_t sd_bytes = (uint32_t)align_up((size_t)kRowsB * pl.ntaps * 32 * 4, 1024);  // D staging
    const int sms = sm_count();
    // band rows: B + kH - 1 fills whole 4-row stages (j stages: 4 by default, 16 gy rows,
    // B = 17 - kH; at least 8 gx rows). The choice depends on the geometry only, never on N —
    // the banding fixes the summation order of gx, so a batch and its single images must band
    // alike (batched == per-image bitwise).
    // A 2-deep derived ring (K-major copy + Xe) decouples the rounding warps from the previous
    // stage's wgrad MMA; one 4-row stage less per band buys the smem for it where needed
    // (VGG-A conv1: j = 3 with 2 derived + 2 TMA stages 0.447 ms vs j = 4 with 1 + 3 0.456 ms;
    // j = 5 0.497 ms)
    int j0 = 4;
    while (4 * j0 - (int)(g.kH - 1) < 8) ++j0;
    auto ring_of = [&](int jj) {
        return (uint32_t)align_up((size_t)g.C * (4 * jj - (int)(g.kH - 1)) * g.W * 4, 1024);
    };
    auto budget_of = [&](int jj) { return kSmemLimitB - 1024 - (int)(wt_bytes + ring_of(jj) + sd_bytes + 1024); };
    auto fits = [&](int jj) {
        const int B = 4 * jj - (int)(g.kH - 1);
        return B >= 1 && budget_of(jj) >= (int)(2 * pl.stage_bytes + pl.dstage_bytes);
    };
    const int two_sd = (int)(2 * pl.stage_bytes + 2 * pl.dstage_bytes);
    int j = j0;
    if (budget_of(j0) < two_sd && 4 * (j0 - 1) - (int)(g.kH - 1) >= 8 && budget_of(j0 - 1) >= two_sd) j = j0 - 1;
    while (j > 1 && !fits(j)) --j;
    if (!fits(j)) return pl;
    pl.B = 4 * j - (int)(g.kH - 1);
    pl.nb = (int)ceil_div(g.H, pl.B);
    pl.rstages = j;
    pl.units = (int)(g.N * pl.nb);
    pl.ctas = std::min(pl.units, sms);
    const uint32_t ring_bytes = ring_of(j);
    const int budget = budget_of(j);
    pl.dstages = budget >= two_sd ? 2 : 1;
    pl.stages = std::min(6, (budget - pl.dstages * (int)pl.dstage_bytes) / (int)pl.stage_bytes);
    if (pl.stages < 2) return pl;
    pl.d_off = (uint32_t)pl.stages * pl.stage_bytes;
    pl.wt_off = pl.d_off + (uint32_t)pl.dstages * pl.dstage_bytes;
    pl.ring_off = pl.wt_off + wt_bytes;
    pl.sd_off = pl.ring_off + ring_bytes;
    pl.bar_off = pl.sd_off + sd_bytes;
    pl.smem = 1024 + (size_t)pl.bar_off + 1024;
    pl.ok = true;
    return pl;
}

bool scbwd_env() {
    static const bool on = [] {
        const char* e = std::getenv("PT_B200_SCBWD");
        return e ? std::atoi(e) != 0 : true;
    }();
    return on;
}

}  // namespace

bool scbwd_ok(const Geo& g) { return scbwd_env() && scplan(g).ok; }

size_t scbwd_workspace(const Geo& g) {
    const SCPlan pl = scplan(g);
    if (!pl.ok) return 0;
    return align_up((size_t)pl.ctas * (128 / pl.Kp) * g.K * 32 * 4, 256) + align_up((size_t)g.K * pl.ctas * 4, 256);
}

void scbwd(const Geo& g, const float* x, const float* gy, const float* w, float* gx, float* gw, float* gb,
           float scale, int accumulate, float bscale, int bacc, void* ws, cudaStream_t st) {
    const SCPlan pl = scplan(g);
    PTB_REQUIRE(pl.ok && scbwd_env(), "scbwd: unsupported geometry");
    PTB_REQUIRE(gx || gw, "scbwd: nothing to compute");
    SCParams p;
    memset(&p, 0, sizeof p);
    {
        const uint64_t dims[4] = {(uint64_t)g.oW, (uint64_t)g.K, (uint64_t)g.oH, (uint64_t)g.N};
        const uint64_t strides[3] = {(uint64_t)(g.oHW * 4), (uint64_t)(g.oW * 4), (uint64_t)(g.K * g.oHW * 4)};
        const uint32_t box[4] = {32, (uint32_t)pl.Kp, (uint32_t)kRowsB, 1};
        tmap_tiled(&p.tmap_gy, gy, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    }
    if (gw) {
        const uint64_t dims[3] = {(uint64_t)g.W, (uint64_t)g.H, (uint64_t)(g.N * g.C)};
        const uint64_t strides[2] = {(uint64_t)(g.W * 4), (uint64_t)(g.HW * 4)};
        const uint32_t box[3] = {32, (uint32_t)(kRowsB + g.kH - 1), (uint32_t)g.C};
        tmap_tiled(&p.tmap_x, x, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    }
    float* part_w = reinterpret_cast<float*>(ws);
    float* part_b = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) +
                                             align_up((size_t)pl.ctas * (128 / pl.Kp) * g.K * 32 * 4, 256));
    p.w = w;
    p.gx = gx;
    p.part_w = part_w;
    p.part_b = part_b;
    p.N = (int)g.N;
    p.C = (int)g.C;
    p.H = (int)g.H;
    p.W = (int)g.W;
    p.K = (int)g.K;
    p.kH = (int)g.kH;
    p.kW = (int)g.kW;
    p.pH = (int)g.pH;
    p.pW = (int)g.pW;
    p.oH = (int)g.oH;
    p.oW = (int)g.oW;
    p.ntaps = pl.ntaps;
    p.B = pl.B;
    p.nb = pl.nb;
    p.rstages = pl.rstages;
    p.jbs = pl.jbs;
    p.per_cta = pl.units / pl.ctas;
    p.rem = pl.units % pl.ctas;
    p.stages = pl.stages;
    p.sz_gyt = pl.sz_gyt;
    p.sz_gyk = pl.sz_gyk;
    p.sz_xe = pl.sz_xe;
    p.sz_x = pl.sz_x;
    p.stage_bytes = pl.stage_bytes;
    p.dstages = pl.dstages;
    p.dstage_bytes = pl.dstage_bytes;
    p.d_off = pl.d_off;
    p.wt_off = pl.wt_off;
    p.ring_off = pl.ring_off;
    p.sd_off = pl.sd_off;
    p.bar_off = pl.bar_off;
    p.do_dg = gx != nullptr;
    p.do_wg = gw != nullptr;
    p.do_bias = gw != nullptr && gb != nullptr;
    p.xbox = pl.xbox;
    p.xoff = (int)(g.pW + 3) / 4 * 4;
    p.tx = pl.sz_gyt + (gw ? (uint32_t)(2 * (kRowsB + g.kH - 1) * g.C * 128) : 0u);

    if (gx && !w) fail_validation("scbwd: gradInput needs the weight");
    if (!gx) p.w = nullptr;
    once_per_device((const void*)umma_scbwd_kernel<32, 0>, [&] {
        for (auto fn : {umma_scbwd_kernel<32, 0>, umma_scbwd_kernel<64, 0>, umma_scbwd_kernel<32, 1>,
                        umma_scbwd_kernel<64, 1>})
            PTB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimitB));
    });
    {
        const double flops = 2.0 * g.M * g.K * g.CRS * ((gx ? 1 : 0) + (gw ? 1 : 0));
        // algorithmic bytes: gy read once, gx written, x read (the HBM roofline of this kernel)
        const double bytes = 4.0 * ((double)g.N * g.K * g.oHW + (gx ? (double)g.N * g.C * g.HW : 0.0) +
                                    (gw ? (double)g.N * g.C * g.HW : 0.0));
        ProfScope prof(gw ? "umma_wgrad" : "umma_conv", st, flops, bytes);
        const bool f3 = g.kH == 3 && g.kW == 3 && g.C == 3;
        const dim3 grid((unsigned)pl.ctas);
        if (pl.Kp == 32 && f3) umma_scbwd_kernel<32, 1><<<grid, kThreadsB, pl.smem, st>>>(p);
        else if (pl.Kp == 32) umma_scbwd_kernel<32, 0><<<grid, kThreadsB, pl.smem, st>>>(p);
        else if (f3) umma_scbwd_kernel<64, 1><<<grid, kThreadsB, pl.smem, st>>>(p);
        else umma_scbwd_kernel<64, 0><<<grid, kThreadsB, pl.smem, st>>>(p);
        after_launch("umma_scbwd");
    }
    if (gw) {
        const int64_t n = g.K * pl.ntaps;
        scbwd_wreduce_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 64), 8 * (int64_t)sm_count()), 256, 0, st>>>(
            part_w, gw, (int)g.K, (int)g.C, (int)g.kH, (int)g.kW, pl.ctas * (128 / pl.Kp), scale, accumulate);
        after_launch("scbwd_wreduce");
        if (gb) {
            scbwd_breduce_kernel<<<(unsigned)g.K, 32, 0, st>>>(part_b, gb, pl.ctas, bscale, bacc);
            after_launch("scbwd_breduce");
        }
    }
}

}  // namespace ptb
