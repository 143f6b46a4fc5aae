// umma_gfold.cu — tensor-core input gradient (updateGradInput) of
// small-channel stride-1 layers with a wide filter (convnet L1: C = 3, 11x11, K = 96), read
// straight from gradOutput's NCHW layout: the gradCol GEMM with the col2im fold in the
// epilogue.
//
//   D[p][n] = sum_k gy[k][p] * W[k][n],         n = (r*C + c)*kW + s   (C*kH*kW <= 384)
//   gx[c][i + r - pH][j + s - pW] += D[(i, j)][n]
//
// Why: as a transposed conv these layers have C = 3 output channels — an N = 3 GEMM that
// the row-expanded form (umma_rowwgrad.cu) only widens to N = kH*C = 33, and that form
// needs gy transposed to NHWC first (a full read + write of the largest tensor of the layer).
// Here N = C*kH*kW (363 -> 3 chunks of 128), the A operand is the NCHW gy tile itself
// (pixels contiguous = MN-major, 128B swizzle with 32-byte atoms; TF32-rounded in place by
// builder warps), and the fold never leaves the SM.
//
// CTA pair (cta_group::2, M = 256): each CTA holds half of W^T (64 of every 128 columns,
// K-major SW128, loaded once by a bulk copy of a pre-swizzled image) and stages its own gy
// tiles of 4 rows x 32 pixels x Kp channels; the two CTAs work on different images (same
// band), so their gx never overlap. A row's box starts at the 16-byte boundary at or before
// the segment (gy rows of convnet L1 are 118 floats: TMA boxes must start 16-byte aligned);
// the builders zero the pixels outside the row and the fold shifts by the offset.
//
// Fold (epilogue warps, lane quarter q = gy row i0 + q, lane = pixel j0 + lane): for each
// (r, c) group the kW taps go to gx columns j + s — a shuffle by s lanes (wrapping lanes
// carry into the 32..32+kW-2 overhang) sums them in registers; the four rows' group sums
// meet in a small staging buffer and one owner thread per gx cell adds them (fixed order)
// into a ring of gx rows in shared memory, flushed to HBM as rows complete.
//
// Banding (batch invariance): an image's gy rows are cut into bands of
// 4*Bb rows (geometry only, 4*Bb >= kH - 1). A band writes the gx rows it owns and its
// kH - 1 overhang rows into a spill buffer; a fixup pass adds each spill to the next band's
// rows. Every gx value is therefore summed in an order fixed by the geometry, whichever
// CTA ran the bands and whatever the batch.
//
// Warps: 0 TMA producer, 1 MMA issuer (pair leader), 2..5 builders (TF32 rounding),
// 6..13 epilogue (fold, ring, flush). TMEM: four 128-column accumulators.
#include <cuda.h>

#include <cstdlib>
#include <type_traits>

#include "kernels.cuh"
#include "tmap.cuh"
#include "umma.cuh"

namespace ptb {

namespace {

using namespace umma;

constexpr int kThreadsG = 448;  // 1 TMA + 1 MMA + 4 builder + 8 epilogue warps
constexpr int kSmemLimitG = 232448;
constexpr int kRB = 16;    // gx ring rows (>= kH + 1)
constexpr int kTB = 4;     // TMEM accumulators of 128 columns (all 512): chunks in flight between
                           // the MMA and the fold cover the commit -> fold -> release round trip

struct GFParams {
    CUtensorMap tmap_gy;  // gy planes flat {oH*oW, K, N}, box {32, Kp, 1}, SW128 32-byte atoms
    const float* wpk;     // W^T halves [2][nch][kcs][64 n][32 k], SW128-swizzled (gfold_pack_kernel)
    float* gx;            // NCHW
    float* spill;         // [N][nb][kH - 1][C][W]
    unsigned long long* tl;  // debug timeline (PT_B200_GFOLD_DBG & 16): [tile][8] globaltimer, CTA pair 0
    int N, C, H, W, K, kH, kW, pH, pW, oH, oW;
    int Kp, kcs, nch, G;
    int Bg, nb, jsegs;    // gy rows per band, bands per image, 128-pixel segments per gy row
    int per_pair, rem;    // pair-units (image pair, band) per CTA pair
    int stages;
    int dbg;  // PT_B200_GFOLD_DBG (timing experiments): 1 no fold, 2 no rounding, 4 no MMA, 8 no gy loads
    uint32_t a_bytes, wt_bytes, wt_off, ring_off, bar_off;
};

__device__ __forceinline__ uint32_t sw16(uint32_t o) { return o ^ (((o >> 7) & 7u) << 4); }  // SW128
__device__ __forceinline__ uint32_t sw32(uint32_t o) { return o ^ (((o >> 7) & 3u) << 5); }  // SW128, 32B atoms
__device__ __forceinline__ float rna(float v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void named_sync(uint32_t id, uint32_t n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define GF_TL(ev)                                                                             \
    if (p.tl && blockIdx.x < 2 && tcount < 64 && lane == 0) p.tl[(tcount * 2 + blockIdx.x) * 8 + (ev)] = gtimer();
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Column layout of a 128-column chunk: group gl (< GPC = 128 / KW) at columns gl*KW .. +KW-1
// (tap s), group g = chunk*GPC + gl = (r*C + c).
template <int KW>
struct Fold {
    static constexpr int GPC = 128 / KW;
    // Groups [GA, GB) of a chunk: their columns' 16-column TMEM blocks
    template <int GA, int GB>
    struct Range {
        static constexpr int NG = GB - GA, b0 = GA * KW / 16, NB = (GB * KW + 15) / 16 - b0;
    };
    template <int GA, int GB>
    static __device__ __forceinline__ void load(uint32_t ta, uint32_t (&v)[Range<GA, GB>::NB][16]) {
        constexpr int b0 = Range<GA, GB>::b0, NB = Range<GA, GB>::NB;
#pragma unroll
        for (int b = 0; b < NB; ++b) tmem_ld_32x32b_x16(ta + (uint32_t)((b0 + b) * 16), v[b]);
        tmem_ld_wait();
    }
    // Every tap s of a group moves s lanes up (pixel j -> gx column j + s, src[s] =
    // (lane - s) & 31); lanes below s wrap into the 32..32+KW-2 overhang (hi). Two groups per
    // step share the shuffle sources and accumulate with one packed add (FADD2): all taps into
    // acc, the wrapped ones also into hi, lo = acc - hi (exact for TF32-exact data, otherwise
    // within one FP32 ulp of the larger part).
    template <int GA, int GB>
    static __device__ __forceinline__ void fold(const uint32_t (&v)[Range<GA, GB>::NB][16], int lane,
                                                const int (&src)[KW], float (&lo)[Range<GA, GB>::NG],
                                                float (&hi)[Range<GA, GB>::NG]) {
        constexpr int b0 = Range<GA, GB>::b0, NG = Range<GA, GB>::NG, NP = (NG + 1) / 2;
        // the pairs' accumulation chains interleaved (s outer): NP independent FADD2 chains
        uint64_t acc[NP], h2[NP];  // {group 2p, group 2p + 1} of the range
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) acc[pp] = h2[pp] = 0;
#pragma unroll
        for (int s = 0; s < KW; ++s) {
            const bool wrap = lane < s;
#pragma unroll
            for (int pp = 0; pp < NP; ++pp) {
                const int gl = GA + 2 * pp;
                const bool two = gl + 1 < GB;
                const int c1 = gl * KW + s - b0 * 16, c2 = c1 + KW;
                const uint32_t x1 = __shfl_sync(0xffffffffu, v[c1 >> 4][c1 & 15], src[s]);
                const uint32_t x2 = two ? __shfl_sync(0xffffffffu, v[c2 >> 4][c2 & 15], src[s]) : 0u;
                asm("{\n\t.reg .b64 x, y;\n\t"
                    "mov.b64 x, {%2, %3};\n\t"
                    "mov.b64 y, {%4, %5};\n\t"
                    "add.rn.f32x2 %0, %0, x;\n\t"
                    "add.rn.f32x2 %1, %1, y;\n\t}"
                    : "+l"(acc[pp]), "+l"(h2[pp])
                    : "r"(x1), "r"(x2), "r"(wrap ? x1 : 0u), "r"(wrap ? x2 : 0u));
            }
        }
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) {
            const int j = 2 * pp;
            uint64_t l2;
            asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(l2) : "l"(acc[pp]), "l"(h2[pp]));
            float a0, a1, c0, c1;
            asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(l2));
            asm("mov.b64 {%0, %1}, %2;" : "=f"(c0), "=f"(c1) : "l"(h2[pp]));
            lo[j] = a0;
            hi[j] = c0;
            if (j + 1 < NG) {
                lo[j + 1] = a1;
                hi[j + 1] = c1;
            }
        }
    }
};

template <int KW>
__global__ void __launch_bounds__(kThreadsG, 1) umma_gfold_kernel(const __grid_constant__ GFParams p) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
    constexpr int GPC = Fold<KW>::GPC;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((((raw + 1023u) & ~1023u)) - raw);
    const int S = p.stages;
    uint8_t* wt = smem + p.wt_off;
    // two gx rings [kRB][C][W]: A takes each quarter's own columns, B the overhang into the
    // next quarter (written by a different warp in the same tile — separate rings keep every
    // update race-free and the order fixed); a flushed row is A + B
    float* ringA = reinterpret_cast<float*>(smem + p.ring_off);
    float* ringB = ringA + kRB * p.C * p.W;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.bar_off);  // own TMA landed
    uint64_t* ready = full + S;    // builders of both CTAs done (leader's copy)
    uint64_t* empty = ready + S;   // MMAs done with the stage (multicast commit)
    uint64_t* tfull = empty + S;           // [kTB]
    uint64_t* tempty = tfull + kTB;        // [kTB] epilogues of both CTAs drained (leader's copy)
    uint64_t* wbar = tempty + kTB;         // own W^T half landed
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(wbar + 1);

    const uint32_t warp = warp_id_uniform(), lane = lane_id();
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int pair = (int)blockIdx.x >> 1;
    const int lo = pair * p.per_pair + (pair < p.rem ? pair : p.rem);
    const int hi = lo + p.per_pair + (pair < p.rem ? 1 : 0);

    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.tmap_gy);
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&ready[i], 8);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < kTB; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 16);
        }
        mbar_init(wbar, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc_cg2(tmem_holder, 128 * kTB);
    if (warp >= 6) {
        const int n = 2 * kRB * p.C * p.W;
        for (int e = (int)threadIdx.x - 192; e < n; e += 256) ringA[e] = 0.f;
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;
    // the pair's tiles: units (image pair, band) [lo, hi), a band's gy rows, 128-px segments
#define GF_FOR_TILES(...)                                                        \
    {                                                                            \
        int tcount = 0;                                                          \
        (void)tcount;                                                            \
        for (int u = lo; u < hi; ++u) {                                          \
            const int np = u / p.nb, band = u - np * p.nb;                      \
            const int i_a = band * p.Bg, i_e = min(i_a + p.Bg, p.oH);            \
            for (int i = i_a; i < i_e; ++i)                                      \
                for (int js = 0; js < p.jsegs; ++js, ++tcount) { __VA_ARGS__ }   \
        }                                                                        \
    }

    if (warp == 0) {
        // ===== TMA producer: W^T half once, then per tile four boxes {32 px, Kp} of one gy
        // row, from the 16-byte boundary at or before the segment start =====
        if (lane == 0) {
            mbar_arrive_expect_tx(wbar, p.wt_bytes);
            bulk_load(wt, p.wpk + (size_t)rank * (p.wt_bytes / 4), p.wt_bytes, wbar);
            int stage = 0;
            uint32_t phase = 0;
            const uint32_t qbytes = p.a_bytes / 4;
            // L2 prefetch kPf tiles ahead (the tall {32 px, Kp planes} boxes have a long DRAM
            // latency and the ring holds two tiles): a cursor over the same tile sequence
            constexpr int kPf = 8;
            int pu = lo, pi = 0, pj = 0, pie = 0;
            bool pf_live = pu < hi;
            auto pf_start = [&]() {
                const int b = pu % p.nb;
                pi = b * p.Bg;
                pie = min(pi + p.Bg, p.oH);
                pj = 0;
            };
            if (pf_live) pf_start();
            auto pf_next = [&]() {
                if (!pf_live) return;
                int n = 2 * (pu / p.nb) + (int)rank;
                if (n >= p.N) n = 0;
                const int f = pi * p.oW;
                const int x0 = f - (f & 3) + 128 * pj;
#pragma unroll
                for (int t = 0; t < 4; ++t) tma_prefetch_3d(&p.tmap_gy, x0 + 32 * t, 0, n);
                if (++pj == p.jsegs) {
                    pj = 0;
                    if (++pi == pie) {
                        if (++pu < hi) pf_start();
                        else pf_live = false;
                    }
                }
            };
            for (int k = 0; k < kPf; ++k) pf_next();
            GF_FOR_TILES({
                pf_next();
                int n = 2 * np + (int)rank;
                if (n >= p.N) n = 0;  // odd N: the spare CTA recomputes image 0 and discards it
                const int f = i * p.oW;
                const int x0 = f - (f & 3) + 128 * js;
                mbar_wait(&empty[stage], phase ^ 1);
                GF_TL(0)
                uint8_t* sb = smem + (size_t)stage * p.a_bytes;
                if (p.dbg & 8) {
                    mbar_arrive(&full[stage]);
                } else {
                    mbar_arrive_expect_tx(&full[stage], p.a_bytes);
#pragma unroll
                    for (int t = 0; t < 4; ++t) tma_load_3d(sb + t * qbytes, &p.tmap_gy, &full[stage], x0 + 32 * t, 0, n);
                }
                if (++stage == S) {
                    stage = 0;
                    phase ^= 1;
                }
            })
        }
    } else if (warp == 1) {
        if (leader) {
            // ===== MMA issuer (whole warp converged, one elected lane issues) =====
            constexpr uint32_t kIdesc = idesc_tf32(256, 128, 1, 0);
            constexpr uint32_t kHiMN = desc_hi(512, kSwizzle128B_Base32B), kHiK = desc_hi(1024, kSwizzle128B);
            const uint32_t wt_lo = desc_lo(smem_u32(wt), 16);
            const int ksteps = p.Kp / 8;
            int stage = 0, buf = 0;
            uint32_t phase = 0, tph = 0;
            GF_FOR_TILES({
                mbar_wait(&ready[stage], phase);
                GF_TL(2)
                tc_fence_after();
                const uint32_t alo = desc_lo(smem_u32(smem + (size_t)stage * p.a_bytes), (uint32_t)p.Kp * 128u);
                for (int ch = 0; ch < p.nch; ++ch) {
                    mbar_wait(&tempty[buf], tph ^ 1);
                    tc_fence_after();
                    const uint32_t bch = wt_lo + (uint32_t)(ch * p.kcs) * 512u;  // 8 KB blocks, 16 B units
                    for (int ks = 0; ks < ((p.dbg & 4) ? 1 : ksteps); ++ks) {
                        // A: k rows 8ks.. of the MN-major tile (1 KB per 8 rows); B: W^T block ks/4, +32 B
                        const uint64_t ad = desc_make(alo + (uint32_t)ks * 64u, kHiMN);
                        const uint64_t bd = desc_make(bch + (uint32_t)(ks >> 2) * 512u + (uint32_t)(ks & 3) * 2u, kHiK);
                        mma_tf32_cg2_warp(tmem + (uint32_t)buf * 128u, ad, bd, kIdesc, ks > 0 ? 1u : 0u);
                    }
                    mma_commit_cg2_warp(&tfull[buf]);
                    if (++buf == kTB) {
                        buf = 0;
                        tph ^= 1;
                    }
                }
                mma_commit_cg2_warp(&empty[stage]);
                if (++stage == S) {
                    stage = 0;
                    phase ^= 1;
                }
            })
        }
    } else if (warp < 6) {
        // ===== builders: round the tile to TF32 in place, zero the pixels outside the row =====
        const int bt = (int)threadIdx.x - 64;
        const int per_q = p.Kp * 8;  // float4s per quarter box
        const uint32_t qbytes = p.a_bytes / 4;
        mbar_wait(wbar, 0);  // this CTA's W^T half is in before its first ready
        int stage = 0;
        uint32_t phase = 0;
        GF_FOR_TILES({
            const int jb = 128 * js - ((i * p.oW) & 3);  // gy column of the tile's first pixel
            mbar_wait(&full[stage], phase);
            if (warp == 2) { GF_TL(1) }
            uint8_t* sb = smem + (size_t)stage * p.a_bytes;
#pragma unroll 1
            for (int t = 0; t < 4; ++t) {
                const int jq = jb + 32 * t;
                const bool inner = jq >= 0 && jq + 32 <= p.oW;
                uint8_t* qb = sb + t * qbytes;
                for (int e = bt; e < ((p.dbg & 2) ? 0 : per_q); e += 128) {
                    const uint32_t o = (uint32_t)e * 16u;
                    float4 v = *reinterpret_cast<const float4*>(qb + o);
                    if (inner) {
                        v.x = rna(v.x);
                        v.y = rna(v.y);
                        v.z = rna(v.z);
                        v.w = rna(v.w);
                    } else {
                        const int j = jq + (int)((sw32(o) & 127u) >> 2);
                        v.x = j >= 0 && j < p.oW ? rna(v.x) : 0.f;
                        v.y = j + 1 >= 0 && j + 1 < p.oW ? rna(v.y) : 0.f;
                        v.z = j + 2 >= 0 && j + 2 < p.oW ? rna(v.z) : 0.f;
                        v.w = j + 3 >= 0 && j + 3 < p.oW ? rna(v.w) : 0.f;
                    }
                    *reinterpret_cast<float4*>(qb + o) = v;
                }
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                if (leader) mbar_arrive(&ready[stage]);
                else mbar_arrive_cluster(&ready[stage], 0);
            }
            if (++stage == S) {
                stage = 0;
                phase ^= 1;
            }
        })
    } else {
        // ===== epilogue (8 warps: TMEM lane quarter q, half of each chunk's groups): fold D
        // into the gx rings, flush rows as they complete =====
        const int q = (int)(warp & 3);          // TMEM lane quarter = 32-pixel quarter of the tile
        const int half = (int)(warp - 6) >> 2;  // groups [0, GPC/2) or [GPC/2, GPC) of each chunk
        const int et = (int)threadIdx.x - 192;
        const int C = p.C, W = p.W, G = p.G;
        const int plane = C * W;
        int src[KW];
#pragma unroll
        for (int t = 0; t < KW; ++t) src[t] = ((int)lane - t) & 31;
        int buf = 0;
        uint32_t tph = 0;
        GF_FOR_TILES({
            const int n = 2 * np + (int)rank;
            const bool live = n < p.N;
            const int colq = 128 * js - ((i * p.oW) & 3) + 32 * q - p.pW;  // gx column of lane 0, s = 0
            const int h0 = i - p.pH;                                        // gx row of r = 0
            const int wa = colq + (int)lane, wb = colq + 32 + (int)lane;
            const bool oka = wa >= 0 && wa < W, okb = (int)lane < p.kW - 1 && wb >= 0 && wb < W;
            for (int ch = 0; ch < p.nch; ++ch) {
                mbar_wait(&tfull[buf], tph);
                if (warp == 6 && ch < 2) { GF_TL(3 + ch) }
                tc_fence_after();
                const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)buf * 128u;
                constexpr int GH = GPC / 2;
                const int g0 = ch * GPC + (half ? GH : 0);
                const uint32_t tb = (uint32_t)buf;
                // load this half's columns, release the accumulator, then fold and update the
                // rings (all ring loads before the stores: the groups' cells are distinct)
                auto process = [&](auto ga, auto gb) {
                    constexpr int GA = decltype(ga)::value, GB = decltype(gb)::value;
                    using R = typename Fold<KW>::template Range<GA, GB>;
                    uint32_t v[R::NB][16];
                    Fold<KW>::template load<GA, GB>(ta, v);
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if (leader) mbar_arrive(&tempty[tb]);
                        else mbar_arrive_cluster(&tempty[tb], 0);
                    }
                    if (p.dbg & 1) return;
                    float lo[R::NG], hi[R::NG];
                    Fold<KW>::template fold<GA, GB>(v, (int)lane, src, lo, hi);
                    int r = g0 / C, c = g0 - r * C;
                    int oa[R::NG];
                    bool ok[R::NG];
#pragma unroll
                    for (int j = 0; j < R::NG; ++j) {
                        const int h = h0 + r;
                        ok[j] = g0 + j < G && h >= 0 && h < p.H;  // groups past G: zero columns
                        oa[j] = (h & (kRB - 1)) * plane + c * W;
                        if (++c == C) {
                            c = 0;
                            ++r;
                        }
                    }
                    float ra[R::NG], rb[R::NG];
#pragma unroll
                    for (int j = 0; j < R::NG; ++j) {
                        ra[j] = ok[j] && oka ? ringA[oa[j] + wa] : 0.f;
                        rb[j] = ok[j] && okb ? ringB[oa[j] + wb] : 0.f;
                    }
#pragma unroll
                    for (int j = 0; j < R::NG; ++j) {
                        if (ok[j] && oka) ringA[oa[j] + wa] = ra[j] + lo[j];
                        if (ok[j] && okb) ringB[oa[j] + wb] = rb[j] + hi[j];
                    }
                };
                if (half == 0) process(std::integral_constant<int, 0>{}, std::integral_constant<int, GH>{});
                else process(std::integral_constant<int, GH>{}, std::integral_constant<int, GPC>{});
                if (++buf == kTB) {
                    buf = 0;
                    tph ^= 1;
                }
            }
            if (warp == 6) { GF_TL(5) }
            if (js == p.jsegs - 1) {
                // all of gy row i's ring updates are in (a barrier per row: the next row's
                // updates touch the same cells)
                named_sync(1, 256);
                if (warp == 6) { GF_TL(6) }
                if (p.dbg & 64) {
                    if (warp == 6) { GF_TL(5) }
                }
                // gx row i - pH is complete within the band; at the band's last row also its
                // kH - 1 overhang rows: -> spill (the next band adds them), or gx for the image's
                // last band. Each element is read, zeroed and stored by one thread; the next row
                // does not touch these ring rows, so no barrier follows (a barrier would wait for
                // the global stores) — except at the band end, whose rows the next band reuses.
                const bool bend = i == i_e - 1;
                const bool last_band = band == p.nb - 1;
                const int f0 = max(0, h0), f1 = bend ? min(p.H, h0 + p.kH) : min(p.H, h0 + 1);
                const int own_end = (bend && last_band) ? p.H : min(p.H, h0 + 1);
                for (int h = f0; h < ((p.dbg & 128) ? f0 : f1); ++h) {
                    const int o = (h & (kRB - 1)) * plane;
                    for (int c = 0; c < C; ++c) {
                        float* gdst = h < own_end
                                          ? p.gx + (((int64_t)n * C + c) * p.H + h) * W
                                          : p.spill + ((((int64_t)n * p.nb + band) * (p.kH - 1) + (h - own_end)) * C + c) * W;
                        for (int w = et; w < W; w += 256) {
                            const int e = o + c * W + w;
                            const float v = ringA[e] + ringB[e];
                            ringA[e] = 0.f;
                            ringB[e] = 0.f;
                            if (live && !(p.dbg & 32)) __stcs(gdst + w, v);
                        }
                    }
                }
                if (bend) named_sync(1, 256);
            }
            if (warp == 6) { GF_TL(7) }
        })
    }
#undef GF_FOR_TILES
    __syncwarp();
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (warp == 1) tmem_dealloc_cg2(tmem, 128 * kTB);
#endif
}

// W^T halves for the CTA pair, as the kernel's smem image: [rank][chunk][k block][64 n][32 k],
// each 8 KB block SW128-swizzled; column n of chunk ch in rank rho is ch*128 + rho*64 + n;
// within a chunk group gl = n / kW (< gpc), tap s = n % kW, group g = ch*gpc + gl = r*C + c.
// TF32-rounded, zero past the groups and K.
__global__ void gfold_pack_kernel(const float* __restrict__ w, float* __restrict__ out, int K, int C, int kH,
                                  int kW, int gpc, int nch, int kcs) {
    const int total = 2 * nch * kcs * 2048;
    const int G = kH * C;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const int blk = idx >> 11, e = idx & 2047;
        const int nl = e >> 5, kl = e & 31;
        const int kc = blk % kcs, t = blk / kcs, ch = t % nch, rho = t / nch;
        const int col = rho * 64 + nl, k = kc * 32 + kl;
        const int gl = col / kW, s = col - gl * kW, g = ch * gpc + gl;
        float v = 0.f;
        if (gl < gpc && g < G && k < K) {
            const int r = g / C, c = g - r * C;
            v = rna(__ldg(w + (((int64_t)k * C + c) * kH + r) * kW + s));
        }
        out[(size_t)blk * 2048 + (sw16((uint32_t)(nl * 128 + kl * 4)) >> 2)] = v;
    }
}

// gx rows [k*Bg - pH, + kH - 1) of band k += band k-1's spill (fixed order: own + spill)
__global__ void gfold_fixup_kernel(float* __restrict__ gx, const float* __restrict__ spill, int N, int nb, int C,
                                   int H, int W, int kH1, int band_rows, int pH) {
    const int64_t total = (int64_t)N * (nb - 1) * kH1 * C * W;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int w = (int)(idx % W);
        int64_t t = idx / W;
        const int c = (int)(t % C);
        t /= C;
        const int tr = (int)(t % kH1);
        t /= kH1;
        const int km1 = (int)(t % (nb - 1));
        const int64_t n = t / (nb - 1);
        const int h = (km1 + 1) * band_rows - pH + tr;
        if (h >= H) continue;
        float* d = gx + ((n * C + c) * H + h) * W + w;
        *d = *d + __ldg(spill + (((n * nb + km1) * kH1 + tr) * C + c) * W + w);
    }
}

struct GFPlan {
    bool ok = false;
    int Kp, kcs, gpc, nch, G, Bg, nb, jsegs, units, pairs, stages;
    uint32_t a_bytes, wt_bytes, wt_off, ring_off, bar_off;
    size_t smem;
    int64_t spill_elems;
};

bool kw_supported(int64_t kW) { return kW == 3 || kW == 5 || kW == 7 || kW == 9 || kW == 11 || kW == 13; }

GFPlan gfplan(const Geo& g) {
    GFPlan pl;
    if (!(g.sH == 1 && g.sW == 1 && g.C <= 4 && g.K <= 128 && g.kH >= 2 && g.kH <= kRB - 1 && kw_supported(g.kW) &&
          g.pH <= g.kH - 1 && g.pW <= g.kW - 1))
        return pl;
    if (g.oHW % 4 != 0 || g.N * g.K * g.oHW >= (1ll << 31) || g.N * g.C * g.HW >= (1ll << 31) || g.N >= 65536)
        return pl;
    pl.G = (int)(g.kH * g.C);
    pl.gpc = (int)(128 / g.kW);
    pl.nch = (pl.G + pl.gpc - 1) / pl.gpc;
    if (pl.nch > 3) return pl;  // one tile's D: <= 3 chunks (TMEM double-buffers 2 x 128 columns)
    pl.Kp = (int)((g.K + 15) / 16 * 16);
    pl.kcs = (pl.Kp + 31) / 32;
    // bands of >= kH - 1 gy rows (a band's overhang reaches only the next band), 12 by default —
    // geometry only, never N (batched == per-image bitwise)
    pl.Bg = (int)std::max<int64_t>(12, g.kH - 1);
    pl.nb = (int)ceil_div(g.oH, pl.Bg);
    // a row box starts up to 3 pixels early (16-byte-aligned start)
    pl.jsegs = (int)ceil_div(g.oW + (g.oW % 4 ? 3 : 0), 128);
    pl.a_bytes = (uint32_t)(4 * pl.Kp * 128);
    pl.wt_bytes = (uint32_t)(pl.nch * pl.kcs * 8192);
    const uint32_t ring_bytes = (uint32_t)align_up((size_t)2 * kRB * g.C * g.W * 4, 1024);
    const int fixed = 1024 + (int)(pl.wt_bytes + ring_bytes) + 1024;
    pl.stages = std::min(4, (kSmemLimitG - fixed) / (int)pl.a_bytes);
    if (pl.stages < 2) return pl;
    pl.wt_off = (uint32_t)pl.stages * pl.a_bytes;
    pl.ring_off = pl.wt_off + pl.wt_bytes;
    pl.bar_off = pl.ring_off + ring_bytes;
    pl.smem = 1024 + (size_t)pl.bar_off + 1024;
    pl.units = (int)(ceil_div(g.N, 2) * pl.nb);
    pl.pairs = std::min(pl.units, sm_count() / 2);
    pl.spill_elems = g.N * pl.nb * (g.kH - 1) * g.C * g.W;
    pl.ok = pl.pairs >= 1;
    return pl;
}

bool gfold_env() {
    static const bool on = [] {
        const char* e = std::getenv("PT_B200_GFOLD");
        return e ? std::atoi(e) != 0 : true;
    }();
    return on;
}

size_t wpk_bytes(const GFPlan& pl) { return align_up((size_t)2 * pl.wt_bytes, 256); }

template <int KW>
void launch_gfold(const GFParams& p, const GFPlan& pl, cudaStream_t st) {
    once_per_device((const void*)umma_gfold_kernel<KW>, [&] {
        PTB_CUDA(cudaFuncSetAttribute(umma_gfold_kernel<KW>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimitG));
    });
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * pl.pairs));
    cfg.blockDim = dim3(kThreadsG);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    PTB_CUDA(cudaLaunchKernelEx(&cfg, umma_gfold_kernel<KW>, p));
}

}  // namespace

unsigned long long*& gfold_timeline_ptr() {
    static unsigned long long* p = nullptr;
    return p;
}

bool gfold_ok(const Geo& g) { return gfold_env() && gfplan(g).ok; }

size_t gfold_workspace(const Geo& g) {
    const GFPlan pl = gfplan(g);
    if (!pl.ok) return 0;
    return wpk_bytes(pl) + align_up((size_t)pl.spill_elems * 4, 256);
}

void gfold(const Geo& g, const float* gy, const float* w, float* gx, void* ws, cudaStream_t st) {
    const GFPlan pl = gfplan(g);
    PTB_REQUIRE(pl.ok && gfold_env(), "gfold: unsupported geometry");
    GFParams p;
    memset(&p, 0, sizeof p);
    float* wpk = reinterpret_cast<float*>(ws);
    float* spill = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + wpk_bytes(pl));
    {
        // gy planes flat: {oH*oW, K, N}; a gy row need not start 16-byte aligned (oW % 4 != 0),
        // a plane must (oHW % 4 == 0)
        const uint64_t dims[3] = {(uint64_t)g.oHW, (uint64_t)g.K, (uint64_t)g.N};
        const uint64_t strides[2] = {(uint64_t)(g.oHW * 4), (uint64_t)(g.K * g.oHW * 4)};
        const uint32_t box[3] = {32, (uint32_t)pl.Kp, 1};
        tmap_tiled(&p.tmap_gy, gy, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    }
    {
        const int total = 2 * pl.nch * pl.kcs * 2048;
        gfold_pack_kernel<<<(unsigned)ceil_div(total, 256), 256, 0, st>>>(w, wpk, (int)g.K, (int)g.C, (int)g.kH,
                                                                           (int)g.kW, pl.gpc, pl.nch, pl.kcs);
        after_launch("gfold_pack");
    }
    p.wpk = wpk;
    p.gx = gx;
    p.spill = spill;
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
    p.Kp = pl.Kp;
    p.kcs = pl.kcs;
    p.nch = pl.nch;
    p.G = pl.G;
    p.Bg = pl.Bg;
    p.nb = pl.nb;
    p.jsegs = pl.jsegs;
    p.per_pair = pl.units / pl.pairs;
    p.rem = pl.units % pl.pairs;
    p.stages = pl.stages;
    {
        static const int dbg = [] {
            const char* e = std::getenv("PT_B200_GFOLD_DBG");
            return e ? std::atoi(e) : 0;
        }();
        p.dbg = dbg;
        if (dbg & 16) {
            static unsigned long long* tl = nullptr;
            if (!tl) {
                PTB_CUDA(cudaMalloc(&tl, 64 * 2 * 8 * sizeof(unsigned long long)));
            }
            PTB_CUDA(cudaMemsetAsync(tl, 0, 64 * 2 * 8 * sizeof(unsigned long long), st));
            p.tl = tl;
            gfold_timeline_ptr() = tl;
        }
    }
    p.a_bytes = pl.a_bytes;
    p.wt_bytes = pl.wt_bytes;
    p.wt_off = pl.wt_off;
    p.ring_off = pl.ring_off;
    p.bar_off = pl.bar_off;
    {
        // algorithmic bytes: gy read once + gx written (the HBM floor of this pass)
        ProfScope prof("umma_conv", st, 2.0 * g.M * g.K * g.CRS,
                       4.0 * ((double)g.N * g.K * g.oHW + (double)g.N * g.C * g.HW));
        switch (g.kW) {
            case 3: launch_gfold<3>(p, pl, st); break;
            case 5: launch_gfold<5>(p, pl, st); break;
            case 7: launch_gfold<7>(p, pl, st); break;
            case 9: launch_gfold<9>(p, pl, st); break;
            case 11: launch_gfold<11>(p, pl, st); break;
            default: launch_gfold<13>(p, pl, st); break;
        }
        after_launch("umma_gfold");
    }
    if (pl.nb > 1) {
        const int64_t total = g.N * (pl.nb - 1) * (g.kH - 1) * g.C * g.W;
        gfold_fixup_kernel<<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 8 * (int64_t)sm_count()), 256, 0,
                             st>>>(gx, spill, (int)g.N, pl.nb, (int)g.C, (int)g.H, (int)g.W, (int)(g.kH - 1), pl.Bg,
                                   (int)g.pH);
        after_launch("gfold_fixup");
    }
    if (p.tl) {  // debug timeline: per tile, ns since the first event of CTA 0
        unsigned long long h[64 * 2 * 8];
        PTB_CUDA(cudaStreamSynchronize(st));
        PTB_CUDA(cudaMemcpy(h, p.tl, sizeof h, cudaMemcpyDeviceToHost));
        const unsigned long long t0 = h[0];
        for (int t = 0; t < 64; ++t)
            for (int b = 0; b < 2; ++b) {
                fprintf(stderr, "tl tile %2d cta %d:", t, b);
                for (int e = 0; e < 8; ++e) {
                    const unsigned long long v = h[(t * 2 + b) * 8 + e];
                    fprintf(stderr, " %8lld", v ? (long long)(v - t0) : -1ll);
                }
                fprintf(stderr, "\n");
            }
    }
}

}  // namespace ptb
