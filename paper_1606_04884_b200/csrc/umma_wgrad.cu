// umma_wgrad.cu — tcgen05 (kind::tf32) weight gradient (accGradParameters).
//
//   gW^T[(r,s,c)][k] = sum_m im2col(x)[m][(r,s,c)] * gy[m][k]      m = output pixel (n,i,j)
//
// CTA-pair GEMM (cta_group::2): M = filter columns (tap, channel) — 256 per pair, 128
// per CTA as four 32-channel im2col boxes; N = output channels k (BN per tile, each
// CTA loads BN/2 of them); reduction over pixels, 64 per pipeline stage. In NHWC both
// operands are MN-major: x by TMA im2col boxes (64 px x 32 ch at filter tap (r,s)),
// gy by tiled TMA boxes (64 px x 32 ch), landing in the MN-major canonical layout
// with 32-byte-atom 128B swizzle (SWIZZLE_128B_BASE32B / TMA SWIZZLE_128B_ATOM_32B).
// The pixel reduction is split over CTA pairs (persistent, static schedule over
// (column-tile, k-tile, split) units); each unit's FP32 tile is drained from TMEM to a
// partial buffer and a fixed-order reduce kernel sums the splits (deterministic),
// applies scale / accumulate and writes KCRS.
#include <cuda.h>

#include <cstdlib>

#include "kernels.cuh"
#include "tmap.cuh"
#include "umma.cuh"

namespace ptb {

namespace {

using namespace umma;

constexpr int kThreadsW = 192;
constexpr int kSmemLimit = 232448;

struct UWgradParams {
    CUtensorMap tmap_gy;  // tiled [M][Kp], box {32 ch, 64 px}
    CUtensorMap tmap_x;   // im2col over x NHWC [N][H][W][Cp], box {32 ch, 64 px}
    int oH, oW, sH, sW, pH, pW, kW;
    int taps, Cp;
    int m_tiles, m_groups, n_tiles, splits;  // a unit covers MT consecutive m-tiles
    int kb_per_split, total_kb;
    int bn, stages;
    uint32_t stage_b, tmem_cols;
    float* part;          // [splits][m_tiles*256][n_tiles*bn]
    int64_t part_ld, part_split;
};

// MT = 2: one unit computes two 256-column m-tiles into two accumulators from the same
// gradOutput (B) stage — B is fetched once for both, and each stage covers 32 pixels so
// the smem ring keeps its depth (opt-in; see wplan).
template <int MT, int KP>  // KP: pixels (reduction rows) per stage
__global__ void __launch_bounds__(kThreadsW, 1) umma_wgrad_kernel(const __grid_constant__ UWgradParams p) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
    constexpr uint32_t BOX = KP * 128;        // one KP-pixel x 32-channel box
    constexpr uint32_t STAGE_A = MT * 4 * BOX;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((((raw + 1023u) & ~1023u)) - raw);
    const int S = p.stages;
    uint8_t* sA = smem;
    uint8_t* sB = smem + (size_t)S * STAGE_A;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + (size_t)S * p.stage_b);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

    const uint32_t warp = warp_id_uniform(), lane = lane_id();
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.tmap_gy);
        tma_prefetch(&p.tmap_x);
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);   // the leader's expect_tx arrive (peer bytes land on it)
            mbar_init(&empty[i], 1);  // one multicast commit
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 8);  // 4 epilogue warps x 2 CTAs
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc_cg2(tmem_holder, p.tmem_cols);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const int units = p.m_groups * p.n_tiles * p.splits;
    const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;

    // unit -> (m-tile, n-tile, split), m fastest: consecutive pairs share a pixel range
    auto decode = [&](int u, int& mt, int& nt, int& sp) {
        mt = (u % p.m_groups) * MT;  // first m-tile of the unit
        const int r = u / p.m_groups;
        nt = r % p.n_tiles;
        sp = r / p.n_tiles;
    };
    auto kb_count = [&](int sp) {
        const int lo = sp * p.kb_per_split;
        const int hi = lo + p.kb_per_split < p.total_kb ? lo + p.kb_per_split : p.total_kb;
        return hi - lo;
    };

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int u = cluster; u < units; u += nclusters) {
                int mt, nt, sp;
                decode(u, mt, nt, sp);
                const int nkb = kb_count(sp);
                // this CTA's filter-column boxes: (tap, channel block) -> (r, s, c0), four per m-tile
                int bc[4 * MT], br[4 * MT], bs[4 * MT];
#pragma unroll
                for (int b = 0; b < 4 * MT; ++b) {
                    const int col = (mt + b / 4) * 256 + (int)rank * 128 + (b % 4) * 32;
                    int tap = col / p.Cp;
                    bc[b] = col - tap * p.Cp;
                    if (tap >= p.taps) {  // columns past the filter are never reduced
                        tap = 0;
                        bc[b] = 0;
                    }
                    br[b] = tap / p.kW;
                    bs[b] = tap - br[b] * p.kW;
                }
                const int kbase = nt * p.bn + (int)rank * (p.bn / 2);
                // pixel cursor (n, i, j) of the first pixel of this split
                int m = sp * p.kb_per_split * KP;
                const int ohw = p.oH * p.oW;
                int n = m / ohw;
                int rem = m - n * ohw;
                int i = rem / p.oW, j = rem - i * p.oW;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* a = sA + (size_t)stage * STAGE_A;
                    uint8_t* b = sB + (size_t)stage * p.stage_b;
                    if (leader) mbar_arrive_expect_tx(&full[stage], 2 * (STAGE_A + p.stage_b));
                    const int wc = j * p.sW - p.pW, hc = i * p.sH - p.pH;
#pragma unroll
                    for (int t = 0; t < 4 * MT; ++t)
                        tma_load_im2col_4d_cg2(a + t * BOX, &p.tmap_x, &full[stage], bc[t], wc, hc, n,
                                               (uint16_t)bs[t], (uint16_t)br[t]);
                    // all of this CTA's gy channel boxes in one 3-D request: {32 ch, KP px, nbB}
                    tma_load_3d_cg2(b, &p.tmap_gy, &full[stage], 0, m, kbase / 32);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                    m += KP;
                    j += KP;
                    while (j >= p.oW) {
                        j -= p.oW;
                        if (++i == p.oH) {
                            i = 0;
                            ++n;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {  // whole warp, converged; one elected lane issues
            const uint32_t idesc = idesc_tf32(256, p.bn, 1, 1);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int u = cluster; u < units; u += nclusters, ++it) {
                int mt, nt, sp;
                decode(u, mt, nt, sp);
                const int nkb = kb_count(sp);
                const uint32_t acc = it & 1;
                mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + acc * MT * p.bn;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    // MN-major: 32-element atoms along M/N at LBO = one box,
                    // 4-row swizzle groups along K at SBO = 512 B; K=8 rows = +1 KB.
                    const uint32_t alo = desc_lo(smem_u32(sA + (size_t)stage * STAGE_A), BOX);
                    const uint32_t blo = desc_lo(smem_u32(sB + (size_t)stage * p.stage_b), BOX);
                    constexpr uint32_t kHi = desc_hi(512, kSwizzle128B_Base32B);
                    const uint32_t acc0 = kb != 0;
#pragma unroll
                    for (int t = 0; t < MT; ++t)
#pragma unroll
                        for (int k = 0; k < KP / 8; ++k)
                            mma_tf32_cg2_warp(d + t * p.bn, desc_make(alo + t * (4 * BOX >> 4) + k * 64, kHi),
                                              desc_make(blo + k * 64, kHi), idesc, k ? 1u : acc0);
                    mma_commit_cg2_warp(&empty[stage]);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                mma_commit_cg2_warp(&tfull[acc]);
            }
        }
    } else {
        const uint32_t q = warp & 3;
        const uint64_t pol = l2_evict_last_policy();
        int it = 0;
        for (int u = cluster; u < units; u += nclusters, ++it) {
            int mt, nt, sp;
            decode(u, mt, nt, sp);
            const uint32_t acc = it & 1;
            mbar_wait(&tfull[acc], (it >> 1) & 1);
            tc_fence_after();
            for (int t = 0; t < MT; ++t) {
                if (mt + t >= p.m_tiles) break;
                const int row = (mt + t) * 256 + (int)rank * 128 + (int)(q * 32 + lane);
                float* dst = p.part + (int64_t)sp * p.part_split + (int64_t)row * p.part_ld +
                             (int64_t)nt * p.bn;
                const uint32_t taddr = tmem_base + ((q * 32u) << 16) + (acc * MT + t) * p.bn;
                for (int c0 = 0; c0 < p.bn; c0 += 16) {
                    uint32_t v[16];
                    tmem_ld_32x32b_x16(taddr + c0, v);
                    tmem_ld_wait();
                    float4* d4 = reinterpret_cast<float4*>(dst + c0);
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj)
                        st_f4_l2hint(d4 + jj,
                                     make_float4(__uint_as_float(v[4 * jj]), __uint_as_float(v[4 * jj + 1]),
                                                 __uint_as_float(v[4 * jj + 2]), __uint_as_float(v[4 * jj + 3])),
                                     pol);
                }
            }
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

// gw[k][c][r][s] = (acc ? gw : 0) + scale * sum_sp part[sp][(r*kW+s)*Cp + c][k]
// (32-bit index math: the caller checks K*CRS < 2^31). Each thread owns four consecutive
// k of one (c, r, s): float4 partial loads, 8 splits' loads in flight (fixed split order).
__global__ void wgrad_reduce_kernel(const float* __restrict__ part, float* __restrict__ gw,
                                    int K, int C, int kH, int kW, int Cp,
                                    int splits, int64_t ld, int64_t split_stride, float scale,
                                    int accumulate, int splits_v, int s_v0) {
    const int K4 = K / 4;
    const int taps = kH * kW;
    const int total = K4 * C * taps;
    const uint64_t pol = l2_evict_first_policy();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int crs = i / K4, k = (i - crs * K4) * 4;
        const int c = crs / taps, rs = crs - c * taps;  // rs = r*kW + s
        const float* src = part + ((int64_t)rs * Cp + c) * ld + k;
        // filter columns s >= s_v0 (umma_hwgrad's vertical quads) carry splits_v partials
        const int ns = rs % kW >= s_v0 ? splits_v : splits;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
        for (int sp = 0; sp < ns; ++sp) {
            const float4 v = ld_f4_l2hint(reinterpret_cast<const float4*>(src + (int64_t)sp * split_stride), pol);
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
        const float a[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t o = (int64_t)(k + u) * C * taps + crs;
            gw[o] = (accumulate ? gw[o] : 0.f) + scale * a[u];
        }
    }
}

// the same for K % 4 != 0 (one k per thread)
__global__ void wgrad_reduce1_kernel(const float* __restrict__ part, float* __restrict__ gw,
                                     int K, int C, int kH, int kW, int Cp,
                                     int splits, int64_t ld, int64_t split_stride, float scale,
                                     int accumulate, int splits_v, int s_v0) {
    const int total = K * C * kH * kW;
    const int taps = kH * kW;
    const uint64_t pol = l2_evict_first_policy();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int crs = i / K, k = i - crs * K;
        const int c = crs / taps, rs = crs - c * taps;
        const float* src = part + ((int64_t)rs * Cp + c) * ld + k;
        const int ns = rs % kW >= s_v0 ? splits_v : splits;
        float acc = 0.f;
#pragma unroll 8
        for (int sp = 0; sp < ns; ++sp) acc += ld_f_l2hint(src + (int64_t)sp * split_stride, pol);
        const int64_t o = (int64_t)k * C * taps + crs;
        gw[o] = (accumulate ? gw[o] : 0.f) + scale * acc;
    }
}

}  // namespace

void wgrad_reduce_launch(const float* part, float* gw, const Geo& g, int64_t Cp, int splits, int64_t ld,
                         int64_t split_stride, float scale, int accumulate, cudaStream_t st, int splits_v,
                         int s_v0) {
    if (s_v0 < 0) {  // one split count for every tap
        splits_v = splits;
        s_v0 = (int)g.kW;
    }
    const int64_t n = g.K * g.CRS;
    PTB_REQUIRE(n < (1ll << 31), "wgrad_reduce: weights too large");
    if (g.K % 4 == 0 && ld % 4 == 0 && split_stride % 4 == 0 && (reinterpret_cast<uintptr_t>(part) & 15) == 0) {
        wgrad_reduce_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n / 4, 256), 8 * (int64_t)sm_count()), 256, 0,
                              st>>>(part, gw, (int)g.K, (int)g.C, (int)g.kH, (int)g.kW, (int)Cp, splits, ld,
                                    split_stride, scale, accumulate, splits_v, s_v0);
    } else {
        wgrad_reduce1_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 8 * (int64_t)sm_count()), 256, 0, st>>>(
            part, gw, (int)g.K, (int)g.C, (int)g.kH, (int)g.kW, (int)Cp, splits, ld, split_stride, scale, accumulate,
            splits_v, s_v0);
    }
    after_launch("wgrad_reduce");
}

namespace {

int wgrad_kp_env() {
    static const int v = [] {
        const char* e = std::getenv("PT_B200_WGRAD_KPIX");
        // 128-pixel boxes: the kernel is bound by TMA requests more than bytes (64 -> 128
        // pixels per box: convnet L2 wgrad 0.99 -> 0.89 ms, L3 0.37 -> 0.32 ms), even though
        // the 96 KB stages leave a 2-deep ring
        const int k = e ? std::atoi(e) : 128;
        return k == 64 ? 64 : 128;
    }();
    return v;
}

int wgrad_sched_env() {
    static const int v = [] {
        const char* e = std::getenv("PT_B200_WGRAD_SCHED");  // 0: ~4 units per pair, rounded up
        return e ? std::atoi(e) : 1;
    }();
    return v;
}

// per-unit fixed cost (k-blocks) in the whole-wave split search
int wgrad_unit_ovh() {
    static const int v = [] {
        const char* e = std::getenv("PT_B200_WGRAD_OVH");
        return e ? std::atoi(e) : 2;
    }();
    return v;
}

struct WPlan {
    int64_t Cp, Kp, kdim;
    int mt;  // m-tiles per unit (1 or 2)
    int kp;  // pixels per pipeline stage
    int bn, m_tiles, m_groups, n_tiles, splits, kb_per_split, total_kb, stages;
    int64_t x_elems, gy_elems, part_elems;
};

WPlan wplan(const Geo& g) {
    WPlan w;
    w.Cp = (g.C + 31) / 32 * 32;
    w.Kp = (g.K + 31) / 32 * 32;
    w.kdim = g.kH * g.kW * w.Cp;
    w.n_tiles = (int)ceil_div(w.Kp, 256);
    w.bn = (int)(ceil_div(ceil_div(w.Kp, w.n_tiles), 64) * 64);
    w.m_tiles = (int)ceil_div(w.kdim, 256);
    // one m-tile per unit (two m-tiles sharing each B stage measured slower in round 1: L2
    // wgrad 1.00 -> 1.42 ms — the 32-pixel boxes needed to keep the ring depth halve the
    // bytes per TMA request — and were removed)
    w.mt = 1;
    w.kp = w.mt == 2 ? 32 : wgrad_kp_env();
    // <= 64 channels (two 32-channel chunks): 64-pixel stages measured faster (AlexNet conv2
    // wgrad 0.110 -> 0.099 ms)
    if (w.kp == 128 && w.Cp <= 64 && std::getenv("PT_B200_WGRAD_KPIX") == nullptr) w.kp = 64;
    // a 128-pixel stage must still leave a 2-deep ring (bn = 256 would get one stage:
    // VGG-A conv4 wgrad 0.33 -> 0.60 ms)
    if (w.kp == 128 && 2 * (4 * 128 * 128 + (w.bn / 64) * 128 * 128) > kSmemLimit - 2048) w.kp = 64;
    w.m_groups = (int)ceil_div(w.m_tiles, w.mt);
    const int kp = w.kp;
    w.total_kb = (int)ceil_div(g.M, kp);
    const int64_t tiles = (int64_t)w.m_groups * w.n_tiles;
    // ~4 units per CTA pair (2 per pair measured slower: convnet L2 wgrad 0.90 -> 1.01 ms)
    const int64_t target_units = 2 * (int64_t)sm_count();
    int64_t splits = ceil_div(target_units, tiles);
    int64_t kbps = ceil_div(w.total_kb, splits);
    if (kbps < 8 * w.mt) kbps = 8 * w.mt;  // >= 512 pixels per unit to amortise the epilogue
    if (wgrad_sched_env()) {
        // units run round-robin over the pairs (static): ~4 per pair rounded UP left a last
        // wave a quarter full on most layers (e.g. 301 units = 4.07 waves of 74). Pick the
        // split count minimising waves x (k-blocks per unit + a per-unit fixed cost of two
        // k-blocks), ties to more units.
        const int64_t pairs = sm_count() / 2;
        double best = 1e30;
        for (int64_t s = 1; s <= 4 * ceil_div(target_units, tiles); ++s) {
            const int64_t kb = std::max<int64_t>(ceil_div(w.total_kb, s), 8 * w.mt);
            const int64_t s2 = ceil_div(w.total_kb, kb);
            const double cost = (double)ceil_div(tiles * s2, pairs) * (double)(kb + wgrad_unit_ovh());
            if (cost <= best) {
                best = cost;
                kbps = kb;
            }
        }
    }
    w.kb_per_split = (int)kbps;
    w.splits = (int)ceil_div(w.total_kb, kbps);
    const int box = kp * 128;
    w.stages = (kSmemLimit - 1024 - 256) / (int)(w.mt * 4 * box + (w.bn / 64) * box);
    if (w.stages > 8) w.stages = 8;
    w.x_elems = g.N * g.HW * w.Cp;
    w.gy_elems = g.M * w.Kp;
    w.part_elems = (int64_t)w.splits * w.m_tiles * 256 * w.n_tiles * w.bn;
    return w;
}

}  // namespace

bool umma_wgrad_ok(const Geo& g) {
    if (g.M >= (1ll << 31) || g.N * g.HW >= (1ll << 31)) return false;
    if (g.pH > 128 || g.pW > 128 || g.kH > 256 || g.kW > 256) return false;
    if (g.pH - (g.kH - 1) < -128 || g.pW - (g.kW - 1) < -128) return false;
    if (g.sH > 8 || g.sW > 8) return false;
    return g.K <= 65536 && g.kH * g.kW * ((g.C + 31) / 32 * 32) < (1ll << 30) && sm_count() >= 2;
}

size_t umma_wgrad_workspace(const Geo& g) {
    const WPlan w = wplan(g);
    const size_t part = std::max((size_t)w.part_elems * 4, hwgrad_ok(g) ? hwgrad_part_bytes(g) : (size_t)0);
    return align_up(w.x_elems * 4, 256) + align_up(w.gy_elems * 4, 256) + align_up(part, 256);
}

int64_t umma_wgrad_kp(const Geo& g) { return (g.K + 31) / 32 * 32; }

void umma_conv_bwd_filter(const Geo& g, const float* x, const float* gy, float* gw, float scale,
                          int accumulate, void* ws, cudaStream_t st, const float* gyh_pre,
                          const float* xh_pre, double alg_flops, int64_t xph, int64_t xpw) {
    if (!xh_pre) xph = xpw = 0;
    const WPlan w = wplan(g);
    char* base = reinterpret_cast<char*>(ws);
    float* xh = reinterpret_cast<float*>(base);
    float* gyh = reinterpret_cast<float*>(base + align_up(w.x_elems * 4, 256));
    float* part = reinterpret_cast<float*>(base + align_up(w.x_elems * 4, 256) +
                                           align_up(w.gy_elems * 4, 256));
    if (!(xh_pre && gyh_pre)) {
        ProfScope prof("layout", st, 0.0,
                       4.0 * ((xh_pre ? 0 : g.N * g.C * g.HW + w.x_elems) +
                              (gyh_pre ? 0 : g.M * g.K + w.gy_elems)));
        if (!xh_pre) nchw_to_nhwc(x, xh, g.N, g.C, g.HW, w.Cp, true, st);
        if (!gyh_pre) nchw_to_nhwc(gy, gyh, g.N, g.K, g.oHW, w.Kp, true, st);
    }
    if (xh_pre) xh = const_cast<float*>(xh_pre);
    if (gyh_pre) gyh = const_cast<float*>(gyh_pre);
    if (xph == 0 && xpw == 0 && hwgrad_ok(g)) {  // wide stride-1 filters: Hankel quads (umma_hwgrad.cu)
        hwgrad_run(g, xh, gyh, gw, scale, accumulate, part, alg_flops, st);
        return;
    }
    UWgradParams p;
    memset(&p, 0, sizeof p);
    {
        // gy NHWC [M][Kp] viewed as {32 ch, M px, Kp/32 channel blocks} so one box carries
        // every 32-channel block a CTA needs, laid out [block][px][32] as the MMA expects
        const uint64_t dims[3] = {32, (uint64_t)g.M, (uint64_t)(w.Kp / 32)};
        const uint64_t strides[2] = {(uint64_t)w.Kp * 4, 128};
        const uint32_t box[3] = {32, (uint32_t)w.kp, (uint32_t)(w.bn / 64)};
        tmap_tiled(&p.tmap_gy, gyh, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    }
    // a zero-bordered copy carries (part of) the padding itself
    const int64_t xH = g.H + 2 * xph, xW = g.W + 2 * xpw, epH = g.pH - xph, epW = g.pW - xpw;
    tmap_im2col(&p.tmap_x, xh, g.N, xH, xW, w.Cp, (int)g.kH, (int)g.kW, (int)epH, (int)epW,
                (int)g.sH, (int)g.sW, 32, w.kp, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    p.oH = (int)g.oH;
    p.oW = (int)g.oW;
    p.sH = (int)g.sH;
    p.sW = (int)g.sW;
    p.pH = (int)epH;
    p.pW = (int)epW;
    p.kW = (int)g.kW;
    p.taps = (int)(g.kH * g.kW);
    p.Cp = (int)w.Cp;
    p.m_tiles = w.m_tiles;
    p.m_groups = w.m_groups;
    p.n_tiles = w.n_tiles;
    p.splits = w.splits;
    p.kb_per_split = w.kb_per_split;
    p.total_kb = w.total_kb;
    p.bn = w.bn;
    p.stages = w.stages;
    p.stage_b = (uint32_t)(w.bn / 64) * (uint32_t)w.kp * 128u;
    p.tmem_cols = 2 * w.mt * w.bn <= 256 ? 256 : 512;
    p.part = part;
    p.part_ld = (int64_t)w.n_tiles * w.bn;
    p.part_split = (int64_t)w.m_tiles * 256 * p.part_ld;
    const size_t smem = 1024 + (size_t)p.stages * (w.mt * 4 * w.kp * 128 + p.stage_b) +
                        (2 * p.stages + 4) * 8 + 16;
    const int units = w.m_groups * w.n_tiles * w.splits;
    const int pairs = std::min(units, sm_count() / 2);
    once_per_device((const void*)umma_wgrad_kernel<1, 64>, [&] {  // the smem limit is a per-device attribute
        PTB_CUDA(cudaFuncSetAttribute(umma_wgrad_kernel<1, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kSmemLimit));
        PTB_CUDA(cudaFuncSetAttribute(umma_wgrad_kernel<1, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kSmemLimit));
    });
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(kThreadsW);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    {
        ProfScope prof("umma_wgrad", st, alg_flops >= 0 ? alg_flops : 2.0 * g.M * g.K * g.CRS, 0.0);
        if (w.kp == 128) PTB_CUDA(cudaLaunchKernelEx(&cfg, umma_wgrad_kernel<1, 128>, p));
        else PTB_CUDA(cudaLaunchKernelEx(&cfg, umma_wgrad_kernel<1, 64>, p));
        after_launch("umma_wgrad");
    }
    wgrad_reduce_launch(part, gw, g, w.Cp, w.splits, p.part_ld, p.part_split, scale, accumulate, st);
}

}  // namespace ptb
