// umma_hwgrad.cu — tcgen05 (kind::tf32) weight gradient of stride-1 layers with wide
// filters (kW >= 7: convnet L2-L4), accGradParameters.
//
//   gW^T[(r,s,c)][k] = sum_{n,i,j} x[n][i+r-pH][j+s-pW][c] * gy[n][i][j][k]
//
// CTA-pair GEMM: M = filter columns, N = output channels k (BN per tile), K = output
// pixels. Both operands are MN-major (NHWC: channels contiguous), so a K step is one
// 128-byte pixel row. The weight-gradient rows of four consecutive taps (r, s..s+3) of one
// 32-channel chunk read the SAME input row shifted by one pixel each: as M atoms of the
// MN-major operand they sit exactly one 128-byte row apart, so one smem descriptor with
// LBO = 128 B addresses all four from ONE staged input-row run (Hankel view; the 128B
// swizzle is a function of the absolute smem address, so any row offset is valid). The
// im2col engine (umma_wgrad.cu) instead fetches a separate box per tap and is bound by the
// L2->SM traffic that re-fetching causes.
//
// A "quad" is 4 taps x 32 channels per CTA (M = 256 rows per pair: CTA 0 takes chunk 2p,
// CTA 1 chunk 2p+1 of the same taps). A unit = (row r, chunk pair, n-tile, pixel split)
// owns ceil(kW/4) quads (taps past kW are computed and dropped), one TMEM accumulator of
// BN columns each, and streams its pixel split in stages of R output rows x KP columns:
// per stage one x box {32 ch, KP + 4*qpr - 1 px, R rows} (CTA's chunk) and one gy box
// {32 k, KP px, R rows, BN/64 blocks}. Partials [split][(r*kW+s)*Cp + c][k] are reduced
// by umma_wgrad.cu's fixed-order wgrad_reduce_kernel (deterministic).
//
// Vertical quads. With kW % 4 != 0 the last quad of every row wastes slots (kW = 9: 12 slots
// for 9 taps). The leftover columns s >= 4*floor(kW/4) are instead covered by quads of four
// consecutive FILTER ROWS r..r+3 of one column s: the same staged data read with LBO = one
// box row (Wbox pixels) instead of one pixel, from a box of R + 3 input rows. A "vertical"
// unit = (band of 4 filter rows, chunk pair, n-tile, split) owns one such quad per leftover
// column; "horizontal" units keep floor(kW/4) quads per row. kW = kH = 9: 21 quads instead
// of 27 (84 slots for 81 taps).
#include <cuda.h>

#include <cstdlib>
#include <cstring>

#include "kernels.cuh"
#include "tmap.cuh"
#include "umma.cuh"

namespace ptb {

namespace {

using namespace umma;

constexpr int kThreadsHW = 320;  // warp 0 TMA, warp 1 MMA, warps 2..9 epilogue (2 per lane quarter)
constexpr int kSmemLimitHW = 232448;

struct HWParams {
    CUtensorMap tmap_x;   // x NHWC 5-D {32, W, H, N, Cp/32}, box {32, Wbox, R, 1, 1}, SW128_32B
    CUtensorMap tmap_gy;  // gy NHWC 5-D {32, oW, oH, N, Kp/32}, box {32, KP, R, 1, BN/64}, SW128_32B
    CUtensorMap tmap_xv;  // vertical units: x box {32, Wbox, R + 3, 1, 1}
    int oH, oW, pH, pW, kW, Cp;
    int qh, ql, nbands;   // vertical quads: horizontal quads per row, leftover columns, 4-row bands (0: off)
    uint32_t tx_v;        // TMA bytes of a vertical unit's stage
    int R, KP, Wbox, jsegs, rgs;
    int qpr;              // quads per filter row
    int cps, n_tiles, splits, kH;
    int items;            // N * rgs * jsegs pixel items
    int per_split, rem;   // split sp covers per_split (+1 for sp < rem) consecutive items
    int splits_v, per_split_v, rem_v;  // the same for the vertical units (their own split count)
    int bn, stages;
    uint32_t stage_a, stage_b, tx, tmem_cols;
    int tbuf;             // TMEM accumulator buffers (1 or 2)
    uint32_t tbuf_cols;   // column offset of buffer 1
    float* part;
    int64_t part_ld, part_split;
};

template <int QPR>
__global__ void __launch_bounds__(kThreadsHW, 1) umma_hwgrad_kernel(const __grid_constant__ HWParams p) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((((raw + 1023u) & ~1023u)) - raw);
    const int S = p.stages;
    const uint32_t stage_bytes = p.stage_a + p.stage_b;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * stage_bytes);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;    // [2]: one per TMEM accumulator buffer
    uint64_t* tempty = tfull + 2;   // [2]
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

    const uint32_t warp = warp_id_uniform(), lane = lane_id();
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.tmap_x);
        tma_prefetch(&p.tmap_gy);
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);   // the leader's expect_tx (the peer's bytes land on it)
            mbar_init(&empty[i], 1);  // one multicast commit
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 16);  // 8 epilogue warps x 2 CTAs
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc_cg2(tmem_holder, p.tmem_cols);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const int units_h = p.kH * p.cps * p.n_tiles * p.splits;
    const int units = units_h + p.nbands * p.cps * p.n_tiles * p.splits_v;
    const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
    // unit -> (r, chunk pair, n-tile, split); r fastest: concurrent pairs share gy stages in L2.
    // Units past units_h are vertical: r = the band's first filter row (4 * band), vt = true.
    auto decode = [&](int u, int& r, int& cp, int& nt, int& sp, bool& vt) {
        vt = u >= units_h;
        const int rows = vt ? p.nbands : p.kH;
        if (vt) u -= units_h;
        r = u % rows;
        int v = u / rows;
        cp = v % p.cps;
        v /= p.cps;
        nt = v % p.n_tiles;
        sp = v / p.n_tiles;
        if (vt) r *= 4;
    };
    // 32-bit only: a 64-bit division is a call, after which the compiler keeps the MMA
    // loop's descriptor state in vector registers (R2UR + elect per MMA)
    auto range = [&](int sp, bool vt, int& lo, int& hi) {
        const int ps = vt ? p.per_split_v : p.per_split, rm = vt ? p.rem_v : p.rem;
        lo = sp * ps + (sp < rm ? sp : rm);
        hi = lo + ps + (sp < rm ? 1 : 0);
    };

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint32_t tx = p.tx;
            for (int u = cluster; u < units; u += nclusters) {
                int r, cp, nt, sp, lo, hi;
                bool vt;
                decode(u, r, cp, nt, sp, vt);
                range(sp, vt, lo, hi);
                const int chunk = 2 * cp + (int)rank;
                const int kb = (nt * p.bn + (int)rank * (p.bn / 2)) / 32;
                for (int it = lo; it < hi; ++it) {
                    const int js = it % p.jsegs;
                    const int rg = (it / p.jsegs) % p.rgs;
                    const int n = it / (p.jsegs * p.rgs);
                    const int j0 = js * p.KP, i0 = rg * p.R;
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* a = smem + (size_t)stage * stage_bytes;
                    if (leader) mbar_arrive_expect_tx(&full[stage], vt ? p.tx_v : tx);
                    // the input-row runs of filter row r (vertical: rows r .. r+3) for the
                    // stage's R output rows
                    tma_load_5d_cg2(a, vt ? &p.tmap_xv : &p.tmap_x, &full[stage], 0, j0 - p.pW, i0 + r - p.pH, n,
                                    chunk);
                    tma_load_5d_cg2(a + p.stage_a, &p.tmap_gy, &full[stage], 0, j0, i0, n, kb);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {  // whole warp, converged; one elected lane issues
            const uint32_t idesc = idesc_tf32(256, p.bn, 1, 1);
            constexpr uint32_t kHi = desc_hi(512, kSwizzle128B_Base32B);
            const uint32_t b_lbo = (uint32_t)(p.R * p.KP * 128);
            // loop-invariant scalars hoisted so the descriptor arithmetic stays in uniform
            // registers (per-MMA R2UR / divergence checks otherwise double the issue cost)
            const int nks = p.R * p.KP / 8, KP = p.KP;
            const uint32_t row_skip = (uint32_t)(p.Wbox - p.KP) * 8u, bn = (uint32_t)p.bn;
            int stage = 0;
            uint32_t phase = 0;
            int it_u = 0;
            for (int u = cluster; u < units; u += nclusters, ++it_u) {
                int r, cp, nt, sp, lo, hi;
                bool vt;
                decode(u, r, cp, nt, sp, vt);
                range(sp, vt, lo, hi);
                // horizontal: quad q = taps 4q..4q+3 one pixel (128 B) apart; vertical: quad q =
                // column 4*qh + q of filter rows r..r+3, one box row (Wbox px) apart
                const int nq = vt ? p.ql : p.qh;
                const uint32_t a_lbo = vt ? (uint32_t)p.Wbox * 128u : 128u;
                const uint32_t q_step = vt ? 8u : 32u, q_base = vt ? (uint32_t)(4 * p.qh) * 8u : 0u;
                // p.tbuf = 2: unit i accumulates in TMEM buffer i & 1, so the epilogue of one
                // unit drains while the next one's MMAs run
                const int tb = p.tbuf == 2 ? (it_u & 1) : 0;
                const uint32_t tpar = p.tbuf == 2 ? (uint32_t)(it_u >> 1) & 1u : (uint32_t)it_u & 1u;
                const uint32_t tacc = tmem_base + (uint32_t)tb * p.tbuf_cols;
                mbar_wait(&tempty[tb], tpar ^ 1);
                tc_fence_after();
                uint32_t accum = 0;
                for (int it = lo; it < hi; ++it) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_addr = smem_u32(smem + (size_t)stage * stage_bytes);
                    // A: taps s..s+3 = M atoms one pixel row (128 B) apart; B: BN/64 k-blocks
                    uint32_t alo = desc_lo(a_addr, a_lbo) + q_base, blo = desc_lo(a_addr + p.stage_a, b_lbo);
                    int k8 = 0;
                    for (int ks = 0; ks < nks; ++ks) {
                        const uint64_t bd = desc_make(blo, kHi);
#pragma unroll
                        for (int q = 0; q < QPR; ++q)
                            if (q < nq)
                                mma_tf32_cg2_warp(tacc + (uint32_t)q * bn, desc_make(alo + q_step * (uint32_t)q, kHi),
                                                  bd, idesc, accum);
                        accum = 1;
                        blo += 64u;  // 8 pixel rows
                        alo += 64u;
                        k8 += 8;
                        if (k8 == KP) {  // next output row of the stage: the next input-row run
                            k8 = 0;
                            alo += row_skip;
                        }
                    }
                    mma_commit_cg2_warp(&empty[stage]);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                mma_commit_cg2_warp(&tfull[tb]);
            }
        }
    } else {
        // ===== epilogue: quad q, lane quarter = tap s = 4q + quarter, lane = channel =====
        const uint32_t qtr = warp & 3;
        const int half = (int)(warp - 2) >> 2;  // column chunks 2*k + half
        int it_u = 0;
        for (int u = cluster; u < units; u += nclusters, ++it_u) {
            int r, cp, nt, sp;
            bool vt;
            decode(u, r, cp, nt, sp, vt);
            const int tb = p.tbuf == 2 ? (it_u & 1) : 0;
            const uint32_t tpar = p.tbuf == 2 ? (uint32_t)(it_u >> 1) & 1u : (uint32_t)it_u & 1u;
            mbar_wait(&tfull[tb], tpar);
            tc_fence_after();
            const int c = (2 * cp + (int)rank) * 32 + (int)lane;
            const int nq = vt ? p.ql : p.qh;
            for (int q = 0; q < nq; ++q) {
                // lane quarter = tap s = 4q + quarter (horizontal) / filter row r + quarter (vertical)
                const int s = vt ? 4 * p.qh + q : 4 * q + (int)qtr, rr = vt ? r + (int)qtr : r;
                const bool valid = s < p.kW && rr < p.kH && c < p.Cp;
                float* dst = p.part + (int64_t)sp * p.part_split +
                             ((int64_t)(rr * p.kW + s) * p.Cp + c) * p.part_ld + (int64_t)nt * p.bn;
                const uint32_t taddr = tmem_base + ((qtr * 32u) << 16) + (uint32_t)tb * p.tbuf_cols + (uint32_t)(q * p.bn);
                for (int c0 = half * 16; c0 < p.bn; c0 += 32) {
                    uint32_t v[16];
                    tmem_ld_32x32b_x16(taddr + c0, v);
                    tmem_ld_wait();
                    if (valid) {
                        // partials stay in L2 for the reduce (umma.cuh: l2_evict_last_policy)
                        const uint64_t pol = l2_evict_last_policy();
                        float4* d4 = reinterpret_cast<float4*>(dst + c0);
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj)
                            st_f4_l2hint(d4 + jj,
                                         make_float4(__uint_as_float(v[4 * jj]), __uint_as_float(v[4 * jj + 1]),
                                                     __uint_as_float(v[4 * jj + 2]), __uint_as_float(v[4 * jj + 3])),
                                         pol);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (leader) mbar_arrive(&tempty[tb]);
                else mbar_arrive_cluster(&tempty[tb], 0);
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

struct HWPlan {
    int Cp, Kp, bn, n_tiles, qpr, KP, R, Wbox, jsegs, rgs, cps, splits, splits_v, stages;
    int qh, ql, nbands;  // horizontal quads per row, leftover columns, vertical bands (0: off)
    int64_t quads;       // MMA quads per (chunk pair, n-tile, split) over all units
    int64_t items;
    uint32_t stage_a, stage_b, tmem_cols, tbuf_cols;
    int tbuf;
    int64_t part_elems;
};

// relative cost per pixel item of a one-quad vertical unit against a one-quad horizontal
// unit (its stage also stages kH-band rows of x: more TMA per MMA)
double hwgrad_vbeta() {
    static const double v = [] {
        // <= 0: one split count for both; 1.2 measured best of 1.0 / 1.2 (convnet L2 wgrad
        // 0.658 -> 0.589 ms, L3 0.254 -> 0.236 ms with the double TMEM buffer)
        const char* e = std::getenv("PT_B200_HWGRAD_VBETA");
        return e ? std::atof(e) : 1.2;
    }();
    return v;
}

int hwgrad_tbuf_env() {
    static const int v = [] {
        const char* e = std::getenv("PT_B200_HWGRAD_TBUF");  // TMEM accumulator buffers: 1 or 2
        return e ? std::atoi(e) : 2;
    }();
    return v;
}

// per-unit fixed cost (pipeline fill, epilogue tail) in pixel items, with the epilogue
// overlapped by the double TMEM buffer
double hwgrad_unit_ovh() {
    static const double v = [] {
        const char* e = std::getenv("PT_B200_HWGRAD_OVH");
        return e ? std::atof(e) : 8.0;
    }();
    return v;
}

int hwgrad_env() {
    static const int v = [] {
        const char* e = std::getenv("PT_B200_HWGRAD");  // 0 off, 1 default rule, 2 force
        return e ? std::atoi(e) : 1;
    }();
    return v;
}

HWPlan hwplan_make(const Geo& g);

// the split search costs ~1 ms of host time; eager callers plan the same layer several times
HWPlan hwplan(const Geo& g) {
    struct Entry {
        int64_t key[12];
        HWPlan plan;
    };
    thread_local Entry cache[8];
    thread_local int next = 0, used = 0;
    const int64_t key[12] = {g.N, g.C, g.H, g.W, g.K, g.kH, g.kW, g.pH, g.pW, g.sH, g.sW, (int64_t)sm_count()};
    for (int i = 0; i < used; ++i)
        if (!memcmp(cache[i].key, key, sizeof key)) return cache[i].plan;
    Entry& e = cache[next];
    memcpy(e.key, key, sizeof key);
    e.plan = hwplan_make(g);
    next = (next + 1) % 8;
    used = std::min(used + 1, 8);
    return e.plan;
}

HWPlan hwplan_make(const Geo& g) {
    HWPlan w;
    w.Cp = (int)((g.C + 31) / 32 * 32);
    w.Kp = (int)((g.K + 31) / 32 * 32);
    w.n_tiles = (int)ceil_div(w.Kp, 256);
    w.bn = (int)(ceil_div(ceil_div(w.Kp, w.n_tiles), 64) * 64);
    w.qpr = (int)ceil_div(g.kW, 4);
    w.qh = w.qpr;
    w.ql = 0;
    w.nbands = 0;
    w.quads = g.kH * w.qpr;
    {
        // vertical quads for the leftover columns when they need fewer MMAs and every unit
        // keeps >= 2 quads per staged box (kW = 5, one horizontal quad per row, measured
        // slower: AlexNet conv2 wgrad, each gy stage then feeds one MMA per K step)
        static const bool vert_on = [] {
            const char* e = std::getenv("PT_B200_HWGRAD_VERT");
            return e ? std::atoi(e) != 0 : true;
        }();
        const int qh = (int)(g.kW / 4), ql = (int)(g.kW % 4), nb = (int)ceil_div(g.kH, 4);
        const int64_t q_new = g.kH * qh + (int64_t)nb * ql;
        if (vert_on && qh >= 2 && ql >= 1 && q_new < w.quads) {
            w.qh = qh;
            w.ql = ql;
            w.nbands = nb;
            w.qpr = std::max(qh, ql);
            w.quads = q_new;
        }
    }
    const int jsegs = (int)ceil_div(g.oW, 128);
    w.jsegs = jsegs;
    w.KP = (int)(ceil_div(ceil_div(g.oW, jsegs), 8) * 8);
    // R output rows per stage (<= 128 pixels), balanced so the last row group is not mostly empty
    const int rmax = std::max(1, 128 / w.KP);
    w.R = (int)ceil_div(g.oH, ceil_div(g.oH, rmax));
    w.Wbox = w.nbands ? w.KP + (int)g.kW - 1 : w.KP + 4 * w.qpr - 1;
    w.rgs = (int)ceil_div(g.oH, w.R);
    w.items = g.N * w.rgs * w.jsegs;
    w.cps = (int)ceil_div(w.Cp / 32, 2);
    w.stage_a = (uint32_t)align_up((size_t)(w.R + (w.nbands ? 3 : 0)) * w.Wbox * 128, 1024);
    w.stage_b = (uint32_t)align_up((size_t)(w.bn / 64) * w.R * w.KP * 128, 1024);
    w.stages = std::min(8, (kSmemLimitHW - 1024 - 256) / (int)(w.stage_a + w.stage_b));
    uint32_t cols = 32;
    while ((int)cols < w.qpr * w.bn) cols <<= 1;
    // two accumulator buffers where they fit the 512 TMEM columns: a unit's epilogue then
    // overlaps the next unit's MMAs
    w.tbuf = hwgrad_tbuf_env() == 2 && 2 * cols <= 512 ? 2 : 1;
    w.tbuf_cols = cols;
    w.tmem_cols = cols * (uint32_t)w.tbuf;
    // pixel splits: enough units for every CTA pair with a small tail (static round-robin
    // schedule: unit i runs on pair i mod P). Vertical units issue ql quads per stage against
    // the horizontal units' qh, so they get their own (smaller) split count: with one count
    // the pairs holding a vertical unit idle for the second half of the launch (convnet L2:
    // 54 two-quad + 18 one-quad units on 74 pairs).
    const int64_t pairs = sm_count() / 2;
    const int64_t bh = g.kH * w.cps * w.n_tiles, bv = (int64_t)w.nbands * w.cps * w.n_tiles;
    const bool sep = w.nbands && hwgrad_vbeta() > 0.0;
    const double beta = sep ? hwgrad_vbeta() * w.ql / w.qh : 1.0;
    int best = 1, best_v = 1;
    double best_cost = 1e30;
    for (int sp = 1; sp <= 96; ++sp) {
        if (sp > w.items) break;
        for (int sv = sep ? 1 : sp; sv <= sp; ++sv) {
            const int64_t uh = bh * sp, uv = bv * sv;
            // time ~ per-pair sum of (work per unit + a per-unit epilogue / pipeline-fill overhead)
            // (the smaller overhead only re-measured with vertical units: the s2d conv1s'
            // split choice stays as it was)
            const double ovh = w.tbuf == 2 && w.nbands ? hwgrad_unit_ovh() : 24.0;
            const double ch = (double)w.items / sp + ovh, cv = beta * w.items / sv + ovh;
            double cost = 0.0;
            for (int64_t c = 0; c < std::min(pairs, uh + uv); ++c) {
                const int64_t nh = c < uh ? (uh - 1 - c) / pairs + 1 : 0;
                // vertical unit indices uh .. uh+uv-1 congruent to c mod pairs
                const int64_t first = uh + ((c - uh % pairs) % pairs + pairs) % pairs;
                const int64_t nv = first < uh + uv ? (uh + uv - 1 - first) / pairs + 1 : 0;
                cost = std::max(cost, nh * ch + nv * cv);
            }
            if (cost < best_cost - 1e-9) {
                best_cost = cost;
                best = sp;
                best_v = sv;
            }
        }
    }
    w.splits = best;
    w.splits_v = best_v;
    w.part_elems = (int64_t)w.splits * g.kH * g.kW * w.Cp * w.n_tiles * w.bn;
    return w;
}

}  // namespace

bool hwgrad_ok(const Geo& g) {
    const int env = hwgrad_env();
    if (env == 0) return false;
    if (g.sH != 1 || g.sW != 1 || g.C < 32) return false;
    // quads of taps: kW = 9 computes 12 tap slots (75%), worth it against the im2col
    // engine's L2->SM bound; 3x3 layers (75%) with >= 128 channels already run near that on
    // the im2col engine, but with <= 64 channels (one chunk pair: VGG-A conv2, the
    // space-to-depth conv1s) the quads win (VGG-A conv2 wgrad 0.27 -> 0.20 ms, AlexNet
    // conv1 0.113 -> 0.064)
    const HWPlan w = hwplan(g);
    if (env != 2 && g.kW < 7 && w.Cp > 64) return false;
    // useful fraction of the MMA work: tap slots x pixel columns x pixel rows computed
    // (convnet L2 0.75, L3 0.72 -> faster than the im2col engine; L4, 10x10 outputs in
    // 16-column stages: 0.55 -> slower, 0.046 -> 0.052 ms)
    const double eff = (double)(g.kH * g.kW) / (4.0 * w.quads) * (double)g.oW / ((double)w.KP * w.jsegs) *
                       (double)g.oH / ((double)w.R * w.rgs);
    if (env != 2 && eff < 0.7) return false;
    if (w.qpr > 4 || w.qpr * w.bn > 512 || w.Wbox > 256 || w.R > 256 || w.stages < 2) return false;
    if (g.pW > 128 || g.pH > 128 || w.items >= (1ll << 31)) return false;
    return g.N * g.HW * w.Cp < (1ll << 31) && g.M * w.Kp < (1ll << 31) && sm_count() >= 2;
}

size_t hwgrad_part_bytes(const Geo& g) { return (size_t)hwplan(g).part_elems * 4; }

void hwgrad_run(const Geo& g, const float* xh, const float* gyh, float* gw, float scale, int accumulate,
                float* part, double alg_flops, cudaStream_t st) {
    const HWPlan w = hwplan(g);
    HWParams p;
    memset(&p, 0, sizeof p);
    {
        const uint64_t dims[5] = {32, (uint64_t)g.W, (uint64_t)g.H, (uint64_t)g.N, (uint64_t)(w.Cp / 32)};
        const uint64_t strides[4] = {(uint64_t)w.Cp * 4, (uint64_t)(g.W * w.Cp * 4), (uint64_t)(g.HW * w.Cp * 4),
                                     128};
        const uint32_t box[5] = {32, (uint32_t)w.Wbox, (uint32_t)w.R, 1, 1};
        tmap_tiled(&p.tmap_x, xh, 5, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
        if (w.nbands) {
            const uint32_t boxv[5] = {32, (uint32_t)w.Wbox, (uint32_t)(w.R + 3), 1, 1};
            tmap_tiled(&p.tmap_xv, xh, 5, dims, strides, boxv, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
        }
    }
    {
        const uint64_t dims[5] = {32, (uint64_t)g.oW, (uint64_t)g.oH, (uint64_t)g.N, (uint64_t)(w.Kp / 32)};
        const uint64_t strides[4] = {(uint64_t)w.Kp * 4, (uint64_t)(g.oW * w.Kp * 4),
                                     (uint64_t)(g.oHW * w.Kp * 4), 128};
        const uint32_t box[5] = {32, (uint32_t)w.KP, (uint32_t)w.R, 1, (uint32_t)(w.bn / 64)};
        tmap_tiled(&p.tmap_gy, gyh, 5, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    }
    p.oH = (int)g.oH;
    p.oW = (int)g.oW;
    p.pH = (int)g.pH;
    p.pW = (int)g.pW;
    p.kW = (int)g.kW;
    p.Cp = w.Cp;
    p.R = w.R;
    p.KP = w.KP;
    p.Wbox = w.Wbox;
    p.jsegs = w.jsegs;
    p.rgs = w.rgs;
    p.qpr = w.qpr;
    p.qh = w.qh;
    p.ql = w.ql;
    p.nbands = w.nbands;
    p.cps = w.cps;
    p.n_tiles = w.n_tiles;
    p.splits = w.splits;
    p.kH = (int)g.kH;
    p.items = (int)w.items;
    p.per_split = (int)(w.items / w.splits);
    p.rem = (int)(w.items % w.splits);
    p.splits_v = w.splits_v;
    p.per_split_v = (int)(w.items / w.splits_v);
    p.rem_v = (int)(w.items % w.splits_v);
    p.bn = w.bn;
    p.stages = w.stages;
    p.stage_a = w.stage_a;
    p.stage_b = w.stage_b;
    p.tx = (uint32_t)(2 * ((size_t)w.R * w.Wbox * 128 + (size_t)(w.bn / 64) * w.R * w.KP * 128));
    p.tx_v = (uint32_t)(2 * ((size_t)(w.R + 3) * w.Wbox * 128 + (size_t)(w.bn / 64) * w.R * w.KP * 128));
    p.tmem_cols = w.tmem_cols;
    p.tbuf = w.tbuf;
    p.tbuf_cols = w.tbuf_cols;
    p.part = part;
    p.part_ld = (int64_t)w.n_tiles * w.bn;
    p.part_split = g.kH * g.kW * w.Cp * p.part_ld;
    const size_t smem = 1024 + (size_t)w.stages * (w.stage_a + w.stage_b) + (2 * w.stages + 4) * 8 + 16;
    const int units = (int)((g.kH * w.splits + w.nbands * w.splits_v) * w.cps * w.n_tiles);
    const int pairs = std::min(units, sm_count() / 2);
    once_per_device((const void*)umma_hwgrad_kernel<1>, [&] {  // the smem limit is a per-device attribute
        PTB_CUDA(cudaFuncSetAttribute(umma_hwgrad_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kSmemLimitHW));
        PTB_CUDA(cudaFuncSetAttribute(umma_hwgrad_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kSmemLimitHW));
        PTB_CUDA(cudaFuncSetAttribute(umma_hwgrad_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kSmemLimitHW));
        PTB_CUDA(cudaFuncSetAttribute(umma_hwgrad_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kSmemLimitHW));
    });
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(kThreadsHW);
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
        if (w.qpr == 1) PTB_CUDA(cudaLaunchKernelEx(&cfg, umma_hwgrad_kernel<1>, p));
        else if (w.qpr == 2) PTB_CUDA(cudaLaunchKernelEx(&cfg, umma_hwgrad_kernel<2>, p));
        else if (w.qpr == 3) PTB_CUDA(cudaLaunchKernelEx(&cfg, umma_hwgrad_kernel<3>, p));
        else PTB_CUDA(cudaLaunchKernelEx(&cfg, umma_hwgrad_kernel<4>, p));
        after_launch("umma_hwgrad");
    }
    wgrad_reduce_launch(part, gw, g, w.Cp, w.splits, p.part_ld, p.part_split, scale, accumulate, st, w.splits_v,
                        w.nbands ? 4 * w.qh : -1);
}

}  // namespace ptb
