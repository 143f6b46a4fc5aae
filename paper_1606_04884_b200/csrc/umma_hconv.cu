// umma_hconv.cu — tcgen05 (kind::tf32) stride-1 convolution over a zero-bordered NHWC
// activation with the im2col operand taken as a Hankel view of ONE pixel run per
// (filter row, channel chunk): fprop (updateOutput) and the stride-1
// input gradient as a transposed conv with the flipped filter.
//
// Position space. The activation is stored padded, xp[n][Hp][Wp][Cp] (Cp = C rounded up
// to 32), flattened to pixels P = (n*Hp + h)*Wp + w. An output position q = i*Wp + j of
// image n (j may run past oW into the right border: those columns are computed and
// discarded) reads, for filter tap (r, s), the pixel n*Hp*Wp + q + r*Wp + s. So for a
// run of 128 consecutive positions the im2col tile of tap (r, s) is the pixel run
// starting at q0 + r*Wp, shifted by s: ONE TMA box of 128 + kW - 1 pixels x 32 channels
// (128B-swizzled, K-major, a pixel = one 128-byte row) feeds all kW taps of filter row r
// — the tcgen05 smem descriptor simply starts s rows (s*128 bytes) further in. The
// im2col-mode kernel (umma_conv.cu) re-fetches the overlapping pixels once per tap, and
// its L2->SM traffic, not the tensor pipe, bounds it (ncu: 13.2 TB/s of TMA reads on
// convnet L2 dgrad at 28% tensor-pipe activity).
//
// Positions are tiled either per image (P_img = oH*Wp rounded up to the 256-position
// pair tile; a tile never crosses images) or flat over the batch (P_img = Hp*Wp; a tile
// may span two images, the pixel index is then just the global position). The host
// picks whichever wastes fewer positions.
//
// CTA pair (cta_group::2): M = 256 positions (128 per CTA), N = BN output channels (each
// CTA stages BN/2 weight rows). Two smem rings: A (pixel runs, one per (r, chunk)) and B
// (weight tiles, one per (r, s, chunk)); the MMA issuer consumes kW B stages per A stage.
// TMEM holds two BN-column accumulators so the epilogue of tile t overlaps tile t+1.
//
// Warp roles (320 threads, 1 CTA/SM, persistent): warp 0 TMA producer, warp 1 TMEM
// allocator + MMA issuer (pair leader), warps 2..9 epilogue (TMEM -> +bias -> NCHW): two
// warps per TMEM lane quarter, each draining half of the column chunks (layers with a
// short reduction are epilogue-paced: AlexNet conv1 as s2d spends ~3x its MMA time there).
#include <cuda.h>

#include <cstdlib>

#include "kernels.cuh"
#include "tmap.cuh"
#include "umma.cuh"

namespace ptb {

namespace {

using namespace umma;

constexpr int kThreadsH = 352;  // + warp 10: the weight (B) producer
constexpr int kSmemLimitH = 232448;
// epilogue neighbour exchange: [tile parity][bn/16 chunks][3 warps][G-1 deltas][G-1 lanes][16]
// floats (two tile buffers: a warp may write tile t+1's slot while its neighbour still
// reads tile t's)
inline int xch_bytes(int G, int bn) { return G > 1 ? 2 * ((bn + 15) / 16) * 3 * (G - 1) * (G - 1) * 16 * 4 : 0; }

struct HConvParams {
    CUtensorMap tmap_a;  // act NHWC [N][aH][aW][Cp], 5-D {32, aW, aH, N, Cp/32}, box {32, Wp, NR, 1, CPS}
    CUtensorMap tmap_a2; // same with NR - 1 rows: runs starting early in a row need one row less
    CUtensorMap tmap_b;  // packed weights, 3-D {32, n_pad, kdim/32}, box {32, rows, CPS}, SW128
    int N, kH, kW, chunks, cin_p;
    int last_k;          // live K=8 steps of the last 32-channel chunk (the rest are zero channels)
    int aph, apw;        // zero border the TMA out-of-bounds fill supplies (top, left)
    int Wp;              // padded row width = position-space row stride
    int oH, oW;          // valid output extent
    int R;               // rows per image half: CTA 0 covers rows [0, R), CTA 1 rows [R, 2R)
    int m;               // positions per half = R * Wp
    int tpi;             // pair tiles per image
    int nr_split;        // runs starting at column < nr_split fit NR - 1 rows
    int tiles;           // N * tpi
    int zero_tap;        // unused (G > 1 packs zero taps into the groups)
    int ngroups;         // G > 1: tap groups per filter row, ceil(kW / G)
    int n_rows, bn, n_tiles;
    int sa, sb;          // ring depths
    uint32_t stage_a, stage_b;  // bytes per stage (CPS boxes)
    uint32_t box_a, box_b;      // bytes per 32-channel box
    uint32_t tmem_cols;
    int nacc;            // TMEM accumulator buffers (2 or 4)
    int a_run;           // 1: A = the exact pixel run by TMA im2col traversal (tmap_run), else NR full rows
    int run_px;          // a_run: pixels per run (128 + kW - 1)
    int flat;            // a_run: CTA tiles are consecutive 129-G position runs of a whole image (pair
                         // = two consecutive CTA tiles), filter rows whose input rows lie entirely in
                         // the zero border are skipped
    int tpc, ctiles, aH; // flat: CTA tiles per image, in total; input rows
    int sbias_n;         // > 0: bias staged in smem (this many floats, zero past n_rows)
    uint32_t xch_bytes_; // bytes of the G > 1 exchange region (the staged bias follows it)
    CUtensorMap tmap_run;  // im2col over the dense NHWC act: {32 ch, run_px positions}, virtual kW = 1
    float* out;
    const float* bias;
};

// CPS: 32-channel chunks per pipeline stage (1 or 2).
// G > 1 (output-shift tap grouping, for <= 128 output channels): one MMA computes taps
// s .. s+G-1 from the SAME pixel run (shift s) with N = G*bn — the weight rows (delta, c)
// are split between the two CTAs. Column group delta then holds tap s+delta's
// contribution to the position delta to the LEFT, so the epilogue forms
// out[q] = sum_delta D_delta[q + delta]; each CTA's last G-1 lanes lack right neighbours
// and are dropped (tiles advance 129 - G positions per CTA). An N <= 128 MMA costs the
// same ~64 cycles whatever N is, so grouping cuts the MMA count up to G-fold.
// RUNS = 2: each unit is two consecutive position tiles sharing every weight stage (their
// A runs sit side by side in the A stage, two accumulators per unit): the weights —
// re-read from L2 per tile, the larger share of the operand traffic for 64-128 channel
// layers — are fetched half as often.
template <int CPS, int G, int RUNS>
__global__ void __launch_bounds__(kThreadsH, 1) umma_hconv_kernel(const __grid_constant__ HConvParams p) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((((raw + 1023u) & ~1023u)) - raw);
    uint8_t* sA = smem;
    uint8_t* sB = sA + (size_t)p.sa * p.stage_a;
    uint64_t* afull = reinterpret_cast<uint64_t*>(sB + (size_t)p.sb * p.stage_b);
    uint64_t* aempty = afull + p.sa;
    uint64_t* bfull = aempty + p.sa;
    uint64_t* bempty = bfull + p.sb;
    uint64_t* tfull = bempty + p.sb;
    uint64_t* tempty = tfull + 4;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 4);
    float* xch = reinterpret_cast<float*>(tmem_holder + 4);  // G > 1: [8 chunks][3 warps][G-1][G-1][16]
    float* sbias = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(xch) + p.xch_bytes_);

    const uint32_t warp = warp_id_uniform(), lane = lane_id();
    const uint32_t crank = cluster_rank();
    const uint32_t rank = crank & 1;          // rank in the CTA pair
    const uint32_t pr = 0;                    // one CTA pair per cluster
    const bool leader = rank == 0;
    const uint16_t pair_mask = (uint16_t)3u;
    const uint16_t bmask = pair_mask;         // who consumes a weight stage
    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.tmap_a);
        tma_prefetch(&p.tmap_a2);
        tma_prefetch(&p.tmap_b);
        for (int i = 0; i < p.sa; ++i) {
            mbar_init(&afull[i], 1);  // armed by the leader only
            mbar_init(&aempty[i], 1);
        }
        for (int i = 0; i < p.sb; ++i) {
            mbar_init(&bfull[i], 1);
            mbar_init(&bempty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 16);  // 8 epilogue warps x 2 CTAs
            mbar_init(&tfull[i + 2], 1);
            mbar_init(&tempty[i + 2], 16);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc_cg2(tmem_holder, p.tmem_cols);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const int num_units = (int)(((int64_t)p.tiles + RUNS - 1) / RUNS) * p.n_tiles;
    const int PPC = 1;  // CTA pairs per cluster
    const int cid = blockIdx.x / (2 * PPC), ncl = gridDim.x / (2 * PPC);
    constexpr int kCtaSpan = 129 - G;  // positions a CTA advances per tile
    // flat tiling: CTA tile c of pair tile t; clamped past the end (a dummy: loads anything
    // valid, stores nothing)
    auto cta_tile = [&](int t, int rk, bool& real) {
        int c = 2 * t + rk;
        real = c < p.ctiles;
        return real ? c : p.ctiles - 1;
    };
    // filter rows with at least one valid input row for the unit's tiles (both CTAs, every run)
    auto unit_rows = [&](int tg, int& r_lo, int& r_hi) {
        r_lo = 0;
        r_hi = p.kH;
        if (!p.flat) return;
        r_lo = p.kH;
        r_hi = 0;
        for (int k = 0; k < RUNS; ++k) {
            int t = tg * RUNS + k;
            if (t >= p.tiles) t = p.tiles - 1;
            for (int rk = 0; rk < 2; ++rk) {
                bool real;
                const int c = cta_tile(t, rk, real);
                const int q0 = (c % p.tpc) * kCtaSpan;
                const int y0 = q0 / p.Wp;
                int y1 = (q0 + kCtaSpan - 1) / p.Wp;
                if (y1 > p.oH - 1) y1 = p.oH - 1;
                r_lo = min(r_lo, max(0, p.aph - y1));
                r_hi = max(r_hi, min(p.kH, p.aH + p.aph - y0));
            }
        }
        if (r_lo >= r_hi) {  // only border rows: one all-zero filter row keeps the output defined
            r_lo = 0;
            r_hi = 1;
        }
    };

    if (warp == 0 || warp == 10) {
        // ===== TMA producers (both CTAs; bytes complete on the leader's barriers): warp 0
        // the pixel runs (A), warp 10 the weights (B), each walking the same stage sequence
        // on its own ring — one thread issuing both let a full B ring stall the A prefetch
        // (the B ring holds only ~2 A stages' worth of taps) =====
        const bool doA = warp == 0, doB = warp == 10;
        if (lane == 0) {
            int as = 0, bs = 0;
            uint32_t aph = 0, bph = 0;
            const uint32_t btx = 2 * p.stage_b;
            const uint32_t run_bytes = (uint32_t)CPS * p.box_a;  // one run's CPS boxes
            for (int uu = cid; uu * PPC < num_units; uu += ncl) {
                const int u0 = uu * PPC + (int)pr;
                const int u = u0 < num_units ? u0 : num_units - 1;  // dummy tile: any valid coordinates
                const int tg = u / p.n_tiles, nt = u - tg * p.n_tiles;
                // per run: image half `rank`, offset qh inside it; both CTAs share the column
                // w0, hence the row count and the byte count
                int n_k[RUNS], row0_k[RUNS];
                bool short_k[RUNS];
                uint32_t atx_t = 0;
                int w0_k[RUNS];
#pragma unroll
                for (int k = 0; k < RUNS; ++k) {
                    int t = tg * RUNS + k;
                    if (t >= p.tiles) t = p.tiles - 1;  // dummy second run past the end
                    if (p.flat) {
                        bool real;
                        const int c = cta_tile(t, (int)rank, real);
                        n_k[k] = c / p.tpc;
                        const int q0 = (c - n_k[k] * p.tpc) * kCtaSpan;
                        row0_k[k] = q0 / p.Wp;
                        w0_k[k] = q0 % p.Wp;
                        short_k[k] = false;
                    } else {
                        n_k[k] = t / p.tpi;
                        const int qh = (t - n_k[k] * p.tpi) * kCtaSpan;
                        row0_k[k] = (int)rank * p.R + qh / p.Wp;
                        w0_k[k] = qh % p.Wp;
                        short_k[k] = qh % p.Wp < p.nr_split;
                    }
                    if (p.a_run) atx_t += 2u * (uint32_t)CPS * (uint32_t)p.run_px * 128u;
                    else atx_t += 2 * (short_k[k] ? run_bytes - (uint32_t)CPS * (uint32_t)p.Wp * 128u : run_bytes);
                }
                const int brow = G > 1 ? 0 : nt * p.bn + (int)rank * (p.bn / 2);
                int r_lo, r_hi;
                unit_rows(tg, r_lo, r_hi);
                for (int r = r_lo; r < r_hi; ++r) {
                    for (int cc = 0; cc < p.chunks; cc += CPS) {
                        if (doA) {
                        mbar_wait(&aempty[as], aph ^ 1);
                        if (leader) mbar_arrive_expect_tx(&afull[as], atx_t);
                        // NR full padded rows from the dense NHWC tensor (out-of-bounds = the zero
                        // border) for the CPS chunks: {32 ch, Wp px, NR rows, 1, CPS}
                        // (one request per chunk: the short map's smaller box would change the
                        // chunk stride inside a multi-chunk box)
#pragma unroll
                        for (int k = 0; k < RUNS; ++k) {
                            if (p.a_run) {
                                // exactly the run: im2col traversal of the padded position space
                                // (row width Wp) from the tile's first position, filter row r
#pragma unroll
                                for (int c = 0; c < CPS; ++c)
                                    // a tile starting in the phantom row 2R-1 = oH (odd oH) has no valid
                                    // position; the im2col start must stay inside the traversal range
                                    tma_load_im2col_4d_cg2(sA + (size_t)as * p.stage_a + k * run_bytes + c * p.box_a,
                                                           &p.tmap_run, &afull[as], (cc + c) * 32, w0_k[k] - p.apw,
                                                           min(row0_k[k], p.oH - 1) - p.aph, n_k[k], 0, (uint16_t)r);
                            } else {
                                const CUtensorMap* amap = short_k[k] ? &p.tmap_a2 : &p.tmap_a;
#pragma unroll
                                for (int c = 0; c < CPS; ++c)
                                    tma_load_5d_cg2(sA + (size_t)as * p.stage_a + k * run_bytes + c * p.box_a, amap,
                                                    &afull[as], 0, -p.apw, row0_k[k] + r - p.aph, n_k[k], cc + c);
                            }
                        }
                        if (++as == p.sa) {
                            as = 0;
                            aph ^= 1;
                        }
                        }  // doA
                        for (int s = 0; doB && s < p.kW; s += G) {
                            mbar_wait(&bempty[bs], bph ^ 1);
                            if (leader) mbar_arrive_expect_tx(&bfull[bs], btx);
                            uint8_t* bdst = sB + (size_t)bs * p.stage_b;
                            if constexpr (G == 1) {
                                tma_load_3d_cg2(bdst, &p.tmap_b, &bfull[bs], 0, brow,
                                                (r * p.kW + s) * (p.cin_p / 32) + cc);
                            } else {
                                // tap-grouped packing: this CTA's G*bn/2 rows of group (r, s/G)
                                // are contiguous — one request for all chunks
                                const int grow = ((r * p.ngroups + s / G) * G) * p.bn + (int)rank * (G * p.bn / 2);
                                tma_load_3d_cg2(bdst, &p.tmap_b, &bfull[bs], 0, grow, cc);
                            }
                            if (++bs == p.sb) {
                                bs = 0;
                                bph ^= 1;
                            }
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {
            // ===== MMA issuer (whole warp, converged; one elected lane issues) =====
            const uint32_t idesc = idesc_tf32(256, G * p.bn, 0, 0);
            constexpr uint32_t kHi = desc_hi(1024, kSwizzle128B);
            int as = 0, bs = 0;
            uint32_t aph = 0, bph = 0;
            int it = 0;
            for (int uu = cid; uu * PPC < num_units; uu += ncl, ++it) {
                const int u0 = uu * PPC + (int)pr;
                const int u = u0 < num_units ? u0 : num_units - 1;
                // nacc (2 or 4) TMEM accumulators: the MMA may run nacc-1 tiles ahead of the
                // epilogue (tiles with little K per tile are otherwise epilogue-paced)
                const uint32_t acc = (uint32_t)(it % p.nacc);
                mbar_wait(&tempty[acc], ((it / p.nacc) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + acc * (RUNS * G * p.bn);
                const int tg = u / p.n_tiles;
                uint32_t w0_k[RUNS];  // run start columns
#pragma unroll
                for (int k = 0; k < RUNS; ++k) {
                    int t = tg * RUNS + k;
                    if (t >= p.tiles) t = p.tiles - 1;
                    w0_k[k] = p.a_run ? 0u : (uint32_t)(((t % p.tpi) * kCtaSpan) % p.Wp);  // a_run: the run starts at the tile
                }
                uint32_t accum = 0;
                const uint32_t box_a16 = p.box_a >> 4, box_b16 = p.box_b >> 4;
                int r_lo, r_hi;
                unit_rows(tg, r_lo, r_hi);
                for (int r = r_lo; r < r_hi; ++r) {
                    for (int cc = 0; cc < p.chunks; cc += CPS) {
                        mbar_wait(&afull[as], aph);
                        tc_fence_after();
                        const uint32_t alo = desc_lo(smem_u32(sA + (size_t)as * p.stage_a), 16);
                        for (int s = 0; s < p.kW; s += G) {
                            mbar_wait(&bfull[bs], bph);
                            tc_fence_after();
                            // tap s: the same pixel run, s rows (s*128 B) further in
                            const uint32_t blo = desc_lo(smem_u32(sB + (size_t)bs * p.stage_b), 16);
#pragma unroll
                            for (int k = 0; k < 4 * CPS; ++k) {
                                // K steps of the last chunk past the real channels multiply zeros
                                if (cc + (k >> 2) == p.chunks - 1 && (k & 3) >= p.last_k) continue;
                                const uint64_t bd = desc_make(blo + (k >> 2) * box_b16 + 2 * (k & 3), kHi);
#pragma unroll
                                for (int q = 0; q < RUNS; ++q) {
                                    const uint32_t a_s = alo + (uint32_t)q * (CPS * box_a16) + (w0_k[q] + (uint32_t)s) * 8u;
                                    mma_tf32_cg2_warp(d + (uint32_t)(q * G) * p.bn,
                                                      desc_make(a_s + (k >> 2) * box_a16 + 2 * (k & 3), kHi), bd, idesc,
                                                      accum);
                                }
                                accum = 1;
                            }
                            mma_commit_cg2_warp_mask(&bempty[bs], bmask);
                            if (++bs == p.sb) {
                                bs = 0;
                                bph ^= 1;
                            }
                        }
                        mma_commit_cg2_warp_mask(&aempty[as], pair_mask);
                        if (++as == p.sa) {
                            as = 0;
                            aph ^= 1;
                        }
                    }
                }
                mma_commit_cg2_warp_mask(&tfull[acc], pair_mask);
            }
        }
    } else if (warp < 10) {
        // ===== epilogue: TMEM -> registers -> (+bias) -> NCHW, border columns dropped =====
        const uint32_t q = warp & 3;            // TMEM lane quarter
        const int half = (int)(warp - 2) >> 2;  // column chunks half, 2*k + half
        const int64_t ohw = (int64_t)p.oH * p.oW;
        if (p.sbias_n > 0) {  // the bias once per CTA (an L2 round trip per chunk per tile otherwise)
            for (int e = (int)((warp - 2) * 32 + lane); e < p.sbias_n; e += 256)
                sbias[e] = e < p.n_rows ? __ldg(p.bias + e) : 0.f;
            asm volatile("bar.sync 3, 256;" ::: "memory");
        }
        const float* sb = p.sbias_n > 0 ? sbias : nullptr;
        int it = 0;
        for (int uu = cid; uu * PPC < num_units; uu += ncl, ++it) {
            const int u0 = uu * PPC + (int)pr;
            const bool real_u = u0 < num_units;  // a dummy tile's accumulator is drained, not stored
            const int u = real_u ? u0 : num_units - 1;
            const uint32_t acc = (uint32_t)(it % p.nacc);
            mbar_wait(&tfull[acc], (it / p.nacc) & 1);
            tc_fence_after();
            const int tg = u / p.n_tiles, nt = u - tg * p.n_tiles;
#pragma unroll 1
            for (int run = 0; run < RUNS; ++run) {
            const int t_raw = tg * RUNS + run;
            bool real = real_u && t_raw < p.tiles;
            const int t = real ? t_raw : p.tiles - 1;
            const int xpar = (it * RUNS + run) & 1;  // exchange-slot parity
            int n, qq, i;
            if (p.flat) {
                bool real_c;
                const int c = cta_tile(t, (int)rank, real_c);
                real = real && real_c;
                n = c / p.tpc;
                qq = (c - n * p.tpc) * kCtaSpan + (int)(q * 32 + lane);  // position in the image
                i = qq / p.Wp;
            } else {
                n = t / p.tpi;
                qq = (t - n * p.tpi) * kCtaSpan + (int)(q * 32 + lane);  // position in the half
                i = (int)rank * p.R + qq / p.Wp;
            }
            const int j = qq % p.Wp;
            const bool valid = real && qq < p.m && i < p.oH && j < p.oW && (int)(q * 32 + lane) < kCtaSpan;
            const int ch0 = nt * p.bn;
            const int64_t base = ((int64_t)n * p.n_rows + ch0) * ohw + (int64_t)i * p.oW + j;
            const uint32_t lane_base = tmem_base + ((q * 32u) << 16);
            if constexpr (G == 1) {
                for (int c0 = half * 16; c0 < p.bn; c0 += 32)
                    store_tmem_columns_nchw(lane_base + (acc * RUNS + run) * p.bn + c0, 16,
                                            p.out + (valid ? base + (int64_t)c0 * ohw : 0), ohw, p.bias,
                                            ch0 + c0, p.n_rows, valid, sb);
            } else {
                const uint32_t taddr = lane_base + (acc * RUNS + run) * G * p.bn;
                for (int c0 = half * 16; c0 < p.bn; c0 += 32) {
                    uint32_t vd[G][16];
                    float acc_v[16];
#pragma unroll
                    for (int dl = 0; dl < G; ++dl) tmem_ld_32x32b_x16(taddr + dl * p.bn + c0, vd[dl]);
                    const int chb = ch0 + c0;
                    const bool full16 = chb + 16 <= p.n_rows;
                    float bv[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        bv[e] = sb ? sb[chb + e] : (p.bias && chb + e < p.n_rows) ? __ldg(p.bias + chb + e) : 0.f;
                    tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 16; ++e) acc_v[e] = __uint_as_float(vd[0][e]);
                    // column group delta: the right neighbour delta lanes over, or (past lane
                    // 31) the next warp's first lanes through shared memory
                    float* slot = xch + (xpar * ((p.bn + 15) >> 4) + (c0 >> 4)) * (3 * (G - 1) * (G - 1) * 16);
#pragma unroll
                    for (int dl = 1; dl < G; ++dl) {
                        float* sd = slot + (dl - 1) * (G - 1) * 16;
#pragma unroll
                        for (int e = 0; e < 16; ++e) {
                            const float v = __uint_as_float(vd[dl][e]);
                            const float nb = __shfl_down_sync(0xffffffffu, v, dl);
                            if (lane < 32 - dl) acc_v[e] += nb;
                            if ((int)lane < dl && q > 0)
                                sd[((q - 1) * (G - 1) * (G - 1) + lane) * 16 + e] = v;
                        }
                    }
                    // the four lane quarters of this column half (named barrier 1 + half)
                    asm volatile("bar.sync %0, 128;" ::"r"(1 + half) : "memory");
                    if (q < 3) {
#pragma unroll
                        for (int dl = 1; dl < G; ++dl) {
                            if ((int)lane >= 32 - dl) {
                                const float* sd = slot + (dl - 1) * (G - 1) * 16 +
                                                  (q * (G - 1) * (G - 1) + (lane + dl - 32)) * 16;
#pragma unroll
                                for (int e = 0; e < 16; ++e) acc_v[e] += sd[e];
                            }
                        }
                    }
                    if (valid) {
                        float* o = p.out + base + (int64_t)c0 * ohw;
                        if (full16) {
#pragma unroll
                            for (int e = 0; e < 16; ++e) {
                                __stcs(o, acc_v[e] + bv[e]);
                                o += ohw;
                            }
                        } else {
#pragma unroll
                            for (int e = 0; e < 16; ++e) {
                                if (chb + e < p.n_rows) __stcs(o, acc_v[e] + bv[e]);
                                o += ohw;
                            }
                        }
                    }
                }
            }
            }  // run
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (leader) mbar_arrive(&tempty[acc]);
                else mbar_arrive_cluster(&tempty[acc], crank & ~1u);
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

}  // namespace

// Tiling: each image's output rows are split into two halves of R rows; CTA 0 of a pair
// walks the top half and CTA 1 the bottom half at the same offset, so both CTAs' pixel
// runs start at the same column and one shared descriptor addresses both.
bool hconv_wrap() {
    static const bool wrap = [] {
        const char* e = std::getenv("PT_B200_HCONV_WRAP");
        return e ? std::atoi(e) != 0 : true;
    }();
    return wrap;
}

HConvTiling hconv_tiling(int64_t N, int64_t Wp, int64_t oH, int64_t cta_span) {
    HConvTiling t;
    const int64_t R = (oH + 1) / 2;
    t.P_img = R * Wp;                                // positions per half
    t.tiles = N * ceil_div(t.P_img, cta_span);       // pair tiles
    return t;
}

void run_hconv(const UmmaPlan& pl, const float* act, const float* wt, int64_t N, int64_t aH,
               int64_t aW, int64_t aph, int64_t apw, int kH, int kW, int64_t oH, int64_t oW,
               float* out, const float* bias, double alg_flops, cudaStream_t st) {
    PTB_REQUIRE(pl.cb == 32 && pl.cg == 2, "hconv: needs the 32-channel CTA-pair plan");
    // Position rows carry only the LEFT border: a tap reading past the right edge of row i
    // wraps into row i+1's left border, which is zero (TMA out-of-bounds) exactly like the
    // right border it replaces — valid because the right border is never wider than the left
    // (symmetric padding). Each row then wastes kW-1-apw junk positions instead of kW-1 (the
    // full-padding transposed conv of a pad-0 layer: none; convnet L2 dgrad 72 -> 64).
    // PT_B200_HCONV_WRAP=0 restores the two-sided border.
    const int64_t Wp = aW + (hconv_wrap() ? 1 : 2) * apw;
    PTB_REQUIRE(Wp <= 256 && kW <= 120, "hconv: padded row too wide for one TMA box");
    const int G = pl.tap_group;
    const bool pair = G > 1;
    const int cta_span = 129 - G;
    // rows a CTA's run (128 + kW - 1 positions from any column) can touch
    const int NR = (int)(1 + (Wp - 1 + 128 + kW - 2) / Wp);
    PTB_REQUIRE(NR <= 256 && N * aH * aW * pl.cin_p < (1ll << 40), "hconv: geometry out of range");
    HConvParams p;
    memset(&p, 0, sizeof p);
    // A: the exact pixel run of a tile (im2col traversal) unless PT_B200_HCONV_A=rows; the
    // NR-full-rows box fetches up to ~2.6x the run for narrow rows (VGG conv2: 3 x 114 px
    // for a 130-pixel run)
    static const int a_env = [] {
        const char* e = std::getenv("PT_B200_HCONV_A");
        return e && std::string(e) == "rows" ? 0 : 1;
    }();
    p.a_run = a_env;
    p.run_px = 128 + kW - 1;
    PTB_REQUIRE(!p.a_run || p.run_px <= 256, "hconv: run too long for one im2col box");
    // CPS: two channel chunks per stage unless the A stage would not leave room for a ring
    const uint32_t box_a = p.a_run ? (uint32_t)align_up((size_t)p.run_px * 128, 1024) : (uint32_t)(NR * Wp) * 128u;
    // B per CTA: G*bn/2 rows of the (delta, c) stack (G > 1), else bn/2 rows of one tap
    const uint32_t box_b = (uint32_t)align_up((size_t)(pair ? G * pl.bn / 2 : pl.bn / 2), 8) * 128u;
    const int sbias_n = (bias && pl.n_rows <= 4096) ? (int)((pl.n_rows + 15) / 16 * 16 + 16) : 0;
    const int budget = kSmemLimitH - 1024 - 512 - xch_bytes(G, pl.bn) - sbias_n * 4;
    // RUNS = 2 (two position tiles per weight stage) for tiles with a short reduction (their
    // per-tile fixed costs dominate: VGG-A conv2 fwd, 72 MMAs per tile, 0.289 -> 0.200 ms;
    // convnet L2 fwd, 648 per tile, unchanged), when both accumulators of a unit still leave
    // TMEM for double buffering (G*bn <= 128). PT_B200_HCONV_RUNS=1|2 forces.
    static const int runs_env = [] {
        const char* e = std::getenv("PT_B200_HCONV_RUNS");
        return e ? std::atoi(e) : 0;
    }();
    const int64_t mmas_per_tile = (int64_t)kH * (pl.cin_p / 32) * ceil_div(kW, G) * 4;
    int runs = ((runs_env == 0 && mmas_per_tile <= 320 && G <= 2 && G * pl.bn <= 128) ||
                (runs_env == 2 && G <= 3 && G * pl.bn <= 256))
                   ? 2
                   : 1;
    if (runs == 2 && 2 * 2 * (int)box_a + 3 * (int)box_b > budget) runs = 1;  // two-run A stages must fit twice
    int cps = (pl.cin_p / 32) % 2 == 0 ? 2 : 1;
    if (cps == 2 && 2 * 2 * runs * (int)box_a + 4 * 2 * (int)box_b > budget) cps = 1;
    PTB_REQUIRE(2 * runs * (int)box_a + 3 * (int)box_b <= budget, "hconv: shared memory too small for the rings");
    {
        const uint64_t dims[5] = {32, (uint64_t)aW, (uint64_t)aH, (uint64_t)N, (uint64_t)(pl.cin_p / 32)};
        const uint64_t strides[4] = {(uint64_t)pl.cin_p * 4, (uint64_t)(aW * pl.cin_p * 4),
                                     (uint64_t)(aH * aW * pl.cin_p * 4), 128};
        const uint32_t box[5] = {32, (uint32_t)Wp, (uint32_t)NR, 1, 1};
        tmap_tiled(&p.tmap_a, act, 5, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
        const uint32_t box2[5] = {32, (uint32_t)Wp, (uint32_t)std::max(1, NR - 1), 1, 1};
        tmap_tiled(&p.tmap_a2, act, 5, dims, strides, box2, CU_TENSOR_MAP_SWIZZLE_128B);
        if (p.a_run)  // positions (i, j < Wp) -> input (i + r - aph, j - apw): a kH x 1 "conv" with pad (aph, apw)
            tmap_im2col(&p.tmap_run, act, N, aH, aW, pl.cin_p, kH, 1, (int)aph, (int)apw, 1, 1, 32, p.run_px,
                        CU_TENSOR_MAP_SWIZZLE_128B, (int)(Wp - aW - apw));
    }
    if (!pair) {
        // {32, weight rows, 32-wide k blocks}: one box = the CPS chunks of one tap
        const uint64_t kdim = (uint64_t)pl.kdim;
        const uint64_t dims[3] = {32, (uint64_t)pl.n_pad, kdim / 32};
        const uint64_t strides[2] = {kdim * 4, 128};
        const uint32_t box[3] = {32, (uint32_t)(pl.bn / 2), (uint32_t)cps};
        tmap_tiled(&p.tmap_b, wt, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    } else {
        // tap-grouped rows [kH*ngroups*G*bn][cin_p] as {32, rows, cin_p/32}: box = one CTA's
        // G*bn/2 rows x CPS chunks
        const int64_t ng = ceil_div(kW, G);
        const uint64_t rows = (uint64_t)(pl.taps / kW * ng * G * pl.bn);
        const uint64_t dims[3] = {32, rows, (uint64_t)(pl.cin_p / 32)};
        const uint64_t strides[2] = {(uint64_t)pl.cin_p * 4, 128};
        const uint32_t box[3] = {32, (uint32_t)(G * pl.bn / 2), (uint32_t)cps};
        tmap_tiled(&p.tmap_b, wt, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
        p.ngroups = (int)ng;
    }
    p.zero_tap = (int)pl.taps;
    PTB_REQUIRE(!pair || (G * pl.bn % 16 == 0 && G * pl.bn <= 256 && (G % 2 == 0 || pl.bn % 16 == 0)),
                "hconv: bad tap group");
    const HConvTiling tl = hconv_tiling(N, Wp, oH, cta_span);
    PTB_REQUIRE(tl.tiles * (int64_t)pl.n_tiles < (1ll << 31) && tl.P_img < (1ll << 30), "hconv: too many tiles");
    p.N = (int)N;
    p.Wp = (int)Wp;
    p.aph = (int)aph;
    p.apw = (int)apw;
    p.kH = kH;
    p.kW = kW;
    p.cin_p = (int)pl.cin_p;
    p.chunks = (int)(pl.cin_p / 32);
    {
        static const bool skip = [] {
            const char* e = std::getenv("PT_B200_HCONV_KSKIP");
            return e ? std::atoi(e) != 0 : true;
        }();
        const int64_t rem = pl.cin_real > 0 ? pl.cin_real - 32 * (p.chunks - 1) : 32;
        p.last_k = skip ? (int)std::min<int64_t>(4, std::max<int64_t>(1, (rem + 7) / 8)) : 4;
    }
    p.oH = (int)oH;
    p.oW = (int)oW;
    p.R = (int)((oH + 1) / 2);
    p.m = (int)tl.P_img;
    p.tpi = (int)ceil_div(tl.P_img, cta_span);
    // a run from column w0 spans rows 0 .. (w0 + 128 + kW - 2) / Wp: one row less below
    p.nr_split = NR > 1 ? (int)std::max<int64_t>(0, (NR - 1) * Wp - (128 + kW - 2)) : 0;
    p.tiles = (int)tl.tiles;
    p.aH = (int)aH;
    p.n_rows = (int)pl.n_rows;
    p.bn = pl.bn;
    p.n_tiles = pl.n_tiles;
    p.box_a = box_a;
    p.box_b = box_b;
    p.stage_a = runs * cps * p.box_a;
    p.stage_b = cps * p.box_b;
    // B ring: enough stages to cover two filter rows' worth of taps; A ring: the rest
    int sb = std::min(16, std::max(4, pair ? 2 * (int)ceil_div(kW, G) : 2 * kW));
    static const int sb_env = [] {
        const char* e = std::getenv("PT_B200_HCONV_SB");
        return e ? std::atoi(e) : 0;
    }();
    if (sb_env >= 2) sb = sb_env;
    while (sb > 3 && budget - sb * (int)p.stage_b < 2 * (int)p.stage_a) --sb;
    int sa = (budget - sb * (int)p.stage_b) / (int)p.stage_a;
    sa = std::min(sa, 8);
    PTB_REQUIRE(sa >= 2, "hconv: shared memory too small for the rings");
    p.sa = sa;
    p.sb = sb;
    p.nacc = 4 * runs * G * pl.bn <= 512 ? 4 : 2 * runs * G * pl.bn <= 512 ? 2 : 1;
    p.tmem_cols = 32;
    while ((int)p.tmem_cols < p.nacc * runs * G * pl.bn) p.tmem_cols <<= 1;
    PTB_REQUIRE(p.tmem_cols <= 512, "hconv: accumulators exceed TMEM");
    p.out = out;
    p.bias = bias;
    const size_t smem = 1024 + (size_t)sa * p.stage_a + (size_t)sb * p.stage_b +
                        (2 * sa + 2 * sb + 8) * 8 + 16 + xch_bytes(G, pl.bn) + (size_t)sbias_n * 4;
    p.sbias_n = sbias_n;
    p.xch_bytes_ = (uint32_t)xch_bytes(G, pl.bn);
    // flat tiling (run mode): consecutive CTA tiles over whole images. It skips the filter
    // rows of a large zero border (convnet L2 dgrad 0.82 -> 0.78 ms) and rounds tiles once
    // per image instead of once per half: interleaved per-launch A/B, flat vs halves: VGG-A
    // conv3 fwd 157 -> 146 us, conv4 fwd/dgrad 293 -> 271 us, AlexNet conv1/conv2 and
    // Overfeat conv1 -2..-3 %; the exception is the row-expanded small-C dgrad (kH = 1:
    // nothing to skip, one filter row per tile), where the image halves stay faster (convnet
    // L1 dgrad 275 vs 284 us). PT_B200_HCONV_FLAT=1 / 2 forces flat / halves.
    static const int flat_env = [] {
        const char* e = std::getenv("PT_B200_HCONV_FLAT");
        return e ? std::atoi(e) : 0;
    }();
    p.flat = (p.a_run && (flat_env == 1 || (flat_env == 0 && kH > 1))) ? 1 : 0;
    if (p.flat) {
        const int64_t P_img = oH * Wp;
        p.m = (int)P_img;
        p.tpc = (int)ceil_div(P_img, cta_span);
        const int64_t ct = N * (int64_t)p.tpc;
        PTB_REQUIRE(ct * pl.n_tiles < (1ll << 31), "hconv: too many tiles");
        p.ctiles = (int)ct;
        p.tiles = (int)ceil_div(ct, 2);
    }
    const int units = (int)ceil_div(p.tiles, runs) * p.n_tiles;
    // (two CTA pairs per cluster sharing each weight stage by TMA multicast measured 1.8x
    // slower — convnet L2 dgrad 0.85 -> 1.51 ms, the pairs' lockstep couples their stalls —
    // and was removed)
    const int cl_ctas = 2;
    const int ncl = std::min(units, sm_count() / cl_ctas);
    once_per_device((const void*)umma_hconv_kernel<1, 1, 1>, [&] {  // the smem limit is a per-device attribute
        for (auto fn : {umma_hconv_kernel<1, 1, 1>, umma_hconv_kernel<1, 2, 1>, umma_hconv_kernel<1, 3, 1>,
                        umma_hconv_kernel<1, 4, 1>, umma_hconv_kernel<2, 1, 1>, umma_hconv_kernel<2, 2, 1>,
                        umma_hconv_kernel<2, 3, 1>, umma_hconv_kernel<2, 4, 1>, umma_hconv_kernel<1, 1, 2>,
                        umma_hconv_kernel<1, 2, 2>, umma_hconv_kernel<2, 1, 2>, umma_hconv_kernel<2, 2, 2>,
                        umma_hconv_kernel<1, 3, 2>, umma_hconv_kernel<2, 3, 2>})
            PTB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimitH));
    });
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl_ctas * ncl);
    cfg.blockDim = dim3(kThreadsH);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl_ctas;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    ProfScope prof("umma_conv", st, alg_flops, 0.0);
#define PTB_HCONV_LAUNCH(CPS_, G_, R_) PTB_CUDA(cudaLaunchKernelEx(&cfg, umma_hconv_kernel<CPS_, G_, R_>, p))
    if (runs == 2) {
        if (cps == 2) {
            if (G == 1) PTB_HCONV_LAUNCH(2, 1, 2);
            else if (G == 2) PTB_HCONV_LAUNCH(2, 2, 2);
            else PTB_HCONV_LAUNCH(2, 3, 2);
        } else {
            if (G == 1) PTB_HCONV_LAUNCH(1, 1, 2);
            else if (G == 2) PTB_HCONV_LAUNCH(1, 2, 2);
            else PTB_HCONV_LAUNCH(1, 3, 2);
        }
    } else if (cps == 2) {
        if (G == 1) PTB_HCONV_LAUNCH(2, 1, 1);
        else if (G == 2) PTB_HCONV_LAUNCH(2, 2, 1);
        else if (G == 3) PTB_HCONV_LAUNCH(2, 3, 1);
        else PTB_HCONV_LAUNCH(2, 4, 1);
    } else {
        if (G == 1) PTB_HCONV_LAUNCH(1, 1, 1);
        else if (G == 2) PTB_HCONV_LAUNCH(1, 2, 1);
        else if (G == 3) PTB_HCONV_LAUNCH(1, 3, 1);
        else PTB_HCONV_LAUNCH(1, 4, 1);
    }
#undef PTB_HCONV_LAUNCH
    after_launch("umma_hconv");
}

}  // namespace ptb
