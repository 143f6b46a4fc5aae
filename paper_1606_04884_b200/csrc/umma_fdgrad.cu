// umma_fdgrad.cu — input gradient of small-channel stride-1 layers (C <= 4: convnet L1;
// updateGradInput) as the SPEC's gradCol GEMM with the col2im fold
// fused into the epilogue:
//
//   gcol[(i,j)][(s,r,c)] = sum_k gy[n][k][i][j] * W[k][c][r][s]          (tensor cores)
//   gx[n][c][i+r-pH][j+s-pW] += gcol[(i,j)][(s,r,c)]                       (epilogue, smem)
//
// M = 128 output pixels of one gy row per CTA (pair: two row bands), N = kH*kW*C filter
// columns (<= 512, up to two MMAs of N <= 256), K = output channels. Unlike the
// transposed-conv engines this computes no zero-padded taps (L1: 118 x 118 pixels instead
// of 128 x 138 positions) and needs no expanded gradient in HBM. The filter (W^T, one CTA's
// half of every N-half) stays resident in smem; each step streams one gy row.
//
// Fold: gy row t of a band contributes to gx rows t+r-pH; a ring of kH gx rows x C
// channels in smem accumulates them, and after row t the ring row of gx row t-pH is
// complete for this band and is written to the band's slab. Adjacent bands overlap in
// kH-1 gx rows; a fixed-order fixup kernel sums the slabs (deterministic). The columns are
// grouped per (r, c) with the kW taps s in 12-column groups, so a lane gathers the 1-D
// fold sum_s gcol[px - s][(r, c, s)] with warp shuffles and does ONE ring update per group;
// the sums that land past its warp's 32 pixels (the next quarter's first kW-1 cells) go to
// a per-quarter spill row added at the flush. Every ring / spill cell has one writer warp.
#include <cuda.h>

#include <cstdlib>

#include "kernels.cuh"
#include "tmap.cuh"
#include "umma.cuh"

namespace ptb {

namespace {

using namespace umma;

constexpr int kThreadsF = 320;  // warp 0 TMA, warp 1 MMA (+ TMEM), warps 2..9 epilogue (2 per lane quarter)
constexpr int kSmemLimitF = 232448;
constexpr int kBand = 16;       // gy rows per CTA unit

struct FDParams {
    CUtensorMap tmap_gy;  // gy NHWC 5-D {32, oW, oH, N, Kp/32}, box {32, 128, 1, 1, 1}, SW128
    CUtensorMap tmap_w;   // W^T packed [Npad][Kp] as {32, Npad, Kp/32}, box {32, nhalf/2, 1}, SW128
    int N, C, H, W, oH, kH, kW, pH, pW;
    int chunks;           // Kp / 32
    int nh, nhalf, ntot;  // N-halves, columns per half, real columns (kH*kW*C)
    int nbands, bands;    // bands per image, N * nbands
    int ring_w;           // 128 (own cells; the spill rows hold the kW-1 cells past each quarter)
    int ngroups, gpr;     // (r, c) groups, groups per N-half region (12 columns each)
    int sa;               // A ring depth
    uint32_t stage_a, b_bytes, b_off, tmem_cols;
    float* slab;          // [bands][C][kBand + kH - 1][W]
};

__global__ void __launch_bounds__(kThreadsF, 1) umma_fdgrad_kernel(const __grid_constant__ FDParams p) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((((raw + 1023u) & ~1023u)) - raw);
    uint8_t* sB = smem;                                 // [nh][chunks][nhalf/2][32] resident
    uint8_t* sA = sB + p.b_off;  // [sa][chunks][128][32]
    float* ring = reinterpret_cast<float*>(sA + (size_t)p.sa * p.stage_a);  // [C][kH][ring_w]
    const int ring_elems = p.C * p.kH * (p.ring_w + 5 * 32);  // own cells, then spill rows
    uint64_t* bars = reinterpret_cast<uint64_t*>(ring + ((ring_elems + 3) & ~3));
    uint64_t* afull = bars;
    uint64_t* aempty = afull + p.sa;
    uint64_t* tfull = aempty + p.sa;  // [2] per N-half region
    uint64_t* tempty = tfull + 2;     // [2]
    uint64_t* wbar = tempty + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(wbar + 1);

    const uint32_t warp = warp_id_uniform(), lane = lane_id();
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.tmap_gy);
        tma_prefetch(&p.tmap_w);
        for (int i = 0; i < p.sa; ++i) {
            mbar_init(&afull[i], 1);
            mbar_init(&aempty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 16);  // 8 epilogue warps x 2 CTAs
        }
        mbar_init(wbar, 1);
        fence_mbar_init();
    }
    for (int e = threadIdx.x; e < ring_elems; e += blockDim.x) ring[e] = 0.f;
    if (warp == 1) tmem_alloc_cg2(tmem_holder, p.tmem_cols);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const int units = (p.bands + 1) / 2;
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    const int rows_per_half = p.nhalf / 2;

    if (warp == 0) {
        if (lane == 0) {
            // resident W^T: this CTA's rows of every N-half, all K chunks
            if (leader) mbar_arrive_expect_tx(wbar, 2 * p.b_bytes);
            for (int h = 0; h < p.nh; ++h)
                for (int c = 0; c < p.chunks; ++c)
                    tma_load_3d_cg2(sB + (size_t)(h * p.chunks + c) * rows_per_half * 128, &p.tmap_w, wbar, 0,
                                    h * p.nhalf + (int)rank * rows_per_half, c);
            int as = 0;
            uint32_t aph = 0;
            for (int u = cid; u < units; u += ncl) {
                const int band = 2 * u + (int)rank;  // this CTA's band (past the end: a dummy, all OOB)
                const int n = band / p.nbands, row0 = (band - n * p.nbands) * kBand;
                for (int t = 0; t < kBand; ++t) {
                    mbar_wait(&aempty[as], aph ^ 1);
                    if (leader) mbar_arrive_expect_tx(&afull[as], 2 * p.stage_a);
                    for (int c = 0; c < p.chunks; ++c)
                        tma_load_5d_cg2(sA + (size_t)as * p.stage_a + (size_t)c * 16384, &p.tmap_gy, &afull[as], 0, 0,
                                        row0 + t, band < p.bands ? n : p.N, c);
                    if (++as == p.sa) {
                        as = 0;
                        aph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {
            const uint32_t idesc = idesc_tf32(256, p.nhalf, 0, 0);
            constexpr uint32_t kHi = desc_hi(1024, kSwizzle128B);
            mbar_wait(wbar, 0);
            tc_fence_after();
            const uint32_t blo0 = desc_lo(smem_u32(sB), 16);
            const uint32_t bchunk16 = (uint32_t)(rows_per_half * 128) >> 4;
            int as = 0;
            uint32_t aph = 0;
            int step = 0;
            for (int u = cid; u < units; u += ncl) {
                for (int t = 0; t < kBand; ++t, ++step) {
                    mbar_wait(&afull[as], aph);
                    tc_fence_after();
                    const uint32_t alo = desc_lo(smem_u32(sA + (size_t)as * p.stage_a), 16);
                    for (int h = 0; h < p.nh; ++h) {
                        mbar_wait(&tempty[h], (step & 1) ^ 1);
                        tc_fence_after();
                        uint32_t accum = 0;
                        for (int c = 0; c < p.chunks; ++c) {
#pragma unroll
                            for (int sub = 0; sub < 4; ++sub) {
                                mma_tf32_cg2_warp(tmem_base + (uint32_t)(h * p.nhalf),
                                                  desc_make(alo + (uint32_t)c * 1024u + 2u * sub, kHi),
                                                  desc_make(blo0 + (uint32_t)(h * p.chunks + c) * bchunk16 + 2u * sub, kHi),
                                                  idesc, accum);
                                accum = 1;
                            }
                        }
                        mma_commit_cg2_warp(&tfull[h]);
                    }
                    mma_commit_cg2_warp(&aempty[as]);
                    if (++as == p.sa) {
                        as = 0;
                        aph ^= 1;
                    }
                }
            }
        }
    } else {
        // ===== epilogue: fold the gcol row into the ring, flush completed gx rows =====
        const uint32_t q = warp & 3;
        const int half = (int)(warp - 2) >> 2;  // this warp folds the groups g = half (mod 2)
        const int px = (int)(q * 32 + lane);  // pixel j of the gy row
        const int slab_rows = kBand + p.kH - 1;
        const int ept = 256;                  // epilogue threads
        const int tid = (int)((warp - 2) * 32 + lane);
        float* spill = ring + p.C * p.kH * p.ring_w;  // [C][kH][5 quarters][32]
        int step = 0;
        for (int u = cid; u < units; u += ncl) {
            const int band = 2 * u + (int)rank;
            const bool real = band < p.bands;
            float* slab = p.slab + (size_t)(real ? band : 0) * p.C * slab_rows * p.W;
            for (int t = 0; t < kBand; ++t, ++step) {
                const int slot0 = t % p.kH;
                for (int h = 0; h < p.nh; ++h) {
                    mbar_wait(&tfull[h], step & 1);
                    tc_fence_after();
                    const uint32_t taddr = tmem_base + ((q * 32u) << 16) + (uint32_t)(h * p.nhalf);
                    const int g0 = h * p.gpr, g_end = min(p.ngroups, g0 + p.gpr);
                    // batches of 4 of this warp's groups: 12 TMEM loads under one wait, then
                    // four independent shuffle folds
                    for (int gb = g0 + half; gb < g_end; gb += 8) {
                        uint32_t v[4][12];
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            const int gl = min(gb + 2 * b, g_end - 1) - g0;
#pragma unroll
                            for (int k = 0; k < 3; ++k)
                                tmem_ld_32x32b_x4(taddr + gl * 12 + 4 * k, *reinterpret_cast<uint32_t(*)[4]>(&v[b][4 * k]));
                        }
                        tmem_ld_wait();
                        // the four groups' folds interleaved (independent shuffle chains)
                        float own[4], spl[4];
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            own[b] = __uint_as_float(v[b][0]);
                            spl[b] = 0.f;
                        }
#pragma unroll
                        for (int s = 1; s < 12; ++s) {
                            if (s < p.kW) {
                                float x[4];
#pragma unroll
                                for (int b = 0; b < 4; ++b)
                                    x[b] = __shfl_sync(0xffffffffu, __uint_as_float(v[b][s]), (lane - s) & 31);
#pragma unroll
                                for (int b = 0; b < 4; ++b) {
                                    if ((int)lane >= s) own[b] += x[b];
                                    else spl[b] += x[b];
                                }
                            }
                        }
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            const int g = gb + 2 * b;
                            if (g < g_end) {
                                const int r = g / p.C, c = g - r * p.C;
                                int slot = slot0 + r;
                                if (slot >= p.kH) slot -= p.kH;
                                ring[(c * p.kH + slot) * p.ring_w + px] += own[b];
                                if ((int)lane < p.kW - 1) spill[((c * p.kH + slot) * 5 + q + 1) * 32 + lane] += spl[b];
                            }
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if (leader) mbar_arrive(&tempty[h]);
                        else mbar_arrive_cluster(&tempty[h], 0);
                    }
                }
                asm volatile("bar.sync 1, 256;" ::: "memory");
                // gx row (band row0 + t - pH) is complete for this band: slab row t
                for (int e = tid; e < p.C * p.W; e += ept) {
                    const int c = e / p.W, w = e - c * p.W;
                    const int x = w + p.pW;
                    const float* rs = ring + (c * p.kH + slot0) * p.ring_w;
                    const float* ss = spill + (c * p.kH + slot0) * 5 * 32;
                    float val = x < 128 ? rs[x] : 0.f;
                    if (x >= 32 && (x & 31) < p.kW - 1) val += ss[(x >> 5) * 32 + (x & 31)];
                    if (real) slab[((size_t)c * slab_rows + t) * p.W + w] = val;
                }
                asm volatile("bar.sync 1, 256;" ::: "memory");
                for (int e = tid; e < p.C * (p.ring_w + 5 * 32); e += ept) {
                    const int c = e / (p.ring_w + 5 * 32), x = e - c * (p.ring_w + 5 * 32);
                    if (x < p.ring_w) ring[(c * p.kH + slot0) * p.ring_w + x] = 0.f;
                    else spill[(c * p.kH + slot0) * 5 * 32 + (x - p.ring_w)] = 0.f;
                }
                asm volatile("bar.sync 1, 256;" ::: "memory");
            }
            // the band's last kH-1 gx rows (completed by the next band's contributions)
            for (int j = 0; j < p.kH - 1; ++j) {
                const int slot = (kBand + j) % p.kH;
                for (int e = tid; e < p.C * p.W; e += ept) {
                    const int c = e / p.W, w = e - c * p.W;
                    const int x = w + p.pW;
                    float val = x < 128 ? ring[(c * p.kH + slot) * p.ring_w + x] : 0.f;
                    if (x >= 32 && (x & 31) < p.kW - 1) val += spill[((c * p.kH + slot) * 5 + (x >> 5)) * 32 + (x & 31)];
                    if (real) slab[((size_t)c * slab_rows + kBand + j) * p.W + w] = val;
                }
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");
            for (int e = tid; e < ring_elems; e += ept) ring[e] = 0.f;
            asm volatile("bar.sync 1, 256;" ::: "memory");
        }
    }
    __syncwarp();
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (warp == 1) tmem_dealloc_cg2(tmem_base, p.tmem_cols);
#endif
}

// W^T packed for the gcol GEMM: row n = region*nhalf + gl*12 + s for the (r, c) group
// g = region*gpr + gl (12 columns per group, the kW taps first, zero past kW / the real
// groups / the channels), column k: wt[n][k] = W[k][c][r][s], TF32-rounded.
__global__ void pack_fdgrad_w_kernel(const float* __restrict__ w, float* __restrict__ wt, int K, int C, int kH,
                                     int kW, int npad, int kp, int nhalf, int gpr, int ngroups) {
    const int total = npad * kp;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int n = i / kp, k = i - n * kp;
        const int region = n / nhalf, nl = n - region * nhalf;
        const int gl = nl / 12, s = nl - gl * 12;
        const int g = region * gpr + gl;
        float v = 0.f;
        if (gl < gpr && g < ngroups && s < kW && k < K) {
            const int r = g / C, c = g - r * C;
            v = __ldg(w + (((int64_t)k * C + c) * kH + r) * kW + s);
        }
        uint32_t u;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(v));
        wt[i] = __uint_as_float(u);
    }
}

// gx[n][c][h][w] = sum over the bands b of image n covering h (in band order) of
// slab[b][c][h - (b*kBand - pH)][w]
__global__ void fdgrad_fixup_kernel(const float* __restrict__ slab, float* __restrict__ gx, int N, int C, int H,
                                    int W, int kH, int pH, int nbands) {
    const int slab_rows = kBand + kH - 1;
    const int64_t total = (int64_t)N * C * H * W;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int w = (int)(e % W);
        const int h = (int)((e / W) % H);
        const int c = (int)((e / ((int64_t)W * H)) % C);
        const int n = (int)(e / ((int64_t)W * H * C));
        // band b covers gx rows [b*kBand - pH, b*kBand - pH + slab_rows)
        int b_lo = (h + pH - slab_rows + 1 + kBand - 1) / kBand;  // ceil((h + pH - slab_rows + 1) / kBand)
        if (h + pH - slab_rows + 1 <= 0) b_lo = 0;
        int b_hi = (h + pH) / kBand;
        if (b_hi > nbands - 1) b_hi = nbands - 1;
        float acc = 0.f;
        for (int b = b_lo; b <= b_hi; ++b) {
            const int rr = h + pH - b * kBand;
            acc += __ldg(slab + ((((int64_t)n * nbands + b) * C + c) * slab_rows + rr) * W + w);
        }
        gx[e] = acc;
    }
}

struct FDPlan {
    int Kp, chunks, ntot, nh, nhalf, npad, nbands, bands, ring_w, sa, ngroups, gpr;
    uint32_t stage_a, b_bytes, tmem_cols;
    size_t smem, wt_bytes, gyh_bytes, slab_bytes;
};

FDPlan fdplan(const Geo& g) {
    FDPlan f;
    f.Kp = (int)((g.K + 31) / 32 * 32);
    f.chunks = f.Kp / 32;
    f.ntot = (int)(g.kH * g.kW * g.C);
    f.ngroups = (int)(g.kH * g.C);  // (r, c) groups of 12 columns (the kW <= 12 taps)
    f.nh = (int)ceil_div(f.ngroups * 12, 256);
    f.gpr = (int)ceil_div(f.ngroups, f.nh);
    f.nhalf = (int)(ceil_div(f.gpr * 12, 16) * 16);
    if (f.nhalf < 32) f.nhalf = 32;
    f.npad = f.nh * f.nhalf;
    f.nbands = (int)ceil_div(g.oH, kBand);
    f.bands = (int)(g.N * f.nbands);
    f.ring_w = 128;
    f.stage_a = (uint32_t)f.chunks * 16384u;
    f.b_bytes = (uint32_t)(f.nh * f.chunks) * (uint32_t)(f.nhalf / 2) * 128u;
    uint32_t cols = 32;
    while ((int)cols < f.npad) cols <<= 1;
    f.tmem_cols = cols;
    const size_t ring = align_up((size_t)g.C * g.kH * (f.ring_w + 5 * 32) * 4, 16);
    const size_t fixed = 1024 + align_up(f.b_bytes, 1024) + ring + 512;
    f.sa = (int)std::min<int64_t>(4, ((int64_t)kSmemLimitF - (int64_t)fixed) / f.stage_a);
    f.smem = fixed + (size_t)f.sa * f.stage_a;
    f.wt_bytes = align_up((size_t)f.npad * f.Kp * 4, 256);
    f.gyh_bytes = align_up((size_t)(g.M * f.Kp) * 4, 256);
    f.slab_bytes = align_up((size_t)f.bands * g.C * (kBand + g.kH - 1) * g.W * 4, 256);
    return f;
}

// Opt-in (PT_B200_FDGRAD=1): correct, but the fold epilogue does not yet keep up with the
// MMAs — convnet L1 dgrad 0.9-1.05 ms against 0.37 + 0.05 ms for the vertically expanded
// Hankel tconv + fold_cols (the MMA/TMA skeleton alone, fold skipped, is 0.21 ms; the
// per-group TMEM loads, shuffles and ring updates each measured cheap when removed alone).
bool fdgrad_env() {
    static const bool on = [] {
        const char* e = std::getenv("PT_B200_FDGRAD");
        return e ? std::atoi(e) != 0 : false;
    }();
    return on;
}

}  // namespace

bool fdgrad_ok(const Geo& g) {
    if (!fdgrad_env()) return false;
    if (!(g.C <= 4 && g.sH == 1 && g.sW == 1 && g.oW <= 128 && g.K <= 512 && g.kW <= 12)) return false;
    const FDPlan f = fdplan(g);
    if (f.npad > 512 || f.nhalf > 256 || f.sa < 2 || f.b_bytes > 160 * 1024) return false;
    if (g.pW + g.W > 128 + g.kW - 1) return false;  // every gx column is a ring or spill cell
    return g.N * g.oHW * f.Kp < (1ll << 31) && (int64_t)f.bands * g.C * (kBand + g.kH) * g.W < (1ll << 31);
}

size_t fdgrad_workspace(const Geo& g) {
    const FDPlan f = fdplan(g);
    return f.wt_bytes + f.gyh_bytes + f.slab_bytes;
}

void fdgrad(const Geo& g, const float* gy, const float* w, float* gx, void* ws, cudaStream_t st,
            const float* gyh_pre) {
    PTB_REQUIRE(fdgrad_ok(g), "fdgrad: unsupported geometry");
    const FDPlan f = fdplan(g);
    char* base = reinterpret_cast<char*>(ws);
    float* wt = reinterpret_cast<float*>(base);
    float* gyh = reinterpret_cast<float*>(base + f.wt_bytes);
    float* slab = reinterpret_cast<float*>(base + f.wt_bytes + f.gyh_bytes);
    if (gyh_pre && f.Kp != (g.K + 31) / 32 * 32) gyh_pre = nullptr;  // not the shared padding
    if (!gyh_pre) {
        ProfScope prof("layout", st, 0.0, 4.0 * (g.M * g.K + g.M * f.Kp));
        nchw_to_nhwc(gy, gyh, g.N, g.K, g.oHW, f.Kp, true, st);
    } else {
        gyh = const_cast<float*>(gyh_pre);
    }
    pack_fdgrad_w_kernel<<<(unsigned)std::min<int64_t>(ceil_div((int64_t)f.npad * f.Kp, 256), 4 * (int64_t)sm_count()),
                           256, 0, st>>>(w, wt, (int)g.K, (int)g.C, (int)g.kH, (int)g.kW, f.npad, f.Kp, f.nhalf,
                                         f.gpr, f.ngroups);
    after_launch("pack_fdgrad_w");
    FDParams p;
    memset(&p, 0, sizeof p);
    {
        const uint64_t dims[5] = {32, (uint64_t)g.oW, (uint64_t)g.oH, (uint64_t)g.N, (uint64_t)f.chunks};
        const uint64_t strides[4] = {(uint64_t)f.Kp * 4, (uint64_t)(g.oW * f.Kp * 4), (uint64_t)(g.oHW * f.Kp * 4),
                                     128};
        const uint32_t box[5] = {32, 128, 1, 1, 1};
        tmap_tiled(&p.tmap_gy, gyh, 5, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    }
    {
        const uint64_t dims[3] = {32, (uint64_t)f.npad, (uint64_t)f.chunks};
        const uint64_t strides[2] = {(uint64_t)f.Kp * 4, 128};
        const uint32_t box[3] = {32, (uint32_t)(f.nhalf / 2), 1};
        tmap_tiled(&p.tmap_w, wt, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    }
    p.N = (int)g.N;
    p.C = (int)g.C;
    p.H = (int)g.H;
    p.W = (int)g.W;
    p.oH = (int)g.oH;
    p.kH = (int)g.kH;
    p.kW = (int)g.kW;
    p.pH = (int)g.pH;
    p.pW = (int)g.pW;
    p.chunks = f.chunks;
    p.nh = f.nh;
    p.nhalf = f.nhalf;
    p.ntot = f.ntot;
    p.nbands = f.nbands;
    p.bands = f.bands;
    p.ring_w = f.ring_w;
    p.ngroups = f.ngroups;
    p.gpr = f.gpr;
    p.sa = f.sa;
    p.stage_a = f.stage_a;
    p.b_bytes = f.b_bytes;
    p.b_off = (uint32_t)align_up(f.b_bytes, 1024);
    p.tmem_cols = f.tmem_cols;
    p.slab = slab;
    once_per_device((const void*)umma_fdgrad_kernel, [&] {  // the smem limit is a per-device attribute
        PTB_CUDA(cudaFuncSetAttribute(umma_fdgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimitF));
    });
    const int units = (f.bands + 1) / 2;
    const int pairs = std::min(units, sm_count() / 2);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(kThreadsF);
    cfg.dynamicSmemBytes = f.smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    {
        ProfScope prof("umma_conv", st, 2.0 * g.M * g.K * g.CRS, 0.0);
        PTB_CUDA(cudaLaunchKernelEx(&cfg, umma_fdgrad_kernel, p));
        after_launch("umma_fdgrad");
    }
    {
        ProfScope prof("layout", st, 0.0, 4.0 * ((double)f.bands * g.C * (kBand + g.kH - 1) * g.W + g.N * g.C * g.HW));
        const int64_t total = g.N * g.C * g.HW;
        fdgrad_fixup_kernel<<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 16 * (int64_t)sm_count()), 256, 0,
                              st>>>(slab, gx, (int)g.N, (int)g.C, (int)g.H, (int)g.W, (int)g.kH, (int)g.pH, f.nbands);
        after_launch("fdgrad_fixup");
    }
}

}  // namespace ptb
