// umma_conv.cu — tcgen05 (kind::tf32) implicit-GEMM convolution for sm_100a.
//
// GEMM view (SPEC.md:389-397 without materialising the unfold):
//   D[m][n] = sum_kd A[m][kd] * B[n][kd]
//   m  = output pixel (n_img, i, j) flattened — 128 per tile (TMEM lanes)
//   n  = output channel — BN per tile (TMEM columns, fp32 accumulators)
//   kd = (r, s, c) — one filter tap x 32 channels per pipeline stage
// A is gathered by TMA in im2col mode straight from an NHWC copy of the
// activation (hardware zero-fill implements the padding), B is the packed
// weight matrix loaded by tiled TMA. Both land 128B-swizzled (K-major) in smem;
// one elected thread issues tcgen05.mma into a double-buffered TMEM accumulator,
// four epilogue warps drain it (tcgen05.ld), add the bias and write NCHW
// directly (a warp stores 32 consecutive pixels of one channel per instruction).
//
// Small-C layers (C % 32 != 0, e.g. C=3 first layers) use 16-byte channel boxes
// (C padded to 4) in the no-swizzle core-matrix layout: 8 (tap,chunk) slots of
// 128 px x 4 ch per stage, one MMA (K=8) spanning two slots.
//
// dgrad (stride 1) is the same kernel on gradOutput with the flipped, transposed
// filter and pad' = k-1-pad (SPEC.md:416-419 gradInput, col2im fused away).
//
// Warp roles (192 threads, 1 CTA/SM, persistent over tiles):
//   warp 0      TMA producer (1 elected lane)
//   warp 1      TMEM allocator + MMA issuer (1 lane)
//   warps 2..5  epilogue (warp w owns TMEM lanes 32*(w%4) .. +31)
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "kernels.cuh"
#include "umma.cuh"

namespace ptb {

namespace {

using namespace umma;

constexpr int kTileM = 128;
constexpr uint32_t kStageA = kTileM * 32 * 4;  // 16 KB: 128 px x 32 fp32
constexpr int kThreadsU = 192;
constexpr int kSmemLimit = 232448;  // 227 KB opt-in per block on sm_100

struct UConvParams {
    CUtensorMap tmap_a;
    CUtensorMap tmap_b;
    int M;             // GEMM rows = output pixels
    int oH, oW;        // output spatial dims of this conv
    int sH, sW, pH, pW;
    int kW;
    int slots;         // taps * chunks (real k-slots)
    int chunks;        // cin_p / cb
    int num_kb;        // pipeline k-blocks per tile
    int n_rows;        // real output channels
    int bn, n_tiles, m_tiles;
    int stages;
    uint32_t stage_b;  // bytes of one B stage (bn * 128)
    uint32_t tmem_cols;
    float* out;
    const float* bias;
    int64_t out_hw;
};

template <int CB>
__global__ void __launch_bounds__(kThreadsU, 1) umma_conv_kernel(const __grid_constant__ UConvParams p) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((((raw + 1023u) & ~1023u)) - raw);
    const int S = p.stages;
    uint8_t* sA = smem;
    uint8_t* sB = smem + (size_t)S * kStageA;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + (size_t)S * p.stage_b);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

    const uint32_t warp = warp_id(), lane = lane_id();
    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.tmap_a);
        tma_prefetch(&p.tmap_b);
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_holder, p.tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const int num_tiles = p.m_tiles * p.n_tiles;
    const int ohw = p.oH * p.oW;

    if (warp == 0) {
        if (lane == 0) {
            // ===== TMA producer =====
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                const int mt = tile / p.n_tiles, nt = tile - mt * p.n_tiles;
                const int m0 = mt * kTileM;
                const int n0 = m0 / ohw;
                const int rem = m0 - n0 * ohw;
                const int i0 = rem / p.oW, j0 = rem - i0 * p.oW;
                const int wc = j0 * p.sW - p.pW, hc = i0 * p.sH - p.pH;
                for (int kb = 0; kb < p.num_kb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* a = sA + (size_t)stage * kStageA;
                    uint8_t* b = sB + (size_t)stage * p.stage_b;
                    mbar_arrive_expect_tx(&full[stage], kStageA + p.stage_b);
                    if constexpr (CB == 32) {
                        const int tap = kb / p.chunks, cc = kb - tap * p.chunks;
                        const int r = tap / p.kW, s = tap - r * p.kW;
                        tma_load_im2col_4d(a, &p.tmap_a, &full[stage], cc * 32, wc, hc, n0,
                                           (uint16_t)s, (uint16_t)r);
                        tma_load_2d(b, &p.tmap_b, &full[stage], kb * 32, nt * p.bn);
                    } else {
#pragma unroll 1
                        for (int t = 0; t < 8; ++t) {
                            int slot = kb * 8 + t;
                            if (slot >= p.slots) slot = 0;  // B is zero there
                            const int tap = slot / p.chunks, cc = slot - tap * p.chunks;
                            const int r = tap / p.kW, s = tap - r * p.kW;
                            tma_load_im2col_4d(a + t * 2048, &p.tmap_a, &full[stage], cc * 4, wc, hc,
                                               n0, (uint16_t)s, (uint16_t)r);
                        }
                        tma_load_3d(b, &p.tmap_b, &full[stage], 0, nt * p.bn, kb * 8);
                    }
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ===== MMA issuer =====
            const uint32_t idesc = idesc_tf32(kTileM, p.bn, 0, 0);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
                const uint32_t acc = it & 1, acc_phase = (it >> 1) & 1;
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + acc * p.bn;
                for (int kb = 0; kb < p.num_kb; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a = smem_u32(sA + (size_t)stage * kStageA);
                    const uint32_t b = smem_u32(sB + (size_t)stage * p.stage_b);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        uint64_t ad, bd;
                        if constexpr (CB == 32) {
                            ad = smem_desc(a + k * 32, 16, 1024, kSwizzle128B);
                            bd = smem_desc(b + k * 32, 16, 1024, kSwizzle128B);
                        } else {
                            ad = smem_desc(a + k * 4096, 2048, 128, kSwizzleNone);
                            bd = smem_desc(b + k * 2 * p.bn * 16, p.bn * 16, 128, kSwizzleNone);
                        }
                        mma_tf32(d, ad, bd, idesc, (kb | k) != 0);
                    }
                    mma_commit(&empty[stage]);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                mma_commit(&tfull[acc]);
            }
        }
    } else {
        // ===== epilogue: TMEM -> registers -> (+bias) -> NCHW =====
        const uint32_t q = warp & 3;
        int it = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
            const uint32_t acc = it & 1;
            mbar_wait(&tfull[acc], (it >> 1) & 1);
            tc_fence_after();
            const int mt = tile / p.n_tiles, nt = tile - mt * p.n_tiles;
            const int m = mt * kTileM + (int)(q * 32 + lane);
            const bool valid = m < p.M;
            int64_t base = 0;
            if (valid) {
                const int64_t n = m / p.out_hw, pix = m - n * p.out_hw;
                base = n * (int64_t)p.n_rows * p.out_hw + pix;
            }
            const int ch0 = nt * p.bn;
            const uint32_t taddr = tmem_base + ((q * 32u) << 16) + acc * p.bn;
            for (int c0 = 0; c0 < p.bn; c0 += 16) {
                uint32_t v[16];
                tmem_ld_32x32b_x16(taddr + c0, v);
                tmem_ld_wait();
                if (valid) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int ch = ch0 + c0 + j;
                        if (ch < p.n_rows) {
                            float val = __uint_as_float(v[j]);
                            if (p.bias) val += __ldg(p.bias + ch);
                            p.out[base + (int64_t)ch * p.out_hw] = val;
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem_base, p.tmem_cols);
#endif
}

// ---- host: TMA descriptor encoding through the driver entry points ----
PFN_cuTensorMapEncodeTiled_v12000 g_encode_tiled = nullptr;
PFN_cuTensorMapEncodeIm2col_v12000 g_encode_im2col = nullptr;
int g_driver_version = 0;

void load_driver_entry_points() {
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q1, q2;
        void* f1 = nullptr;
        void* f2 = nullptr;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f1, 12000, cudaEnableDefault,
                                             &q1) != cudaSuccess ||
            q1 != cudaDriverEntryPointSuccess ||
            cudaGetDriverEntryPointByVersion("cuTensorMapEncodeIm2col", &f2, 12000,
                                             cudaEnableDefault, &q2) != cudaSuccess ||
            q2 != cudaDriverEntryPointSuccess) {
            err = "cuTensorMapEncode* driver entry points unavailable";
            return;
        }
        g_encode_tiled = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f1);
        g_encode_im2col = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(f2);
        cudaDriverGetVersion(&g_driver_version);
    });
    if (!g_encode_tiled || !g_encode_im2col) fail_backend(err);
}

// Driver releases <= 13.1 mis-handle a descriptor flag for tensors under 128 KiB
// (the same workaround CUTLASS applies in copy_traits_sm90_im2col.hpp).
void small_tensor_fixup(CUtensorMap* m, size_t bytes) {
    if (g_driver_version <= 13010 && bytes < 131072)
        reinterpret_cast<uint64_t*>(m)[1] &= ~(1ull << 21);
}

void encode_im2col(CUtensorMap* m, const float* act, int64_t N, int64_t H, int64_t W, int64_t Cp,
                   int kH, int kW, int pH, int pW, int sH, int sW, int cb) {
    cuuint64_t dims[4] = {(cuuint64_t)Cp, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)(Cp * 4), (cuuint64_t)(W * Cp * 4),
                             (cuuint64_t)(H * W * Cp * 4)};
    int lower[2] = {-pW, -pH};
    int upper[2] = {pW - (kW - 1), pH - (kH - 1)};
    cuuint32_t estr[4] = {1, (cuuint32_t)sW, (cuuint32_t)sH, 1};
    CUresult r = g_encode_im2col(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(act), dims,
                                 strides, lower, upper, (cuuint32_t)cb, kTileM, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 cb == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail_backend("cuTensorMapEncodeIm2col failed (" + std::to_string((int)r) + ")");
    small_tensor_fixup(m, (size_t)(N * H * W * Cp * 4));
}

void encode_weights(CUtensorMap* m, const float* wt, const UmmaPlan& pl) {
    CUresult r;
    if (pl.cb == 32) {
        const int64_t kdim = pl.taps * pl.cin_p;
        cuuint64_t dims[2] = {(cuuint64_t)kdim, (cuuint64_t)pl.n_pad};
        cuuint64_t strides[1] = {(cuuint64_t)(kdim * 4)};
        cuuint32_t box[2] = {32, (cuuint32_t)pl.bn};
        cuuint32_t estr[2] = {1, 1};
        r = g_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(wt), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        cuuint64_t dims[3] = {4, (cuuint64_t)pl.n_pad, (cuuint64_t)pl.slots_p};
        cuuint64_t strides[2] = {16, (cuuint64_t)(pl.n_pad * 16)};
        cuuint32_t box[3] = {4, (cuuint32_t)pl.bn, 8};
        cuuint32_t estr[3] = {1, 1, 1};
        r = g_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(wt), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) fail_backend("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    small_tensor_fixup(m, (size_t)pl.wt_elems * 4);
}

int stages_for(int bn) {
    const int per = (int)kStageA + bn * 128;
    int s = (kSmemLimit - 1024 - 256) / per;
    return s > 8 ? 8 : s;
}

uint32_t tmem_cols_for(int bn) {
    const int need = 2 * bn;
    uint32_t c = 32;
    while ((int)c < need) c <<= 1;
    return c;
}

void launch(const UConvParams& p, int cb, cudaStream_t st) {
    const size_t smem = 1024 + (size_t)p.stages * (kStageA + p.stage_b) + (2 * p.stages + 4) * 8 + 16;
    const int num_tiles = p.m_tiles * p.n_tiles;
    const int grid = num_tiles < sm_count() ? num_tiles : sm_count();
    if (cb == 32) {
        static bool attr = false;
        if (!attr) {
            PTB_CUDA(cudaFuncSetAttribute(umma_conv_kernel<32>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit));
            attr = true;
        }
        umma_conv_kernel<32><<<grid, kThreadsU, smem, st>>>(p);
    } else {
        static bool attr = false;
        if (!attr) {
            PTB_CUDA(cudaFuncSetAttribute(umma_conv_kernel<4>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit));
            attr = true;
        }
        umma_conv_kernel<4><<<grid, kThreadsU, smem, st>>>(p);
    }
    after_launch("umma_conv");
}

// Shared body of fprop / dgrad: act is NHWC [N][aH][aW][cin_p] in the workspace.
void run_umma(const UmmaPlan& pl, const float* act, const float* wt, int64_t N, int64_t aH,
              int64_t aW, int kH, int kW, int pH, int pW, int sH, int sW, int64_t oH, int64_t oW,
              float* out, const float* bias, double alg_flops, cudaStream_t st) {
    load_driver_entry_points();
    UConvParams p;
    memset(&p, 0, sizeof p);
    encode_im2col(&p.tmap_a, act, N, aH, aW, pl.cin_p, kH, kW, pH, pW, sH, sW, pl.cb);
    encode_weights(&p.tmap_b, wt, pl);
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
    p.num_kb = pl.cb == 32 ? p.slots : (int)(pl.slots_p / 8);
    p.n_rows = (int)pl.n_rows;
    p.bn = pl.bn;
    p.n_tiles = pl.n_tiles;
    p.m_tiles = (int)ceil_div(M, kTileM);
    p.stages = stages_for(pl.bn);
    p.stage_b = (uint32_t)pl.bn * 128u;
    p.tmem_cols = tmem_cols_for(pl.bn);
    p.out = out;
    p.bias = bias;
    p.out_hw = oH * oW;
    ProfScope prof("umma_conv", st, alg_flops, 0.0);
    launch(p, pl.cb, st);
}

}  // namespace

UmmaPlan umma_plan(const Geo& g, bool dgrad) {
    UmmaPlan pl;
    const int64_t cin = dgrad ? g.K : g.C;
    pl.n_rows = dgrad ? g.C : g.K;
    pl.taps = g.kH * g.kW;
    if (dgrad) {
        // transposed conv as a stride-1 conv on gy: needs stride 1 and pad <= k-1
        if (g.sH != 1 || g.sW != 1 || g.pH > g.kH - 1 || g.pW > g.kW - 1) return pl;
    }
    // TMA im2col limits (rank-4 corners in [-128,127], filter offsets in [0,255]).
    const int64_t pad_h = dgrad ? g.kH - 1 - g.pH : g.pH, pad_w = dgrad ? g.kW - 1 - g.pW : g.pW;
    if (pad_h > 128 || pad_w > 128 || g.kH > 256 || g.kW > 256) return pl;
    if (pad_h - (g.kH - 1) < -128 || pad_w - (g.kW - 1) < -128) return pl;
    if ((!dgrad && (g.sH > 8 || g.sW > 8))) return pl;
    if (pl.n_rows > 65536) return pl;
    const int64_t c32 = (cin + 31) / 32 * 32;
    if (cin % 32 == 0 || c32 * 3 <= cin * 4) {
        pl.cb = 32;
        pl.cin_p = c32;
    } else {
        pl.cb = 4;
        pl.cin_p = (cin + 3) / 4 * 4;
    }
    const int64_t nt = (pl.n_rows + 255) / 256;
    pl.bn = (int)(((pl.n_rows + nt - 1) / nt + 15) / 16 * 16);
    pl.n_tiles = (int)ceil_div(pl.n_rows, pl.bn);
    pl.n_pad = (int64_t)pl.n_tiles * pl.bn;
    pl.slots_p = ceil_div(pl.taps * (pl.cin_p / 4), 8) * 8;
    const int64_t aHW = dgrad ? g.oHW : g.HW;
    pl.act_elems = g.N * aHW * pl.cin_p;
    pl.wt_elems = pl.cb == 32 ? pl.n_pad * pl.taps * pl.cin_p : pl.slots_p * pl.n_pad * 4;
    if (pl.taps * pl.cin_p > (1ll << 31) / 4) return pl;
    pl.ws_bytes = align_up(pl.act_elems * 4, 256) + align_up(pl.wt_elems * 4, 256);
    pl.ok = true;
    return pl;
}

void umma_conv_fwd(const Geo& g, const UmmaPlan& pl, const float* x, const float* w,
                   const float* b, float* y, void* ws, cudaStream_t st) {
    float* act = reinterpret_cast<float*>(ws);
    float* wt = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + align_up(pl.act_elems * 4, 256));
    {
        ProfScope prof("layout", st, 0.0, 4.0 * (g.N * g.C * g.HW + g.N * g.HW * pl.cin_p));
        nchw_to_nhwc(x, act, g.N, g.C, g.HW, pl.cin_p, true, st);
    }
    pack_weights(w, wt, g.K, g.C, g.kH, g.kW, false, pl.cb, pl.n_pad, pl.cin_p, pl.slots_p, true, st);
    run_umma(pl, act, wt, g.N, g.H, g.W, (int)g.kH, (int)g.kW, (int)g.pH, (int)g.pW, (int)g.sH,
             (int)g.sW, g.oH, g.oW, y, b, 2.0 * g.M * g.K * g.CRS, st);
}

void umma_conv_bwd_data(const Geo& g, const UmmaPlan& pl, const float* gy, const float* w,
                        float* gx, void* ws, cudaStream_t st) {
    float* act = reinterpret_cast<float*>(ws);
    float* wt = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + align_up(pl.act_elems * 4, 256));
    {
        ProfScope prof("layout", st, 0.0, 4.0 * (g.N * g.K * g.oHW + g.N * g.oHW * pl.cin_p));
        nchw_to_nhwc(gy, act, g.N, g.K, g.oHW, pl.cin_p, true, st);
    }
    pack_weights(w, wt, g.K, g.C, g.kH, g.kW, true, pl.cb, pl.n_pad, pl.cin_p, pl.slots_p, true, st);
    run_umma(pl, act, wt, g.N, g.oH, g.oW, (int)g.kH, (int)g.kW, (int)(g.kH - 1 - g.pH),
             (int)(g.kW - 1 - g.pW), 1, 1, g.H, g.W, gx, nullptr, 2.0 * g.M * g.K * g.CRS, st);
}

}  // namespace ptb
