// umma_gemm.cu — batched tcgen05 (kind::tf32) GEMM for sm_100a:
//
//   D[b][n][m] = alpha * sum_k A[b][m][k] * B[b][n][k]  (+ beta * D[b][n][m])
//
// the contraction under the SPEC gemm (clBLAS SGEMM in cltorch)
// in TF32 mode and under the Winograd entry's 16 transform-domain GEMMs (winograd.cu).
// Either operand may be K-major (k contiguous: 128B-swizzled boxes of 32 k x rows) or
// MN-major (m / n contiguous: 32-element atoms, 128B swizzle with 32-byte atoms), chosen
// at compile time; TMA zero-fills every out-of-range row / column / k, so any M, N, K work.
//
// CTA pair (cta_group::2), persistent over (batch, m-tile, n-tile): M = 256 rows per pair
// (128 per CTA = TMEM lanes), N = bn <= 256 columns (each CTA loads bn/2 rows of B),
// 32-deep K per pipeline stage, 4 MMAs (K = 8) per stage, a double-buffered TMEM
// accumulator drained by four epilogue warps. D is written "n-major": for a fixed column n
// a warp stores 32 consecutive m — coalesced — which is row-major C for the SPEC gemm (m
// = C's column) and the [component][channel][tile] layout the Winograd output transform
// reads.
//
// Warp roles (192 threads, 1 CTA/SM): warp 0 TMA producer, warp 1 TMEM allocator + MMA
// issuer (pair leader), warps 2..5 epilogue (warp w drains TMEM lanes 32*(w%4)..+31).
#include <cuda.h>

#include "kernels.cuh"
#include "tmap.cuh"
#include "umma.cuh"

namespace ptb {

namespace {

using namespace umma;

constexpr int kThreadsG = 192;
constexpr int kSmemLimitG = 232448;
constexpr uint32_t kStageA = 128 * 32 * 4;  // 128 rows x 32 k x fp32 per CTA
constexpr uint32_t kAtom = 32 * 32 * 4;     // MN-major box: 32 rows x 32 k

struct GemmParams {
    CUtensorMap tmap_a;  // K-major: {K, M, batch} box {32, 128, 1}; MN-major: {M, K, batch} box {32, 32, 1}
    CUtensorMap tmap_b;  // K-major: {K, N, batch} box {32, bn/2, 1}; MN-major: {N, K, batch} box {32, 32, 1}
    int M, N, batch;
    int bn, m_tiles, n_tiles, num_kb, stages;
    uint32_t stage_b, tmem_cols;
    float* d;
    int64_t ldd, batch_d;
    float alpha, beta;
};

template <int AMN, int BMN>
__global__ void __launch_bounds__(kThreadsG, 1) umma_gemm_kernel(const __grid_constant__ GemmParams p) {
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

    const uint32_t warp = warp_id_uniform(), lane = lane_id();
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.tmap_a);
        tma_prefetch(&p.tmap_b);
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
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
    const int per_batch = p.m_tiles * p.n_tiles;
    const int num_tiles = p.batch * per_batch;
    const int cid = blockIdx.x / 2, ncl = gridDim.x / 2;
    const int half_bn = p.bn / 2;

    if (warp == 0) {
        if (lane == 0) {
            // ===== TMA producer (both CTAs: own 128 rows of A, own bn/2 rows of B) =====
            int stage = 0;
            uint32_t phase = 0;
            const uint32_t tx = 2 * (kStageA + p.stage_b);
            for (int tile = cid; tile < num_tiles; tile += ncl) {
                const int b = tile / per_batch, r = tile - b * per_batch;
                const int mt = r / p.n_tiles, nt = r - mt * p.n_tiles;
                const int m0 = mt * 256 + (int)rank * 128;
                const int n0 = nt * p.bn + (int)rank * half_bn;
                for (int kb = 0; kb < p.num_kb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* a = sA + (size_t)stage * kStageA;
                    uint8_t* bb = sB + (size_t)stage * p.stage_b;
                    if (leader) mbar_arrive_expect_tx(&full[stage], tx);
                    if constexpr (AMN) {
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            tma_load_3d_cg2(a + i * kAtom, &p.tmap_a, &full[stage], m0 + 32 * i, kb * 32, b);
                    } else {
                        tma_load_3d_cg2(a, &p.tmap_a, &full[stage], kb * 32, m0, b);
                    }
                    if constexpr (BMN) {
                        for (int i = 0; i < half_bn / 32; ++i)
                            tma_load_3d_cg2(bb + i * kAtom, &p.tmap_b, &full[stage], n0 + 32 * i, kb * 32, b);
                    } else {
                        tma_load_3d_cg2(bb, &p.tmap_b, &full[stage], kb * 32, n0, b);
                    }
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {  // whole warp converged; one elected lane issues
            // ===== MMA issuer =====
            const uint32_t idesc = idesc_tf32(256, p.bn, AMN, BMN);
            constexpr uint32_t kHiK = desc_hi(1024, kSwizzle128B);        // K-major SW128
            constexpr uint32_t kHiMN = desc_hi(512, kSwizzle128B_Base32B);  // MN-major, 32B atoms
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int tile = cid; tile < num_tiles; tile += ncl, ++it) {
                const uint32_t acc = it & 1;
                mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + acc * p.bn;
                for (int kb = 0; kb < p.num_kb; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a = smem_u32(sA + (size_t)stage * kStageA);
                    const uint32_t b = smem_u32(sB + (size_t)stage * p.stage_b);
                    // K-major: +32 B per K=8 slab; MN-major: +1 KB (8 k-rows of 128 B),
                    // 32-row atoms one box (LBO) apart
                    const uint32_t alo = AMN ? desc_lo(a, kAtom) : desc_lo(a, 16);
                    const uint32_t blo = BMN ? desc_lo(b, kAtom) : desc_lo(b, 16);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint64_t ad = desc_make(alo + (AMN ? 64u * k : 2u * k), AMN ? kHiMN : kHiK);
                        const uint64_t bd = desc_make(blo + (BMN ? 64u * k : 2u * k), BMN ? kHiMN : kHiK);
                        mma_tf32_cg2_warp(d, ad, bd, idesc, (kb | k) ? 1u : 0u);
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
    } else {
        // ===== epilogue: TMEM -> registers -> alpha/beta -> D[b][n][m] =====
        const uint32_t q = warp & 3;
        int it = 0;
        for (int tile = cid; tile < num_tiles; tile += ncl, ++it) {
            const uint32_t acc = it & 1;
            mbar_wait(&tfull[acc], (it >> 1) & 1);
            tc_fence_after();
            const int b = tile / per_batch, r = tile - b * per_batch;
            const int mt = r / p.n_tiles, nt = r - mt * p.n_tiles;
            const int m = mt * 256 + (int)rank * 128 + (int)(q * 32 + lane);
            const bool valid = m < p.M;
            const int n0 = nt * p.bn;
            float* dst = p.d + (int64_t)b * p.batch_d + (valid ? m : 0);
            const uint32_t taddr = tmem_base + ((q * 32u) << 16) + acc * p.bn;
            for (int c0 = 0; c0 < p.bn; c0 += 16) {
                uint32_t v[16];
                tmem_ld_32x32b_x16(taddr + c0, v);
                tmem_ld_wait();
                if (valid) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int n = n0 + c0 + j;
                        if (n < p.N) {
                            float* o = dst + (int64_t)n * p.ldd;
                            float val = p.alpha * __uint_as_float(v[j]);
                            if (p.beta != 0.f) val = fmaf(p.beta, *o, val);
                            *o = val;
                        }
                    }
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

template <int AMN, int BMN>
void launch_gemm(const GemmParams& p, int grid, size_t smem, cudaStream_t st) {
    once_per_device((const void*)umma_gemm_kernel<AMN, BMN>, [&] {  // per-device attribute
        PTB_CUDA(cudaFuncSetAttribute(umma_gemm_kernel<AMN, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kSmemLimitG));
    });
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreadsG);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    PTB_CUDA(cudaLaunchKernelEx(&cfg, umma_gemm_kernel<AMN, BMN>, p));
}

// TMA strides must be non-zero multiples of 16 bytes: a single matrix (batch 1, or a
// broadcast operand with batch stride 0 over batch 1) gets its own extent as the stride.
uint64_t batch_bytes(int64_t batch, int64_t batch_stride, int64_t extent) {
    const int64_t s = (batch > 1 && batch_stride > 0) ? batch_stride : extent;
    return (uint64_t)((s * 4 + 15) / 16 * 16);
}

void encode_operand(CUtensorMap* m, const float* base, bool mn_major, int64_t rows, int64_t K,
                    int64_t ld, int64_t batch, int64_t batch_stride, int box_rows) {
    if (mn_major) {  // element (row, k) at k*ld + row
        const uint64_t dims[3] = {(uint64_t)rows, (uint64_t)K, (uint64_t)batch};
        const uint64_t strides[2] = {(uint64_t)ld * 4, batch_bytes(batch, batch_stride, ld * K)};
        const uint32_t box[3] = {32, 32, 1};
        tmap_tiled(m, base, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    } else {         // element (row, k) at row*ld + k
        const uint64_t dims[3] = {(uint64_t)K, (uint64_t)rows, (uint64_t)batch};
        const uint64_t strides[2] = {(uint64_t)ld * 4, batch_bytes(batch, batch_stride, ld * rows)};
        const uint32_t box[3] = {32, (uint32_t)box_rows, 1};
        tmap_tiled(m, base, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    }
}

bool tma_addressable(const void* p, int64_t ld, int64_t batch_stride) {
    return (reinterpret_cast<uintptr_t>(p) & 15) == 0 && ld % 4 == 0 && ld >= 4 &&
           batch_stride % 4 == 0;
}

}  // namespace

bool umma_gemm_supported(const UmmaGemm& g) {
    return tma_addressable(g.a, g.lda, g.batch_a) && tma_addressable(g.b, g.ldb, g.batch_b) &&
           g.M >= 1 && g.N >= 1 && g.K >= 1 && g.batch >= 1 &&
           (g.batch == 1 || (g.batch_a > 0 && g.batch_b > 0)) && g.M < (1ll << 31) &&
           g.N < (1ll << 31) && g.K < (1ll << 31);
}

void umma_gemm(const UmmaGemm& g, cudaStream_t st) {
    PTB_REQUIRE(umma_gemm_supported(g),
                "gemm (TF32 tensor cores): operands must be 16-byte aligned with leading dimensions "
                "and batch strides that are multiples of 4 floats");
    GemmParams p;
    memset(&p, 0, sizeof p);
    p.bn = g.N > 128 ? 256 : (g.N > 64 ? 128 : 64);
    encode_operand(&p.tmap_a, g.a, g.a_mn, g.M, g.K, g.lda, g.batch, g.batch_a, 128);
    encode_operand(&p.tmap_b, g.b, g.b_mn, g.N, g.K, g.ldb, g.batch, g.batch_b, p.bn / 2);
    p.M = (int)g.M;
    p.N = (int)g.N;
    p.batch = (int)g.batch;
    p.m_tiles = (int)ceil_div(g.M, 256);
    p.n_tiles = (int)ceil_div(g.N, p.bn);
    p.num_kb = (int)ceil_div(g.K, 32);
    p.stage_b = (uint32_t)(p.bn / 2) * 128u;
    const int s = (kSmemLimitG - 1024 - 256) / (int)(kStageA + p.stage_b);
    p.stages = s > 8 ? 8 : s;
    p.tmem_cols = 2 * p.bn < 32 ? 32 : 2 * p.bn;
    p.d = g.d;
    p.ldd = g.ldd;
    p.batch_d = g.batch_d;
    p.alpha = g.alpha;
    p.beta = g.beta;
    const size_t smem = 1024 + (size_t)p.stages * (kStageA + p.stage_b) + (2 * p.stages + 4) * 8 + 16;
    const int64_t tiles = (int64_t)p.batch * p.m_tiles * p.n_tiles;
    const int clusters = (int)std::min<int64_t>(tiles, sm_count() / 2);
    ProfScope prof("umma_conv", st, 2.0 * g.M * g.N * g.K * g.batch, 0.0);
    if (g.a_mn && g.b_mn) launch_gemm<1, 1>(p, 2 * clusters, smem, st);
    else if (g.a_mn) launch_gemm<1, 0>(p, 2 * clusters, smem, st);
    else if (g.b_mn) launch_gemm<0, 1>(p, 2 * clusters, smem, st);
    else launch_gemm<0, 0>(p, 2 * clusters, smem, st);
    after_launch("umma_gemm");
}

}  // namespace ptb
