// mma_bench.cu — microbenchmark of tcgen05.mma kind::tf32 issue throughput on B200
// (not product code): one persistent CTA (or CTA pair) per SM issues back-to-back
// MMAs from shared memory into TMEM, committing to an mbarrier every `per_commit`
// MMAs, and optionally waiting on that barrier (a consumer-release round trip).
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -Iinclude -o tests/mma_bench tests/mma_bench.cu
//   tests/mma_bench <N> <cg 1|2> <per_commit> <shift 0|1> [iters]
#include <cstdio>
#include <cstdlib>

#include "../paper_1606_04884_b200/csrc/umma.cuh"

using namespace ptb::umma;

struct P {
    int n, cg, per_commit, shift, iters;
};

template <int CG>
__global__ void __launch_bounds__(128, 1) bench(P p, unsigned long long* cyc) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((((raw + 1023u) & ~1023u)) - raw);
    uint8_t* sA = smem;                 // 64 KB
    uint8_t* sB = smem + 65536;         // 64 KB
    __shared__ uint64_t bar, dummy;
    __shared__ uint32_t holder;
    const uint32_t rank = CG == 2 ? cluster_rank() : 0;
    for (int i = threadIdx.x; i < 32768; i += blockDim.x)
        reinterpret_cast<float*>(smem)[i] = p.shift == 3 ? 0.f : (float)((i * 2654435761u) >> 20) * 1e-3f - 2.f;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&dummy, 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) {
        if (CG == 2) tmem_alloc_cg2(&holder, 512);
        else tmem_alloc(&holder, 512);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    if (CG == 2) cluster_sync();
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = holder;
    if (threadIdx.x == 0 && rank == 0) {
        const uint32_t idesc = idesc_tf32(128 * p.cg, p.n, 0, 0);
        const uint32_t a = smem_u32(sA), b = smem_u32(sB);
        uint32_t phase = 0;
        const unsigned long long t0 = clock64();
        if (p.shift == 4) {
            // the im2col kernel's stage pattern: 8 MMAs over two 16 KB boxes, commit per stage
            for (int i = 0; i < p.iters; i += 8) {
                const uint32_t st = (uint32_t)((i >> 3) & 1) * 32768u;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t ao = st + (k >> 2) * 16384u + (k & 3) * 32u;
                    const uint32_t bo = st / 2 + (k >> 2) * 8192u + (k & 3) * 32u;
                    if (CG == 2) mma_tf32_cg2(tmem, smem_desc(a + ao, 16, 1024, kSwizzle128B),
                                             smem_desc(b + bo, 16, 1024, kSwizzle128B), idesc, 1);
                    else mma_tf32(tmem, smem_desc(a + ao, 16, 1024, kSwizzle128B),
                                  smem_desc(b + bo, 16, 1024, kSwizzle128B), idesc, 1);
                }
                if (CG == 2) mma_commit_cg2(&dummy);
                else mma_commit(&dummy);
            }
        }
        if (p.shift == 5 || p.shift == 6) {
            // rowconv pattern: A no-swizzle Hankel (LBO 16, SBO 128, K=8 per MMA = two 16-B
            // taps, start +32 B per MMA); B no-swizzle [N/2][4] blocks (LBO = N/2*16).
            // shift 6: the same with non-overlapping A (LBO 2048 = standard core-matrix layout)
            const uint32_t lbo_b = (uint32_t)(p.n / CG) * 16u;
            constexpr uint32_t kHi = desc_hi(128, kSwizzleNone);
            const uint32_t alo = desc_lo(a, p.shift == 5 ? 16 : 2048), blo = desc_lo(b, lbo_b);
            for (int i = 0; i < p.iters; i += 6) {
#pragma unroll
                for (int k = 0; k < 6; ++k) {
                    const uint32_t ao = p.shift == 5 ? 2u * k : 256u * k;
                    if (CG == 2) mma_tf32_cg2(tmem, desc_make(alo + ao, kHi), desc_make(blo + k * ((2 * lbo_b) >> 4), kHi), idesc, 1);
                    else mma_tf32(tmem, desc_make(alo + ao, kHi), desc_make(blo + k * ((2 * lbo_b) >> 4), kHi), idesc, 1);
                }
                if (CG == 2) mma_commit_cg2(&dummy);
                else mma_commit(&dummy);
            }
        }
        if (p.shift >= 7 && p.shift <= 9) {
            // MN-major tf32 (SW128 with 32-byte atoms; the wgrad operands): K step = 8 pixel
            // rows = 1 KB. shift 7: A atoms 16 KB apart (one box per 32 channels); shift 8: A
            // atoms 128 B apart (Hankel taps, overlapping); shift 9: A MN-major, B K-major SW128
            const uint32_t idesc2 = idesc_tf32(128 * p.cg, p.n, 1, p.shift == 9 ? 0 : 1);
            constexpr uint32_t kHiM = desc_hi(512, kSwizzle128B_Base32B), kHiK = desc_hi(1024, kSwizzle128B);
            const uint32_t alo = desc_lo(a, p.shift == 8 ? 128 : 16384), blo = desc_lo(b, p.shift == 9 ? 16 : 16384);
            for (int i = 0; i < p.iters; i += 8) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint64_t ad = desc_make(alo + (uint32_t)k * 64u, kHiM);
                    const uint64_t bd = p.shift == 9 ? desc_make(blo + (uint32_t)(k & 3) * 2u, kHiK)
                                                     : desc_make(blo + (uint32_t)k * 64u, kHiM);
                    if (CG == 2) mma_tf32_cg2(tmem, ad, bd, idesc2, 1);
                    else mma_tf32(tmem, ad, bd, idesc2, 1);
                }
                if (CG == 2) mma_commit_cg2(&dummy);
                else mma_commit(&dummy);
            }
        }
        for (int i = 0; i < (p.shift >= 4 ? 0 : p.iters); ++i) {
            // shift 1: Hankel-style row shifts; shift 2: walk 4 distinct 16 KB A stages
            const uint32_t sh = p.shift == 1 ? (uint32_t)(i % 9) * 128u
                                : p.shift == 2 ? (uint32_t)((i >> 2) & 3) * 16384u : 0u;
            const uint64_t ad = smem_desc(a + sh + (i & 3) * 32u, 16, 1024, kSwizzle128B);
            const uint64_t bd = smem_desc(b + (p.shift == 2 ? sh / 2 : 0u) + (i & 3) * 32u, 16, 1024, kSwizzle128B);
            if (CG == 2) mma_tf32_cg2(tmem, ad, bd, idesc, 1);
            else mma_tf32(tmem, ad, bd, idesc, 1);
            if ((i + 1) % p.per_commit == 0) {
                if (CG == 2) mma_commit_cg2(&dummy);
                else mma_commit(&dummy);
            }
        }
        if (CG == 2) mma_commit_cg2(&bar);
        else mma_commit(&bar);
        mbar_wait(&bar, phase);
        const unsigned long long t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    if (CG == 2) cluster_sync();
    else __syncthreads();
    tc_fence_after();
    if (threadIdx.x < 32) {
        if (CG == 2) tmem_dealloc_cg2(tmem, 512);
        else tmem_dealloc(tmem, 512);
    }
}

int main(int argc, char** argv) {
    P p{argc > 1 ? atoi(argv[1]) : 128, argc > 2 ? atoi(argv[2]) : 2, argc > 3 ? atoi(argv[3]) : 4,
        argc > 4 ? atoi(argv[4]) : 0, argc > 5 ? atoi(argv[5]) : 20000};
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* d;
    cudaMalloc(&d, sizeof(unsigned long long) * sms);
    cudaMemset(d, 0, sizeof(unsigned long long) * sms);
    const size_t smem = 132 * 1024 + 1024;
    cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(bench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms / p.cg * p.cg);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = p.cg;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = p.cg == 2 ? 1 : 0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        cudaError_t err = p.cg == 2 ? cudaLaunchKernelEx(&cfg, bench<2>, p, d)
                                    : cudaLaunchKernelEx(&cfg, bench<1>, p, d);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
            printf("launch failed: %s\n", cudaGetErrorString(err));
            return 1;
        }
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[256];
    cudaMemcpy(h, d, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
    const double flops = 2.0 * 128 * p.cg * p.n * 8 * (double)p.iters * (sms / p.cg);
    printf("N=%d cg=%d per_commit=%d shift=%d: %.1f cycles/MMA (leader 0), %.1f TFLOP/s\n", p.n, p.cg,
           p.per_commit, p.shift, (double)h[0] / p.iters, flops / (ms * 1e-3) / 1e12);
    return 0;
}
