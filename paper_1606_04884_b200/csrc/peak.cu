// peak.cu — measured TF32 tensor-pipe ceiling of this GPU at its current clocks, for the
// roofline denominator (bench.py). One CTA pair per SM pair issues back-to-back
// kind::tf32 M=256 N=256 K=8 MMAs from shared memory (no global traffic, converged-warp
// issue with constant descriptors), which is the rate a perfectly fed conv kernel could
// reach. MEASURED_PEAKS.json carries only bf16 (cuBLAS); bf16/2 under-states TF32 here
// (tests/mma_bench.cu: 4096 TF32 flop/clk/SM at N=256).
#include "common.cuh"
#include "umma.cuh"

namespace ptb {

namespace {

using namespace umma;

constexpr int kPeakIters = 16384;  // MMAs per CTA pair (multiple of 8)

__global__ void __launch_bounds__(128, 1) tf32_peak_kernel(int iters) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((((raw + 1023u) & ~1023u)) - raw);
    __shared__ uint64_t bar;
    __shared__ uint32_t holder;
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
    const uint32_t warp = warp_id_uniform();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc_cg2(&holder, 256);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = holder;
    if (warp == 0 && cluster_rank() == 0) {
        const uint32_t idesc = idesc_tf32(256, 256, 0, 0);
        constexpr uint32_t kHi = desc_hi(1024, kSwizzle128B);
        const uint32_t alo = desc_lo(smem_u32(smem), 16), blo = desc_lo(smem_u32(smem + 32768), 16);
        for (int i = 0; i < iters; i += 8) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                mma_tf32_cg2_warp(tmem, desc_make(alo + (k & 3) * 2, kHi), desc_make(blo + (k & 3) * 2, kHi),
                                  idesc, 1);
        }
        mma_commit_cg2_warp(&bar);
        mbar_wait(&bar, 0);
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (warp == 0) tmem_dealloc_cg2(tmem, 256);
#endif
}

}  // namespace

}  // namespace ptb

using namespace ptb;

extern "C" double pt_b200_tf32_mma_peak(void) {
    try {
        const int sms = sm_count();
        const size_t smem = 64 * 1024 + 1024;
        PTB_CUDA(cudaFuncSetAttribute(tf32_peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(sms / 2 * 2);
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaEvent_t e0, e1;
        PTB_CUDA(cudaEventCreate(&e0));
        PTB_CUDA(cudaEventCreate(&e1));
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
            PTB_CUDA(cudaEventRecord(e0, cfg.stream));
            PTB_CUDA(cudaLaunchKernelEx(&cfg, tf32_peak_kernel, kPeakIters));
            PTB_CUDA(cudaEventRecord(e1, cfg.stream));
            PTB_CUDA(cudaEventSynchronize(e1));
            float ms = 0.f;
            PTB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            if (rep > 0 && ms < best) best = ms;  // rep 0 warms up
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        const double flops = 2.0 * 256 * 256 * 8 * (double)kPeakIters * (sms / 2);
        return flops / (best * 1e-3) / 1e12;
    } catch (const std::exception&) {
        return -1.0;
    }
}
