// split3.cu — operand splitting for the 3xTF32 math mode (PT_MATH_3XTF32).
//
// v = hi + lo with hi = tf32_rna(v) and lo = tf32_rna(v - hi); a product a*b is then
// a_hi*b_hi + a_lo*b_hi + a_hi*b_lo up to the dropped a_lo*b_lo (|.| <= 2^-22 |a*b|) and the
// rounding of lo (<= 2^-23 |v|), i.e. FP32-level accuracy from TF32 tensor-core MMAs.
// Instead of three MMA streams inside every engine, the three products become one TF32
// convolution over a 3x larger reduction, so every tensor-core engine serves unchanged:
//   forward / gradInput: concatenate along the reduced channel axis
//     x3 = [x_hi | x_lo | x_hi],  w3 = [w_hi | w_hi | w_lo]   (C' = 3C for fwd, K' = 3K for dgrad)
//   gradWeight: concatenate along the batch (the reduction over pixels and images)
//     x3 = [x_hi ; x_hi ; x_lo], gy3 = [gy_hi ; gy_lo ; gy_hi] (N' = 3N)
// split3() writes dst[o][b][i] = part(pattern bit b)(src[o][i]) for b = 0, 1, 2, i < blk.
#include "kernels.cuh"

namespace ptb {

namespace {

__device__ __forceinline__ float tf32_rna(float v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
}

// pattern bit b set: block b takes lo, else hi. float4 path when blk % 4 == 0 and both
// pointers are 16-byte aligned.
__global__ void split3_kernel(const float* __restrict__ src, float* __restrict__ dst, int64_t outer,
                              int64_t blk, int pattern) {
    const int64_t total = outer * blk;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = i / blk, j = i - o * blk;
        const float v = __ldg(src + i);
        const float hi = tf32_rna(v), lo = tf32_rna(v - hi);
        float* d = dst + o * 3 * blk + j;
#pragma unroll
        for (int b = 0; b < 3; ++b) __stcs(d + b * blk, (pattern >> b) & 1 ? lo : hi);
    }
}

__global__ void split3_kernel4(const float4* __restrict__ src, float4* __restrict__ dst, int64_t outer,
                               int64_t blk4, int pattern) {
    const int64_t total = outer * blk4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = i / blk4, j = i - o * blk4;
        const float4 v = __ldg(src + i);
        float4 hi, lo;
        hi.x = tf32_rna(v.x); lo.x = tf32_rna(v.x - hi.x);
        hi.y = tf32_rna(v.y); lo.y = tf32_rna(v.y - hi.y);
        hi.z = tf32_rna(v.z); lo.z = tf32_rna(v.z - hi.z);
        hi.w = tf32_rna(v.w); lo.w = tf32_rna(v.w - hi.w);
        float4* d = dst + o * 3 * blk4 + j;
#pragma unroll
        for (int b = 0; b < 3; ++b) __stcs(d + b * blk4, (pattern >> b) & 1 ? lo : hi);
    }
}

}  // namespace

void split3(const float* src, float* dst, int64_t outer, int64_t blk, int pattern, cudaStream_t st) {
    const int64_t total = outer * blk;
    if (total <= 0) return;
    ProfScope prof("layout", st, 0.0, 16.0 * total);
    const bool vec = blk % 4 == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
    const int64_t items = vec ? total / 4 : total;
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(items, 256), 8 * (int64_t)sm_count());
    if (vec)
        split3_kernel4<<<grid, 256, 0, st>>>(reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst),
                                             outer, blk / 4, pattern);
    else
        split3_kernel<<<grid, 256, 0, st>>>(src, dst, outer, blk, pattern);
    after_launch("split3");
}

}  // namespace ptb
