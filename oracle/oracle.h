/*
 * oracle.h — CPU restatement of the reference's SpatialConvolutionMM path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker or the timed CPU baseline. The product path
 * (paper_1606_04884_b200, libpt_b200.so) never links or calls it.
 *
 * Every function cites the reference file:line whose behaviour it restates.
 * Paths are relative to /root/reference. The reference ships no conv code
 * (SURVEY.md §0): conv/gemm/col2im semantics come from SPEC.md, the unfold
 * index maths from proj/templates/im2col.kt.tmpl, and apply/reduce from
 * proj/src/reference_backend.cpp + proj/src/expression.cpp.
 */
#ifndef PT_ORACLE_H
#define PT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Field order mirrors conv::ConvGeometry (proj/include/portten/conv_geometry.hpp:29-39). */
typedef struct or_geom {
    int64_t N, C, H, W, K, kH, kW, padH, padW, strideH, strideW;
} or_geom;

/* Strided float view (Tensor sizes/strides/storageOffset, proj/include/portten/tensor.hpp:56-120). */
typedef struct or_view {
    int32_t ndim;
    int64_t sizes[8];
    int64_t strides[8];
    int64_t offset;
} or_view;

enum { OR_SUM = 0, OR_MAX = 1, OR_MIN = 2 }; /* codegen::ReduceOp order */

/* conv_geometry.hpp:41-46 floor rule; :49 patchSize; :51 outSpatial. */
int64_t or_out_h(const or_geom* g);
int64_t or_out_w(const or_geom* g);
/* conv_geometry.hpp:53-63. Returns 0 when valid, 2 (ValidationError) otherwise. */
int or_validate(const or_geom* g);

/* Counter-based synthetic inputs: v[i] = lo + (hi-lo) * u(splitmix64(seed + i)),
 * u in [0,1) from the top 24 bits. Identical to pt_b200_fill_uniform on device. */
void or_fill_uniform(float* dst, int64_t n, uint64_t seed, float lo, float hi);

/* SPEC.md:353-361 conv_direct: cross-correlation, zero padding, per-output
 * float accumulation in (c, r, s) order, bias added first (b may be NULL). */
void or_conv_direct(const or_geom* g, const float* x, const float* w, const float* b, float* y);
/* Same contraction accumulated in double, rounded once: the high-precision
 * reference the tolerance checks measure against. */
void or_conv_direct_f64(const or_geom* g, const float* x, const float* w, const float* b, float* y);

/* proj/templates/im2col.kt.tmpl:9-21 (one image): col[(c*kH*kW + r*kW + s)*oHW + i*oW + j]
 * = inside ? img[c*H*W + h*W + w] : 0.0f with h = i*sH - pH + r, w = j*sW - pW + s. */
void or_im2col(const or_geom* g, const float* img, float* col);
/* SPEC.md:371-379 col2im (one image): zero img, then scatter-add every column
 * entry into its source position in (c, r, s, i, j) order; pad positions dropped. */
void or_col2im(const or_geom* g, const float* col, float* img);

/* SPEC.md:347-350, 380-388 gemm, row-major: C <- alpha*op(A)*op(B) + beta*C. */
void or_gemm_naive(int transA, int transB, int64_t M, int64_t N, int64_t K, float alpha,
                   const float* A, int64_t lda, const float* B, int64_t ldb, float beta,
                   float* C, int64_t ldc);
/* Tiled/blocked variant ("tiled/blocked variant (default)"),
 * OpenMP over `threads` (<=0: all). Equal to naive within 1e-5 relative. */
void or_gemm_blocked(int transA, int transB, int64_t M, int64_t N, int64_t K, float alpha,
                     const float* A, int64_t lda, const float* B, int64_t ldb, float beta,
                     float* C, int64_t ldc, int threads);

/* SPEC.md:389-397 conv_im2col_forward / :398-406 conv_im2col_batched:
 * per chunk of `chunk` images, lower to (CRS) x (chunk*oHW), one GEMM
 * W(K x CRS) * col, then bias per output channel. chunk<=0 means 1. */
void or_conv_forward(const or_geom* g, const float* x, const float* w, const float* b, float* y,
                     int64_t chunk, int threads);
/* SPEC.md:416-419 conv_backward_input: gcol = W^T * gy[n], col2im -> gx[n]. */
void or_conv_backward_input(const or_geom* g, const float* gy, const float* w, float* gx,
                            int threads);
/* SPEC.md:416-424 conv_backward_weight + gradBias, with Torch accGradParameters
 * semantics: gw (+)= scale * sum_n gy[n] * im2col(x[n])^T, gb (+)= scale * sum gy.
 * accumulate=0 overwrites (SPEC "fresh" gradients). gb may be NULL. */
void or_conv_backward_weight(const or_geom* g, const float* x, const float* gy, float* gw,
                             float* gb, float scale, int accumulate, int threads);

/* proj/src/reference_backend.cpp:115-127 runReduceAll: sequential fold in
 * logical row-major order; Sum/Max/Min with fmaxf/fminf. */
float or_reduce_all(int op, const float* base, const or_view* v);
/* proj/src/reference_backend.cpp:129-156 runReduceDim: out has v's sizes with
 * sizes[dim]=1, contiguous; each output folds its strided run sequentially. */
void or_reduce_dim(int op, const float* base, const or_view* v, int dim, float* out);

/* proj/src/expression.cpp:340-402 Program::eval over RPN bytecode (see
 * pt_b200.h PT_OP_*), applied elementwise over 1..3 same-shaped strided views
 * in logical order (reference_backend.cpp:80-113). bases[0] is the destination. */
void or_apply(const int32_t* code, int32_t ncode, int arity, float* const* bases,
              const or_view* views, float scalar);

/* Library build stamp (tests check the oracle they load is the one built). */
const char* or_version(void);

#ifdef __cplusplus
}
#endif
#endif
