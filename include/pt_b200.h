/*
 * pt_b200.h — C ABI of libpt_b200.so, the sm_100a SpatialConvolutionMM hot path.
 *
 * This is the drop-in boundary. Plain pointers, sizes and an
 * opaque stream handle only: no C++ or torch types cross it, no exceptions
 * escape it. Every entry point is stream-ordered on `stream` (a cudaStream_t
 * passed as void*; NULL = legacy default stream) and reentrant across
 * streams; only the per-device plan cache (TMA descriptors, tile choice) is
 * global, under a mutex.
 *
 * Return codes mirror the reference's error classes / CLI exit codes
 * (proj/include/portten/errors.hpp:24-40):
 *   PT_OK (0), PT_EVALIDATION (2) = ValidationError, PT_EBACKEND (3) = BackendError.
 * The message of the last failure on the calling thread is pt_b200_last_error().
 *
 * Device tensors are float32, dense, row-major (NCHW activations, KCRS weights),
 * 16-byte aligned. The C++ wrapper (include/portten/ headers) rethrows the codes as
 * portten::ValidationError / portten::BackendError.
 */
#ifndef PT_B200_H
#define PT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PT_B200_ABI_VERSION 1

enum pt_status { PT_OK = 0, PT_EVALIDATION = 2, PT_EBACKEND = 3 };

/* Conv problem descriptor. Field order == conv::ConvGeometry
 * (proj/include/portten/conv_geometry.hpp:29-39): batch, inChannels, inHeight,
 * inWidth, outChannels, kernelH, kernelW, padH, padW, strideH, strideW.
 * Output dims use the floor rule of conv_geometry.hpp:41-46. */
typedef struct pt_conv_geom {
    int64_t N, C, H, W, K, kH, kW, padH, padW, strideH, strideW;
} pt_conv_geom;

/* Contraction mode. TF32: tcgen05 tensor cores, operands rounded to TF32
 * (cvt.rna), FP32 accumulate in TMEM. FP32: CUDA-core FFMA implicit GEMM,
 * the tight-tolerance mode (north_star "FP32-FFMA mode for tight checks"). */
/* PT_MATH_3XTF32: FP32-accurate on the tensor cores. Each operand is split v = hi + lo
 * (both TF32) and the three products hi*hi + lo*hi + hi*lo run as one TF32 convolution over
 * a 3x reduction (SURVEY.md §5 PORTTEN_CONV_MATH=3xtf32; the reference's arithmetic is FP32
 * SGEMM). Convolutions only; pt_b200_gemm rejects it. */
enum pt_math { PT_MATH_TF32 = 0, PT_MATH_FP32 = 1, PT_MATH_3XTF32 = 2 };

/* Which conv pass a workspace query is for. */
enum pt_conv_op { PT_CONV_FWD = 0, PT_CONV_BWD_DATA = 1, PT_CONV_BWD_FILTER = 2, PT_CONV_BWD = 3 };

/* Strided view (Tensor sizes/strides/storageOffset, proj/include/portten/tensor.hpp:56-120).
 * Rank 1..8 (kMaxDims, tensor.hpp:29); strides in elements, non-negative. */
typedef struct pt_view {
    int32_t ndim;
    int64_t sizes[8];
    int64_t strides[8];
    int64_t offset;
} pt_view;

/* Reduction op, same order as codegen::ReduceOp (proj/include/portten/kernel_codegen.hpp:70). */
enum pt_reduce_op { PT_REDUCE_SUM = 0, PT_REDUCE_MAX = 1, PT_REDUCE_MIN = 2 };

/* Apply bytecode: the RPN form of expr::Program (proj/src/expression.cpp:340-402).
 * One int32 per instruction (low byte = opcode); PT_OP_CONST is followed by one
 * int32 holding the float bit pattern. Max stack depth 32 (expression.cpp track()). */
enum pt_apply_op {
    PT_OP_CONST = 0, PT_OP_X = 1, PT_OP_Y = 2, PT_OP_Z = 3, PT_OP_S = 4,
    PT_OP_ADD = 5, PT_OP_SUB = 6, PT_OP_MUL = 7, PT_OP_DIV = 8, PT_OP_NEG = 9,
    PT_OP_ABS = 10, PT_OP_EXP = 11, PT_OP_LOG = 12, PT_OP_SQRT = 13, PT_OP_TANH = 14,
    PT_OP_MAX = 15, PT_OP_MIN = 16
};

/* Device capability record (BackendDescriptor, proj/include/portten/backend.hpp:35-40). */
typedef struct pt_device_desc {
    char name[64];            /* "b200:<ordinal>" */
    int32_t maxWorkgroupSize; /* max threads per block */
    int64_t localMemBytes;    /* max opt-in shared memory per block */
    int32_t smCount;
    int32_t ccMajor, ccMinor;
    int64_t globalMemBytes;
} pt_device_desc;

/* ---- library / device plumbing (replaces opencl_probe_devices, proj/src/opencl_backend.hpp:29) ---- */
int pt_b200_abi_version(void);
const char* pt_b200_last_error(void);
/* Number of usable sm_100 devices; 0 when no driver/GPU (never an error). */
int pt_b200_device_count(void);
int pt_b200_device_info(int device, pt_device_desc* out);
int pt_b200_set_device(int device);
int pt_b200_get_device(int* device);
int pt_b200_malloc(void** ptr, size_t bytes);
int pt_b200_free(void* ptr);
/* device_upload / device_download (proj/src/backend.cpp:163-181): contiguous staging copies. */
int pt_b200_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream);
int pt_b200_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream);
int pt_b200_stream_sync(void* stream);
/* Non-blocking completion check of `stream`: PT_OK when all its work is done, 1 while work
 * is pending, PT_EBACKEND on a device error (used to poll NCCL's async error meanwhile). */
int pt_b200_stream_query(void* stream);
/* Same generator as oracle or_fill_uniform (counter-based splitmix64). */
int pt_b200_fill_uniform(float* dst, int64_t n, uint64_t seed, float lo, float hi, void* stream);

/* ---- convolution (Torch SpatialConvolutionMM) ---- */
/* Validates like conv::ConvGeometry::validate (conv_geometry.hpp:53-63). */
int pt_b200_conv_validate(const pt_conv_geom* g);
/* Bytes of device scratch the pass needs (caller allocates; 0 is possible). */
size_t pt_b200_conv_workspace_bytes(const pt_conv_geom* g, int op, int math);
/* updateOutput == conv_im2col_forward: y = W (K x CRS) * im2col(x) + b.
 * b may be NULL (no bias). */
int pt_b200_conv_fwd(const pt_conv_geom* g, const float* x, const float* w, const float* b,
                     float* y, int math, void* ws, size_t ws_bytes, void* stream);
/* updateGradInput == conv_backward_input: gx = col2im(W^T * gy). */
int pt_b200_conv_bwd_data(const pt_conv_geom* g, const float* gy, const float* w, float* gx,
                          int math, void* ws, size_t ws_bytes, void* stream);
/* accGradParameters == conv_backward_weight + gradBias:
 * gw (+)= scale * sum_n gy[n] im2col(x[n])^T ; gb (+)= scale * sum gy. accumulate=0
 * overwrites (SPEC's fresh gradients), 1 accumulates (Torch). gb may be NULL. */
int pt_b200_conv_bwd_filter(const pt_conv_geom* g, const float* x, const float* gy, float* gw,
                            float* gb, float scale, int accumulate, int math, void* ws,
                            size_t ws_bytes, void* stream);
/* Torch backward() = updateGradInput + accGradParameters in one call: one NHWC
 * transform of gy (with gradBias fused) feeds both tensor-core passes. gx may be NULL
 * (first layer: no gradInput), gw may be NULL (gradInput only); gb may be NULL. */
int pt_b200_conv_bwd(const pt_conv_geom* g, const float* x, const float* gy, const float* w,
                     float* gx, float* gw, float* gb, float scale, int accumulate, int math,
                     void* ws, size_t ws_bytes, void* stream);
/* Torch's `finput` (nn.SpatialConvolutionMM keeps the input unfold of updateOutput for
 * accGradParameters): the forward engine's channels-last copy of x, which the weight
 * gradient can reuse instead of re-laying x out. finput_bytes is 0 when the engines do
 * not share a layout for this geometry (the *_finput calls then ignore the buffer).
 * Contract as in Torch: x must be unchanged between the two calls. */
size_t pt_b200_conv_finput_bytes(const pt_conv_geom* g, int math);
int pt_b200_conv_fwd_finput(const pt_conv_geom* g, const float* x, const float* w, const float* b,
                            float* y, int math, void* ws, size_t ws_bytes, float* finput,
                            void* stream);
int pt_b200_conv_bwd_finput(const pt_conv_geom* g, const float* x, const float* gy, const float* w,
                            float* gx, float* gw, float* gb, float scale, int accumulate, int math,
                            void* ws, size_t ws_bytes, const float* finput, void* stream);
/* Winograd F(2x2,3x3) registry entry (conv_winograd_2x2_3x3): 3x3 stride-1
 * layers only (gradInput: padding <= 2), otherwise PT_EVALIDATION "unsupported geometry".
 * Weight / input transforms, 16 transform-domain TF32 GEMMs on the tensor cores (channel
 * sums in the transform domain), output transform + bias. Same argument meaning as
 * pt_b200_conv_fwd / _bwd_data; scratch from pt_b200_winograd_workspace_bytes(g, op), op =
 * PT_CONV_FWD or PT_CONV_BWD_DATA ((size_t)-1 for an unsupported geometry). */
size_t pt_b200_winograd_workspace_bytes(const pt_conv_geom* g, int op);
int pt_b200_conv_fwd_winograd(const pt_conv_geom* g, const float* x, const float* w, const float* b,
                              float* y, void* ws, size_t ws_bytes, void* stream);
int pt_b200_conv_bwd_data_winograd(const pt_conv_geom* g, const float* gy, const float* w, float* gx,
                                   void* ws, size_t ws_bytes, void* stream);
/* Standalone unfold of ONE image, bit-exact with proj/templates/im2col.kt.tmpl:9-21. */
int pt_b200_im2col(const pt_conv_geom* g, const float* img, float* col, void* stream);
/* Batched unfold: images [n0, n0+count) into (CRS) x (count*oHW). */
int pt_b200_im2col_batched(const pt_conv_geom* g, const float* x, int64_t n0, int64_t count,
                           float* col, void* stream);
/* Scatter-add inverse of im2col for ONE image. img is overwritten. */
int pt_b200_col2im(const pt_conv_geom* g, const float* col, float* img, void* stream);
/* SPEC gemm, row-major, device pointers:
 * C <- alpha*op(A)*op(B) + beta*C (beta == 0: C is not read). math = PT_MATH_FP32: CUDA-core
 * FFMA; PT_MATH_TF32: the tcgen05 tensor-core GEMM, which needs A, B 16-byte aligned with
 * lda, ldb multiples of 4 (TMA), else PT_EVALIDATION. */
int pt_b200_gemm(int transA, int transB, int64_t M, int64_t N, int64_t K, float alpha,
                 const float* A, int64_t lda, const float* B, int64_t ldb, float beta, float* C,
                 int64_t ldc, int math, void* stream);

/* ---- pointwise apply / reduce on the conv path (Backend::runApply / runReduce*) ---- */
/* Compiles an apply expression "x = <expr>" (the grammar of expr::Program::parse,
 * proj/include/portten/expression.hpp:29-45: operands x y z up to `arity`, scalar s, float
 * literals, + - * /, unary minus, parentheses, abs exp log sqrt tanh max min, stack depth
 * <= 32) to the pt_apply_op bytecode pt_b200_apply runs. On a grammar error returns
 * PT_EVALIDATION with the reference's message (pt_b200_last_error). code may be NULL (then
 * only *ncode is set); *referenced = highest operand index used + 1; statement (optional)
 * receives the canonical kernel-language text, e.g. "x = (x * 2);" (kernelStatement()). */
int pt_b200_expression_compile(const char* text, int arity, int32_t* code, int32_t capacity,
                               int32_t* ncode, int32_t* referenced, char* statement,
                               size_t statement_cap);
/* Elementwise program over 1..3 same-shaped strided views; bases[0]/views[0] is x
 * (the destination). Mirrors ReferenceBackend::runApply (proj/src/reference_backend.cpp:80-113). */
int pt_b200_apply(const int32_t* code, int32_t ncode, int arity, float* const* bases,
                  const pt_view* views, float scalar, void* stream);
/* Per-channel bias add over an NCHW tensor: y[n,k,:,:] += b[k] (the conv-path
 * "x = x + s" on y.narrow(1,k,1), as one launch). */
int pt_b200_bias_add(float* y, const float* b, int64_t N, int64_t K, int64_t HW, void* stream);
/* Reduce-all into *out_dev (device float). Tree order; <=1e-5 rel of the sequential fold. */
int pt_b200_reduce_all(int op, const float* base, const pt_view* view, float* out_dev,
                       void* stream);
/* Reduce along `dim` into a contiguous tensor with sizes[dim]=1 (reference_backend.cpp:129-156). */
int pt_b200_reduce_dim(int op, const float* base, const pt_view* view, int dim, float* out,
                       void* stream);

/* ---- the other layers of the model-stack bench (ModelSpec layers
 * conv / pool-max / relu; bench_model :484-492). NCHW float32, device pointers. ---- */
/* y = max(x, 0) (in place allowed); backward gx = y > 0 ? gy : 0 (Torch threshold). */
int pt_b200_relu_fwd(const float* x, float* y, int64_t n, void* stream);
int pt_b200_relu_bwd(const float* y, const float* gy, float* gx, int64_t n, void* stream);
/* Max pooling, window kH x kW, stride sH x sW, zero-or-more padding (never selected);
 * oH = (H + 2pH - kH)/sH + 1 (floor, Torch's default). argmax (int32 index into the input
 * plane, may be NULL in inference) feeds the backward, a deterministic gather that sums the
 * gradients of every window whose arg-max a pixel is. */
int pt_b200_maxpool_fwd(const float* x, float* y, int32_t* argmax, int64_t N, int64_t C, int64_t H,
                        int64_t W, int kH, int kW, int sH, int sW, int pH, int pW, void* stream);
int pt_b200_maxpool_bwd(const float* gy, const int32_t* argmax, float* gx, int64_t N, int64_t C,
                        int64_t H, int64_t W, int kH, int kW, int sH, int sW, int pH, int pW,
                        void* stream);

/* ---- data-parallel helpers (batch sharding) ---- */
/* Number of kernels this library launched on the calling process (bench gpu_launches). */
int64_t pt_b200_launch_count(void);

/* Plan cache: TMA descriptors are cached per thread, keyed by every encode argument
 * (buffer address, extents, strides, box, swizzle), so re-running a layer on the same
 * buffers skips the driver encodes. Counts since process start (either may be null). */
void pt_b200_plan_cache_stats(int64_t* hits, int64_t* encodes);

/* Measured TF32 tensor-pipe ceiling (TFLOP/s) of the current device at its current
 * clocks: back-to-back M=256 N=256 K=8 kind::tf32 MMAs from shared memory on every SM
 * pair (the roofline denominator bench.py reports against). < 0 on failure. */
double pt_b200_tf32_mma_peak(void);

/* ---- live kernel timing (bench.py roofline) ----
 * When enabled, the library brackets each launch of its hot kernels with CUDA events
 * on the launching stream and records the algorithmic work of that launch. Reading
 * synchronises the recorded events. Kernel classes: "umma_conv" (tcgen05 fprop/dgrad),
 * "umma_wgrad" (tcgen05 wgrad), "simt_conv" (FFMA passes), "layout" (NHWC/pack passes). */
int pt_b200_profile_enable(int on);
/* Scheduling of the combined backward (pt_b200_conv_bwd / _finput): 1 (default) runs the
 * weight gradient on an internal per-device stream concurrently with the input gradient
 * (fork/join with events on the caller's stream, results unchanged); 0 serialises them on
 * the caller's stream (per-launch event timings then measure each kernel alone). */
int pt_b200_set_bwd_streams(int on);
int pt_b200_profile_reset(void);
/* Label for the launches the calling thread records next (e.g. the layer name); each
 * launch is also accumulated under "<class>@<tag>.<pass>", pass = fwd | dgrad | wgrad. */
int pt_b200_profile_tag(const char* tag);
/* kernel_class: a class name or a "<class>@<tag>.<pass>" key.
 * total_ms = summed event durations, launches = count, flops = algorithmic FLOPs,
 * bytes = algorithmic HBM bytes (for memory-bound classes). */
int pt_b200_profile_read(const char* kernel_class, double* total_ms, int64_t* launches,
                         double* flops, double* bytes);

#ifdef __cplusplus
}
#endif
#endif
