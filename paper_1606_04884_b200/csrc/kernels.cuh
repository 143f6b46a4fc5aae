// kernels.cuh — internal (C++) entry points shared between the .cu files of
// libpt_b200.so. None of these cross the ABI; include/pt_b200.h is the boundary.
#pragma once

#include "common.cuh"

namespace ptb {

// ---- simt_conv.cu: FP32-FFMA implicit GEMM on NCHW / KCRS ----
void simt_conv_fwd(const Geo& g, const float* x, const float* w, const float* b, float* y,
                   cudaStream_t st);
void simt_conv_bwd_data(const Geo& g, const float* gy, const float* w, float* gx, cudaStream_t st);
int simt_wgrad_splits(const Geo& g);
size_t simt_wgrad_workspace(const Geo& g);
void simt_conv_bwd_filter(const Geo& g, const float* x, const float* gy, float* gw, float scale,
                          int accumulate, float* ws, cudaStream_t st);
void simt_gemm(int transA, int transB, int64_t M, int64_t N, int64_t K, float alpha,
               const float* A, int64_t lda, const float* B, int64_t ldb, float beta, float* C,
               int64_t ldc, cudaStream_t st);

// ---- layout.cu: HBM layout transforms feeding the tensor-core path ----
// NCHW [N][C][HW] -> NHWC [N][HW][Cp] (channels zero-padded to Cp), optionally
// rounded to TF32 (cvt.rna).
void nchw_to_nhwc(const float* src, float* dst, int64_t N, int64_t C, int64_t HW, int64_t Cp,
                  bool round_tf32, cudaStream_t st);
// Same transform (TF32-rounded) of gradOutput with gradBias fused: per-block channel
// sums of the unrounded values land in `part` (nhwc_bias_partials_bytes) and a
// fixed-order reduce writes gb (+)= scale * sum. gb may be null (no bias).
size_t nhwc_bias_partials_bytes(int64_t N, int64_t C, int64_t HW);
// Destination of an NCHW -> NHWC transform: pixel (h, w) of an H x W image lands at
// (h + ph) * Wp + (w + pw) of an image of `img` pixels (dense: Wp = W, img = H*W).
struct NhwcDst {
    float* p = nullptr;
    int64_t W = 1, Wp = 1, ph = 0, pw = 0, img = 0;
    static NhwcDst dense(float* p, int64_t HW) { return NhwcDst{p, HW, HW, 0, 0, HW}; }
    static NhwcDst padded(float* p, int64_t H, int64_t W, int64_t ph, int64_t pw) {
        return NhwcDst{p, W, W + 2 * pw, ph, pw, (H + 2 * ph) * (W + 2 * pw)};
    }
    __host__ __device__ int64_t pixel(int64_t p_) const {
        if (Wp == W) return p_ + ph * Wp;
        const int64_t h = p_ / W;
        return (h + ph) * Wp + (p_ - h * W) + pw;
    }
};
// NCHW -> one or two NHWC copies (TF32-rounded, channels zero-padded to Cp), the
// spatial border of padded destinations zeroed; gradBias fused as in nchw_to_nhwc_bias
// when gb is set.
void nchw_to_nhwc_padded(const float* src, const NhwcDst& d0, const NhwcDst& d1, int64_t N,
                         int64_t C, int64_t H, int64_t W, int64_t Cp, float* gb, float scale,
                         int accumulate, float* part, cudaStream_t st);
// defer_bias: the partials are written but the gradBias reduce is left to the caller
// (bias_from_nhwc_partials, e.g. on another stream ordered after this one)
void nchw_to_nhwc_bias(const float* src, float* dst, int64_t N, int64_t C, int64_t HW, int64_t Cp,
                       float* gb, float scale, int accumulate, float* part, cudaStream_t st,
                       bool defer_bias = false);
void bias_from_nhwc_partials(const float* part, int64_t N, int64_t C, int64_t HW, float* gb, float scale,
                             int accumulate, cudaStream_t st);
// Weight packing for the implicit GEMM B operand. W is KCRS [K][C][kH][kW].
//  kPackFprop     : row n = k,         tap (r,s),           channel = c  (cin = C)
//  kPackDgradFlip : row n = c,         tap (kH-1-r,kW-1-s), channel = k  (cin = K)
//  kPackGcol      : row n = (c,r,s),   single tap,          channel = k  (cin = K)
// layout 32: B[n_pad][taps][cin_p]           (Kdim-contiguous rows, SW128 tiles)
// layout 4 : B[slots_p][n_pad][4], slot = tap*(cin_p/4) + chunk (core-matrix tiles)
enum PackMode { kPackFprop = 0, kPackDgradFlip = 1, kPackGcol = 2 };
void pack_weights(const float* w, float* dst, int64_t K, int64_t C, int64_t kH, int64_t kW,
                  int mode, int layout, int64_t n_pad, int64_t cin_p, int64_t slots_p,
                  int64_t total_elems, bool round_tf32, cudaStream_t st);
// Hankel tap groups: [kH][ceil(kW/G)][G][bn][cin_p] (see layout.cu:pack_grouped_kernel).
void pack_grouped(const float* w, float* dst, int64_t K, int64_t C, int64_t kH, int64_t kW, bool dgrad,
                  int G, int bn, int64_t cin_p, cudaStream_t st);
// gb[k] = (acc ? gb[k] : 0) + scale * sum_{n,p} gy[n][k][p] (fixed-order, deterministic).
void bias_grad(const float* gy, float* gb, int64_t N, int64_t K, int64_t HW, float scale,
               int accumulate, float* ws, size_t ws_bytes, cudaStream_t st);
size_t bias_grad_workspace(int64_t N, int64_t K, int64_t HW);

// ---- split3.cu: 3xTF32 operand split, dst[o][b][i] = (pattern bit b ? lo : hi)(src[o][i]) ----
void split3(const float* src, float* dst, int64_t outer, int64_t blk, int pattern, cudaStream_t st);

// ---- umma_conv.cu: tcgen05 kind::tf32 implicit GEMM (fprop, stride-1 dgrad) ----
struct UmmaPlan {
    enum Mode { kFprop = 0, kDgradTconv = 1, kDgradGcol = 2 };
    bool ok = false;      // geometry supported by the tensor-core path
    int mode = kFprop;
    int64_t extra_elems = 0;  // gcol scratch (kDgradGcol)
    int cb = 32;          // channel chunk per TMA im2col box (32: SW128, 4: no swizzle)
    int cg = 1;           // CTAs per MMA (2: cta_group::2 pair, M = 256)
    int64_t cin_p = 0;    // padded input channels of the NHWC operand
    int64_t cin_real = 0; // the real ones (the rest of the last 32-channel chunk is zero)
    int64_t taps = 0;     // kH*kW
    int64_t slots_p = 0;  // layout-4 slot count padded to 8
    int64_t n_rows = 0;   // GEMM N (output channels)
    int bn = 0;           // N tile
    int n_tiles = 0;
    int64_t n_pad = 0;    // n_tiles * bn
    int64_t act_elems = 0, wt_elems = 0;  // workspace floats
    size_t ws_bytes = 0;
    // Hankel pixel-run engine (umma_hconv.cu): stride 1, 32-channel chunks, CTA pair. The
    // activation stays dense NHWC; the (aph, apw) border is TMA out-of-bounds fill.
    bool hankel = false;
    int64_t aH = 0, aW = 0, aph = 0, apw = 0, aHp = 0, aWp = 0;
    // <= 128 output rows: group G taps (s .. s+G-1) in one N = G*bn MMA (umma_hconv.cu);
    // the packed weights then carry one extra all-zero tap (index `taps`) for kW % G != 0
    int tap_group = 1;  // taps per MMA (1, or 2..4: output-shift grouping)
    int64_t kdim = 0;  // packed weight row length (floats)
};
struct HConvTiling {
    int64_t P_img = 0;  // positions per image
    int64_t tiles = 0;  // 256-position pair tiles
};
// position rows carry only the left zero border (a right-edge tap wraps into the next
// row's left border); PT_B200_HCONV_WRAP=0: both borders
bool hconv_wrap();
HConvTiling hconv_tiling(int64_t N, int64_t Wp, int64_t oH, int64_t cta_span = 128);
// act: dense NHWC [N][aH][aW][cin_p]; the (aph, apw) zero border comes from TMA
// out-of-bounds fill. Stride-1 kH x kW conv -> oH x oW NCHW.
void run_hconv(const UmmaPlan& pl, const float* act, const float* wt, int64_t N, int64_t aH,
               int64_t aW, int64_t aph, int64_t apw, int kH, int kW, int64_t oH, int64_t oW,
               float* out, const float* bias, double alg_flops, cudaStream_t st);
// fprop: act = x (C channels, HxW), n_rows = K.
// dgrad, kDgradTconv: act = gy (K channels, oHxoW), n_rows = C, flipped weights,
//   pad' = k-1-pad (stride 1).  kDgradGcol (small C / strided): gcol = W^T gy as a
//   1x1 conv over gy (n_rows = CRS) then a gather col2im.
UmmaPlan umma_plan(const Geo& g, bool dgrad);
// act_out: where the NHWC activation copy goes (Torch's finput, reused by the weight
// gradient); null = the workspace.
// act_ready: act_out already holds that copy (x unused).
void umma_conv_fwd(const Geo& g, const UmmaPlan& pl, const float* x, const float* w,
                   const float* b, float* y, void* ws, cudaStream_t st, float* act_out = nullptr,
                   bool act_ready = false);
// gyh_pre: gy already in the plan's NHWC layout (TF32-rounded; zero-bordered when
// pl.hankel), or null to transform here.
void umma_conv_bwd_data(const Geo& g, const UmmaPlan& pl, const float* gy, const float* w,
                        float* gx, void* ws, cudaStream_t st, const float* gyh_pre = nullptr,
                        double alg_flops = -1.0);

// ---- umma_rowwgrad.cu: small-C dgrad = tconv of the (kH x 1) row-expanded layer + 1-D fold ----
bool rowdgrad_ok(const Geo& g, UmmaPlan* plan = nullptr);
size_t rowdgrad_workspace(const Geo& g);
// gyh_pre: gy NHWC (round_up(K,32) channels), zero-bordered for the expanded layer's
// Hankel plan when pre_padded; used only if it matches the plan's layout.
void rowdgrad(const Geo& g, const float* gy, const float* w, float* gx, void* ws, cudaStream_t st,
              const float* gyh_pre = nullptr, bool pre_padded = false);
size_t rowdgrad_act_offset(const Geo& g);  // byte offset of the engine's activation buffer in ws

// ---- umma_rowconv.cu: small-C (<=4), stride-1 forward via the Hankel row view ----
// x NCHW -> zero-bordered NHWC4 xp[n][Hp][Wa][4] (TF32-rounded)
void pad_nhwc4(const float* x, float* xp, const Geo& g, int Hp, int Wa, cudaStream_t st);
bool rowconv_ok(const Geo& g);
size_t rowconv_workspace(const Geo& g);
void rowconv_fwd(const Geo& g, const float* x, const float* w, const float* b, float* y, void* ws,
                 cudaStream_t st);

// ---- umma_rowwgrad.cu: small-C (<=4), stride-1 weight gradient via the Hankel row view ----
bool rowwgrad_ok(const Geo& g);
size_t rowwgrad_workspace(const Geo& g);
// gyh: gradOutput NHWC [N*oH*oW][round_up(K,32)], TF32-rounded
void rowwgrad(const Geo& g, const float* x, const float* gyh, float* gw, float scale, int accumulate,
              void* ws, cudaStream_t st);

// ---- umma_wgrad.cu: tcgen05 kind::tf32 weight gradient (MN-major operands, split-K) ----
bool umma_wgrad_ok(const Geo& g);
size_t umma_wgrad_workspace(const Geo& g);
// gyh_pre: gy already in NHWC [M][round_up(K,32)] (TF32-rounded), or null.
// xh_pre: x already NHWC [N][H+2*xph][W+2*xpw][round_up(C,32)] (TF32-rounded, zero border
// of (xph, xpw) — the forward pass's copy), or null.
// alg_flops: algorithmic FLOPs recorded for the live roofline (default 2*M*K*CRS of g).
void umma_conv_bwd_filter(const Geo& g, const float* x, const float* gy, float* gw, float scale,
                          int accumulate, void* ws, cudaStream_t st, const float* gyh_pre = nullptr,
                          const float* xh_pre = nullptr, double alg_flops = -1.0, int64_t xph = 0,
                          int64_t xpw = 0);
int64_t umma_wgrad_kp(const Geo& g);  // channel padding of the wgrad gy operand

// ---- umma_hwgrad.cu: stride-1 wide-filter weight gradient (Hankel tap quads) ----
bool hwgrad_ok(const Geo& g);
size_t hwgrad_part_bytes(const Geo& g);
// xh: x NHWC dense with (C+31)/32*32 channels; gyh: gy NHWC with (K+31)/32*32 channels
void hwgrad_run(const Geo& g, const float* xh, const float* gyh, float* gw, float scale, int accumulate,
                float* part, double alg_flops, cudaStream_t st);
// fixed-order split reduce of [split][(r*kW+s)*Cp + c][k] partials into KCRS gw; filter
// columns s >= s_v0 sum splits_v partials instead of splits (s_v0 < 0: all columns splits)
void wgrad_reduce_launch(const float* part, float* gw, const Geo& g, int64_t Cp, int splits, int64_t ld,
                         int64_t split_stride, float scale, int accumulate, cudaStream_t st, int splits_v = 0,
                         int s_v0 = -1);

// ---- umma_swgrad.cu: small-C stride-1 weight gradient (planes of horizontal taps) ----
bool swgrad_ok(const Geo& g);
size_t swgrad_workspace(const Geo& g);
// gyh: gy NHWC with (K+31)/32*32 channels, TF32-rounded (the shared backward transform)
void swgrad(const Geo& g, const float* x, const float* gyh, float* gw, float scale, int accumulate, void* ws,
            cudaStream_t st);

// ---- umma_scbwd.cu: fused backward of small-C stride-1 layers (C*kH*kW <= 32, K <= 64) ----
// One NCHW gy read feeds gradInput (gcol GEMM + in-smem fold), gradWeight and gradBias;
// gx / gw may be null (that product skipped); gb only with gw. gw takes (scale, accumulate),
// gb (bscale, bacc).
bool scbwd_ok(const Geo& g);
size_t scbwd_workspace(const Geo& g);
void scbwd(const Geo& g, const float* x, const float* gy, const float* w, float* gx, float* gw, float* gb,
           float scale, int accumulate, float bscale, int bacc, void* ws, cudaStream_t st);

// ---- s2d.cu: space-to-depth for strided small-C layers ----
bool s2d_applies(const Geo& g);
Geo s2d_geo(const Geo& g);  // the equivalent stride-1 conv over C*s*s channels
void s2d_input(const Geo& g, const float* x, float* xs, cudaStream_t st);
// x' directly in NHWC with Cp (zero-padded, TF32-rounded) channels: the engines' layout
bool s2d_nhwc_ok(const Geo& g, int64_t Cp);
void s2d_input_nhwc(const Geo& g, const float* x, float* xh, int64_t Cp, cudaStream_t st);
void s2d_weight(const Geo& g, const float* w, float* ws, cudaStream_t st);
void d2s_grad(const Geo& g, const float* gxs, float* gx, cudaStream_t st);
void d2s_weight_grad(const Geo& g, const float* gws, float* gw, float scale, int accumulate,
                     cudaStream_t st);

// ---- unfold.cu ----
void im2col_launch(const Geo& g, const float* x, int64_t n0, int64_t count, float* col,
                   cudaStream_t st);
void col2im_launch(const Geo& g, const float* col, float* img, cudaStream_t st);
// gcol [N][CRS][oHW] -> gx [N][C][H][W]
void col2im_batched_launch(const Geo& g, const float* col, float* img, cudaStream_t st);

// ---- pointwise.cu ----
void fill_uniform(float* dst, int64_t n, uint64_t seed, float lo, float hi, cudaStream_t st);
void apply_launch(const int32_t* code, int32_t ncode, int arity, float* const* bases,
                  const pt_view* views, float scalar, cudaStream_t st);
void bias_add_launch(float* y, const float* b, int64_t N, int64_t K, int64_t HW, cudaStream_t st);
void reduce_all_launch(int op, const float* base, const pt_view& v, float* out, cudaStream_t st);
void reduce_dim_launch(int op, const float* base, const pt_view& v, int dim, float* out,
                       cudaStream_t st);

// ---- umma_gemm.cu: batched tcgen05 TF32 GEMM D[b][n][m] = alpha*sum_k A[b][m][k] B[b][n][k] (+beta*D) ----
struct UmmaGemm {
    const float* a;
    const float* b;
    float* d;
    int64_t M, N, K, batch;
    bool a_mn, b_mn;  // operand stored MN-major (row index contiguous) instead of K-major
    int64_t lda, ldb, ldd, batch_a, batch_b, batch_d;
    float alpha, beta;
};
bool umma_gemm_supported(const UmmaGemm& g);
void umma_gemm(const UmmaGemm& g, cudaStream_t st);

// ---- winograd.cu: F(2x2,3x3) registry entry ----
bool winograd_applies(const Geo& g, int op);  // op: PT_CONV_FWD / PT_CONV_BWD_DATA
size_t winograd_workspace(const Geo& g, int op);
void winograd_fwd(const Geo& g, const float* x, const float* w, const float* b, float* y, void* ws,
                  cudaStream_t st);
void winograd_bwd_data(const Geo& g, const float* gy, const float* w, float* gx, void* ws, cudaStream_t st);

// ---- nnlayers.cu (model-stack bench layers) ----
void relu_fwd(const float* x, float* y, int64_t n, cudaStream_t st);
void relu_bwd(const float* y, const float* gy, float* gx, int64_t n, cudaStream_t st);
void maxpool_fwd(const float* x, float* y, int32_t* arg, int64_t N, int64_t C, int64_t H, int64_t W,
                 int kH, int kW, int sH, int sW, int pH, int pW, cudaStream_t st);
void maxpool_bwd(const float* gy, const int32_t* arg, float* gx, int64_t N, int64_t C, int64_t H,
                 int64_t W, int kH, int kW, int sH, int sW, int pH, int pW, cudaStream_t st);

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace ptb
