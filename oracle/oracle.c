/*
 * oracle.c — CPU restatement of the reference's conv path. TEST INFRASTRUCTURE:
 * loaded only by tests/, __graft_entry__.smoke() and bench.py's CPU legs, as the
 * checker or the timed CPU baseline — never by the product library.
 *
 * Citations are /root/reference-relative. See oracle.h for the contract.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../include/pt_b200.h"

const char* or_version(void) { return "pt-oracle-1"; }

/* conv_geometry.hpp:41-46 */
int64_t or_out_h(const or_geom* g) { return (g->H + 2 * g->padH - g->kH) / g->strideH + 1; }
int64_t or_out_w(const or_geom* g) { return (g->W + 2 * g->padW - g->kW) / g->strideW + 1; }

/* conv_geometry.hpp:53-63 */
int or_validate(const or_geom* g) {
    if (!(g->N >= 1 && g->C >= 1 && g->H >= 1 && g->W >= 1 && g->K >= 1 && g->kH >= 1 &&
          g->kW >= 1 && g->strideH >= 1 && g->strideW >= 1))
        return 2;
    if (g->padH < 0 || g->padW < 0) return 2;
    if (g->kH > g->H + 2 * g->padH || g->kW > g->W + 2 * g->padW) return 2;
    if (or_out_h(g) < 1 || or_out_w(g) < 1) return 2;
    return 0;
}

static uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void or_fill_uniform(float* dst, int64_t n, uint64_t seed, float lo, float hi) {
    const float span = hi - lo;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t r = splitmix64(seed + (uint64_t)i);
        const float u = (float)(r >> 40) * (1.0f / 16777216.0f);
        dst[i] = lo + span * u;
    }
}

/* out[n,k,i,j] = bias[k] + sum_{c,r,s} in[n,c,i*sH+r-pH,j*sW+s-pW]*w[k,c,r,s] */
void or_conv_direct(const or_geom* g, const float* x, const float* w, const float* b, float* y) {
    const int64_t oH = or_out_h(g), oW = or_out_w(g);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t n = 0; n < g->N; ++n)
        for (int64_t k = 0; k < g->K; ++k)
            for (int64_t i = 0; i < oH; ++i)
                for (int64_t j = 0; j < oW; ++j) {
                    float acc = b ? b[k] : 0.0f;
                    for (int64_t c = 0; c < g->C; ++c)
                        for (int64_t r = 0; r < g->kH; ++r) {
                            const int64_t h = i * g->strideH + r - g->padH;
                            if (h < 0 || h >= g->H) continue;
                            for (int64_t s = 0; s < g->kW; ++s) {
                                const int64_t ww = j * g->strideW + s - g->padW;
                                if (ww < 0 || ww >= g->W) continue;
                                acc += x[((n * g->C + c) * g->H + h) * g->W + ww] *
                                       w[((k * g->C + c) * g->kH + r) * g->kW + s];
                            }
                        }
                    y[((n * g->K + k) * oH + i) * oW + j] = acc;
                }
}

void or_conv_direct_f64(const or_geom* g, const float* x, const float* w, const float* b, float* y) {
    const int64_t oH = or_out_h(g), oW = or_out_w(g);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t n = 0; n < g->N; ++n)
        for (int64_t k = 0; k < g->K; ++k)
            for (int64_t i = 0; i < oH; ++i)
                for (int64_t j = 0; j < oW; ++j) {
                    double acc = b ? (double)b[k] : 0.0;
                    for (int64_t c = 0; c < g->C; ++c)
                        for (int64_t r = 0; r < g->kH; ++r) {
                            const int64_t h = i * g->strideH + r - g->padH;
                            if (h < 0 || h >= g->H) continue;
                            for (int64_t s = 0; s < g->kW; ++s) {
                                const int64_t ww = j * g->strideW + s - g->padW;
                                if (ww < 0 || ww >= g->W) continue;
                                acc += (double)x[((n * g->C + c) * g->H + h) * g->W + ww] *
                                       (double)w[((k * g->C + c) * g->kH + r) * g->kW + s];
                            }
                        }
                    y[((n * g->K + k) * oH + i) * oW + j] = (float)acc;
                }
}

/* im2col.kt.tmpl:9-21 — one work item per (c,i,j); row (c*kH*kW + r*kW + s), col i*oW + j. */
static void im2col_into(const or_geom* g, const float* img, float* col, int64_t ld, int64_t col0) {
    const int64_t oH = or_out_h(g), oW = or_out_w(g);
    const int64_t oHW = oH * oW;
    const int64_t patch = g->kH * g->kW;
    (void)oHW;
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < g->C; ++c)
        for (int64_t i = 0; i < oH; ++i)
            for (int64_t j = 0; j < oW; ++j) {
                const int64_t h0 = i * g->strideH - g->padH;
                const int64_t w0 = j * g->strideW - g->padW;
                const int64_t img_base = c * g->H * g->W;
                const int64_t col_pos = col0 + i * oW + j;
                for (int64_t r = 0; r < g->kH; ++r)
                    for (int64_t s = 0; s < g->kW; ++s) {
                        const int64_t h = h0 + r, ww = w0 + s;
                        const int inside = (h >= 0) && (h < g->H) && (ww >= 0) && (ww < g->W);
                        col[(c * patch + r * g->kW + s) * ld + col_pos] =
                            inside ? img[img_base + h * g->W + ww] : 0.0f;
                    }
            }
}

void or_im2col(const or_geom* g, const float* img, float* col) {
    im2col_into(g, img, col, or_out_h(g) * or_out_w(g), 0);
}

/* scatter-add, (c, r, s, i, j) order, pads dropped. */
static void col2im_from(const or_geom* g, const float* col, int64_t ld, int64_t col0, float* img) {
    const int64_t oH = or_out_h(g), oW = or_out_w(g);
    const int64_t patch = g->kH * g->kW;
    memset(img, 0, sizeof(float) * (size_t)(g->C * g->H * g->W));
    /* Channels are independent: parallel over c keeps each image plane's order fixed. */
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < g->C; ++c)
        for (int64_t r = 0; r < g->kH; ++r)
            for (int64_t s = 0; s < g->kW; ++s) {
                const float* row = col + (c * patch + r * g->kW + s) * ld + col0;
                for (int64_t i = 0; i < oH; ++i) {
                    const int64_t h = i * g->strideH - g->padH + r;
                    if (h < 0 || h >= g->H) continue;
                    for (int64_t j = 0; j < oW; ++j) {
                        const int64_t ww = j * g->strideW - g->padW + s;
                        if (ww < 0 || ww >= g->W) continue;
                        img[(c * g->H + h) * g->W + ww] += row[i * oW + j];
                    }
                }
            }
}

void or_col2im(const or_geom* g, const float* col, float* img) {
    col2im_from(g, col, or_out_h(g) * or_out_w(g), 0, img);
}

/* SPEC.md:380-388 naive triple loop. */
void or_gemm_naive(int transA, int transB, int64_t M, int64_t N, int64_t K, float alpha,
                   const float* A, int64_t lda, const float* B, int64_t ldb, float beta,
                   float* C, int64_t ldc) {
    for (int64_t i = 0; i < M; ++i)
        for (int64_t j = 0; j < N; ++j) {
            float acc = 0.0f;
            for (int64_t k = 0; k < K; ++k) {
                const float a = transA ? A[k * lda + i] : A[i * lda + k];
                const float bb = transB ? B[j * ldb + k] : B[k * ldb + j];
                acc += a * bb;
            }
            C[i * ldc + j] = (beta == 0.0f ? 0.0f : beta * C[i * ldc + j]) + alpha * acc;
        }
}

/* Blocked GEMM: pack op(A) rows / op(B) panels, i-k-j inner order so the j loop
 * vectorises; OpenMP over (row block, column block) tiles. */
enum { GB_M = 64, GB_N = 256, GB_K = 256 };

void or_gemm_blocked(int transA, int transB, int64_t M, int64_t N, int64_t K, float alpha,
                     const float* A, int64_t lda, const float* B, int64_t ldb, float beta,
                     float* C, int64_t ldc, int threads) {
    const int64_t mb = (M + GB_M - 1) / GB_M, nb = (N + GB_N - 1) / GB_N;
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#else
    (void)threads;
#endif
#pragma omp parallel for collapse(2) schedule(dynamic, 1) num_threads(threads)
    for (int64_t bi = 0; bi < mb; ++bi)
        for (int64_t bj = 0; bj < nb; ++bj) {
            const int64_t i0 = bi * GB_M, i1 = i0 + GB_M < M ? i0 + GB_M : M;
            const int64_t j0 = bj * GB_N, j1 = j0 + GB_N < N ? j0 + GB_N : N;
            const int64_t nn = j1 - j0;
            float acc[GB_M][GB_N];
            float bp[GB_K][GB_N];
            float ap[GB_M][GB_K];
            for (int64_t i = 0; i < i1 - i0; ++i)
                for (int64_t j = 0; j < nn; ++j) acc[i][j] = 0.0f;
            for (int64_t k0 = 0; k0 < K; k0 += GB_K) {
                const int64_t k1 = k0 + GB_K < K ? k0 + GB_K : K;
                for (int64_t k = k0; k < k1; ++k)
                    for (int64_t j = 0; j < nn; ++j)
                        bp[k - k0][j] = transB ? B[(j0 + j) * ldb + k] : B[k * ldb + j0 + j];
                for (int64_t i = i0; i < i1; ++i)
                    for (int64_t k = k0; k < k1; ++k)
                        ap[i - i0][k - k0] = transA ? A[k * lda + i] : A[i * lda + k];
                for (int64_t i = 0; i < i1 - i0; ++i)
                    for (int64_t k = 0; k < k1 - k0; ++k) {
                        const float a = ap[i][k];
                        float* __restrict__ ci = acc[i];
                        const float* __restrict__ bk = bp[k];
                        for (int64_t j = 0; j < nn; ++j) ci[j] += a * bk[j];
                    }
            }
            for (int64_t i = i0; i < i1; ++i)
                for (int64_t j = j0; j < j1; ++j) {
                    float* cij = &C[i * ldc + j];
                    *cij = (beta == 0.0f ? 0.0f : beta * *cij) + alpha * acc[i - i0][j - j0];
                }
        }
}

/* per chunk lower `chunk` images, one GEMM, bias per channel. */
void or_conv_forward(const or_geom* g, const float* x, const float* w, const float* b, float* y,
                     int64_t chunk, int threads) {
    const int64_t oHW = or_out_h(g) * or_out_w(g);
    const int64_t crs = g->C * g->kH * g->kW;
    if (chunk <= 0) chunk = 1;
    float* col = (float*)malloc(sizeof(float) * (size_t)(crs * chunk * oHW));
    float* tmp = (float*)malloc(sizeof(float) * (size_t)(g->K * chunk * oHW));
    for (int64_t n0 = 0; n0 < g->N; n0 += chunk) {
        const int64_t cnt = n0 + chunk <= g->N ? chunk : g->N - n0;
        const int64_t ld = cnt * oHW;
        for (int64_t t = 0; t < cnt; ++t)
            im2col_into(g, x + (n0 + t) * g->C * g->H * g->W, col, ld, t * oHW);
        or_gemm_blocked(0, 0, g->K, ld, crs, 1.0f, w, crs, col, ld, 0.0f, tmp, ld, threads);
        /* scatter the K x (cnt*oHW) result into NCHW and add the bias (apply x = x + s). */
#pragma omp parallel for collapse(2) schedule(static)
        for (int64_t t = 0; t < cnt; ++t)
            for (int64_t k = 0; k < g->K; ++k) {
                float* dst = y + ((n0 + t) * g->K + k) * oHW;
                const float* src = tmp + k * ld + t * oHW;
                const float bias = b ? b[k] : 0.0f;
                for (int64_t p = 0; p < oHW; ++p) dst[p] = src[p] + bias;
            }
    }
    free(col);
    free(tmp);
}

/* gcol = W^T (CRS x K) * gy[n] (K x oHW); col2im -> gx[n]. */
void or_conv_backward_input(const or_geom* g, const float* gy, const float* w, float* gx,
                            int threads) {
    const int64_t oHW = or_out_h(g) * or_out_w(g);
    const int64_t crs = g->C * g->kH * g->kW;
    float* gcol = (float*)malloc(sizeof(float) * (size_t)(crs * oHW));
    for (int64_t n = 0; n < g->N; ++n) {
        or_gemm_blocked(1, 0, crs, oHW, g->K, 1.0f, w, crs, gy + n * g->K * oHW, oHW, 0.0f, gcol,
                        oHW, threads);
        col2im_from(g, gcol, oHW, 0, gx + n * g->C * g->H * g->W);
    }
    free(gcol);
}

/* SPEC.md:416-424 + Torch accGradParameters (scale, +=). */
void or_conv_backward_weight(const or_geom* g, const float* x, const float* gy, float* gw,
                             float* gb, float scale, int accumulate, int threads) {
    const int64_t oHW = or_out_h(g) * or_out_w(g);
    const int64_t crs = g->C * g->kH * g->kW;
    float* col = (float*)malloc(sizeof(float) * (size_t)(crs * oHW));
    if (!accumulate) {
        memset(gw, 0, sizeof(float) * (size_t)(g->K * crs));
        if (gb) memset(gb, 0, sizeof(float) * (size_t)g->K);
    }
    for (int64_t n = 0; n < g->N; ++n) {
        im2col_into(g, x + n * g->C * g->H * g->W, col, oHW, 0);
        /* gw += scale * gy[n] (K x oHW) * col^T (oHW x CRS) */
        or_gemm_blocked(0, 1, g->K, crs, oHW, scale, gy + n * g->K * oHW, oHW, col, oHW, 1.0f, gw,
                        crs, threads);
        if (gb) {
            for (int64_t k = 0; k < g->K; ++k) {
                const float* row = gy + (n * g->K + k) * oHW;
                float acc = 0.0f;
                for (int64_t p = 0; p < oHW; ++p) acc += row[p];
                gb[k] += scale * acc;
            }
        }
    }
    free(col);
}

/* ---- apply / reduce (reference_backend.cpp) ---- */

/* Logical row-major odometer over one view (reference_backend.cpp:29-63). */
static int64_t view_offset(const or_view* v, int64_t linear) {
    int64_t off = v->offset;
    for (int d = v->ndim - 1; d >= 0; --d) {
        const int64_t idx = linear % v->sizes[d];
        linear /= v->sizes[d];
        off += idx * v->strides[d];
    }
    return off;
}

static int64_t view_numel(const or_view* v) {
    int64_t n = 1;
    for (int d = 0; d < v->ndim; ++d) n *= v->sizes[d];
    return n;
}

static float red_identity(int op) {
    return op == OR_SUM ? 0.0f : (op == OR_MAX ? -INFINITY : INFINITY);
}
static float red_combine(int op, float a, float b) {
    return op == OR_SUM ? a + b : (op == OR_MAX ? fmaxf(a, b) : fminf(a, b));
}

/* reference_backend.cpp:115-127 */
float or_reduce_all(int op, const float* base, const or_view* v) {
    const int64_t n = view_numel(v);
    float acc = red_identity(op);
    for (int64_t i = 0; i < n; ++i) acc = red_combine(op, acc, base[view_offset(v, i)]);
    return acc;
}

/* reference_backend.cpp:129-156 */
void or_reduce_dim(int op, const float* base, const or_view* v, int dim, float* out) {
    or_view outer = *v;
    outer.sizes[dim] = 1;
    const int64_t count = view_numel(&outer);
    for (int64_t o = 0; o < count; ++o) {
        const int64_t start = view_offset(&outer, o);
        float acc = red_identity(op);
        for (int64_t j = 0; j < v->sizes[dim]; ++j)
            acc = red_combine(op, acc, base[start + j * v->strides[dim]]);
        out[o] = acc;
    }
}

/* expression.cpp:340-402 */
static float eval_rpn(const int32_t* code, int32_t ncode, const float* ops, float s) {
    float st[32];
    int top = 0;
    for (int32_t pc = 0; pc < ncode; ++pc) {
        switch (code[pc] & 0xff) {
            case PT_OP_CONST: {
                float c;
                memcpy(&c, &code[++pc], sizeof c);
                st[top++] = c;
                break;
            }
            case PT_OP_X: st[top++] = ops[0]; break;
            case PT_OP_Y: st[top++] = ops[1]; break;
            case PT_OP_Z: st[top++] = ops[2]; break;
            case PT_OP_S: st[top++] = s; break;
            case PT_OP_ADD: --top; st[top - 1] += st[top]; break;
            case PT_OP_SUB: --top; st[top - 1] -= st[top]; break;
            case PT_OP_MUL: --top; st[top - 1] *= st[top]; break;
            case PT_OP_DIV: --top; st[top - 1] /= st[top]; break;
            case PT_OP_NEG: st[top - 1] = -st[top - 1]; break;
            case PT_OP_ABS: st[top - 1] = fabsf(st[top - 1]); break;
            case PT_OP_EXP: st[top - 1] = expf(st[top - 1]); break;
            case PT_OP_LOG: st[top - 1] = logf(st[top - 1]); break;
            case PT_OP_SQRT: st[top - 1] = sqrtf(st[top - 1]); break;
            case PT_OP_TANH: st[top - 1] = tanhf(st[top - 1]); break;
            case PT_OP_MAX: --top; st[top - 1] = fmaxf(st[top - 1], st[top]); break;
            case PT_OP_MIN: --top; st[top - 1] = fminf(st[top - 1], st[top]); break;
            default: return NAN;
        }
    }
    return st[0];
}

/* reference_backend.cpp:80-113: read all operands, evaluate, store to x, logical order. */
void or_apply(const int32_t* code, int32_t ncode, int arity, float* const* bases,
              const or_view* views, float scalar) {
    const int64_t n = view_numel(&views[0]);
    float ops[3] = {0, 0, 0};
    for (int64_t i = 0; i < n; ++i) {
        for (int t = 0; t < arity; ++t) ops[t] = bases[t][view_offset(&views[t], i)];
        bases[0][view_offset(&views[0], i)] = eval_rpn(code, ncode, ops, scalar);
    }
}
