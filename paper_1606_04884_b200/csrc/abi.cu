// abi.cu — the extern "C" boundary of libpt_b200.so (include/pt_b200.h).
// Validation mirrors the reference's checks (conv_geometry.hpp:53-63,
// backend.cpp:115-161); every exception is converted to a status code here.
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "kernels.cuh"
#include "tmap.cuh"

namespace ptb {

std::atomic<int64_t> g_launches{0};

namespace {
thread_local std::string g_last_error;
}  // namespace

void set_last_error(const char* msg) { g_last_error = msg ? msg : ""; }

namespace {

template <class F>
int guarded(F&& f) {
    try {
        f();
        return PT_OK;
    } catch (const AbiError& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return PT_EBACKEND;
    }
}

std::string geom_str(const pt_conv_geom& g) {
    char b[256];
    snprintf(b, sizeof b, "N%lld C%lld H%lld W%lld K%lld k%lldx%lld p%lldx%lld s%lldx%lld",
             (long long)g.N, (long long)g.C, (long long)g.H, (long long)g.W, (long long)g.K,
             (long long)g.kH, (long long)g.kW, (long long)g.padH, (long long)g.padW,
             (long long)g.strideH, (long long)g.strideW);
    return b;
}

void require_math(int math) {
    PTB_REQUIRE(math == PT_MATH_TF32 || math == PT_MATH_FP32 || math == PT_MATH_3XTF32,
                "conv: unknown math mode " + std::to_string(math));
}

void require_ptr(const void* p, const char* what) {
    PTB_REQUIRE(p != nullptr, std::string("conv: null ") + what);
}

void require_view(const pt_view& v, const char* what) {
    PTB_REQUIRE(v.ndim >= 1 && v.ndim <= 8, std::string(what) + ": rank must be 1..8");
    for (int d = 0; d < v.ndim; ++d) {
        PTB_REQUIRE(v.sizes[d] >= 1, std::string(what) + ": sizes must be >= 1");
        PTB_REQUIRE(v.strides[d] >= 0, std::string(what) + ": negative strides unsupported");
    }
    PTB_REQUIRE(v.offset >= 0, std::string(what) + ": negative storage offset");
}

// small-C stride-1 layers: the fused one-read backward (umma_scbwd.cu)
bool sc_on(const Geo& g, int math) { return math == PT_MATH_TF32 && scbwd_ok(g); }

bool fwd_rowconv(const Geo& g, int math) {
    static const bool off = std::getenv("PT_B200_NO_ROWCONV") != nullptr;  // A/B switch for tests
    return math == PT_MATH_TF32 && !off && rowconv_ok(g);
}
size_t fwd_ws(const Geo& g, int math) {
    if (fwd_rowconv(g, math)) return rowconv_workspace(g);
    if (math == PT_MATH_TF32) {
        const UmmaPlan pl = umma_plan(g, false);
        if (pl.ok) return pl.ws_bytes;
    }
    return 0;
}
// small-C stride-1 dgrad: tconv of the row-expanded (kH x 1) layer + 1-D fold
bool dgrad_row(const Geo& g, int math) {
    static const bool off = std::getenv("PT_B200_NO_ROWCONV") != nullptr;
    return math == PT_MATH_TF32 && !off && rowdgrad_ok(g);
}
size_t bwd_data_ws(const Geo& g, int math) {
    if (sc_on(g, math)) return scbwd_workspace(g);
    if (dgrad_row(g, math)) return rowdgrad_workspace(g);
    if (math == PT_MATH_TF32) {
        const UmmaPlan pl = umma_plan(g, true);
        if (pl.ok) return pl.ws_bytes;
    }
    return 0;
}
// updateGradInput body. gyh_pre (gy NHWC, round_up(K,32) channels) is used when the
// chosen engine reads that layout.
void bwd_data_impl(const Geo& g, const float* gy, const float* w, float* gx, int math, void* ws,
                   cudaStream_t st, const float* gyh_pre = nullptr, bool pre_padded = false) {
    PassScope pass("dgrad");
    if (sc_on(g, math)) {
        scbwd(g, nullptr, gy, w, gx, nullptr, nullptr, 1.f, 0, 1.f, 0, ws, st);
        return;
    }
    if (dgrad_row(g, math)) {
        rowdgrad(g, gy, w, gx, ws, st, gyh_pre, pre_padded);
        return;
    }
    if (math == PT_MATH_TF32) {
        const UmmaPlan pl = umma_plan(g, true);
        if (pl.ok) {
            const bool same_layout = pl.cb == 32 && pl.cin_p == umma_wgrad_kp(g);
            umma_conv_bwd_data(g, pl, gy, w, gx, ws, st, same_layout ? gyh_pre : nullptr);
            return;
        }
    }
    simt_conv_bwd_data(g, gy, w, gx, st);
}
// Tensor-core wgrad engines, both fed by gy in NHWC (round_up(K,32) channels):
// the Hankel row kernel for small-C stride-1 layers, else the im2col-TMA kernel.
bool wgrad_row(const Geo& g, int math) {
    static const bool off = std::getenv("PT_B200_NO_ROWCONV") != nullptr;
    return math == PT_MATH_TF32 && !off && rowwgrad_ok(g);
}
bool wgrad_tc(const Geo& g, int math) {
    return math == PT_MATH_TF32 && (wgrad_row(g, math) || umma_wgrad_ok(g));
}
size_t wgrad_tc_ws(const Geo& g, int math) {
    return align_up(wgrad_row(g, math) ? rowwgrad_workspace(g) : umma_wgrad_workspace(g), 256);
}
void wgrad_tc_run(const Geo& g, const float* x, const float* gy, const float* gyh, float* gw, float scale,
                  int accumulate, int math, char* ws, cudaStream_t st, const float* xh_pre = nullptr,
                  int64_t xph = 0, int64_t xpw = 0) {
    PassScope pass("wgrad");
    if (wgrad_row(g, math)) rowwgrad(g, x, gyh, gw, scale, accumulate, ws, st);
    else umma_conv_bwd_filter(g, x, gy, gw, scale, accumulate, ws, st, gyh, xh_pre, -1.0, xph, xpw);
}
size_t gyh_bytes(const Geo& g) { return align_up((size_t)(g.M * umma_wgrad_kp(g)) * 4, 256); }
size_t bias_part_bytes(const Geo& g) { return align_up(nhwc_bias_partials_bytes(g.N, g.K, g.oHW), 256); }
// TF32 wgrad workspace: [gy NHWC + fused gradBias partials][wgrad kernel scratch]
// FP32 wgrad workspace: [split-K partials][gradBias partials]
size_t bwd_filter_ws(const Geo& g, int math) {
    if (sc_on(g, math)) return scbwd_workspace(g);
    if (wgrad_tc(g, math)) return gyh_bytes(g) + bias_part_bytes(g) + wgrad_tc_ws(g, math);
    return align_up(simt_wgrad_workspace(g), 256) + align_up(bias_grad_workspace(g.N, g.K, g.oHW), 256);
}
// Combined backward: one gy NHWC transform (+ fused gradBias) feeds the tensor-core
// wgrad and, when its engine reads the same layout, the dgrad.
bool bwd_shared(const Geo& g, int math) { return wgrad_tc(g, math); }
size_t bwd_ws(const Geo& g, int math) {
    if (sc_on(g, math)) return scbwd_workspace(g);
    if (bwd_shared(g, math))
        return gyh_bytes(g) + bias_part_bytes(g) + align_up(bwd_data_ws(g, math), 256) + wgrad_tc_ws(g, math);
    return std::max(bwd_data_ws(g, math), bwd_filter_ws(g, math));
}

// accGradParameters body; ws laid out as bwd_filter_ws describes. gw takes (scale,
// accumulate), gb takes (bscale, bacc) — equal except under the s2d wrapper, whose remap
// applies the caller's scale to gw.
void bwd_filter_impl(const Geo& g, const float* x, const float* gy, float* gw, float* gb, float scale,
                     int accumulate, int math, char* ws, cudaStream_t st, float bscale, int bacc,
                     const float* xh_pre = nullptr) {
    PassScope pass("wgrad");
    if (sc_on(g, math)) {
        scbwd(g, x, gy, nullptr, nullptr, gw, gb, scale, accumulate, bscale, bacc, ws, st);
        return;
    }
    if (wgrad_tc(g, math)) {
        float* gyh = reinterpret_cast<float*>(ws);
        float* part = reinterpret_cast<float*>(ws + gyh_bytes(g));
        {
            ProfScope prof("layout", st, 0.0, 4.0 * (g.M * g.K + g.M * umma_wgrad_kp(g)));
            nchw_to_nhwc_bias(gy, gyh, g.N, g.K, g.oHW, umma_wgrad_kp(g), gb, bscale, bacc, part, st);
        }
        wgrad_tc_run(g, x, gy, gyh, gw, scale, accumulate, math, ws + gyh_bytes(g) + bias_part_bytes(g),
                     st, xh_pre);
        return;
    }
    simt_conv_bwd_filter(g, x, gy, gw, scale, accumulate, reinterpret_cast<float*>(ws), st);
    if (gb) {
        float* bws = reinterpret_cast<float*>(ws + align_up(simt_wgrad_workspace(g), 256));
        bias_grad(gy, gb, g.N, g.K, g.oHW, bscale, bacc, bws,
                  align_up(bias_grad_workspace(g.N, g.K, g.oHW), 256), st);
    }
}

bool s2d_on(const Geo& g, int math);

// Torch's `finput`: the relaid input updateOutput prepares and accGradParameters reuses.
// Here it is the forward engine's NHWC copy of x, shareable when the weight-gradient
// kernel reads the same layout (32-channel chunks; a Hankel forward's copy carries its
// zero border, which the wgrad im2col descriptor absorbs). 0 = not shareable.
int64_t s2d_fwd_cp(const Geo& g, int math);
size_t finput_layout(const Geo& g, int math, int64_t* ph = nullptr, int64_t* pw = nullptr) {
    if (s2d_on(g, math)) {
        // the space-to-depth input x', NHWC (written by the forward, read by the wgrad)
        const Geo e = s2d_geo(g);
        return s2d_fwd_cp(g, math) ? finput_layout(e, math, ph, pw) : 0;
    }
    if (math != PT_MATH_TF32 || fwd_rowconv(g, math) || wgrad_row(g, math) ||
        !umma_wgrad_ok(g))
        return 0;
    const UmmaPlan pl = umma_plan(g, false);
    if (!pl.ok || pl.cb != 32 || pl.cin_p != (g.C + 31) / 32 * 32) return 0;
    if (ph) *ph = 0;  // every engine keeps x dense (a Hankel border is TMA out-of-bounds fill)
    if (pw) *pw = 0;
    return align_up((size_t)pl.act_elems * 4, 256);
}

void fwd_core(const Geo& g, const float* x, const float* w, const float* b, float* y, int math,
              void* ws, cudaStream_t st, float* finput = nullptr) {
    if (fwd_rowconv(g, math)) {
        rowconv_fwd(g, x, w, b, y, ws, st);
        return;
    }
    if (math == PT_MATH_TF32) {
        const UmmaPlan pl = umma_plan(g, false);
        if (pl.ok) {
            umma_conv_fwd(g, pl, x, w, b, y, ws, st,
                          finput && finput_layout(g, math) ? finput : nullptr);
            return;
        }
    }
    simt_conv_fwd(g, x, w, b, y, st);
}

// ---- strided small-C layers: space-to-depth into a stride-1 conv (s2d.cu) ----
bool s2d_on(const Geo& g, int math) {
    static const bool off = std::getenv("PT_B200_NO_S2D") != nullptr;  // A/B switch
    return math == PT_MATH_TF32 && !off && s2d_applies(g);
}
size_t s2d_x_bytes(const Geo& g) {  // x' as NCHW or as NHWC with 32-padded channels
    const Geo e = s2d_geo(g);
    return align_up((size_t)(e.N * (e.C + 31) / 32 * 32 * e.HW) * 4, 256);
}
// Cp of the NHWC x' the stride-1 plan reads when s2d_input_nhwc can write it directly
// (32-channel-chunk tensor-core plan), else 0 (x' as NCHW, relaid by the engine).
int64_t s2d_fwd_cp(const Geo& g, int math) {
    const Geo e = s2d_geo(g);
    if (fwd_rowconv(e, math)) return 0;
    const UmmaPlan pl = umma_plan(e, false);
    if (!pl.ok || pl.cb != 32 || !s2d_nhwc_ok(g, pl.cin_p)) return 0;
    return pl.cin_p;
}
size_t s2d_w_bytes(const Geo& g) {
    const Geo e = s2d_geo(g);
    return align_up((size_t)(e.K * e.CRS) * 4, 256);
}
size_t fwd_ws_top(const Geo& g, int math) {
    if (s2d_on(g, math)) return s2d_x_bytes(g) + s2d_w_bytes(g) + fwd_ws(s2d_geo(g), math);
    return fwd_ws(g, math);
}
size_t bwd_data_ws_top(const Geo& g, int math) {
    if (s2d_on(g, math)) return s2d_w_bytes(g) + s2d_x_bytes(g) + bwd_data_ws(s2d_geo(g), math);
    return bwd_data_ws(g, math);
}
size_t bwd_filter_ws_top(const Geo& g, int math) {
    if (s2d_on(g, math)) return s2d_x_bytes(g) + s2d_w_bytes(g) + bwd_filter_ws(s2d_geo(g), math);
    return bwd_filter_ws(g, math);
}
size_t bwd_ws_top(const Geo& g, int math) {
    if (s2d_on(g, math)) return 2 * s2d_x_bytes(g) + 2 * s2d_w_bytes(g) + bwd_ws(s2d_geo(g), math);
    return bwd_ws(g, math);
}

void require_ws(size_t have, size_t need, const void* ws) {
    PTB_REQUIRE(have >= need && (need == 0 || ws != nullptr),
                "conv: workspace too small (" + std::to_string(have) + " < " +
                    std::to_string(need) + " bytes)");
    PTB_REQUIRE((reinterpret_cast<uintptr_t>(ws) & 255) == 0, "conv: workspace must be 256-byte aligned");
}

// Combined backward body (pt_b200_conv_bwd). inner_gw_plain: write gw with unit scale and
// overwrite (the s2d wrapper applies the caller's scale / accumulate in its remap) while
// gradBias still takes the caller's scale / accumulate.
// The combined backward runs the weight gradient on an internal stream (Fork slot 0)
// concurrently with the input gradient: they only share the transformed gy, and each
// kernel's last partial wave then overlaps the other's (each is a persistent kernel sized
// to the whole GPU). pt_b200_set_bwd_streams(0) serialises (the bench's per-launch timing
// pass).
void bwd_core(const Geo& g, const float* x, const float* gy, const float* w, float* gx, float* gw,
              float* gb, float scale, int accumulate, int math, char* ws, cudaStream_t st,
              bool inner_gw_plain, const float* finput = nullptr) {
    int64_t fph = 0, fpw = 0;
    if (finput && !finput_layout(g, math, &fph, &fpw)) finput = nullptr;
    char* base = ws;
    if (gx && gw && sc_on(g, math)) {  // one gy read for gradInput, gradWeight and gradBias
        PassScope pass("bwd");
        if (inner_gw_plain) scbwd(g, x, gy, w, gx, gw, gb, 1.f, 0, scale, accumulate, ws, st);
        else scbwd(g, x, gy, w, gx, gw, gb, scale, accumulate, scale, accumulate, ws, st);
        return;
    }
    if (gx && gw && bwd_shared(g, math)) {
        // one gy NHWC transform (+ fused gradBias) feeds both tensor-core passes
        float* gyh = reinterpret_cast<float*>(base);
        float* part = reinterpret_cast<float*>(base + gyh_bytes(g));
        char* dws = base + gyh_bytes(g) + bias_part_bytes(g);
        char* wws = dws + align_up(bwd_data_ws(g, math), 256);
        {
            PassScope pass("bwd");
            ProfScope prof("layout", st, 0.0, 4.0 * (g.M * g.K + g.M * umma_wgrad_kp(g)));
            nchw_to_nhwc_bias(gy, gyh, g.N, g.K, g.oHW, umma_wgrad_kp(g), gb, scale, accumulate, part,
                              st, /*defer_bias=*/true);
        }
        Fork fk(st, 0);  // fork: the weight gradient waits for the gy transform only
        if (inner_gw_plain) wgrad_tc_run(g, x, gy, gyh, gw, 1.f, 0, math, wws, fk.side, finput, fph, fpw);
        else wgrad_tc_run(g, x, gy, gyh, gw, scale, accumulate, math, wws, fk.side, finput, fph, fpw);
        // gradBias from the transform's partials, behind the weight gradient on the side
        // stream: off the input gradient's path
        if (gb) bias_from_nhwc_partials(part, g.N, g.K, g.oHW, gb, scale, accumulate, fk.side);
        bwd_data_impl(g, gy, w, gx, math, dws, st, gyh);
        fk.join();  // the caller's stream sees both gradients
        return;
    }
    if (gx) bwd_data_impl(g, gy, w, gx, math, ws, st);
    if (gw) {
        if (inner_gw_plain)
            bwd_filter_impl(g, x, gy, gw, gb, 1.f, 0, math, base, st, scale, accumulate, finput);
        else
            bwd_filter_impl(g, x, gy, gw, gb, scale, accumulate, math, base, st, scale, accumulate, finput);
    }
}


}  // namespace

void validate_geom(const pt_conv_geom* gp) {
    PTB_REQUIRE(gp != nullptr, "conv geometry: null");
    const pt_conv_geom& g = *gp;
    PTB_REQUIRE(g.N >= 1 && g.C >= 1 && g.H >= 1 && g.W >= 1 && g.K >= 1 && g.kH >= 1 &&
                    g.kW >= 1 && g.strideH >= 1 && g.strideW >= 1,
                "conv geometry: counts, dims, kernel and stride must be >= 1");
    PTB_REQUIRE(g.padH >= 0 && g.padW >= 0, "conv geometry: padding must be >= 0");
    PTB_REQUIRE(g.kH <= g.H + 2 * g.padH && g.kW <= g.W + 2 * g.padW,
                "conv geometry: kernel exceeds padded input (" + geom_str(g) + ")");
    const Geo d(g);
    PTB_REQUIRE(d.oH >= 1 && d.oW >= 1, "conv geometry: empty output (" + geom_str(g) + ")");
    // device kernels index spatial/channel extents in 32-bit
    PTB_REQUIRE(g.C < (1 << 24) && g.K < (1 << 24) && g.H < (1 << 20) && g.W < (1 << 20) &&
                    g.kH < 4096 && g.kW < 4096 && d.M < (1ll << 31),
                "conv geometry: extents exceed device limits (" + geom_str(g) + ")");
}

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && cached[dev]) return cached[dev];
    int n = 148;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) n = 148;
    if (dev >= 0 && dev < 64) cached[dev] = n;
    return n;
}


void fwd_top(const Geo& g, const float* x, const float* w, const float* b, float* y, int math, void* ws,
             cudaStream_t st, float* finput);
void bwd_data_top(const Geo& g, const float* gy, const float* w, float* gx, int math, void* ws, cudaStream_t st);
void bwd_filter_top(const Geo& g, const float* x, const float* gy, float* gw, float* gb, float scale,
                    int accumulate, int math, void* ws, cudaStream_t st);

// Top-level bodies of the conv entry points (space-to-depth wrapper, then the engines).
void fwd_top(const Geo& g, const float* x, const float* w, const float* b, float* y, int math, void* ws,
             cudaStream_t st, float* finput) {
    {
        if (s2d_on(g, math)) {
            const Geo e = s2d_geo(g);
            char* base = reinterpret_cast<char*>(ws);
            float* xs = reinterpret_cast<float*>(base);
            float* wsd = reinterpret_cast<float*>(base + s2d_x_bytes(g));
            char* inner = base + s2d_x_bytes(g) + s2d_w_bytes(g);
            if (const int64_t cp = s2d_fwd_cp(g, math)) {
                // x' straight into the engine's NHWC layout (into finput when shareable)
                float* xh = finput && finput_layout(g, math) ? finput : xs;
                s2d_input_nhwc(g, x, xh, cp, st);
                s2d_weight(g, w, wsd, st);
                umma_conv_fwd(e, umma_plan(e, false), nullptr, wsd, b, y, inner, st, xh, true);
                return;
            }
            s2d_input(g, x, xs, st);
            s2d_weight(g, w, wsd, st);
            fwd_core(e, xs, wsd, b, y, math, inner, st);
            return;
        }
        fwd_core(g, x, w, b, y, math, ws, st, finput);
    }
}

void bwd_data_top(const Geo& g, const float* gy, const float* w, float* gx, int math, void* ws, cudaStream_t st) {
    if (s2d_on(g, math)) {
        const Geo e = s2d_geo(g);
        char* base = reinterpret_cast<char*>(ws);
        float* wsd = reinterpret_cast<float*>(base);
        float* gxs = reinterpret_cast<float*>(base + s2d_w_bytes(g));
        s2d_weight(g, w, wsd, st);
        bwd_data_impl(e, gy, wsd, gxs, math, base + s2d_w_bytes(g) + s2d_x_bytes(g), st);
        d2s_grad(g, gxs, gx, st);
        return;
    }
    bwd_data_impl(g, gy, w, gx, math, ws, st);
}

void bwd_filter_top(const Geo& g, const float* x, const float* gy, float* gw, float* gb, float scale,
                    int accumulate, int math, void* ws, cudaStream_t st) {
    if (s2d_on(g, math)) {
        const Geo e = s2d_geo(g);
        char* base = reinterpret_cast<char*>(ws);
        float* xs = reinterpret_cast<float*>(base);
        float* gws = reinterpret_cast<float*>(base + s2d_x_bytes(g));
        const int64_t cp = finput_layout(g, math) ? s2d_fwd_cp(g, math) : 0;
        if (cp) s2d_input_nhwc(g, x, xs, cp, st);
        else s2d_input(g, x, xs, st);
        bwd_filter_impl(e, xs, gy, gws, gb, 1.f, 0, math, base + s2d_x_bytes(g) + s2d_w_bytes(g), st,
                        scale, accumulate, cp ? xs : nullptr);
        d2s_weight_grad(g, gws, gw, scale, accumulate, st);
        return;
    }
    bwd_filter_impl(g, x, gy, gw, gb, scale, accumulate, math, reinterpret_cast<char*>(ws), st, scale,
                    accumulate);
}

// ---- 3xTF32 (split3.cu): the TF32 engines over a 3x reduction ----
namespace {
constexpr int kHiLoHi = 2, kHiHiLo = 4;  // split3 patterns (bit b set: block b holds lo)
enum Axis { kAxisC, kAxisK, kAxisN };
Geo scaled3(const Geo& g, Axis a) {
    pt_conv_geom e{g.N, g.C, g.H, g.W, g.K, g.kH, g.kW, g.pH, g.pW, g.sH, g.sW};
    if (a == kAxisC) e.C *= 3;
    if (a == kAxisK) e.K *= 3;
    if (a == kAxisN) e.N *= 3;
    validate_geom(&e);
    return Geo(e);
}
size_t fbytes(int64_t n) { return align_up((size_t)n * 4, 256); }
// [x3 | w3 | inner(C' = 3C)]
size_t fwd_3x_ws(const Geo& g) {
    return fbytes(3 * g.N * g.C * g.HW) + fbytes(3 * g.K * g.CRS) + fwd_ws_top(scaled3(g, kAxisC), PT_MATH_TF32);
}
// [gy3 | w3 | inner(K' = 3K)]
size_t bwd_data_3x_ws(const Geo& g) {
    return fbytes(3 * g.M * g.K) + fbytes(3 * g.K * g.CRS) + bwd_data_ws_top(scaled3(g, kAxisK), PT_MATH_TF32);
}
// [x3 | gy3 | gradBias scratch | inner(N' = 3N)]
size_t bwd_filter_3x_ws(const Geo& g) {
    return fbytes(3 * g.N * g.C * g.HW) + fbytes(3 * g.M * g.K) + align_up(bias_grad_workspace(g.N, g.K, g.oHW), 256) +
           bwd_filter_ws_top(scaled3(g, kAxisN), PT_MATH_TF32);
}
}  // namespace

size_t ws_3x(const Geo& g, int op) {
    switch (op) {
        case PT_CONV_FWD: return fwd_3x_ws(g);
        case PT_CONV_BWD_DATA: return bwd_data_3x_ws(g);
        case PT_CONV_BWD_FILTER: return bwd_filter_3x_ws(g);
        default: return std::max(bwd_data_3x_ws(g), bwd_filter_3x_ws(g));
    }
}

// y = conv([x_hi | x_lo | x_hi], [w_hi | w_hi | w_lo]) + b over 3C input channels
void fwd_3x(const Geo& g, const float* x, const float* w, const float* b, float* y, char* ws, cudaStream_t st) {
    const Geo e = scaled3(g, kAxisC);
    float* x3 = reinterpret_cast<float*>(ws);
    float* w3 = reinterpret_cast<float*>(ws + fbytes(3 * g.N * g.C * g.HW));
    char* inner = ws + fbytes(3 * g.N * g.C * g.HW) + fbytes(3 * g.K * g.CRS);
    split3(x, x3, g.N, g.C * g.HW, kHiLoHi, st);
    split3(w, w3, g.K, g.CRS, kHiHiLo, st);
    fwd_top(e, x3, w3, b, y, PT_MATH_TF32, inner, st, nullptr);
}

// gx = tconv([gy_hi | gy_lo | gy_hi], [w_hi ; w_hi ; w_lo]) over 3K gradient channels
void bwd_data_3x(const Geo& g, const float* gy, const float* w, float* gx, char* ws, cudaStream_t st) {
    const Geo e = scaled3(g, kAxisK);
    float* gy3 = reinterpret_cast<float*>(ws);
    float* w3 = reinterpret_cast<float*>(ws + fbytes(3 * g.M * g.K));
    char* inner = ws + fbytes(3 * g.M * g.K) + fbytes(3 * g.K * g.CRS);
    split3(gy, gy3, g.N, g.K * g.oHW, kHiLoHi, st);
    split3(w, w3, 1, g.K * g.CRS, kHiHiLo, st);
    bwd_data_top(e, gy3, w3, gx, PT_MATH_TF32, inner, st);
}

// gw (+)= scale * wgrad([x_hi ; x_hi ; x_lo], [gy_hi ; gy_lo ; gy_hi]) over 3N images;
// gradBias from gy itself (fixed-order FP32 reduction)
void bwd_filter_3x(const Geo& g, const float* x, const float* gy, float* gw, float* gb, float scale, int accumulate,
                   char* ws, cudaStream_t st) {
    const Geo e = scaled3(g, kAxisN);
    const size_t xb = fbytes(3 * g.N * g.C * g.HW), gb3 = fbytes(3 * g.M * g.K);
    const size_t bb = align_up(bias_grad_workspace(g.N, g.K, g.oHW), 256);
    float* x3 = reinterpret_cast<float*>(ws);
    float* gy3 = reinterpret_cast<float*>(ws + xb);
    float* bws = reinterpret_cast<float*>(ws + xb + gb3);
    char* inner = ws + xb + gb3 + bb;
    split3(x, x3, 1, g.N * g.C * g.HW, kHiHiLo, st);
    split3(gy, gy3, 1, g.M * g.K, kHiLoHi, st);
    bwd_filter_top(e, x3, gy3, gw, nullptr, scale, accumulate, PT_MATH_TF32, inner, st);
    if (gb) bias_grad(gy, gb, g.N, g.K, g.oHW, scale, accumulate, bws, bb, st);
}

}  // namespace ptb

using namespace ptb;

extern "C" {

int pt_b200_abi_version(void) { return PT_B200_ABI_VERSION; }

const char* pt_b200_last_error(void) { return g_last_error.c_str(); }

int pt_b200_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int usable = 0;
    for (int i = 0; i < n; ++i) {
        cudaDeviceProp p;
        if (cudaGetDeviceProperties(&p, i) == cudaSuccess && p.major == 10 && p.minor == 0) ++usable;
    }
    return usable;
}

int pt_b200_device_info(int device, pt_device_desc* out) {
    return guarded([&] {
        PTB_REQUIRE(out != nullptr, "device_info: null output");
        cudaDeviceProp p;
        PTB_CUDA(cudaGetDeviceProperties(&p, device));
        memset(out, 0, sizeof *out);
        snprintf(out->name, sizeof out->name, "b200:%d", device);
        out->maxWorkgroupSize = p.maxThreadsPerBlock;
        out->localMemBytes = (int64_t)p.sharedMemPerBlockOptin;
        out->smCount = p.multiProcessorCount;
        out->ccMajor = p.major;
        out->ccMinor = p.minor;
        out->globalMemBytes = (int64_t)p.totalGlobalMem;
    });
}

int pt_b200_set_device(int device) { return guarded([&] { PTB_CUDA(cudaSetDevice(device)); }); }
int pt_b200_get_device(int* device) {
    return guarded([&] {
        PTB_REQUIRE(device != nullptr, "get_device: null output");
        PTB_CUDA(cudaGetDevice(device));
    });
}

int pt_b200_malloc(void** ptr, size_t bytes) {
    return guarded([&] {
        PTB_REQUIRE(ptr != nullptr, "malloc: null output");
        *ptr = nullptr;
        if (bytes) PTB_CUDA(cudaMalloc(ptr, bytes));
    });
}

int pt_b200_free(void* ptr) { return guarded([&] { if (ptr) PTB_CUDA(cudaFree(ptr)); }); }

int pt_b200_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream) {
    return guarded([&] {
        if (bytes) PTB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, as_stream(stream)));
    });
}

int pt_b200_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream) {
    return guarded([&] {
        if (bytes) PTB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, as_stream(stream)));
    });
}

int pt_b200_stream_query(void* stream) {
    const cudaError_t e = cudaStreamQuery(as_stream(stream));
    if (e == cudaSuccess) return PT_OK;
    if (e == cudaErrorNotReady) return 1;
    set_last_error(cudaGetErrorString(e));
    return PT_EBACKEND;
}

int pt_b200_stream_sync(void* stream) {
    return guarded([&] { PTB_CUDA(cudaStreamSynchronize(as_stream(stream))); });
}

int pt_b200_fill_uniform(float* dst, int64_t n, uint64_t seed, float lo, float hi, void* stream) {
    return guarded([&] {
        PTB_REQUIRE(n >= 0 && (n == 0 || dst), "fill_uniform: bad arguments");
        fill_uniform(dst, n, seed, lo, hi, as_stream(stream));
    });
}

int pt_b200_conv_validate(const pt_conv_geom* g) { return guarded([&] { validate_geom(g); }); }

size_t pt_b200_conv_workspace_bytes(const pt_conv_geom* gp, int op, int math) {
    size_t r = 0;
    const int st = guarded([&] {
        validate_geom(gp);
        require_math(math);
        const Geo g(*gp);
        if (op < PT_CONV_FWD || op > PT_CONV_BWD) fail_validation("workspace: unknown conv op " + std::to_string(op));
        if (math == PT_MATH_3XTF32) {
            r = ws_3x(g, op);
            return;
        }
        switch (op) {
            case PT_CONV_FWD: r = fwd_ws_top(g, math); break;
            case PT_CONV_BWD_DATA: r = bwd_data_ws_top(g, math); break;
            case PT_CONV_BWD_FILTER: r = bwd_filter_ws_top(g, math); break;
            default: r = bwd_ws_top(g, math); break;
        }
    });
    return st == PT_OK ? r : (size_t)-1;
}

static int conv_fwd_entry(const pt_conv_geom* gp, const float* x, const float* w, const float* b,
                          float* y, int math, void* ws, size_t ws_bytes, float* finput, void* stream) {
    return guarded([&] {
        validate_geom(gp);
        require_math(math);
        require_ptr(x, "input");
        require_ptr(w, "weight");
        require_ptr(y, "output");
        const Geo g(*gp);
        cudaStream_t st = as_stream(stream);
        PassScope pass("fwd");
        if (math == PT_MATH_3XTF32) {
            require_ws(ws_bytes, ws_3x(g, PT_CONV_FWD), ws);
            fwd_3x(g, x, w, b, y, reinterpret_cast<char*>(ws), st);
            return;
        }
        require_ws(ws_bytes, fwd_ws_top(g, math), ws);
        fwd_top(g, x, w, b, y, math, ws, st, finput);
    });
}


int pt_b200_conv_fwd(const pt_conv_geom* gp, const float* x, const float* w, const float* b,
                     float* y, int math, void* ws, size_t ws_bytes, void* stream) {
    return conv_fwd_entry(gp, x, w, b, y, math, ws, ws_bytes, nullptr, stream);
}

int pt_b200_conv_fwd_finput(const pt_conv_geom* gp, const float* x, const float* w, const float* b,
                            float* y, int math, void* ws, size_t ws_bytes, float* finput, void* stream) {
    return conv_fwd_entry(gp, x, w, b, y, math, ws, ws_bytes, finput, stream);
}

size_t pt_b200_conv_finput_bytes(const pt_conv_geom* gp, int math) {
    size_t r = 0;
    const int st = guarded([&] {
        validate_geom(gp);
        require_math(math);
        r = finput_layout(Geo(*gp), math);
    });
    return st == PT_OK ? r : 0;
}

size_t pt_b200_winograd_workspace_bytes(const pt_conv_geom* gp, int op) {
    size_t r = 0;
    const int st = guarded([&] {
        validate_geom(gp);
        const Geo g(*gp);
        PTB_REQUIRE(op == PT_CONV_FWD || op == PT_CONV_BWD_DATA, "winograd: op must be FWD or BWD_DATA");
        PTB_REQUIRE(winograd_applies(g, op), "winograd: unsupported geometry " + geom_str(*gp) +
                                                 " (3x3 stride 1; padding <= 2 for gradInput)");
        r = winograd_workspace(g, op);
    });
    return st == PT_OK ? r : (size_t)-1;
}

int pt_b200_conv_fwd_winograd(const pt_conv_geom* gp, const float* x, const float* w, const float* b,
                              float* y, void* ws, size_t ws_bytes, void* stream) {
    return guarded([&] {
        validate_geom(gp);
        require_ptr(x, "input");
        require_ptr(w, "weight");
        require_ptr(y, "output");
        const Geo g(*gp);
        PTB_REQUIRE(winograd_applies(g, PT_CONV_FWD),
                    "winograd: unsupported geometry " + geom_str(*gp) + " (3x3 stride 1 only)");
        require_ws(ws_bytes, winograd_workspace(g, PT_CONV_FWD), ws);
        winograd_fwd(g, x, w, b, y, ws, as_stream(stream));
    });
}

int pt_b200_conv_bwd_data_winograd(const pt_conv_geom* gp, const float* gy, const float* w, float* gx,
                                   void* ws, size_t ws_bytes, void* stream) {
    return guarded([&] {
        validate_geom(gp);
        require_ptr(gy, "gradOutput");
        require_ptr(w, "weight");
        require_ptr(gx, "gradInput");
        const Geo g(*gp);
        PTB_REQUIRE(winograd_applies(g, PT_CONV_BWD_DATA),
                    "winograd: unsupported geometry " + geom_str(*gp) + " (3x3 stride 1, padding <= 2)");
        require_ws(ws_bytes, winograd_workspace(g, PT_CONV_BWD_DATA), ws);
        winograd_bwd_data(g, gy, w, gx, ws, as_stream(stream));
    });
}

int pt_b200_conv_bwd_data(const pt_conv_geom* gp, const float* gy, const float* w, float* gx,
                          int math, void* ws, size_t ws_bytes, void* stream) {
    return guarded([&] {
        validate_geom(gp);
        require_math(math);
        require_ptr(gy, "gradOutput");
        require_ptr(w, "weight");
        require_ptr(gx, "gradInput");
        const Geo g(*gp);
        cudaStream_t st = as_stream(stream);
        if (math == PT_MATH_3XTF32) {
            require_ws(ws_bytes, ws_3x(g, PT_CONV_BWD_DATA), ws);
            bwd_data_3x(g, gy, w, gx, reinterpret_cast<char*>(ws), st);
            return;
        }
        require_ws(ws_bytes, bwd_data_ws_top(g, math), ws);
        bwd_data_top(g, gy, w, gx, math, ws, st);
    });
}


int pt_b200_conv_bwd_filter(const pt_conv_geom* gp, const float* x, const float* gy, float* gw,
                            float* gb, float scale, int accumulate, int math, void* ws,
                            size_t ws_bytes, void* stream) {
    return guarded([&] {
        validate_geom(gp);
        require_math(math);
        require_ptr(x, "input");
        require_ptr(gy, "gradOutput");
        require_ptr(gw, "gradWeight");
        const Geo g(*gp);
        cudaStream_t st = as_stream(stream);
        if (math == PT_MATH_3XTF32) {
            require_ws(ws_bytes, ws_3x(g, PT_CONV_BWD_FILTER), ws);
            bwd_filter_3x(g, x, gy, gw, gb, scale, accumulate, reinterpret_cast<char*>(ws), st);
            return;
        }
        require_ws(ws_bytes, bwd_filter_ws_top(g, math), ws);
        bwd_filter_top(g, x, gy, gw, gb, scale, accumulate, math, ws, st);
    });
}


static int conv_bwd_entry(const pt_conv_geom* gp, const float* x, const float* gy, const float* w,
                          float* gx, float* gw, float* gb, float scale, int accumulate, int math,
                          void* ws, size_t ws_bytes, const float* finput, void* stream) {
    return guarded([&] {
        validate_geom(gp);
        require_math(math);
        require_ptr(gy, "gradOutput");
        PTB_REQUIRE(gx || gw, "conv bwd: nothing to compute (gradInput and gradWeight both null)");
        if (gx) require_ptr(w, "weight");
        if (gw) require_ptr(x, "input");
        const Geo g(*gp);
        cudaStream_t st = as_stream(stream);
        if (math == PT_MATH_3XTF32) {
            require_ws(ws_bytes, ws_3x(g, PT_CONV_BWD), ws);
            // the two products are independent 3x problems; the gradient parts run in turn
            if (gx) bwd_data_3x(g, gy, w, gx, reinterpret_cast<char*>(ws), st);
            if (gw) bwd_filter_3x(g, x, gy, gw, gb, scale, accumulate, reinterpret_cast<char*>(ws), st);
            return;
        }
        require_ws(ws_bytes, bwd_ws_top(g, math), ws);
        if (s2d_on(g, math)) {
            const Geo e = s2d_geo(g);
            char* base = reinterpret_cast<char*>(ws);
            float* xs = reinterpret_cast<float*>(base);
            float* wsd = reinterpret_cast<float*>(base + s2d_x_bytes(g));
            float* gxs = reinterpret_cast<float*>(base + s2d_x_bytes(g) + s2d_w_bytes(g));
            float* gws = reinterpret_cast<float*>(base + 2 * s2d_x_bytes(g) + s2d_w_bytes(g));
            char* inner = base + 2 * s2d_x_bytes(g) + 2 * s2d_w_bytes(g);
            // x' for the wgrad: the forward's NHWC copy (finput), else made here
            const float* xh = nullptr;
            if (gw && finput_layout(g, math)) {
                if (finput) {
                    xh = finput;
                } else {
                    s2d_input_nhwc(g, x, xs, s2d_fwd_cp(g, math), st);
                    xh = xs;
                }
            } else if (gw) {
                s2d_input(g, x, xs, st);
            }
            if (gx) s2d_weight(g, w, wsd, st);
            bwd_core(e, xs, gy, wsd, gx ? gxs : nullptr, gw ? gws : nullptr, gb, scale, accumulate, math,
                     inner, st, /*inner_gw_plain=*/true, xh);
            if (gx) d2s_grad(g, gxs, gx, st);
            if (gw) d2s_weight_grad(g, gws, gw, scale, accumulate, st);
            return;
        }
        bwd_core(g, x, gy, w, gx, gw, gb, scale, accumulate, math, reinterpret_cast<char*>(ws), st, false,
                 finput);
    });
}

int pt_b200_set_bwd_streams(int on) {
    set_concurrency(on);
    return PT_OK;
}

int pt_b200_conv_bwd(const pt_conv_geom* gp, const float* x, const float* gy, const float* w,
                     float* gx, float* gw, float* gb, float scale, int accumulate, int math,
                     void* ws, size_t ws_bytes, void* stream) {
    return conv_bwd_entry(gp, x, gy, w, gx, gw, gb, scale, accumulate, math, ws, ws_bytes, nullptr,
                          stream);
}

int pt_b200_conv_bwd_finput(const pt_conv_geom* gp, const float* x, const float* gy, const float* w,
                            float* gx, float* gw, float* gb, float scale, int accumulate, int math,
                            void* ws, size_t ws_bytes, const float* finput, void* stream) {
    return conv_bwd_entry(gp, x, gy, w, gx, gw, gb, scale, accumulate, math, ws, ws_bytes, finput,
                          stream);
}

int pt_b200_im2col(const pt_conv_geom* gp, const float* img, float* col, void* stream) {
    return guarded([&] {
        validate_geom(gp);
        require_ptr(img, "image");
        require_ptr(col, "columns");
        im2col_launch(Geo(*gp), img, 0, 1, col, as_stream(stream));
    });
}

int pt_b200_im2col_batched(const pt_conv_geom* gp, const float* x, int64_t n0, int64_t count,
                           float* col, void* stream) {
    return guarded([&] {
        validate_geom(gp);
        require_ptr(x, "input");
        require_ptr(col, "columns");
        PTB_REQUIRE(count >= 1 && n0 >= 0 && n0 + count <= gp->N,
                    "im2col_batched: invalid batch chunk");
        im2col_launch(Geo(*gp), x, n0, count, col, as_stream(stream));
    });
}

int pt_b200_col2im(const pt_conv_geom* gp, const float* col, float* img, void* stream) {
    return guarded([&] {
        validate_geom(gp);
        require_ptr(img, "image");
        require_ptr(col, "columns");
        col2im_launch(Geo(*gp), col, img, as_stream(stream));
    });
}

int pt_b200_gemm(int transA, int transB, int64_t M, int64_t N, int64_t K, float alpha,
                 const float* A, int64_t lda, const float* B, int64_t ldb, float beta, float* C,
                 int64_t ldc, int math, void* stream) {
    return guarded([&] {
        require_math(math);
        PTB_REQUIRE(math != PT_MATH_3XTF32, "gemm: math 3xtf32 is a convolution mode (use tf32 or fp32)");
        PTB_REQUIRE(M >= 1 && N >= 1 && K >= 1, "gemm: dims must be >= 1");
        PTB_REQUIRE(lda >= (transA ? M : K) && ldb >= (transB ? K : N) && ldc >= N,
                    "gemm: leading dimensions smaller than the matrix extent");
        PTB_REQUIRE(A && B && C, "gemm: null matrix");
        PTB_REQUIRE(M < (1ll << 31) / 64 * 64, "gemm: M too large");
        if (math == PT_MATH_FP32) {
            simt_gemm(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, as_stream(stream));
            return;
        }
        // TF32: the tcgen05 GEMM computes C^T's columns as its rows (D[n][m] with m = C's
        // column j, n = C's row i): its A operand is op(B) (row j, K-major iff transB), its
        // B operand is op(A) (row i, K-major iff !transA), D = C with ldd = ldc.
        UmmaGemm gm{};
        gm.a = B;
        gm.b = A;
        gm.d = C;
        gm.M = N;
        gm.N = M;
        gm.K = K;
        gm.batch = 1;
        gm.a_mn = !transB;
        gm.b_mn = transA != 0;
        gm.lda = ldb;
        gm.ldb = lda;
        gm.ldd = ldc;
        gm.alpha = alpha;
        gm.beta = beta;
        umma_gemm(gm, as_stream(stream));
    });
}

int pt_b200_apply(const int32_t* code, int32_t ncode, int arity, float* const* bases,
                  const pt_view* views, float scalar, void* stream) {
    return guarded([&] {
        PTB_REQUIRE(arity >= 1 && arity <= 3, "apply takes 1..3 operands, got " + std::to_string(arity));
        PTB_REQUIRE(code && bases && views, "apply: null argument");
        for (int t = 0; t < arity; ++t) {
            require_view(views[t], "apply operand");
            PTB_REQUIRE(bases[t] != nullptr, "apply operand is undefined");
            PTB_REQUIRE(views[t].ndim == views[0].ndim, "apply operands must share sizes");
            for (int d = 0; d < views[0].ndim; ++d)
                PTB_REQUIRE(views[t].sizes[d] == views[0].sizes[d], "apply operands must share sizes");
        }
        // stack discipline check (the program must leave exactly one value)
        int depth = 0;
        for (int32_t pc = 0; pc < ncode; ++pc) {
            const int op = code[pc] & 0xff;
            if (op == PT_OP_CONST) { ++depth; ++pc; }
            else if (op >= PT_OP_X && op <= PT_OP_S) {
                PTB_REQUIRE(op - PT_OP_X < arity || op == PT_OP_S, "apply: operand beyond arity");
                ++depth;
            } else if (op == PT_OP_ADD || op == PT_OP_SUB || op == PT_OP_MUL || op == PT_OP_DIV ||
                       op == PT_OP_MAX || op == PT_OP_MIN) --depth;
            else PTB_REQUIRE(op >= PT_OP_NEG && op <= PT_OP_TANH, "apply: bad opcode");
            PTB_REQUIRE(depth >= 1 && depth <= 32, "apply: malformed program");
        }
        PTB_REQUIRE(depth == 1, "apply: malformed program");
        apply_launch(code, ncode, arity, bases, views, scalar, as_stream(stream));
    });
}

int pt_b200_bias_add(float* y, const float* b, int64_t N, int64_t K, int64_t HW, void* stream) {
    return guarded([&] {
        PTB_REQUIRE(y && b && N >= 1 && K >= 1 && HW >= 1, "bias_add: bad arguments");
        bias_add_launch(y, b, N, K, HW, as_stream(stream));
    });
}

int pt_b200_relu_fwd(const float* x, float* y, int64_t n, void* stream) {
    return guarded([&] {
        PTB_REQUIRE(x && y && n >= 1, "relu: bad arguments");
        relu_fwd(x, y, n, as_stream(stream));
    });
}

int pt_b200_relu_bwd(const float* y, const float* gy, float* gx, int64_t n, void* stream) {
    return guarded([&] {
        PTB_REQUIRE(y && gy && gx && n >= 1, "relu backward: bad arguments");
        relu_bwd(y, gy, gx, n, as_stream(stream));
    });
}

int pt_b200_maxpool_fwd(const float* x, float* y, int32_t* argmax, int64_t N, int64_t C, int64_t H,
                        int64_t W, int kH, int kW, int sH, int sW, int pH, int pW, void* stream) {
    return guarded([&] {
        PTB_REQUIRE(x && y, "maxpool: null tensor");
        maxpool_fwd(x, y, argmax, N, C, H, W, kH, kW, sH, sW, pH, pW, as_stream(stream));
    });
}

int pt_b200_maxpool_bwd(const float* gy, const int32_t* argmax, float* gx, int64_t N, int64_t C,
                        int64_t H, int64_t W, int kH, int kW, int sH, int sW, int pH, int pW,
                        void* stream) {
    return guarded([&] {
        PTB_REQUIRE(gy && argmax && gx, "maxpool backward: null tensor");
        maxpool_bwd(gy, argmax, gx, N, C, H, W, kH, kW, sH, sW, pH, pW, as_stream(stream));
    });
}

int pt_b200_reduce_all(int op, const float* base, const pt_view* view, float* out_dev, void* stream) {
    return guarded([&] {
        PTB_REQUIRE(op >= 0 && op <= 2, "reduce: unknown op");
        PTB_REQUIRE(base && view && out_dev, "reduce on an undefined tensor");
        require_view(*view, "reduce");
        reduce_all_launch(op, base, *view, out_dev, as_stream(stream));
    });
}

int pt_b200_reduce_dim(int op, const float* base, const pt_view* view, int dim, float* out,
                       void* stream) {
    return guarded([&] {
        PTB_REQUIRE(op >= 0 && op <= 2, "reduce: unknown op");
        PTB_REQUIRE(base && view && out, "reduce on an undefined tensor");
        require_view(*view, "reduce");
        PTB_REQUIRE(dim >= 0 && dim < view->ndim,
                    "reduce dim " + std::to_string(dim) + " out of range for rank " +
                        std::to_string(view->ndim));
        reduce_dim_launch(op, base, *view, dim, out, as_stream(stream));
    });
}

int64_t pt_b200_launch_count(void) { return g_launches.load(); }

void pt_b200_plan_cache_stats(int64_t* hits, int64_t* encodes) { tmap_cache_stats(hits, encodes); }

}  // extern "C"
