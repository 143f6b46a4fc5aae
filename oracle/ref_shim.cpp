// ref_shim.cpp — extern "C" access to the REFERENCE's own code, compiled in place
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/libportten_ref.so.
//
// TEST INFRASTRUCTURE: used by tests/ and tests/golden/make_golden.py to pin the
// oracle restatement against the reference itself. Nothing here is product code
// and no reference source is copied: this file only calls the reference's public
// API (portten::Tensor, dispatch_apply/reduce on reference_backend(),
// expr::Program, tmpl::Template, codegen::gen_im2col_kernel).
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "portten/backend.hpp"
#include "portten/conv_geometry.hpp"
#include "portten/embedded_templates.hpp"
#include "portten/expression.hpp"
#include "portten/kernel_codegen.hpp"
#include "portten/template_engine.hpp"
#include "portten/tensor.hpp"

using namespace portten;

// The backend the dispatch entry points run on: the reference's host interpreter here;
// integration/Makefile recompiles this file with SHIM_BACKEND=select_backend("device") to
// drive the reference's dispatch through the B200 plug-in (integration/b200_backend.cpp).
#ifndef SHIM_BACKEND
#define SHIM_BACKEND reference_backend()
#endif

namespace {

struct GeomC {
    int64_t N, C, H, W, K, kH, kW, padH, padW, strideH, strideW;
};

conv::ConvGeometry toGeom(const GeomC* g) {
    conv::ConvGeometry c;
    c.batch = g->N; c.inChannels = g->C; c.inHeight = g->H; c.inWidth = g->W;
    c.outChannels = g->K; c.kernelH = g->kH; c.kernelW = g->kW; c.padH = g->padH;
    c.padW = g->padW; c.strideH = g->strideH; c.strideW = g->strideW;
    return c;
}

int fail(char* err, int cap, const std::string& msg, int code) {
    if (err && cap > 0) {
        std::strncpy(err, msg.c_str(), static_cast<size_t>(cap - 1));
        err[cap - 1] = 0;
    }
    return code;
}

template <class F>
int guarded(char* err, int cap, F&& f) {
    try {
        f();
        return 0;
    } catch (const ValidationError& e) {
        return fail(err, cap, e.what(), 2);
    } catch (const BackendError& e) {
        return fail(err, cap, e.what(), 3);
    } catch (const std::exception& e) {
        return fail(err, cap, e.what(), 4);
    }
}

// A view is described as a contiguous base tensor plus a chain of
// narrow(dim,start,len) [kind 0] / select(dim,index) [kind 1] ops.
Tensor makeView(const Tensor& base, const int64_t* ops, int nops) {
    Tensor v = base;
    for (int i = 0; i < nops; ++i) {
        const int64_t* o = ops + 4 * i;
        if (o[0] == 0) v = v.narrow(static_cast<int>(o[1]), o[2], o[3]);
        else v = v.select(static_cast<int>(o[1]), o[2]);
    }
    return v;
}

Tensor makeBase(const float* data, const int64_t* sizes, int ndim) {
    Tensor t = Tensor::create(std::vector<int64_t>(sizes, sizes + ndim));
    std::memcpy(t.data(), data, sizeof(float) * static_cast<size_t>(t.numel()));
    return t;
}

}  // namespace

extern "C" {

// Reference defect D1: gen_im2col_kernel as shipped. Returns 0
// and the text if it renders, else the error class and message.
int ref_gen_im2col_kernel(const GeomC* g, char* out, int cap) {
    return guarded(out, cap, [&] {
        const auto src = codegen::gen_im2col_kernel(toGeom(g));
        fail(out, cap, src.text, 0);
    });
}

// The reference's own im2col template (proj/templates/im2col.kt.tmpl) rendered
// by the reference's template engine with the bindings of
// proj/src/kernel_codegen.cpp:255-272, but with the two flags bound as
// tmpl::Value(bool) so the D1 overload-resolution defect is bypassed.
int ref_render_im2col(const GeomC* g, char* out, int cap) {
    return guarded(out, cap, [&] {
        const conv::ConvGeometry geom = toGeom(g);
        geom.validate();
        const int64_t outH = geom.outHeight(), outW = geom.outWidth();
        tmpl::RenderContext ctx;
        ctx.bind("entry", "portten_im2col");
        ctx.bind("n_items", tmpl::Value(geom.inChannels * outH * outW));
        ctx.bind("outH", tmpl::Value(outH));
        ctx.bind("outW", tmpl::Value(outW));
        ctx.bind("out_spatial", tmpl::Value(outH * outW));
        ctx.bind("strideH", tmpl::Value(geom.strideH));
        ctx.bind("strideW", tmpl::Value(geom.strideW));
        ctx.bind("padH", tmpl::Value(geom.padH));
        ctx.bind("padW", tmpl::Value(geom.padW));
        ctx.bind("channel_stride", tmpl::Value(geom.inHeight * geom.inWidth));
        ctx.bind("H", tmpl::Value(geom.inHeight));
        ctx.bind("W", tmpl::Value(geom.inWidth));
        ctx.bind("kH", tmpl::Value(geom.kernelH));
        ctx.bind("kW", tmpl::Value(geom.kernelW));
        ctx.bind("patch", tmpl::Value(geom.kernelH * geom.kernelW));
        ctx.bind("unrolled", tmpl::Value(geom.kernelH * geom.kernelW <= 25));
        ctx.bind("has_pad", tmpl::Value(geom.padH > 0 || geom.padW > 0));
        static const tmpl::Template t = tmpl::Template::parse(embedded::kIm2colTemplate);
        const std::string text = t.render(ctx);
        if (static_cast<int>(text.size()) + 1 > cap) throw BackendError("render buffer too small");
        std::memcpy(out, text.c_str(), text.size() + 1);
    });
}

// expr::Program::parse validation (proj/src/expression.cpp:336-338): returns 0 and
// the canonical kernel statement, or the error class and message.
int ref_parse_expr(const char* text, int arity, char* out, int cap) {
    return guarded(out, cap, [&] {
        const auto p = expr::Program::parse(text, arity);
        fail(out, cap, p.kernelStatement(), 0);
    });
}

// dispatch_apply on reference_backend() (proj/src/backend.cpp:115-141).
// Operand t: base data/sizes/ndim + view op chain. Base storages are written back.
int ref_apply(const char* expr, int arity, float** data, const int64_t* sizes /*[arity*8]*/,
              const int32_t* ndim, const int64_t* ops /*[arity*16*4]*/, const int32_t* nops,
              float scalar, char* err, int cap) {
    return guarded(err, cap, [&] {
        std::vector<Tensor> bases, views;
        for (int t = 0; t < arity; ++t) {
            bases.push_back(makeBase(data[t], sizes + 8 * t, ndim[t]));
            views.push_back(makeView(bases.back(), ops + 64 * t, nops[t]));
        }
        dispatch_apply(expr, std::span<Tensor>(views.data(), views.size()), scalar,
                       SHIM_BACKEND);
        for (int t = 0; t < arity; ++t)
            std::memcpy(data[t], bases[t].data(), sizeof(float) * bases[t].numel());
    });
}

int ref_reduce_all(int op, const float* data, const int64_t* sizes, int ndim, const int64_t* ops,
                   int nops, float* out, char* err, int cap) {
    return guarded(err, cap, [&] {
        Tensor base = makeBase(data, sizes, ndim);
        *out = dispatch_reduce_all(static_cast<ReduceOp>(op), makeView(base, ops, nops),
                                   SHIM_BACKEND);
    });
}

int ref_reduce_dim(int op, const float* data, const int64_t* sizes, int ndim, const int64_t* ops,
                   int nops, int dim, float* out, int64_t out_cap, char* err, int cap) {
    return guarded(err, cap, [&] {
        Tensor base = makeBase(data, sizes, ndim);
        Tensor r = dispatch_reduce_dim(static_cast<ReduceOp>(op), makeView(base, ops, nops), dim,
                                       SHIM_BACKEND);
        if (r.numel() > out_cap) throw BackendError("reduce_dim output buffer too small");
        Tensor c = r.contiguous();
        std::memcpy(out, c.data(), sizeof(float) * c.numel());
    });
}

// device_upload of a view, then device_download into a fresh contiguous tensor
// (proj/src/backend.cpp:163-181): the round trip the reference promises is bitwise identity.
int ref_roundtrip(const float* data, const int64_t* sizes, int ndim, const int64_t* ops, int nops,
                  float* out, int64_t out_cap, char* err, int cap) {
    return guarded(err, cap, [&] {
        Tensor base = makeBase(data, sizes, ndim);
        Tensor v = makeView(base, ops, nops);
        Backend& b = SHIM_BACKEND;
        const DeviceBuffer buf = device_upload(v, b);
        Tensor back = Tensor::create(v.sizes());
        device_download(buf, back, b);
        if (back.numel() > out_cap) throw BackendError("roundtrip output buffer too small");
        std::memcpy(out, back.data(), sizeof(float) * back.numel());
    });
}

// Name / isDevice of the backend SHIM_BACKEND resolves to, and of every backend_enumerate() entry.
int ref_backend_info(char* out, int cap) {
    return guarded(out, cap, [&] {
        std::string s = SHIM_BACKEND.descriptor().name;
        s += SHIM_BACKEND.descriptor().isDevice ? " device" : " host";
        for (Backend* b : backend_enumerate()) s += ";" + b->descriptor().name;
        fail(out, cap, s, 0);
    });
}

// choose_launch (proj/src/backend.cpp:25-33).
int ref_choose_launch(int64_t n, int maxwg, int64_t* global, int* wg, char* err, int cap) {
    return guarded(err, cap, [&] {
        BackendDescriptor d;
        d.name = "probe";
        d.maxWorkgroupSize = maxwg;
        const LaunchConfig lc = choose_launch(n, d);
        *global = lc.globalSize;
        *wg = lc.workgroupSize;
    });
}

// ConvGeometry::validate (conv_geometry.hpp:53-63).
int ref_geom_validate(const GeomC* g, char* err, int cap) {
    return guarded(err, cap, [&] { toGeom(g).validate(); });
}

}  // extern "C"
