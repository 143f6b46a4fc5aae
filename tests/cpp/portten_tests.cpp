// portten_tests — C++ test driver for the portten-b200 operator API (include/portten/).
//   portten_tests          host-only checks (no GPU needed): Tensor views, expression
//                          grammar, geometry, choose_launch, registry, backend selection
//   portten_tests --gpu    device parity through the C++ API vs the C oracle
//                          (oracle/liboracle.so — the checker, linked by tests only)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "../../oracle/oracle.h"
#include "portten/backend.hpp"
#include "portten/convolution.hpp"
#include "portten/data_parallel.hpp"

using namespace portten;

static int g_fail = 0, g_pass = 0;
#define EXPECT(cond)                                                              \
    do {                                                                          \
        if (cond) ++g_pass;                                                       \
        else {                                                                    \
            ++g_fail;                                                             \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                         \
    } while (0)

template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static Tensor seeded(std::vector<std::int64_t> sizes, uint64_t seed, float lo = -1, float hi = 1) {
    Tensor t = Tensor::create(sizes);
    or_fill_uniform(t.data(), t.numel(), seed, lo, hi);
    return t;
}

static double rel_err(const Tensor& a, const std::vector<float>& r) {
    double n = 0, d = 0;
    for (std::size_t i = 0; i < r.size(); ++i) {
        const double e = (double)a.data()[i] - r[i];
        n += e * e;
        d += (double)r[i] * r[i];
    }
    return std::sqrt(n / (d > 0 ? d : 1e-30));
}

// ---------------------------------------------------------------- host-only
static void test_tensor_views() {
    Tensor t = Tensor::create({2, 3, 4});
    for (int i = 0; i < 24; ++i) t.data()[i] = (float)i;
    EXPECT(t.isContiguous() && t.numel() == 24);
    Tensor n = t.narrow(2, 1, 2);
    EXPECT(n.storageOffset() == 1 && n.size(2) == 2 && !n.isContiguous());
    EXPECT(n.at({1, 2, 1}) == 12 + 8 + 2);
    Tensor s = t.select(1, 2);
    EXPECT(s.dim() == 2 && s.storageOffset() == 8 && s.at({1, 3}) == 12 + 8 + 3);
    Tensor c = n.contiguous();
    EXPECT(c.isContiguous() && c.at({1, 2, 1}) == 22);
    EXPECT(throws<ValidationError>([&] { t.narrow(0, 1, 2); }));
    EXPECT(throws<ValidationError>([&] { Tensor::create({2, 0}); }));
    // copy between overlapping views of one storage is rejected (tensor.cpp:153-160)
    EXPECT(throws<ValidationError>([&] { t.narrow(2, 0, 2).copyFrom(t.narrow(2, 1, 2)); }));
    Tensor dst = t.narrow(0, 0, 1), src = t.narrow(0, 1, 1);
    dst.copyFrom(src);
    EXPECT(t.at({0, 0, 0}) == 12);
    t.select(0, 1).fill(-1);
    EXPECT(t.at({1, 2, 3}) == -1 && t.at({0, 2, 3}) == 23);
    EXPECT(Tensor::create({1}).item() == 0.0f);
}

static void test_geometry() {
    conv::ConvGeometry g{16, 3, 32, 32, 64, 3, 3, 1, 1, 1, 1};
    EXPECT(g.outHeight() == 32 && g.patchSize() == 27 && g.outSpatial() == 1024);
    EXPECT(g.toString() == "N16 C3 H32 W32 K64 k3x3 p1x1 s1x1");
    g.validate();
    conv::ConvGeometry bad{1, 1, 3, 3, 1, 5, 5, 0, 0, 1, 1};
    EXPECT(throws<ValidationError>([&] { bad.validate(); }));
    const pt_conv_geom a = bad.abi();
    EXPECT(pt_b200_conv_validate(&a) == PT_EVALIDATION);
    or_geom og{1, 1, 3, 3, 1, 5, 5, 0, 0, 1, 1};
    EXPECT(or_validate(&og) == 2);
}

static void test_expression() {
    auto p = expr::Program::parse("x = max(x, y) * 2.5", 2);
    EXPECT(p.kernelStatement() == "x = (fmax(x, y) * 2.5f);");
    EXPECT(p.referencedOperands() == 2);
    EXPECT(p.code().size() == 5 + 1);  // X Y MAX CONST(bits) MUL
    const char* bad[] = {"y = x", "x = w", "x = (x", "x = x +", "x = 1.2.3", "x = foo(x)"};
    for (const char* b : bad) EXPECT(throws<ValidationError>([&] { expr::Program::parse(b, 1); }));
    EXPECT(throws<ValidationError>([&] { expr::Program::parse("x = y", 1); }));
}

static void test_launch_and_selection() {
    BackendDescriptor d{"b200:0", 1024, 232448, true};
    auto lc = choose_launch(1000, d);
    EXPECT(lc.workgroupSize == 256 && lc.globalSize == 1024);
    EXPECT(throws<ValidationError>([&] { choose_launch(0, d); }));
    EXPECT(throws<BackendError>([&] { select_backend("reference"); }));
    EXPECT(throws<ValidationError>([&] { select_backend("opencl"); }));
    if (pt_b200_device_count() == 0) {
        EXPECT(backend_enumerate().empty());
        EXPECT(throws<BackendError>([&] { select_backend("device"); }));
    }
}

static void test_registry() {
    BackendDescriptor dev{"b200:0", 1024, 232448, true}, host{"host", 256, 32768, false};
    conv::ConvGeometry g{2, 8, 9, 9, 16, 3, 3, 1, 1, 1, 1};
    EXPECT(conv::conv_registry_select(g, dev).name == "implicitgemm-sm100a");
    EXPECT(throws<ValidationError>([&] { conv::conv_registry_select(g, host); }));
    conv::ConvImplEntry e;
    e.name = "custom";
    e.priority = 999;
    e.supports = [](const conv::ConvGeometry&, const BackendDescriptor& d) { return !d.isDevice; };
    conv::conv_registry_register(e);
    EXPECT(conv::conv_registry_select(g, host).name == "custom");
    EXPECT(conv::conv_registry_select(g, dev).name == "implicitgemm-sm100a");
    EXPECT(throws<ValidationError>([&] { conv::conv_registry_register(e); }));
    // the Winograd entry is registered, supports only 3x3 stride 1, and
    // ranks below the implicit GEMM (measured slower on B200)
    bool has_wino = false;
    for (const auto& n : conv::conv_registry_names()) has_wino = has_wino || n == "winograd-sm100a";
    EXPECT(has_wino);
    conv::ConvGeometry g5{2, 8, 9, 9, 16, 5, 5, 2, 2, 1, 1};
    EXPECT(conv::conv_registry_select(g5, dev).name == "implicitgemm-sm100a");
}

// ---------------------------------------------------------------- GPU
// TF32-exact integer tensors: x, gy in [-8, 8], w in {-1, 0, 1}, b in [-4, 4]
static Tensor exact(std::vector<std::int64_t> sizes, uint64_t seed, int a) {
    Tensor t = seeded(sizes, seed, -a - 0.5f, a + 0.5f);
    for (std::int64_t i = 0; i < t.numel(); ++i) {
        const float v = std::nearbyint(t.data()[i]);
        t.data()[i] = v > a ? a : (v < -a ? -a : v);
    }
    return t;
}

static bool same_bits(const Tensor& a, const std::vector<float>& r) {
    return static_cast<std::size_t>(a.numel()) == r.size() &&
           std::memcmp(a.data(), r.data(), sizeof(float) * r.size()) == 0;
}

// Every layer bench.py times, at its real per-image shape (batch 1), through the C++
// operator API: the registry's selected entry, the Winograd entry where it applies and the
// Torch-style SpatialConvolutionMM; TF32-exact inputs -> bitwise equal to the C oracle.
static void test_gpu_bench_layers_exact() {
    Backend& be = select_backend("device");
    struct L { const char* name; conv::ConvGeometry g; };
    const L layers[] = {
        {"convnet/L1", {1, 3, 128, 128, 96, 11, 11, 0, 0, 1, 1}}, {"convnet/L2", {1, 64, 64, 64, 128, 9, 9, 0, 0, 1, 1}},
        {"convnet/L3", {1, 128, 32, 32, 128, 9, 9, 0, 0, 1, 1}}, {"convnet/L4", {1, 128, 16, 16, 128, 7, 7, 0, 0, 1, 1}},
        {"convnet/L5", {1, 384, 13, 13, 384, 3, 3, 0, 0, 1, 1}},
        {"alexnet/c1", {1, 3, 224, 224, 64, 11, 11, 2, 2, 4, 4}}, {"alexnet/c2", {1, 64, 27, 27, 192, 5, 5, 2, 2, 1, 1}},
        {"alexnet/c3", {1, 192, 13, 13, 384, 3, 3, 1, 1, 1, 1}}, {"alexnet/c4", {1, 384, 13, 13, 256, 3, 3, 1, 1, 1, 1}},
        {"alexnet/c5", {1, 256, 13, 13, 256, 3, 3, 1, 1, 1, 1}},
        {"overfeat/c1", {1, 3, 231, 231, 96, 11, 11, 0, 0, 4, 4}}, {"overfeat/c2", {1, 96, 24, 24, 256, 5, 5, 0, 0, 1, 1}},
        {"overfeat/c3", {1, 256, 12, 12, 512, 3, 3, 1, 1, 1, 1}}, {"overfeat/c4", {1, 512, 12, 12, 1024, 3, 3, 1, 1, 1, 1}},
        {"overfeat/c5", {1, 1024, 12, 12, 1024, 3, 3, 1, 1, 1, 1}},
        {"vgga/c1", {1, 3, 224, 224, 64, 3, 3, 1, 1, 1, 1}}, {"vgga/c2", {1, 64, 112, 112, 128, 3, 3, 1, 1, 1, 1}},
        {"vgga/c3", {1, 128, 56, 56, 256, 3, 3, 1, 1, 1, 1}}, {"vgga/c4", {1, 256, 56, 56, 256, 3, 3, 1, 1, 1, 1}},
        {"vgga/c5", {1, 256, 28, 28, 512, 3, 3, 1, 1, 1, 1}}, {"vgga/c6", {1, 512, 28, 28, 512, 3, 3, 1, 1, 1, 1}},
        {"vgga/c7", {1, 512, 14, 14, 512, 3, 3, 1, 1, 1, 1}}, {"vgga/c8", {1, 512, 14, 14, 512, 3, 3, 1, 1, 1, 1}},
    };
    int checked = 0;
    for (const auto& l : layers) {
        const auto& g = l.g;
        or_geom og{g.batch, g.inChannels, g.inHeight, g.inWidth, g.outChannels, g.kernelH, g.kernelW,
                   g.padH, g.padW, g.strideH, g.strideW};
        Tensor x = exact({g.batch, g.inChannels, g.inHeight, g.inWidth}, 11, 8);
        Tensor w = exact({g.outChannels, g.inChannels, g.kernelH, g.kernelW}, 12, 1);
        Tensor b = exact({g.outChannels}, 13, 4);
        Tensor gy = exact({g.batch, g.outChannels, g.outHeight(), g.outWidth()}, 14, 8);
        std::vector<float> ry(g.batch * g.outChannels * g.outSpatial()), rgx(x.numel()), rgw(w.numel()),
            rgb(g.outChannels);
        or_conv_forward(&og, x.data(), w.data(), b.data(), ry.data(), 1, 0);
        or_conv_backward_input(&og, gy.data(), w.data(), rgx.data(), 0);
        or_conv_backward_weight(&og, x.data(), gy.data(), rgw.data(), rgb.data(), 1.0f, 0, 0);
        const auto& impl = conv::conv_registry_select(g, be.descriptor());
        bool ok = same_bits(impl.run(x, w, &b, g), ry);
        ok = same_bits(impl.backward_input(gy, w, g), rgx) && ok;
        Tensor gb;
        ok = same_bits(impl.backward_weight(x, gy, g, &gb), rgw) && same_bits(gb, rgb) && ok;
        // Torch-style layer over device tensors: updateOutput (keeps finput) + backward()
        conv::SpatialConvolutionMM layer((int)g.inChannels, (int)g.outChannels, (int)g.kernelW,
                                         (int)g.kernelH, (int)g.strideW, (int)g.strideH, (int)g.padW,
                                         (int)g.padH);
        layer.weight = DeviceTensor::upload(w);
        layer.bias = DeviceTensor::upload(b);
        layer.zeroGradParameters();
        DeviceTensor dx = DeviceTensor::upload(x), dgy = DeviceTensor::upload(gy);
        ok = same_bits(layer.updateOutput(dx).download(), ry) && ok;
        ok = same_bits(layer.backward(dx, dgy).download(), rgx) && ok;
        ok = same_bits(layer.gradWeight.download(), rgw) && same_bits(layer.gradBias.download(), rgb) && ok;
        if (g.kernelH == 3 && g.kernelW == 3 && g.strideH == 1 && g.strideW == 1) {
            ok = same_bits(conv::conv_winograd_2x2_3x3(x, w, &b, g), ry) && ok;
            ok = same_bits(conv::conv_backward_input_winograd(gy, w, g), rgx) && ok;
        }
        if (!ok) std::fprintf(stderr, "FAIL bench layer %s: not bitwise equal to the oracle\n", l.name);
        EXPECT(ok);
        ++checked;
    }
    EXPECT(checked == 23);
    // the Winograd entry rejects what it does not support
    conv::ConvGeometry g5{1, 8, 9, 9, 8, 5, 5, 2, 2, 1, 1};
    Tensor x5 = seeded({1, 8, 9, 9}, 1), w5 = seeded({8, 8, 5, 5}, 2);
    EXPECT(throws<ValidationError>([&] { conv::conv_winograd_2x2_3x3(x5, w5, nullptr, g5); }));
}
static void test_gpu_conv() {
    Backend& be = select_backend("auto");
    EXPECT(be.descriptor().isDevice && be.descriptor().name.rfind("b200:", 0) == 0);
    const conv::ConvGeometry geoms[] = {{16, 3, 32, 32, 64, 3, 3, 1, 1, 1, 1},
                                        {2, 64, 14, 14, 96, 5, 5, 2, 2, 1, 1},
                                        {2, 3, 31, 31, 32, 11, 11, 2, 2, 4, 4}};
    for (const auto& g : geoms) {
        or_geom og{g.batch, g.inChannels, g.inHeight, g.inWidth, g.outChannels, g.kernelH, g.kernelW,
                   g.padH, g.padW, g.strideH, g.strideW};
        Tensor x = seeded({g.batch, g.inChannels, g.inHeight, g.inWidth}, 1);
        Tensor w = seeded({g.outChannels, g.inChannels, g.kernelH, g.kernelW}, 2, -0.2f, 0.2f);
        Tensor b = seeded({g.outChannels}, 3, -0.1f, 0.1f);
        Tensor gy = seeded({g.batch, g.outChannels, g.outHeight(), g.outWidth()}, 4);
        const auto& impl = conv::conv_registry_select(g, be.descriptor());
        for (auto m : {conv::Math::TF32, conv::Math::FP32}) {
            Tensor y = m == conv::Math::TF32 ? impl.run(x, w, &b, g) : conv::conv_im2col_forward(x, w, &b, g, m);
            std::vector<float> ry(y.numel());
            or_conv_direct_f64(&og, x.data(), w.data(), b.data(), ry.data());
            const double tol = m == conv::Math::TF32 ? 5e-3 : 1e-5;
            EXPECT(rel_err(y, ry) < tol);
            Tensor gx = conv::conv_backward_input(gy, w, g, m);
            std::vector<float> rgx(gx.numel());
            or_conv_backward_input(&og, gy.data(), w.data(), rgx.data(), 0);
            EXPECT(rel_err(gx, rgx) < tol);
            Tensor gb;
            Tensor gw = conv::conv_backward_weight(x, gy, g, &gb, m);
            std::vector<float> rgw(gw.numel()), rgb(gb.numel());
            or_conv_backward_weight(&og, x.data(), gy.data(), rgw.data(), rgb.data(), 1.0f, 0, 0);
            EXPECT(rel_err(gw, rgw) < tol);
            EXPECT(rel_err(gb, rgb) < 1e-5);
        }
        // batched lowering == unbatched
        Tensor y1 = conv::conv_im2col_forward(x, w, &b, g);
        Tensor y2 = conv::conv_im2col_batched(x, w, &b, g, g.batch);
        EXPECT(std::memcmp(y1.data(), y2.data(), sizeof(float) * y1.numel()) == 0);
    }
}

static void test_gpu_layer_and_ops() {
    Backend& be = select_backend("device");
    // SpatialConvolutionMM: backward() == updateGradInput + accGradParameters (x2 accumulates)
    conv::SpatialConvolutionMM layer(64, 128, 3, 3, 1, 1, 1);
    Tensor xh = seeded({4, 64, 12, 12}, 5), gyh = seeded({4, 128, 12, 12}, 6);
    DeviceTensor x = DeviceTensor::upload(xh), gy = DeviceTensor::upload(gyh);
    layer.updateOutput(x);
    layer.backward(x, gy);
    Tensor gw1 = layer.gradWeight.download(), gx1 = layer.gradInput.download();
    layer.accGradParameters(x, gy);
    Tensor gw2 = layer.gradWeight.download();
    double md = 0;
    for (std::int64_t i = 0; i < gw1.numel(); ++i)
        md = std::max(md, (double)std::fabs(gw2.data()[i] - 2 * gw1.data()[i]));
    EXPECT(md < 1e-3);
    Tensor gx2 = layer.updateGradInput(x, gy).download();
    EXPECT(std::memcmp(gx1.data(), gx2.data(), sizeof(float) * gx1.numel()) == 0);
    // apply on aliasing host views (in-place destination semantics of runApply)
    Tensor t = seeded({4, 6}, 7);
    Tensor before = t.contiguous();
    before = Tensor::create({4, 6});
    before.copyFrom(t);
    Tensor ops[2] = {t.narrow(1, 0, 3), t.narrow(1, 3, 3)};
    dispatch_apply("x = x * s + y", std::span<Tensor>(ops, 2), 2.0f, be);
    bool ok = true;
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 3; ++c) {
            const float want = before.at({r, c}) * 2.0f + before.at({r, c + 3});
            ok = ok && t.at({r, c}) == want && t.at({r, c + 3}) == before.at({r, c + 3});
        }
    EXPECT(ok);
    const float s = dispatch_reduce_all(ReduceOp::Sum, before, be);
    or_view v{2, {4, 6}, {6, 1}, 0};
    EXPECT(std::fabs(s - or_reduce_all(OR_SUM, before.data(), &v)) < 1e-4);
    Tensor rd = dispatch_reduce_dim(ReduceOp::Max, before.select(1, 2), 0, be);
    EXPECT(rd.numel() == 1);
    DeviceBuffer buf = device_upload(before.narrow(1, 1, 2), be);
    Tensor back = Tensor::create({4, 2});
    device_download(buf, back, be);
    EXPECT(back.at({3, 1}) == before.at({3, 2}));
    // im2col bit-exact vs the oracle
    conv::ConvGeometry g{1, 3, 9, 10, 4, 3, 3, 1, 1, 2, 1};
    or_geom og{1, 3, 9, 10, 4, 3, 3, 1, 1, 2, 1};
    Tensor img = seeded({3, 9, 10}, 8);
    Tensor col = conv::im2col(img, g);
    std::vector<float> rcol(col.numel());
    or_im2col(&og, img.data(), rcol.data());
    EXPECT(std::memcmp(col.data(), rcol.data(), sizeof(float) * col.numel()) == 0);
}

// ---------------------------------------------------------------- data parallelism
static void test_shard_range() {
    for (std::int64_t n : {128, 64, 7, 1}) {
        for (int world = 1; world <= 8; ++world) {
            std::int64_t next = 0;
            for (int r = 0; r < world; ++r) {
                const dp::ShardRange s = dp::shard_range(n, r, world);
                EXPECT(s.start == next);  // contiguous, in rank order
                const std::int64_t len = s.stop - s.start;
                EXPECT(len == n / world + (r < n % world ? 1 : 0));  // remainder to the low ranks
                next = s.stop;
            }
            EXPECT(next == n);
        }
    }
    EXPECT(throws<ValidationError>([] { dp::shard_range(8, 2, 2); }));
    EXPECT(throws<ValidationError>([] { dp::shard_range(8, 0, 0); }));
}

// one GPU: the shards' gradients sum to the full batch's (the DP identity), and a world-1 NCCL
// communicator's allreduce + error-polling synchronize leave the gradients bitwise unchanged
static void test_gpu_dp() {
    const conv::ConvGeometry full(4, 32, 12, 12, 48, 3, 3, 1, 1, 1, 1);
    Tensor x = seeded({4, 32, 12, 12}, 31), gy = seeded({4, 48, 12, 12}, 32);
    DeviceTensor dx = DeviceTensor::upload(x), dgy = DeviceTensor::upload(gy);
    DeviceTensor gw = DeviceTensor::empty({48, 32, 3, 3}), gb = DeviceTensor::empty({48});
    conv::conv_backward_weight(full, dx, dgy, gw, &gb);
    // two emulated ranks: each its shard, accumulated into one buffer (= the allreduce's sum)
    DeviceTensor sw = DeviceTensor::empty({48, 32, 3, 3}), sb = DeviceTensor::empty({48});
    for (int r = 0; r < 2; ++r) {
        const dp::ShardRange s = dp::shard_range(4, r, 2);
        const conv::ConvGeometry part(s.stop - s.start, 32, 12, 12, 48, 3, 3, 1, 1, 1, 1);
        conv::conv_backward_weight(part, dx.narrow(0, s.start, s.stop - s.start),
                                   dgy.narrow(0, s.start, s.stop - s.start), sw, &sb, 1.0f, r > 0);
    }
    Tensor hf = gw.download(), hs = sw.download();
    std::vector<float> ref(hf.data(), hf.data() + hf.numel());
    EXPECT(rel_err(hs, ref) < 1e-5);  // same TF32 products, two fp32 partial sums
    Tensor hb = gb.download(), hsb = sb.download();
    std::vector<float> refb(hb.data(), hb.data() + hb.numel());
    EXPECT(rel_err(hsb, refb) < 1e-6);
    dp::Communicator comm(dp::new_unique_id(), 0, 1, 0);
    EXPECT(comm.rank() == 0 && comm.world() == 1);
    comm.allreduceGradients(gw, &gb, nullptr);
    comm.synchronize(nullptr, 60.0);
    Tensor aw = gw.download(), ab = gb.download();
    EXPECT(std::memcmp(aw.data(), hf.data(), sizeof(float) * hf.numel()) == 0);
    EXPECT(std::memcmp(ab.data(), hb.data(), sizeof(float) * hb.numel()) == 0);
}

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "--gpu") == 0;
    test_tensor_views();
    test_geometry();
    test_expression();
    test_launch_and_selection();
    test_registry();
    test_shard_range();
    if (gpu) {
        test_gpu_dp();
        test_gpu_conv();
        test_gpu_layer_and_ops();
        test_gpu_bench_layers_exact();
    }
    std::printf("portten_tests: %d passed, %d failed%s\n", g_pass, g_fail, gpu ? " (gpu)" : "");
    return g_fail ? 1 : 0;
}
