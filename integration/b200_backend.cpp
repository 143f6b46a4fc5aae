// b200_backend.cpp — the B200 device backend as the REFERENCE's own plug-in.
//
// Compiled against the reference's headers (proj/include/portten/backend.hpp,
// proj/src/opencl_backend.hpp), not ours: B200Backend derives from the reference's
// portten::Backend and implements its exact vtable
//   descriptor(), runApply(const codegen::ApplySpec&, const expr::Program&,
//   std::span<Tensor>, float, const LaunchConfig&), runReduceAll / runReduceDim
//   (codegen::ReduceOp), uploadContiguous / downloadContiguous
// (proj/include/portten/backend.hpp:67-81) over the libpt_b200 C ABI (include/pt_b200.h).
//
// It plugs into the reference's device slot unchanged: built with PORTTEN_HAVE_OPENCL
// defined, the reference's probedBackends() (proj/src/backend.cpp:45-60) calls
// opencl_probe_devices() — defined here — and lists one B200Backend per sm_100 GPU after
// reference_backend(); select_backend("device"/"auto"), dispatch_apply / dispatch_reduce_*
// and device_upload / device_download (backend.cpp:78-181) then run on the B200 with the
// reference's own validation and launch-config checks in front. No reference source is
// modified or copied (integration/Makefile compiles backend.cpp in place).
//
// The reference's Tensor lives in host memory, so each dispatch stages the operands'
// storages to the device, runs the library's kernel on the same views (sizes, strides,
// storage offsets) and copies the destination storage back. The expression is compiled
// from ApplySpec::expression by the library's compiler (pt_b200_expression_compile), which
// accepts exactly the reference's grammar; the reference's own Program has already
// validated it by then (dispatch_apply parses before runApply).
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "opencl_backend.hpp"
#include "portten/backend.hpp"
#include "../include/pt_b200.h"

namespace portten {

namespace {

void ok(int st, const char* what) {
    if (st == PT_OK) return;
    const std::string msg = std::string(what) + ": " + pt_b200_last_error();
    if (st == PT_EVALIDATION) throw ValidationError(msg);
    throw BackendError(msg);
}

struct DevMem {
    void* p = nullptr;
    explicit DevMem(std::size_t bytes) { ok(pt_b200_malloc(&p, bytes), "b200 malloc"); }
    ~DevMem() { pt_b200_free(p); }
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
};

pt_view view_of(const Tensor& t) {
    pt_view v{};
    v.ndim = t.dim();
    for (int d = 0; d < t.dim(); ++d) {
        v.sizes[d] = t.size(d);
        v.strides[d] = t.stride(d);
    }
    v.offset = t.storageOffset();
    return v;
}

int reduce_code(ReduceOp op) {
    switch (op) {
        case ReduceOp::Sum: return PT_REDUCE_SUM;
        case ReduceOp::Max: return PT_REDUCE_MAX;
        case ReduceOp::Min: return PT_REDUCE_MIN;
    }
    throw ValidationError("unknown reduce op");
}

// Device copies of the storages behind a set of views; views sharing a Storage share
// one device copy, so aliasing between operands is preserved.
class Staged {
public:
    float* base(const Tensor& t) {
        Storage* s = t.storage().get();
        auto it = bufs_.find(s);
        if (it != bufs_.end()) return static_cast<float*>(it->second->p);
        const std::size_t bytes = sizeof(float) * static_cast<std::size_t>(s->length());
        auto m = std::make_unique<DevMem>(bytes);
        ok(pt_b200_memcpy_h2d(m->p, s->data(), bytes, nullptr), "b200 upload");
        float* p = static_cast<float*>(m->p);
        bufs_.emplace(s, std::move(m));
        return p;
    }
    void write_back(const Tensor& t) {
        Storage* s = t.storage().get();
        ok(pt_b200_memcpy_d2h(s->data(), bufs_.at(s)->p, sizeof(float) * s->length(), nullptr),
           "b200 download");
        ok(pt_b200_stream_sync(nullptr), "b200 sync");
    }

private:
    std::map<Storage*, std::unique_ptr<DevMem>> bufs_;
};

class B200Backend final : public Backend {
public:
    explicit B200Backend(int device) : device_(device) {
        pt_device_desc d{};
        ok(pt_b200_device_info(device, &d), "b200 device info");
        desc_.name = d.name;                      // "b200:<ordinal>"
        desc_.maxWorkgroupSize = d.maxWorkgroupSize;
        desc_.localMemBytes = d.localMemBytes;
        desc_.isDevice = true;
    }

    const BackendDescriptor& descriptor() const override { return desc_; }

    void runApply(const codegen::ApplySpec& spec, const expr::Program& program,
                  std::span<Tensor> operands, float scalar, const LaunchConfig&) override {
        (void)program;  // validated by dispatch_apply; compiled from spec.expression below
        std::lock_guard<std::mutex> lk(mu_);  // device queue submission is serialised
        ok(pt_b200_set_device(device_), "b200 set device");
        std::int32_t n = 0;
        ok(pt_b200_expression_compile(spec.expression.c_str(), spec.arity, nullptr, 0, &n, nullptr,
                                      nullptr, 0), "apply expression");
        std::vector<std::int32_t> code(static_cast<std::size_t>(n));
        ok(pt_b200_expression_compile(spec.expression.c_str(), spec.arity, code.data(), n, &n,
                                      nullptr, nullptr, 0), "apply expression");
        Staged st;
        float* bases[3] = {nullptr, nullptr, nullptr};
        pt_view views[3] = {};
        for (int t = 0; t < spec.arity; ++t) {
            bases[t] = st.base(operands[static_cast<std::size_t>(t)]);
            views[t] = view_of(operands[static_cast<std::size_t>(t)]);
        }
        ok(pt_b200_apply(code.data(), n, spec.arity, bases, views, scalar, nullptr), "b200 apply");
        st.write_back(operands[0]);
    }

    float runReduceAll(ReduceOp op, const Tensor& t) override {
        std::lock_guard<std::mutex> lk(mu_);
        ok(pt_b200_set_device(device_), "b200 set device");
        Staged st;
        const float* base = st.base(t);
        const pt_view v = view_of(t);
        DevMem out(sizeof(float));
        ok(pt_b200_reduce_all(reduce_code(op), base, &v, static_cast<float*>(out.p), nullptr),
           "b200 reduce_all");
        float r = 0.f;
        ok(pt_b200_memcpy_d2h(&r, out.p, sizeof(float), nullptr), "b200 download");
        ok(pt_b200_stream_sync(nullptr), "b200 sync");
        return r;
    }

    Tensor runReduceDim(ReduceOp op, const Tensor& t, int dim) override {
        std::lock_guard<std::mutex> lk(mu_);
        ok(pt_b200_set_device(device_), "b200 set device");
        std::vector<std::int64_t> sizes = t.sizes();
        sizes[static_cast<std::size_t>(dim)] = 1;
        Tensor r = Tensor::create(sizes);
        Staged st;
        const float* base = st.base(t);
        const pt_view v = view_of(t);
        DevMem out(sizeof(float) * static_cast<std::size_t>(r.numel()));
        ok(pt_b200_reduce_dim(reduce_code(op), base, &v, dim, static_cast<float*>(out.p), nullptr),
           "b200 reduce_dim");
        ok(pt_b200_memcpy_d2h(r.data(), out.p, sizeof(float) * r.numel(), nullptr), "b200 download");
        ok(pt_b200_stream_sync(nullptr), "b200 sync");
        return r;
    }

    DeviceBuffer uploadContiguous(const Tensor& t) override {
        PORTTEN_CHECK(t.isContiguous(), "upload expects a contiguous tensor");
        ok(pt_b200_set_device(device_), "b200 set device");
        const std::size_t bytes = sizeof(float) * static_cast<std::size_t>(t.numel());
        void* p = nullptr;
        ok(pt_b200_malloc(&p, bytes), "b200 malloc");
        DeviceBuffer buf;
        buf.impl = std::shared_ptr<void>(p, [](void* q) { pt_b200_free(q); });
        ok(pt_b200_memcpy_h2d(p, t.data(), bytes, nullptr), "b200 upload");
        ok(pt_b200_stream_sync(nullptr), "b200 sync");
        buf.elems = t.numel();
        buf.backendName = desc_.name;
        return buf;
    }

    void downloadContiguous(const DeviceBuffer& buf, Tensor& dst) override {
        PORTTEN_CHECK(dst.isContiguous(), "download expects a contiguous tensor");
        PORTTEN_CHECK(buf.backendName == desc_.name, "buffer belongs to another backend");
        PORTTEN_CHECK(buf.impl != nullptr && buf.elems == dst.numel(), "download size mismatch");
        ok(pt_b200_set_device(device_), "b200 set device");
        ok(pt_b200_memcpy_d2h(dst.data(), buf.impl.get(), sizeof(float) * dst.numel(), nullptr),
           "b200 download");
        ok(pt_b200_stream_sync(nullptr), "b200 sync");
    }

private:
    int device_;
    BackendDescriptor desc_;
    std::mutex mu_;
};

}  // namespace

// The reference's device slot (proj/src/opencl_backend.hpp:29): one backend per usable
// sm_100 GPU, process-lifetime singletons like reference_backend(); an empty list when
// there is no driver or GPU (pt_b200_device_count() == 0 is not an error).
std::vector<Backend*> opencl_probe_devices() {
    static std::vector<std::unique_ptr<B200Backend>> owned = [] {
        std::vector<std::unique_ptr<B200Backend>> v;
        const int n = pt_b200_device_count();
        for (int i = 0; i < n; ++i) v.push_back(std::make_unique<B200Backend>(i));
        return v;
    }();
    std::vector<Backend*> out;
    for (auto& b : owned) out.push_back(b.get());
    return out;
}

}  // namespace portten
