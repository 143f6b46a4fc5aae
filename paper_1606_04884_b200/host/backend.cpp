// backend.cpp — the Backend boundary for B200 (include/portten/backend.hpp).
//
// B200Backend fills the reference's device slot (opencl_probe_devices,
// proj/src/opencl_backend.hpp:29 / proj/src/backend.cpp:50-57). Host-Tensor dispatches
// keep the reference's semantics — in-place update of the destination view, views may
// alias one storage — by staging each distinct Storage once to the device, running the
// op there on the original sizes/strides/offsets, and copying the destination storage
// back. No host compute path exists: a missing device is a BackendError.
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>

#include "portten/backend.hpp"

namespace portten {

LaunchConfig choose_launch(std::int64_t n, const BackendDescriptor& d) {
    PORTTEN_CHECK(n >= 1, "choose_launch requires at least one work item");
    PORTTEN_CHECK(d.maxWorkgroupSize >= 1, "backend reports no workgroup capacity");
    LaunchConfig lc;
    lc.workgroupSize = std::min(256, d.maxWorkgroupSize);
    lc.globalSize = (n + lc.workgroupSize - 1) / lc.workgroupSize * lc.workgroupSize;
    return lc;
}

namespace {

std::shared_ptr<void> dev_alloc(std::size_t bytes) {
    void* p = nullptr;
    throw_if_error(pt_b200_malloc(&p, bytes ? bytes : 4));
    return std::shared_ptr<void>(p, [](void* q) { pt_b200_free(q); });
}

class B200Backend final : public Backend {
public:
    explicit B200Backend(int ordinal) : ordinal_(ordinal) {
        pt_device_desc dd{};
        throw_if_error(pt_b200_device_info(ordinal, &dd));
        desc_.name = dd.name;
        desc_.maxWorkgroupSize = dd.maxWorkgroupSize;
        desc_.localMemBytes = dd.localMemBytes;
        desc_.isDevice = true;
    }

    const BackendDescriptor& descriptor() const override { return desc_; }

    void runApply(const expr::Program& program, std::span<Tensor> operands, float scalar,
                  const LaunchConfig&) override {
        std::lock_guard<std::mutex> lk(mu_);  // device queue submission is serialised
        throw_if_error(pt_b200_set_device(ordinal_));
        std::map<const Storage*, std::shared_ptr<void>> staged;
        float* bases[3] = {nullptr, nullptr, nullptr};
        pt_view views[3] = {};
        for (std::size_t t = 0; t < operands.size(); ++t) {
            const Storage* s = operands[t].storage().get();
            auto it = staged.find(s);
            if (it == staged.end()) {
                auto buf = dev_alloc(sizeof(float) * s->length());
                throw_if_error(pt_b200_memcpy_h2d(buf.get(), s->data(), sizeof(float) * s->length(), nullptr));
                it = staged.emplace(s, std::move(buf)).first;
            }
            bases[t] = static_cast<float*>(it->second.get());
            views[t] = operands[t].view();
        }
        const auto& code = program.code();
        throw_if_error(pt_b200_apply(code.data(), static_cast<std::int32_t>(code.size()),
                                     static_cast<int>(operands.size()), bases, views, scalar, nullptr));
        Storage* dst = operands[0].storage().get();
        throw_if_error(pt_b200_memcpy_d2h(dst->data(), bases[0], sizeof(float) * dst->length(), nullptr));
        throw_if_error(pt_b200_stream_sync(nullptr));
    }

    float runReduceAll(ReduceOp op, const Tensor& t) override {
        std::lock_guard<std::mutex> lk(mu_);
        throw_if_error(pt_b200_set_device(ordinal_));
        auto buf = stage(t);
        auto out = dev_alloc(sizeof(float));
        const pt_view v = t.view();
        throw_if_error(pt_b200_reduce_all(static_cast<int>(op), static_cast<float*>(buf.get()), &v,
                                          static_cast<float*>(out.get()), nullptr));
        float r = 0.0f;
        throw_if_error(pt_b200_memcpy_d2h(&r, out.get(), sizeof r, nullptr));
        throw_if_error(pt_b200_stream_sync(nullptr));
        return r;
    }

    Tensor runReduceDim(ReduceOp op, const Tensor& t, int dim) override {
        std::lock_guard<std::mutex> lk(mu_);
        throw_if_error(pt_b200_set_device(ordinal_));
        std::vector<std::int64_t> os = t.sizes();
        os[dim] = 1;
        Tensor out = Tensor::create(os);
        auto buf = stage(t);
        auto dout = dev_alloc(sizeof(float) * out.numel());
        const pt_view v = t.view();
        throw_if_error(pt_b200_reduce_dim(static_cast<int>(op), static_cast<float*>(buf.get()), &v, dim,
                                          static_cast<float*>(dout.get()), nullptr));
        throw_if_error(pt_b200_memcpy_d2h(out.data(), dout.get(), sizeof(float) * out.numel(), nullptr));
        throw_if_error(pt_b200_stream_sync(nullptr));
        return out;
    }

    DeviceBuffer uploadContiguous(const Tensor& t) override {
        PORTTEN_CHECK(t.isContiguous(), "upload expects a contiguous tensor");
        throw_if_error(pt_b200_set_device(ordinal_));
        auto buf = dev_alloc(sizeof(float) * t.numel());
        throw_if_error(pt_b200_memcpy_h2d(buf.get(), t.data(), sizeof(float) * t.numel(), nullptr));
        throw_if_error(pt_b200_stream_sync(nullptr));
        return DeviceBuffer{buf, t.numel(), desc_.name};
    }

    void downloadContiguous(const DeviceBuffer& buf, Tensor& dst) override {
        PORTTEN_CHECK(dst.isContiguous(), "download expects a contiguous tensor");
        PORTTEN_CHECK(buf.backendName == desc_.name, "buffer belongs to another backend");
        PORTTEN_CHECK(buf.impl && buf.elems == dst.numel(), "download size mismatch");
        throw_if_error(pt_b200_set_device(ordinal_));
        throw_if_error(pt_b200_memcpy_d2h(dst.data(), buf.impl.get(), sizeof(float) * dst.numel(), nullptr));
        throw_if_error(pt_b200_stream_sync(nullptr));
    }

private:
    int ordinal_;
    BackendDescriptor desc_;
    std::mutex mu_;

    std::shared_ptr<void> stage(const Tensor& t) {
        const Storage* s = t.storage().get();
        auto buf = dev_alloc(sizeof(float) * s->length());
        throw_if_error(pt_b200_memcpy_h2d(buf.get(), s->data(), sizeof(float) * s->length(), nullptr));
        return buf;
    }
};

std::string backend_env() {
    const char* e = std::getenv("PORTTEN_BACKEND");
    return (e && *e) ? e : "auto";
}

std::string shape_of(const Tensor& t) {
    std::string s = "[";
    for (int d = 0; d < t.dim(); ++d) s += (d ? "," : "") + std::to_string(t.size(d));
    return s + "]";
}

}  // namespace

std::vector<Backend*> cuda_probe_devices() {
    static std::vector<Backend*> devices = [] {
        std::vector<Backend*> v;
        const int n = pt_b200_device_count();
        for (int i = 0; i < n; ++i) v.push_back(new B200Backend(i));
        return v;
    }();
    return devices;
}

std::vector<Backend*> backend_enumerate() {
    if (backend_env() == "reference") return {};
    return cuda_probe_devices();
}

Backend& select_backend(std::string_view requested) {
    std::string mode(requested.empty() ? "auto" : requested);
    if (mode == "auto") {
        mode = backend_env();
        if (mode != "reference" && mode != "device") mode = "auto";
    }
    if (mode == "reference")
        throw BackendError("the host reference interpreter is not part of portten-b200 (it is the "
                           "test oracle); select 'device' or 'auto'");
    if (mode != "device" && mode != "auto")
        throw ValidationError("unknown backend selector '" + mode +
                              "' (expected reference, device, or auto)");
    const auto devs = cuda_probe_devices();
    if (devs.empty())
        throw BackendError("no device backend available (no sm_100 GPU visible to libpt_b200)");
    std::int64_t index = 0;
    if (const char* env = std::getenv("PORTTEN_DEVICE"); env && *env) index = std::atoll(env);
    if (index < 0 || index >= static_cast<std::int64_t>(devs.size()))
        throw BackendError("PORTTEN_DEVICE index " + std::to_string(index) + " out of range, " +
                           std::to_string(devs.size()) + " device(s) present");
    return *devs[static_cast<std::size_t>(index)];
}

void dispatch_apply(std::string_view expression, std::span<Tensor> operands, float scalar,
                    Backend& backend) {
    PORTTEN_CHECK(!operands.empty() && operands.size() <= 3,
                  "apply takes 1..3 operands, got " + std::to_string(operands.size()));
    for (const Tensor& t : operands) {
        PORTTEN_CHECK(t.defined(), "apply operand is undefined");
        PORTTEN_CHECK(t.sizes() == operands[0].sizes(), "apply operands must share sizes: " +
                                                            shape_of(operands[0]) + " vs " + shape_of(t));
    }
    const expr::Program program = expr::Program::parse(expression, static_cast<int>(operands.size()));
    const LaunchConfig lc = choose_launch(operands[0].numel(), backend.descriptor());
    PORTTEN_CHECK(lc.workgroupSize <= backend.descriptor().maxWorkgroupSize,
                  "launch config exceeds device workgroup limit");
    backend.runApply(program, operands, scalar, lc);
}

void dispatch_apply(std::string_view expression, std::span<DeviceTensor> operands, float scalar) {
    PORTTEN_CHECK(!operands.empty() && operands.size() <= 3,
                  "apply takes 1..3 operands, got " + std::to_string(operands.size()));
    float* bases[3] = {nullptr, nullptr, nullptr};
    pt_view views[3] = {};
    for (std::size_t t = 0; t < operands.size(); ++t) {
        PORTTEN_CHECK(operands[t].defined(), "apply operand is undefined");
        PORTTEN_CHECK(operands[t].sizes() == operands[0].sizes(), "apply operands must share sizes");
        bases[t] = operands[t].base();
        views[t] = operands[t].view();
    }
    const expr::Program program = expr::Program::parse(expression, static_cast<int>(operands.size()));
    throw_if_error(pt_b200_apply(program.code().data(), static_cast<std::int32_t>(program.code().size()),
                                 static_cast<int>(operands.size()), bases, views, scalar, nullptr));
}

float dispatch_reduce_all(ReduceOp op, const Tensor& t, Backend& backend) {
    PORTTEN_CHECK(t.defined(), "reduce on an undefined tensor");
    PORTTEN_CHECK(t.numel() >= 1, "reduce on an empty tensor");
    const LaunchConfig lc = choose_launch(t.numel(), backend.descriptor());
    PORTTEN_CHECK(lc.workgroupSize <= backend.descriptor().maxWorkgroupSize,
                  "launch config exceeds device workgroup limit");
    return backend.runReduceAll(op, t);
}

Tensor dispatch_reduce_dim(ReduceOp op, const Tensor& t, int dim, Backend& backend) {
    PORTTEN_CHECK(t.defined(), "reduce on an undefined tensor");
    PORTTEN_CHECK(dim >= 0 && dim < t.dim(), "reduce dim " + std::to_string(dim) +
                                                 " out of range for rank " + std::to_string(t.dim()));
    const LaunchConfig lc = choose_launch(t.numel(), backend.descriptor());
    PORTTEN_CHECK(lc.workgroupSize <= backend.descriptor().maxWorkgroupSize,
                  "launch config exceeds device workgroup limit");
    return backend.runReduceDim(op, t, dim);
}

DeviceBuffer device_upload(const Tensor& t, Backend& backend) {
    PORTTEN_CHECK(t.defined(), "upload of an undefined tensor");
    return backend.uploadContiguous(t.contiguous());
}

void device_download(const DeviceBuffer& buf, Tensor& dst, Backend& backend) {
    PORTTEN_CHECK(dst.defined(), "download into an undefined tensor");
    PORTTEN_CHECK(buf.elems == dst.numel(), "download size mismatch: buffer holds " +
                                                std::to_string(buf.elems) + " element(s), destination expects " +
                                                std::to_string(dst.numel()));
    if (dst.isContiguous()) {
        backend.downloadContiguous(buf, dst);
        return;
    }
    Tensor staged = Tensor::create(dst.sizes());
    backend.downloadContiguous(buf, staged);
    dst.copyFrom(staged);
}

}  // namespace portten
