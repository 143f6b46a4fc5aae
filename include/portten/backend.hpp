// Backend — the execution-backend boundary of the reference
// (proj/include/portten/backend.hpp:31-112): BackendDescriptor, LaunchConfig /
// choose_launch, DeviceBuffer, the abstract Backend, enumeration/selection by
// PORTTEN_BACKEND / PORTTEN_DEVICE, and the validating dispatch_* wrappers.
//
// B200 build: the device slot (the reference's opencl_probe_devices,
// proj/src/opencl_backend.hpp:29) is filled by cuda_probe_devices() — one B200Backend
// per sm_100 GPU, all work in libpt_b200.so. The host interpreter ("reference") is NOT
// part of this library: it is the oracle (oracle/), never a fallback; selecting it
// throws BackendError.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <string>
#include <string_view>
#include <vector>

#include "portten/expression.hpp"
#include "portten/tensor.hpp"

namespace portten {

struct BackendDescriptor {
    std::string name;
    int maxWorkgroupSize = 1;
    std::int64_t localMemBytes = 0;
    bool isDevice = false;
};

struct LaunchConfig {
    std::int64_t globalSize = 0;
    int workgroupSize = 0;
};

/// workgroupSize = min(256, device max); globalSize = n rounded up (backend.cpp:25-33).
LaunchConfig choose_launch(std::int64_t n, const BackendDescriptor& d);

struct DeviceBuffer {
    std::shared_ptr<void> impl;
    std::int64_t elems = 0;
    std::string backendName;
};

enum class ReduceOp { Sum = PT_REDUCE_SUM, Max = PT_REDUCE_MAX, Min = PT_REDUCE_MIN };

class Backend {
public:
    virtual ~Backend() = default;
    virtual const BackendDescriptor& descriptor() const = 0;
    virtual void runApply(const expr::Program& program, std::span<Tensor> operands, float scalar,
                          const LaunchConfig& lc) = 0;
    virtual float runReduceAll(ReduceOp op, const Tensor& t) = 0;
    virtual Tensor runReduceDim(ReduceOp op, const Tensor& t, int dim) = 0;
    virtual DeviceBuffer uploadContiguous(const Tensor& t) = 0;
    virtual void downloadContiguous(const DeviceBuffer& buf, Tensor& dst) = 0;
};

/// One backend per usable sm_100 device (empty when none). Replaces the reference's
/// opencl_probe_devices() slot.
std::vector<Backend*> cuda_probe_devices();
std::vector<Backend*> backend_enumerate();
/// "auto" | "device": the B200 device (PORTTEN_DEVICE index); "reference" -> BackendError.
Backend& select_backend(std::string_view requested);

void dispatch_apply(std::string_view expression, std::span<Tensor> operands, float scalar,
                    Backend& backend);
float dispatch_reduce_all(ReduceOp op, const Tensor& t, Backend& backend);
Tensor dispatch_reduce_dim(ReduceOp op, const Tensor& t, int dim, Backend& backend);
DeviceBuffer device_upload(const Tensor& t, Backend& backend);
void device_download(const DeviceBuffer& buf, Tensor& dst, Backend& backend);

/// Device-resident overloads (no host round trip).
void dispatch_apply(std::string_view expression, std::span<DeviceTensor> operands, float scalar);

}  // namespace portten
