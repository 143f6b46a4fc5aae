// common.cuh — shared plumbing for libpt_b200.so (error state, launch accounting,
// geometry helpers). No kernel here depends on torch; all entry points are the
// extern "C" functions of include/pt_b200.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <functional>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/pt_b200.h"

namespace ptb {

// Thrown inside the library, converted to a status code at the ABI edge.
struct AbiError : std::runtime_error {
    int code;
    AbiError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail_validation(const std::string& m) { throw AbiError(PT_EVALIDATION, m); }
[[noreturn]] inline void fail_backend(const std::string& m) { throw AbiError(PT_EBACKEND, m); }

#define PTB_REQUIRE(cond, msg)                     \
    do {                                           \
        if (!(cond)) ::ptb::fail_validation(msg);  \
    } while (0)

#define PTB_CUDA(call)                                                                        \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            ::ptb::fail_backend(std::string(#call) + ": " + cudaGetErrorString(e_));          \
    } while (0)

extern std::atomic<int64_t> g_launches;

// Every kernel launch goes through this so bench.py can report gpu_launches and
// launch errors surface at the call that caused them.
inline void after_launch(const char* what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail_backend(std::string("launch ") + what + ": " + cudaGetErrorString(e));
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Derived conv sizes (conv_geometry.hpp:41-51).
struct Geo {
    int64_t N, C, H, W, K, kH, kW, pH, pW, sH, sW;
    int64_t oH, oW, oHW, CRS, HW, M;  // M = N*oH*oW (GEMM pixels)
    explicit Geo(const pt_conv_geom& g)
        : N(g.N), C(g.C), H(g.H), W(g.W), K(g.K), kH(g.kH), kW(g.kW), pH(g.padH), pW(g.padW),
          sH(g.strideH), sW(g.strideW) {
        oH = (H + 2 * pH - kH) / sH + 1;
        oW = (W + 2 * pW - kW) / sW + 1;
        oHW = oH * oW;
        CRS = C * kH * kW;
        HW = H * W;
        M = N * oHW;
    }
};

void validate_geom(const pt_conv_geom* g);  // throws AbiError(PT_EVALIDATION)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

int sm_count();  // of the current device (cached)

}  // namespace ptb

namespace ptb {
// Live kernel timing for bench.py (pt_b200_profile_*). When disabled this is a
// single relaxed atomic load per launch.
bool prof_enabled();
struct ProfScope {
    const char* cls;
    cudaStream_t st;
    double flops, bytes;
    cudaEvent_t e0 = nullptr;
    ProfScope(const char* c, cudaStream_t s, double f, double b);
    ~ProfScope();
};
// Concurrency of independent work inside one API call (pt_b200_set_bwd_streams): internal
// non-blocking streams per (device, caller stream) (slot 0: the backward's weight gradient,
// slot 1: weight packs next to layout passes) joined back to the caller's stream with events.
bool concurrency_on();
void set_concurrency(int on);
cudaStream_t aux_stream(cudaStream_t caller, int slot);
// Runs `set` once per (current device, key) and makes concurrent callers wait until it has
// run: kernel attributes such as the dynamic shared-memory limit are per device.
void once_per_device(const void* key, const std::function<void()>& set);
// fork(st, slot): work submitted to .side after this waits for everything already on st;
// join(): st waits for everything submitted to .side. side == st when concurrency is off.
struct Fork {
    cudaStream_t st, side;
    Fork(cudaStream_t s, int slot);
    Fork(const Fork&) = delete;
    Fork& operator=(const Fork&) = delete;
    // An error thrown between fork and join still leaves st ordered after the side work,
    // so the caller never frees or reuses buffers the side stream is still reading.
    ~Fork();
    void join();
};
// Labels the launches recorded while alive with the conv pass ("fwd", "dgrad", "wgrad").
struct PassScope {
    const char* prev;
    explicit PassScope(const char* pass);
    ~PassScope();
};
}  // namespace ptb
