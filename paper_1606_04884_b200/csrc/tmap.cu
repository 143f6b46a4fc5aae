// tmap.cu — host-side TMA descriptor encoding (cuTensorMapEncodeTiled / Im2col)
// through the runtime's driver-entry-point query (no link-time libcuda dependency).
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "tmap.cuh"

namespace ptb {

namespace {
PFN_cuTensorMapEncodeTiled_v12000 g_encode_tiled = nullptr;
PFN_cuTensorMapEncodeIm2col_v12000 g_encode_im2col = nullptr;
int g_driver_version = 0;
std::string g_err;

void load() {
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q1, q2;
        void* f1 = nullptr;
        void* f2 = nullptr;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f1, 12000, cudaEnableDefault,
                                             &q1) != cudaSuccess ||
            q1 != cudaDriverEntryPointSuccess ||
            cudaGetDriverEntryPointByVersion("cuTensorMapEncodeIm2col", &f2, 12000,
                                             cudaEnableDefault, &q2) != cudaSuccess ||
            q2 != cudaDriverEntryPointSuccess) {
            g_err = "cuTensorMapEncode* driver entry points unavailable";
            return;
        }
        g_encode_tiled = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f1);
        g_encode_im2col = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(f2);
        cudaDriverGetVersion(&g_driver_version);
    });
    if (!g_encode_tiled || !g_encode_im2col) fail_backend(g_err);
}

// Driver releases <= 13.1 mis-handle a descriptor flag for tensors under 128 KiB
// (the same workaround CUTLASS applies in copy_traits_sm90_im2col.hpp).
void small_tensor_fixup(CUtensorMap* m, size_t bytes) {
    if (g_driver_version <= 13010 && bytes < 131072) reinterpret_cast<uint64_t*>(m)[1] &= ~(1ull << 21);
}

// ---- descriptor cache ----
// A tensor map is a pure function of its encode arguments, so repeated calls with the same
// buffers (a training loop re-running a layer on the same activations / workspace) reuse the
// encoded descriptor instead of calling into the driver again (the encodes were most of the
// host time of an eager conv call). Per thread: no locking on the launch path; bounded.
struct TmapKey {
    uint64_t w[24];
    bool operator==(const TmapKey& o) const { return std::memcmp(w, o.w, sizeof w) == 0; }
};
struct TmapKeyHash {
    size_t operator()(const TmapKey& k) const {
        uint64_t h = 1469598103934665603ull;
        for (uint64_t v : k.w) h = (h ^ v) * 1099511628211ull;
        return (size_t)h;
    }
};
std::unordered_map<TmapKey, CUtensorMap, TmapKeyHash>& tmap_cache() {
    thread_local std::unordered_map<TmapKey, CUtensorMap, TmapKeyHash> c;
    if (c.size() > 4096) c.clear();
    return c;
}
std::atomic<int64_t> g_tmap_hits{0}, g_tmap_encodes{0};
bool tmap_cache_on() {
    static const bool on = std::getenv("PT_B200_NO_TMAP_CACHE") == nullptr;
    return on;
}
}  // namespace

void tmap_cache_stats(int64_t* hits, int64_t* encodes) {
    if (hits) *hits = g_tmap_hits.load();
    if (encodes) *encodes = g_tmap_encodes.load();
}

void tmap_im2col(CUtensorMap* m, const float* act, int64_t N, int64_t H, int64_t W, int64_t Cp,
                 int kH, int kW, int pH, int pW, int sH, int sW, int channels, int pixels,
                 CUtensorMapSwizzle swizzle, int pW_right) {
    TmapKey key{};
    const uint64_t a[] = {1, (uint64_t)(uintptr_t)act, (uint64_t)N, (uint64_t)H, (uint64_t)W, (uint64_t)Cp,
                          (uint64_t)kH, (uint64_t)kW, (uint64_t)pH, (uint64_t)pW, (uint64_t)sH, (uint64_t)sW,
                          (uint64_t)channels, (uint64_t)pixels, (uint64_t)swizzle, (uint64_t)(int64_t)pW_right};
    std::memcpy(key.w, a, sizeof a);
    if (tmap_cache_on()) {
        auto& c = tmap_cache();
        auto it = c.find(key);
        if (it != c.end()) {
            *m = it->second;
            g_tmap_hits.fetch_add(1, std::memory_order_relaxed);
            return;
        }
        tmap_im2col_encode(m, act, N, H, W, Cp, kH, kW, pH, pW, sH, sW, channels, pixels, swizzle, pW_right);
        c.emplace(key, *m);
        return;
    }
    tmap_im2col_encode(m, act, N, H, W, Cp, kH, kW, pH, pW, sH, sW, channels, pixels, swizzle, pW_right);
}

void tmap_im2col_encode(CUtensorMap* m, const float* act, int64_t N, int64_t H, int64_t W, int64_t Cp,
                        int kH, int kW, int pH, int pW, int sH, int sW, int channels, int pixels,
                        CUtensorMapSwizzle swizzle, int pW_right) {
    load();
    g_tmap_encodes.fetch_add(1, std::memory_order_relaxed);
    cuuint64_t dims[4] = {(cuuint64_t)Cp, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)(Cp * 4), (cuuint64_t)(W * Cp * 4),
                             (cuuint64_t)(H * W * Cp * 4)};
    int lower[2] = {-pW, -pH};
    int upper[2] = {(pW_right < 0 ? pW : pW_right) - (kW - 1), pH - (kH - 1)};
    cuuint32_t estr[4] = {1, (cuuint32_t)sW, (cuuint32_t)sH, 1};
    CUresult r = g_encode_im2col(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(act), dims,
                                 strides, lower, upper, (cuuint32_t)channels, (cuuint32_t)pixels, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail_backend("cuTensorMapEncodeIm2col failed (" + std::to_string((int)r) + ")");
    small_tensor_fixup(m, (size_t)(N * H * W * Cp * 4));
}

void tmap_tiled(CUtensorMap* m, const float* base, int rank, const uint64_t* dims,
                const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swizzle) {
    if (tmap_cache_on() && rank >= 1 && rank <= 5) {
        TmapKey key{};
        key.w[0] = 2;
        key.w[1] = (uint64_t)(uintptr_t)base;
        key.w[2] = (uint64_t)rank | ((uint64_t)swizzle << 8);
        for (int i = 0; i < rank; ++i) {
            key.w[3 + i] = dims[i];
            key.w[8 + i] = box[i];
            if (i + 1 < rank) key.w[13 + i] = strides_bytes[i];
        }
        auto& c = tmap_cache();
        auto it = c.find(key);
        if (it != c.end()) {
            *m = it->second;
            g_tmap_hits.fetch_add(1, std::memory_order_relaxed);
            return;
        }
        tmap_tiled_encode(m, base, rank, dims, strides_bytes, box, swizzle);
        c.emplace(key, *m);
        return;
    }
    tmap_tiled_encode(m, base, rank, dims, strides_bytes, box, swizzle);
}

void tmap_tiled_encode(CUtensorMap* m, const float* base, int rank, const uint64_t* dims,
                       const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swizzle) {
    load();
    g_tmap_encodes.fetch_add(1, std::memory_order_relaxed);
    cuuint64_t d[5], s[4];
    cuuint32_t b[5], e[5];
    size_t bytes = 4;
    for (int i = 0; i < rank; ++i) {
        d[i] = dims[i];
        b[i] = box[i];
        e[i] = 1;
        if (i + 1 < rank) s[i] = strides_bytes[i];
    }
    // footprint of the whole view (strides need not be monotone, e.g. a channel-block dim)
    bytes = (size_t)dims[0] * 4;
    for (int i = 1; i < rank; ++i) bytes += (size_t)(dims[i] - 1) * strides_bytes[i - 1];
    CUresult r = g_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<float*>(base), d, s,
                                b, e, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail_backend("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    small_tensor_fixup(m, bytes);
}

}  // namespace ptb
