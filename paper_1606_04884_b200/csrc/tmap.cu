// tmap.cu — host-side TMA descriptor encoding (cuTensorMapEncodeTiled / Im2col)
// through the runtime's driver-entry-point query (no link-time libcuda dependency).
#include <cudaTypedefs.h>

#include <mutex>
#include <string>

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
}  // namespace

void tmap_im2col(CUtensorMap* m, const float* act, int64_t N, int64_t H, int64_t W, int64_t Cp,
                 int kH, int kW, int pH, int pW, int sH, int sW, int channels, int pixels,
                 CUtensorMapSwizzle swizzle) {
    load();
    cuuint64_t dims[4] = {(cuuint64_t)Cp, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)(Cp * 4), (cuuint64_t)(W * Cp * 4),
                             (cuuint64_t)(H * W * Cp * 4)};
    int lower[2] = {-pW, -pH};
    int upper[2] = {pW - (kW - 1), pH - (kH - 1)};
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
    load();
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
