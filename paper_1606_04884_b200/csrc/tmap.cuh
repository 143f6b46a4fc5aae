// tmap.cuh — TMA descriptor helpers (host). Activations are NHWC float32.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace ptb {

// im2col-mode descriptor over an NHWC tensor [N][H][W][Cp] for a kH x kW conv with
// padding (pH,pW) and stride (sH,sW): each box is `pixels` consecutive output
// pixels x `channels` channels of one filter tap.
// pW_right >= 0: right padding differing from the left one (default: symmetric)
void tmap_im2col(CUtensorMap* m, const float* act, int64_t N, int64_t H, int64_t W, int64_t Cp,
                 int kH, int kW, int pH, int pW, int sH, int sW, int channels, int pixels,
                 CUtensorMapSwizzle swizzle, int pW_right = -1);

// Tiled descriptor: dims innermost-first (elements), strides of dims 1.. in bytes.
void tmap_tiled(CUtensorMap* m, const float* base, int rank, const uint64_t* dims,
                const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swizzle);

// The two above go through a per-thread descriptor cache keyed by every encode argument
// (PT_B200_NO_TMAP_CACHE=1 disables it); the *_encode forms always call the driver.
void tmap_im2col_encode(CUtensorMap* m, const float* act, int64_t N, int64_t H, int64_t W, int64_t Cp,
                        int kH, int kW, int pH, int pW, int sH, int sW, int channels, int pixels,
                        CUtensorMapSwizzle swizzle, int pW_right = -1);
void tmap_tiled_encode(CUtensorMap* m, const float* base, int rank, const uint64_t* dims,
                       const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swizzle);
void tmap_cache_stats(int64_t* hits, int64_t* encodes);

}  // namespace ptb
