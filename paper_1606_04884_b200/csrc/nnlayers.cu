// nnlayers.cu — the non-conv layers of the model-stack bench (bench_model
// :484-492: ModelSpec layers conv / pool-max / relu): ReLU and max pooling, forward and
// backward, NCHW float32. Both are HBM-bound streaming passes: ReLU moves float4 vectors
// with a grid sized to the SMs; max pooling reads each window from L2-resident rows and
// records the arg-max (int32 index within the input plane) for the backward, which is a
// deterministic gather (every input pixel sums, in ascending window order, the gradients
// of the windows whose arg-max it is — no atomics, so results do not depend on scheduling).
#include "kernels.cuh"

namespace ptb {

namespace {

int stream_grid(int64_t work) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, 256), 8 * (int64_t)sm_count()));
}

__global__ void relu_fwd_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t n, int vec) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t start = 0;
    if (vec) {
        const int64_t n4 = n / 4;
        for (int64_t i = tid; i < n4; i += stride) {
            float4 v = reinterpret_cast<const float4*>(x)[i];
            v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
            reinterpret_cast<float4*>(y)[i] = v;
        }
        start = n4 * 4;
    }
    for (int64_t i = start + tid; i < n; i += stride) y[i] = fmaxf(x[i], 0.f);
}

// gx = gy where the forward output is positive (Torch threshold backward), else 0
__global__ void relu_bwd_kernel(const float* __restrict__ y, const float* __restrict__ gy,
                                float* __restrict__ gx, int64_t n, int vec) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t start = 0;
    if (vec) {
        const int64_t n4 = n / 4;
        for (int64_t i = tid; i < n4; i += stride) {
            const float4 o = reinterpret_cast<const float4*>(y)[i];
            float4 g = reinterpret_cast<const float4*>(gy)[i];
            g.x = o.x > 0.f ? g.x : 0.f; g.y = o.y > 0.f ? g.y : 0.f;
            g.z = o.z > 0.f ? g.z : 0.f; g.w = o.w > 0.f ? g.w : 0.f;
            reinterpret_cast<float4*>(gx)[i] = g;
        }
        start = n4 * 4;
    }
    for (int64_t i = start + tid; i < n; i += stride) gx[i] = y[i] > 0.f ? gy[i] : 0.f;
}

struct PoolGeo {
    int64_t planes;  // N*C
    int32_t H, W, oH, oW, kH, kW, sH, sW, pH, pW;
};

// one block-stride loop over (plane, output row) — the only 64-bit division is per row and
// block-uniform — with the threads along the output row; padding positions never win
// (-inf); NaN propagates
__global__ void maxpool_fwd_kernel(const float* __restrict__ x, float* __restrict__ y,
                                   int32_t* __restrict__ arg, const PoolGeo g) {
    const int64_t rows = g.planes * g.oH;
    for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
        const int64_t plane = row / g.oH;
        const int oh = (int)(row - plane * g.oH);
        const float* xp = x + plane * g.H * g.W;
        const int h0 = oh * g.sH - g.pH;
        const int64_t ob = row * g.oW;
        for (int ow = threadIdx.x; ow < g.oW; ow += blockDim.x) {
            const int w0 = ow * g.sW - g.pW;
            float best = -INFINITY;
            int32_t bi = -1;
            for (int r = 0; r < g.kH; ++r) {
                const int h = h0 + r;
                if (h < 0 || h >= g.H) continue;
                for (int s = 0; s < g.kW; ++s) {
                    const int w = w0 + s;
                    if (w < 0 || w >= g.W) continue;
                    const float v = __ldg(xp + h * g.W + w);
                    if (v > best || bi < 0 || (v != v && best == best)) {
                        best = v;
                        bi = h * g.W + w;
                    }
                }
            }
            y[ob + ow] = best;
            if (arg) arg[ob + ow] = bi;
        }
    }
}

// gather form: input pixel (h, w) receives gy of every window (oh, ow) covering it whose
// arg-max is (h, w), summed in ascending (oh, ow) order; (plane, input row) per block step
__global__ void maxpool_bwd_kernel(const float* __restrict__ gy, const int32_t* __restrict__ arg,
                                   float* __restrict__ gx, const PoolGeo g) {
    const int64_t rows = g.planes * g.H;
    for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
        const int64_t plane = row / g.H;
        const int h = (int)(row - plane * g.H);
        // windows with oh*sH - pH <= h <= oh*sH - pH + kH - 1
        const int oh_lo = max(0, (h + g.pH - g.kH + g.sH) / g.sH);
        const int oh_hi = min(g.oH - 1, (h + g.pH) / g.sH);
        const int64_t ob = plane * g.oH * g.oW;
        for (int w = threadIdx.x; w < g.W; w += blockDim.x) {
            const int32_t me = h * g.W + w;
            const int ow_lo = max(0, (w + g.pW - g.kW + g.sW) / g.sW);
            const int ow_hi = min(g.oW - 1, (w + g.pW) / g.sW);
            float acc = 0.f;
            for (int oh = oh_lo; oh <= oh_hi; ++oh)
                for (int ow = ow_lo; ow <= ow_hi; ++ow) {
                    const int64_t o = ob + (int64_t)oh * g.oW + ow;
                    if (__ldg(arg + o) == me) acc += __ldg(gy + o);
                }
            gx[row * g.W + w] = acc;
        }
    }
}

int row_block(int64_t len) { return len >= 192 ? 256 : (len >= 96 ? 128 : 64); }
int row_grid(int64_t rows) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(rows, 32 * (int64_t)sm_count()));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

PoolGeo pool_geo(int64_t N, int64_t C, int64_t H, int64_t W, int kH, int kW, int sH, int sW,
                 int pH, int pW) {
    PTB_REQUIRE(N >= 1 && C >= 1 && H >= 1 && W >= 1 && kH >= 1 && kW >= 1 && sH >= 1 && sW >= 1 &&
                    pH >= 0 && pW >= 0, "maxpool: counts, dims, window and stride must be >= 1");
    PTB_REQUIRE(2 * pH <= kH && 2 * pW <= kW, "maxpool: padding must be at most half the window");
    PTB_REQUIRE(H < (1 << 15) && W < (1 << 15), "maxpool: plane too large");
    PoolGeo g;
    g.planes = N * C;
    g.H = (int)H; g.W = (int)W; g.kH = kH; g.kW = kW; g.sH = sH; g.sW = sW; g.pH = pH; g.pW = pW;
    const int64_t oH = (H + 2 * pH - kH) / sH + 1, oW = (W + 2 * pW - kW) / sW + 1;
    PTB_REQUIRE(H + 2 * pH >= kH && W + 2 * pW >= kW && oH >= 1 && oW >= 1, "maxpool: empty output");
    g.oH = (int)oH;
    g.oW = (int)oW;
    return g;
}

}  // namespace

void relu_fwd(const float* x, float* y, int64_t n, cudaStream_t st) {
    const int vec = aligned16(x) && aligned16(y);
    ProfScope ps("layout", st, 0.0, 8.0 * n);
    relu_fwd_kernel<<<stream_grid(vec ? n / 4 + 1 : n), 256, 0, st>>>(x, y, n, vec);
    after_launch("relu_fwd");
}

void relu_bwd(const float* y, const float* gy, float* gx, int64_t n, cudaStream_t st) {
    const int vec = aligned16(y) && aligned16(gy) && aligned16(gx);
    ProfScope ps("layout", st, 0.0, 12.0 * n);
    relu_bwd_kernel<<<stream_grid(vec ? n / 4 + 1 : n), 256, 0, st>>>(y, gy, gx, n, vec);
    after_launch("relu_bwd");
}

void maxpool_fwd(const float* x, float* y, int32_t* arg, int64_t N, int64_t C, int64_t H, int64_t W,
                 int kH, int kW, int sH, int sW, int pH, int pW, cudaStream_t st) {
    const PoolGeo g = pool_geo(N, C, H, W, kH, kW, sH, sW, pH, pW);
    const int64_t out = g.planes * g.oH * g.oW;
    ProfScope ps("layout", st, 0.0, 4.0 * (g.planes * H * W + out * (arg ? 2 : 1)));
    maxpool_fwd_kernel<<<row_grid(g.planes * g.oH), row_block(g.oW), 0, st>>>(x, y, arg, g);
    after_launch("maxpool_fwd");
}

void maxpool_bwd(const float* gy, const int32_t* arg, float* gx, int64_t N, int64_t C, int64_t H,
                 int64_t W, int kH, int kW, int sH, int sW, int pH, int pW, cudaStream_t st) {
    const PoolGeo g = pool_geo(N, C, H, W, kH, kW, sH, sW, pH, pW);
    const int64_t in = g.planes * H * W;
    ProfScope ps("layout", st, 0.0, 4.0 * (in + 2 * g.planes * g.oH * g.oW));
    maxpool_bwd_kernel<<<row_grid(g.planes * H), row_block(W), 0, st>>>(gy, arg, gx, g);
    after_launch("maxpool_bwd");
}

}  // namespace ptb
