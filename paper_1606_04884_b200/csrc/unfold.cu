// unfold.cu — the standalone unfold / fold ops of the SPEC convolution module.
//   im2col : proj/templates/im2col.kt.tmpl:9-21 (index maths, zero pad) — pure
//            copies, so bit-exact with the reference kernel; one thread per
//            column-matrix element so stores are coalesced along output pixels.
//   col2im : SPEC.md:371-379 scatter-add, computed in gather form (one thread per
//            image element, taps summed in (r, s) order from 0.0f) — no atomics,
//            deterministic, and the same summation order as the oracle's scatter.
#include "kernels.cuh"

namespace ptb {

namespace {

__global__ void im2col_kernel(const float* __restrict__ x, float* __restrict__ col, int C, int H,
                              int W, int kH, int kW, int pH, int pW, int sH, int sW, int oH,
                              int oW, int64_t n0, int64_t count) {
    const int64_t oHW = (int64_t)oH * oW;
    const int64_t ld = count * oHW;
    const int64_t rows = (int64_t)C * kH * kW;
    const int64_t total = rows * ld;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = e / ld, colpos = e - row * ld;
        const int64_t t = colpos / oHW, pos = colpos - t * oHW;
        const int c = (int)(row / (kH * kW));
        const int rs = (int)(row - (int64_t)c * kH * kW);
        const int r = rs / kW, s = rs - r * kW;
        const int i = (int)(pos / oW), j = (int)(pos - (int64_t)i * oW);
        const int h = i * sH - pH + r, w = j * sW - pW + s;
        const bool inside = (h >= 0) && (h < H) && (w >= 0) && (w < W);
        const float* img = x + (n0 + t) * (int64_t)C * H * W;
        col[e] = inside ? img[((int64_t)c * H + h) * W + w] : 0.0f;
    }
}

// img[n] = col2im(col[n]) for n in [0, N): one thread per image element.
__global__ void col2im_kernel(const float* __restrict__ colb, float* __restrict__ imgb, int C, int H,
                              int W, int kH, int kW, int pH, int pW, int sH, int sW, int oH,
                              int oW, int64_t N) {
    const int64_t oHW = (int64_t)oH * oW;
    const int64_t per = (int64_t)C * H * W;
    const int64_t total = per * N;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t n = e / per;
        const int64_t ei = e - n * per;
        const float* col = colb + n * (int64_t)C * kH * kW * oHW;
        float* img = imgb + n * per;
        const int c = (int)(ei / ((int64_t)H * W));
        const int hw = (int)(ei - (int64_t)c * H * W);
        const int h = hw / W, w = hw - h * W;
        float acc = 0.0f;
        for (int r = 0; r < kH; ++r) {
            const int hn = h + pH - r;
            if (hn < 0) break;
            const int i = hn / sH;
            if (i * sH != hn || i >= oH) continue;
            for (int s = 0; s < kW; ++s) {
                const int wn = w + pW - s;
                if (wn < 0) break;
                const int j = wn / sW;
                if (j * sW != wn || j >= oW) continue;
                acc += col[((int64_t)(c * kH + r) * kW + s) * oHW + (int64_t)i * oW + j];
            }
        }
        img[ei] = acc;
    }
}

// Stride-1 fast path: one image row (n, c, h) per (blockIdx.x, threadIdx.y), threads
// sweep w; taps are independent predicated loads (same (r, s) summation order as above,
// so results are bitwise identical). The general kernel's data-dependent break/continue
// serialises the loads (1.3 TB/s on VGG-A conv1's 347 MB gcol).
__global__ void col2im_s1_kernel(const float* __restrict__ colb, float* __restrict__ imgb, int C, int H,
                                 int W, int kH, int kW, int pH, int pW, int oH, int oW, int rows) {
    const int row = blockIdx.x * blockDim.y + threadIdx.y;  // (n, c, h)
    if (row >= rows) return;
    const int h = row % H;
    const int c = (row / H) % C;
    const int n = row / (H * C);
    const int64_t oHW = (int64_t)oH * oW;
    const float* col = colb + ((int64_t)n * C + c) * kH * kW * oHW;
    float* img = imgb + (int64_t)row * W;
    for (int w = threadIdx.x; w < W; w += blockDim.x) {
        float acc = 0.0f;
        for (int r = 0; r < kH; ++r) {
            const int i = h + pH - r;
            if (i < 0 || i >= oH) continue;  // uniform across the row's threads
            const float* cr = col + (int64_t)r * kW * oHW + (int64_t)i * oW;
#pragma unroll 4
            for (int s = 0; s < kW; ++s) {
                const int j = w + pW - s;
                if (j >= 0 && j < oW) acc += __ldg(cr + s * oHW + j);
            }
        }
        img[w] = acc;
    }
}

}  // namespace

void im2col_launch(const Geo& g, const float* x, int64_t n0, int64_t count, float* col,
                   cudaStream_t st) {
    const int64_t total = g.CRS * count * g.oHW;
    if (total == 0) return;
    const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 16 * (int64_t)sm_count());
    im2col_kernel<<<blocks, 256, 0, st>>>(x, col, (int)g.C, (int)g.H, (int)g.W, (int)g.kH,
                                          (int)g.kW, (int)g.pH, (int)g.pW, (int)g.sH, (int)g.sW,
                                          (int)g.oH, (int)g.oW, n0, count);
    after_launch("im2col");
}

static void col2im_n(const Geo& g, const float* col, float* img, int64_t n, cudaStream_t st) {
    const int64_t total = g.C * g.HW * n;
    if (g.sH == 1 && g.sW == 1 && n * g.C * g.H < (1ll << 31)) {
        const int rows = (int)(n * g.C * g.H);
        const int tx = g.W >= 128 ? 128 : g.W >= 64 ? 64 : 32;
        const int ty = 256 / tx;
        col2im_s1_kernel<<<(unsigned)ceil_div(rows, ty), dim3(tx, ty), 0, st>>>(
            col, img, (int)g.C, (int)g.H, (int)g.W, (int)g.kH, (int)g.kW, (int)g.pH, (int)g.pW,
            (int)g.oH, (int)g.oW, rows);
        after_launch("col2im");
        return;
    }
    const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 16 * (int64_t)sm_count());
    col2im_kernel<<<blocks, 256, 0, st>>>(col, img, (int)g.C, (int)g.H, (int)g.W, (int)g.kH,
                                          (int)g.kW, (int)g.pH, (int)g.pW, (int)g.sH, (int)g.sW,
                                          (int)g.oH, (int)g.oW, n);
    after_launch("col2im");
}

void col2im_launch(const Geo& g, const float* col, float* img, cudaStream_t st) {
    col2im_n(g, col, img, 1, st);
}

void col2im_batched_launch(const Geo& g, const float* col, float* img, cudaStream_t st) {
    col2im_n(g, col, img, g.N, st);
}

}  // namespace ptb
