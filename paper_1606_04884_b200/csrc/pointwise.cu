// pointwise.cu — the apply / reduce kernels that sit on the conv path
// (Backend::runApply / runReduceAll / runReduceDim, proj/include/portten/backend.hpp:75-78).
//
// The reference renders one OpenCL kernel per (expression, strides, offsets)
// (proj/src/kernel_codegen.cpp:131-245). Here there is no runtime codegen: the
// expression arrives as RPN bytecode (expr::Program's instruction stream,
// proj/src/expression.cpp:340-402) and one compiled kernel interprets it per
// element, with a vectorised float4 path for contiguous operands and fused
// fast paths for the conv-path statements (x = x + s, x = s, x = x * s, x = y,
// x = x + y). Reductions are warp-shuffle trees with a fixed two-stage order.
#include <cstring>

#include "kernels.cuh"

namespace ptb {

namespace {

constexpr int kMaxCode = 192;

struct ApplyArgs {
    int32_t code[kMaxCode];
    int32_t ncode;
    int32_t arity;
    float scalar;
    int32_t ndim;
    int64_t sizes[8];
    int64_t strides[3][8];
    int64_t offset[3];
    float* base[3];
    int64_t n;
};

__device__ __forceinline__ float vm_eval(const ApplyArgs& a, float x, float y, float z) {
    float st[32];
    int top = 0;
    for (int pc = 0; pc < a.ncode; ++pc) {
        const int32_t ins = a.code[pc];
        switch (ins & 0xff) {
            case PT_OP_CONST: st[top++] = __int_as_float(a.code[++pc]); break;
            case PT_OP_X: st[top++] = x; break;
            case PT_OP_Y: st[top++] = y; break;
            case PT_OP_Z: st[top++] = z; break;
            case PT_OP_S: st[top++] = a.scalar; break;
            case PT_OP_ADD: --top; st[top - 1] = __fadd_rn(st[top - 1], st[top]); break;
            case PT_OP_SUB: --top; st[top - 1] = __fsub_rn(st[top - 1], st[top]); break;
            case PT_OP_MUL: --top; st[top - 1] = __fmul_rn(st[top - 1], st[top]); break;
            case PT_OP_DIV: --top; st[top - 1] = __fdiv_rn(st[top - 1], st[top]); break;
            case PT_OP_NEG: st[top - 1] = -st[top - 1]; break;
            case PT_OP_ABS: st[top - 1] = fabsf(st[top - 1]); break;
            case PT_OP_EXP: st[top - 1] = expf(st[top - 1]); break;
            case PT_OP_LOG: st[top - 1] = logf(st[top - 1]); break;
            case PT_OP_SQRT: st[top - 1] = __fsqrt_rn(st[top - 1]); break;
            case PT_OP_TANH: st[top - 1] = tanhf(st[top - 1]); break;
            case PT_OP_MAX: --top; st[top - 1] = fmaxf(st[top - 1], st[top]); break;
            case PT_OP_MIN: --top; st[top - 1] = fminf(st[top - 1], st[top]); break;
            default: break;
        }
    }
    return st[0];
}

__device__ __forceinline__ int64_t view_off(const ApplyArgs& a, int t, int64_t i) {
    int64_t off = a.offset[t];
    for (int d = a.ndim - 1; d >= 0; --d) {
        const int64_t sz = a.sizes[d];
        const int64_t q = i / sz;
        off += (i - q * sz) * a.strides[t][d];
        i = q;
    }
    return off;
}

__global__ void apply_strided_kernel(const __grid_constant__ ApplyArgs a) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float v[3] = {0.f, 0.f, 0.f};
        int64_t off0 = 0;
        for (int t = 0; t < a.arity; ++t) {
            const int64_t o = view_off(a, t, i);
            if (t == 0) off0 = o;
            v[t] = a.base[t][o];
        }
        a.base[0][off0] = vm_eval(a, v[0], v[1], v[2]);
    }
}

// All operands contiguous (offsets honoured): flat index; when every operand is 16-byte
// aligned (vec), float4 loads/stores with four independent evaluations per thread, then a
// scalar tail.
__global__ void apply_contig_kernel(const __grid_constant__ ApplyArgs a, int vec) {
    float* x = a.base[0] + a.offset[0];
    const float* y = a.arity > 1 ? a.base[1] + a.offset[1] : nullptr;
    const float* z = a.arity > 2 ? a.base[2] + a.offset[2] : nullptr;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t start = 0;
    if (vec) {
        const int64_t n4 = a.n / 4;
        float4* x4 = reinterpret_cast<float4*>(x);
        const float4* y4 = reinterpret_cast<const float4*>(y);
        const float4* z4 = reinterpret_cast<const float4*>(z);
        const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t i = tid; i < n4; i += stride) {
            float4 xv = x4[i];
            const float4 yv = y4 ? y4[i] : zero;
            const float4 zv = z4 ? z4[i] : zero;
            xv.x = vm_eval(a, xv.x, yv.x, zv.x);
            xv.y = vm_eval(a, xv.y, yv.y, zv.y);
            xv.z = vm_eval(a, xv.z, yv.z, zv.z);
            xv.w = vm_eval(a, xv.w, yv.w, zv.w);
            x4[i] = xv;
        }
        start = n4 * 4;
    }
    for (int64_t i = start + tid; i < a.n; i += stride) {
        x[i] = vm_eval(a, x[i], y ? y[i] : 0.f, z ? z[i] : 0.f);
    }
}

// Fast paths for the conv-path statements, float4 vectorised.
enum FastOp { kFill = 1, kScale = 2, kAddS = 3, kCopy = 4, kAdd = 5 };

__global__ void apply_fast_kernel(float* __restrict__ x, const float* __restrict__ y, int64_t n,
                                  float s, int op) {
    const int64_t n4 = n / 4;
    float4* x4 = reinterpret_cast<float4*>(x);
    const float4* y4 = reinterpret_cast<const float4*>(y);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 v;
        switch (op) {
            case kFill: v = make_float4(s, s, s, s); break;
            case kScale: v = x4[i]; v.x *= s; v.y *= s; v.z *= s; v.w *= s; break;
            case kAddS: v = x4[i]; v.x += s; v.y += s; v.z += s; v.w += s; break;
            case kCopy: v = y4[i]; break;
            default: {
                v = x4[i];
                const float4 u = y4[i];
                v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w;
            }
        }
        x4[i] = v;
    }
    for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        switch (op) {
            case kFill: x[i] = s; break;
            case kScale: x[i] = x[i] * s; break;
            case kAddS: x[i] = x[i] + s; break;
            case kCopy: x[i] = y[i]; break;
            default: x[i] = x[i] + y[i];
        }
    }
}

int match_fast(const int32_t* c, int32_t n, int arity) {
    auto is = [&](std::initializer_list<int32_t> ops) {
        if ((int32_t)ops.size() != n) return false;
        int i = 0;
        for (int32_t o : ops)
            if ((c[i++] & 0xff) != o) return false;
        return true;
    };
    if (is({PT_OP_S})) return kFill;
    if (is({PT_OP_X, PT_OP_S, PT_OP_MUL})) return kScale;
    if (is({PT_OP_X, PT_OP_S, PT_OP_ADD})) return kAddS;
    if (arity >= 2 && is({PT_OP_Y})) return kCopy;
    if (arity >= 2 && is({PT_OP_X, PT_OP_Y, PT_OP_ADD})) return kAdd;
    return 0;
}

bool contiguous(const pt_view& v) {
    int64_t expect = 1;
    for (int d = v.ndim - 1; d >= 0; --d) {
        if (v.sizes[d] != 1 && v.strides[d] != expect) return false;
        expect *= v.sizes[d];
    }
    return true;
}

int64_t numel(const pt_view& v) {
    int64_t n = 1;
    for (int d = 0; d < v.ndim; ++d) n *= v.sizes[d];
    return n;
}

int grid_for(int64_t n) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 8 * (int64_t)sm_count()));
}

__global__ void fill_uniform_kernel(float* __restrict__ dst, int64_t n, uint64_t seed, float lo,
                                    float span) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t z = seed + (uint64_t)i + 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const float u = (float)(z >> 40) * (1.0f / 16777216.0f);
        dst[i] = __fadd_rn(lo, __fmul_rn(span, u));
    }
}

__global__ void bias_add_kernel(float* __restrict__ y, const float* __restrict__ b, int64_t K,
                                int64_t HW, int64_t rows) {
    // one block-stride loop over (n,k) rows; inner loop coalesced along HW
    for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
        const float bias = __ldg(b + row % K);
        float* r = y + row * HW;
        if ((HW & 3) == 0 && ((reinterpret_cast<uintptr_t>(r) & 15) == 0)) {
            float4* r4 = reinterpret_cast<float4*>(r);
            for (int64_t i = threadIdx.x; i < HW / 4; i += blockDim.x) {
                float4 v = r4[i];
                v.x += bias; v.y += bias; v.z += bias; v.w += bias;
                r4[i] = v;
            }
        } else {
            for (int64_t i = threadIdx.x; i < HW; i += blockDim.x) r[i] += bias;
        }
    }
}

__device__ __forceinline__ float red_id(int op) {
    return op == PT_REDUCE_SUM ? 0.f : (op == PT_REDUCE_MAX ? -INFINITY : INFINITY);
}
__device__ __forceinline__ float red_op(int op, float a, float b) {
    return op == PT_REDUCE_SUM ? a + b : (op == PT_REDUCE_MAX ? fmaxf(a, b) : fminf(a, b));
}
__device__ __forceinline__ float warp_red(int op, float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = red_op(op, v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ float block_red(int op, float v) {
    __shared__ float sh[32];
    v = warp_red(op, v);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    v = threadIdx.x < blockDim.x / 32 ? sh[threadIdx.x] : red_id(op);
    if (threadIdx.x < 32) v = warp_red(op, v);
    __syncthreads();
    return v;
}

struct RedView {
    int32_t ndim;
    int64_t sizes[8];
    int64_t strides[8];
    int64_t offset;
};

__device__ __forceinline__ int64_t rv_off(const RedView& v, int64_t i) {
    int64_t off = v.offset;
    for (int d = v.ndim - 1; d >= 0; --d) {
        const int64_t q = i / v.sizes[d];
        off += (i - q * v.sizes[d]) * v.strides[d];
        i = q;
    }
    return off;
}

__global__ void reduce_all_partial(const float* __restrict__ base, const __grid_constant__ RedView v,
                                   int64_t n, int op, float* __restrict__ part) {
    float acc = red_id(op);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        acc = red_op(op, acc, base[rv_off(v, i)]);
    acc = block_red(op, acc);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void reduce_final(const float* __restrict__ part, int n, int op, float* __restrict__ out) {
    float acc = red_id(op);
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc = red_op(op, acc, part[i]);
    acc = block_red(op, acc);
    if (threadIdx.x == 0) *out = acc;
}

// One block per output element: fold the strided run along `dim`.
__global__ void reduce_dim_kernel(const float* __restrict__ base, const __grid_constant__ RedView outer,
                                  int64_t count, int64_t len, int64_t stride, int op,
                                  float* __restrict__ out) {
    for (int64_t o = blockIdx.x; o < count; o += gridDim.x) {
        const int64_t start = rv_off(outer, o);
        float acc = red_id(op);
        for (int64_t j = threadIdx.x; j < len; j += blockDim.x)
            acc = red_op(op, acc, base[start + j * stride]);
        acc = block_red(op, acc);
        if (threadIdx.x == 0) out[o] = acc;
    }
}

RedView to_rv(const pt_view& v) {
    RedView r;
    r.ndim = v.ndim;
    for (int d = 0; d < 8; ++d) {
        r.sizes[d] = d < v.ndim ? v.sizes[d] : 1;
        r.strides[d] = d < v.ndim ? v.strides[d] : 0;
    }
    r.offset = v.offset;
    return r;
}

}  // namespace

void fill_uniform(float* dst, int64_t n, uint64_t seed, float lo, float hi, cudaStream_t st) {
    if (n <= 0) return;
    fill_uniform_kernel<<<grid_for(n), 256, 0, st>>>(dst, n, seed, lo, hi - lo);
    after_launch("fill_uniform");
}

void apply_launch(const int32_t* code, int32_t ncode, int arity, float* const* bases,
                  const pt_view* views, float scalar, cudaStream_t st) {
    PTB_REQUIRE(ncode >= 1 && ncode <= kMaxCode, "apply: program length out of range");
    const int64_t n = numel(views[0]);
    bool contig = true;
    for (int t = 0; t < arity; ++t) contig = contig && contiguous(views[t]);
    if (contig) {
        const int fast = match_fast(code, ncode, arity);
        float* x = bases[0] + views[0].offset;
        const float* y = arity > 1 ? bases[1] + views[1].offset : nullptr;
        const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                             (!y || (reinterpret_cast<uintptr_t>(y) & 15) == 0);
        if (fast && aligned) {
            apply_fast_kernel<<<grid_for(n / 4 + 1), 256, 0, st>>>(x, y, n, scalar, fast);
            after_launch("apply_fast");
            return;
        }
    }
    ApplyArgs a;
    memset(&a, 0, sizeof a);
    memcpy(a.code, code, sizeof(int32_t) * ncode);
    a.ncode = ncode;
    a.arity = arity;
    a.scalar = scalar;
    a.ndim = views[0].ndim;
    for (int d = 0; d < 8; ++d) a.sizes[d] = d < a.ndim ? views[0].sizes[d] : 1;
    for (int t = 0; t < arity; ++t) {
        for (int d = 0; d < a.ndim; ++d) a.strides[t][d] = views[t].strides[d];
        a.offset[t] = views[t].offset;
        a.base[t] = bases[t];
    }
    a.n = n;
    if (contig) {
        bool vec = true;
        for (int t = 0; t < arity; ++t)
            vec = vec && (reinterpret_cast<uintptr_t>(bases[t] + views[t].offset) & 15) == 0;
        apply_contig_kernel<<<grid_for(vec ? n / 4 + 1 : n), 256, 0, st>>>(a, vec ? 1 : 0);
    }
    else apply_strided_kernel<<<grid_for(n), 256, 0, st>>>(a);
    after_launch("apply");
}

void bias_add_launch(float* y, const float* b, int64_t N, int64_t K, int64_t HW, cudaStream_t st) {
    const int64_t rows = N * K;
    if (rows == 0 || HW == 0) return;
    const int blocks = (int)std::min<int64_t>(rows, 16 * (int64_t)sm_count());
    bias_add_kernel<<<blocks, 256, 0, st>>>(y, b, K, HW, rows);
    after_launch("bias_add");
}

void reduce_all_launch(int op, const float* base, const pt_view& v, float* out, cudaStream_t st) {
    const int64_t n = numel(v);
    constexpr int kParts = 1024;
    // stream-ordered scratch: safe for concurrent calls on distinct streams
    float* part = nullptr;
    PTB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&part), kParts * sizeof(float), st));
    const int blocks = (int)std::min<int64_t>(kParts, std::max<int64_t>(1, ceil_div(n, 1024)));
    reduce_all_partial<<<blocks, 256, 0, st>>>(base, to_rv(v), n, op, part);
    after_launch("reduce_all_partial");
    reduce_final<<<1, 1024, 0, st>>>(part, blocks, op, out);
    after_launch("reduce_all_final");
    PTB_CUDA(cudaFreeAsync(part, st));
}

void reduce_dim_launch(int op, const float* base, const pt_view& v, int dim, float* out,
                       cudaStream_t st) {
    pt_view outer = v;
    outer.sizes[dim] = 1;
    const int64_t count = numel(outer);
    const int blocks = (int)std::min<int64_t>(count, 32 * (int64_t)sm_count());
    reduce_dim_kernel<<<std::max(blocks, 1), 128, 0, st>>>(base, to_rv(outer), count, v.sizes[dim],
                                                           v.strides[dim], op, out);
    after_launch("reduce_dim");
}

}  // namespace ptb
