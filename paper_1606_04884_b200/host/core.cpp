// core.cpp — errors, ConvGeometry, host Tensor views and DeviceTensor for the
// portten-b200 operator API (include/portten/*.hpp).
#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>

#include "portten/conv_geometry.hpp"
#include "portten/tensor.hpp"

namespace portten {

void throw_if_error(int status) {
    if (status == PT_OK) return;
    const std::string msg = pt_b200_last_error();
    if (status == PT_EVALIDATION) throw ValidationError(msg);
    throw BackendError(msg);
}

// ---------------------------------------------------------------- ConvGeometry
namespace conv {

void ConvGeometry::validate() const {
    PORTTEN_CHECK(batch >= 1 && inChannels >= 1 && inHeight >= 1 && inWidth >= 1 &&
                      outChannels >= 1 && kernelH >= 1 && kernelW >= 1 && strideH >= 1 &&
                      strideW >= 1,
                  "conv geometry: counts, dims, kernel and stride must be >= 1");
    PORTTEN_CHECK(padH >= 0 && padW >= 0, "conv geometry: padding must be >= 0");
    PORTTEN_CHECK(kernelH <= inHeight + 2 * padH && kernelW <= inWidth + 2 * padW,
                  "conv geometry: kernel exceeds padded input (" + toString() + ")");
    PORTTEN_CHECK(outHeight() >= 1 && outWidth() >= 1,
                  "conv geometry: empty output (" + toString() + ")");
}

std::string ConvGeometry::toString() const {
    auto s = [](std::int64_t v) { return std::to_string(v); };
    return "N" + s(batch) + " C" + s(inChannels) + " H" + s(inHeight) + " W" + s(inWidth) + " K" +
           s(outChannels) + " k" + s(kernelH) + "x" + s(kernelW) + " p" + s(padH) + "x" + s(padW) +
           " s" + s(strideH) + "x" + s(strideW);
}

}  // namespace conv

// ---------------------------------------------------------------- Storage / Tensor
Storage::Storage(std::int64_t length) : elems_(static_cast<std::size_t>(length), 0.0f) {
    PORTTEN_CHECK(length >= 0, "storage length must be >= 0");
}

std::vector<std::int64_t> rowMajorStrides(const std::vector<std::int64_t>& sizes) {
    std::vector<std::int64_t> st(sizes.size(), 1);
    for (int d = static_cast<int>(sizes.size()) - 2; d >= 0; --d) st[d] = st[d + 1] * sizes[d + 1];
    return st;
}

namespace {
std::string shape_str(const std::vector<std::int64_t>& s) {
    std::string r = "[";
    for (std::size_t i = 0; i < s.size(); ++i) r += (i ? "," : "") + std::to_string(s[i]);
    return r + "]";
}

void check_sizes(const std::vector<std::int64_t>& sizes) {
    PORTTEN_CHECK(!sizes.empty() && sizes.size() <= static_cast<std::size_t>(kMaxDims),
                  "tensor rank must be 1.." + std::to_string(kMaxDims));
    for (auto s : sizes) PORTTEN_CHECK(s >= 1, "tensor sizes must be >= 1, got " + shape_str(sizes));
}

std::int64_t prod(const std::vector<std::int64_t>& s) {
    return std::accumulate(s.begin(), s.end(), std::int64_t{1}, std::multiplies<>());
}
}  // namespace

Tensor Tensor::create(std::vector<std::int64_t> sizes) {
    check_sizes(sizes);
    Tensor t;
    t.storage_ = std::make_shared<Storage>(prod(sizes));
    t.strides_ = rowMajorStrides(sizes);
    t.sizes_ = std::move(sizes);
    return t;
}

Tensor Tensor::create(std::initializer_list<std::int64_t> sizes) {
    return create(std::vector<std::int64_t>(sizes));
}

void Tensor::requireDefined() const { PORTTEN_CHECK(defined(), "operation on an undefined tensor"); }

std::int64_t Tensor::size(int d) const {
    PORTTEN_CHECK(d >= 0 && d < dim(), "dimension out of range");
    return sizes_[d];
}
std::int64_t Tensor::stride(int d) const {
    PORTTEN_CHECK(d >= 0 && d < dim(), "dimension out of range");
    return strides_[d];
}
std::int64_t Tensor::numel() const { return defined() ? prod(sizes_) : 0; }
bool Tensor::isContiguous() const { return strides_ == rowMajorStrides(sizes_); }

Tensor Tensor::narrow(int d, std::int64_t start, std::int64_t length) const {
    requireDefined();
    PORTTEN_CHECK(d >= 0 && d < dim(), "narrow: dimension out of range");
    PORTTEN_CHECK(start >= 0 && length >= 1 && start + length <= sizes_[d],
                  "narrow: range out of bounds");
    Tensor v = *this;
    v.offset_ += start * strides_[d];
    v.sizes_[d] = length;
    return v;
}

Tensor Tensor::select(int d, std::int64_t index) const {
    requireDefined();
    PORTTEN_CHECK(dim() >= 2, "select needs rank >= 2");
    PORTTEN_CHECK(d >= 0 && d < dim() && index >= 0 && index < sizes_[d], "select: out of range");
    Tensor v = *this;
    v.offset_ += index * strides_[d];
    v.sizes_.erase(v.sizes_.begin() + d);
    v.strides_.erase(v.strides_.begin() + d);
    return v;
}

std::int64_t Tensor::maxReachableIndex() const {
    std::int64_t m = offset_;
    for (int d = 0; d < dim(); ++d) m += (sizes_[d] - 1) * strides_[d];
    return m;
}

namespace {
// visit every logical element (row-major order) with its storage offset
template <class F>
void for_each_offset(const std::vector<std::int64_t>& sizes, const std::vector<std::int64_t>& strides,
                     std::int64_t offset, F&& f) {
    const int r = static_cast<int>(sizes.size());
    std::vector<std::int64_t> idx(r, 0);
    const std::int64_t n = prod(sizes);
    std::int64_t off = offset;
    for (std::int64_t i = 0; i < n; ++i) {
        f(i, off);
        for (int d = r - 1; d >= 0; --d) {
            off += strides[d];
            if (++idx[d] < sizes[d]) break;
            off -= sizes[d] * strides[d];
            idx[d] = 0;
        }
    }
}
}  // namespace

void Tensor::copyFrom(const Tensor& src) {
    requireDefined();
    src.requireDefined();
    PORTTEN_CHECK(src.sizes_ == sizes_, "copy: size mismatch, dst " + shape_str(sizes_) +
                                            " vs src " + shape_str(src.sizes_));
    if (src.storage_ == storage_) {  // same rule as proj/src/tensor.cpp:153-160
        const bool disjoint = src.maxReachableIndex() < offset_ || maxReachableIndex() < src.offset_;
        PORTTEN_CHECK(disjoint, "copy between overlapping views of the same storage is not supported");
    }
    std::vector<float> tmp(static_cast<std::size_t>(numel()));
    const float* s = src.storage_->data();
    for_each_offset(src.sizes_, src.strides_, src.offset_, [&](std::int64_t i, std::int64_t o) { tmp[i] = s[o]; });
    float* d = storage_->data();
    for_each_offset(sizes_, strides_, offset_, [&](std::int64_t i, std::int64_t o) { d[o] = tmp[i]; });
}

Tensor Tensor::contiguous() const {
    requireDefined();
    if (isContiguous()) return *this;
    Tensor t = create(sizes_);
    t.copyFrom(*this);
    return t;
}

void Tensor::fill(float value) {
    requireDefined();
    float* d = storage_->data();
    for_each_offset(sizes_, strides_, offset_, [&](std::int64_t, std::int64_t o) { d[o] = value; });
}

float* Tensor::data() {
    requireDefined();
    return storage_->data() + offset_;
}
const float* Tensor::data() const {
    requireDefined();
    return storage_->data() + offset_;
}

std::int64_t Tensor::indexOffset(std::span<const std::int64_t> index) const {
    requireDefined();
    PORTTEN_CHECK(static_cast<int>(index.size()) == dim(), "at: index rank mismatch");
    std::int64_t o = offset_;
    for (int d = 0; d < dim(); ++d) {
        PORTTEN_CHECK(index[d] >= 0 && index[d] < sizes_[d], "at: index out of range");
        o += index[d] * strides_[d];
    }
    return o;
}
float& Tensor::at(std::span<const std::int64_t> i) { return storage_->data()[indexOffset(i)]; }
float Tensor::at(std::span<const std::int64_t> i) const { return storage_->data()[indexOffset(i)]; }
float& Tensor::at(std::initializer_list<std::int64_t> i) {
    return at(std::span<const std::int64_t>(i.begin(), i.size()));
}
float Tensor::at(std::initializer_list<std::int64_t> i) const {
    return at(std::span<const std::int64_t>(i.begin(), i.size()));
}
float Tensor::item() const {
    PORTTEN_CHECK(numel() == 1, "item() needs a single-element tensor");
    return storage_->data()[offset_];
}

pt_view Tensor::view() const {
    pt_view v{};
    v.ndim = dim();
    for (int d = 0; d < dim(); ++d) {
        v.sizes[d] = sizes_[d];
        v.strides[d] = strides_[d];
    }
    v.offset = offset_;
    return v;
}

// ---------------------------------------------------------------- DeviceTensor
DeviceTensor DeviceTensor::empty(std::vector<std::int64_t> sizes) {
    check_sizes(sizes);
    DeviceTensor t;
    t.capacity_ = prod(sizes);
    void* p = nullptr;
    throw_if_error(pt_b200_malloc(&p, static_cast<size_t>(t.capacity_) * sizeof(float)));
    t.buf_ = std::shared_ptr<void>(p, [](void* q) { pt_b200_free(q); });
    t.strides_ = rowMajorStrides(sizes);
    t.sizes_ = std::move(sizes);
    return t;
}

DeviceTensor DeviceTensor::upload(const Tensor& host, void* stream) {
    const Tensor c = host.contiguous();
    DeviceTensor t = empty(c.sizes());
    throw_if_error(pt_b200_memcpy_h2d(t.base(), c.data(), sizeof(float) * c.numel(), stream));
    throw_if_error(pt_b200_stream_sync(stream));
    return t;
}

Tensor DeviceTensor::download(void* stream) const {
    PORTTEN_CHECK(defined(), "download of an undefined device tensor");
    PORTTEN_CHECK(isContiguous(), "download expects a contiguous device tensor");
    Tensor h = Tensor::create(sizes_);
    throw_if_error(pt_b200_memcpy_d2h(h.data(), data(), sizeof(float) * numel(), stream));
    throw_if_error(pt_b200_stream_sync(stream));
    return h;
}

float* DeviceTensor::data() const { return base() + offset_; }
std::int64_t DeviceTensor::numel() const { return defined() ? prod(sizes_) : 0; }
bool DeviceTensor::isContiguous() const { return strides_ == rowMajorStrides(sizes_); }

DeviceTensor DeviceTensor::narrow(int d, std::int64_t start, std::int64_t length) const {
    PORTTEN_CHECK(defined() && d >= 0 && d < dim() && start >= 0 && length >= 1 &&
                      start + length <= sizes_[d],
                  "narrow: range out of bounds");
    DeviceTensor v = *this;
    v.offset_ += start * strides_[d];
    v.sizes_[d] = length;
    return v;
}

DeviceTensor DeviceTensor::select(int d, std::int64_t index) const {
    PORTTEN_CHECK(defined() && dim() >= 2 && d >= 0 && d < dim() && index >= 0 && index < sizes_[d],
                  "select: out of range");
    DeviceTensor v = *this;
    v.offset_ += index * strides_[d];
    v.sizes_.erase(v.sizes_.begin() + d);
    v.strides_.erase(v.strides_.begin() + d);
    return v;
}

pt_view DeviceTensor::view() const {
    pt_view v{};
    v.ndim = dim();
    for (int d = 0; d < dim(); ++d) {
        v.sizes[d] = sizes_[d];
        v.strides[d] = strides_[d];
    }
    v.offset = offset_;
    return v;
}

}  // namespace portten
