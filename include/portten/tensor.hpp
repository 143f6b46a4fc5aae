// Tensor — strided float32 views with storageOffset, the reference's operand model
// (proj/include/portten/tensor.hpp:26-123): host Storage, narrow/select views sharing
// storage, copyFrom with overlap rejection, contiguous, fill, at.
//
// DeviceTensor is the B200 addition SURVEY.md §1 calls for: the same view model over a
// device allocation (libpt_b200), so conv stacks stay resident in HBM between layers.
#pragma once

#include <cstdint>
#include <initializer_list>
#include <memory>
#include <span>
#include <vector>

#include "../pt_b200.h"
#include "portten/errors.hpp"

namespace portten {

inline constexpr int kMaxDims = 8;

class Storage {
public:
    explicit Storage(std::int64_t length);
    std::int64_t length() const { return static_cast<std::int64_t>(elems_.size()); }
    float* data() { return elems_.data(); }
    const float* data() const { return elems_.data(); }

private:
    std::vector<float> elems_;
};

std::vector<std::int64_t> rowMajorStrides(const std::vector<std::int64_t>& sizes);

class Tensor {
public:
    Tensor() = default;
    static Tensor create(std::vector<std::int64_t> sizes);
    static Tensor create(std::initializer_list<std::int64_t> sizes);

    bool defined() const { return storage_ != nullptr; }
    const std::shared_ptr<Storage>& storage() const { return storage_; }
    std::int64_t storageOffset() const { return offset_; }
    int dim() const { return static_cast<int>(sizes_.size()); }
    const std::vector<std::int64_t>& sizes() const { return sizes_; }
    const std::vector<std::int64_t>& strides() const { return strides_; }
    std::int64_t size(int d) const;
    std::int64_t stride(int d) const;
    std::int64_t numel() const;
    bool isContiguous() const;

    Tensor narrow(int dim, std::int64_t start, std::int64_t length) const;
    Tensor select(int dim, std::int64_t index) const;
    void copyFrom(const Tensor& src);
    Tensor contiguous() const;
    void fill(float value);

    float* data();
    const float* data() const;
    float& at(std::span<const std::int64_t> index);
    float at(std::span<const std::int64_t> index) const;
    float& at(std::initializer_list<std::int64_t> index);
    float at(std::initializer_list<std::int64_t> index) const;
    float item() const;
    std::int64_t maxReachableIndex() const;

    /// C-ABI view descriptor (sizes / strides / offset) of this tensor.
    pt_view view() const;

private:
    std::shared_ptr<Storage> storage_;
    std::int64_t offset_ = 0;
    std::vector<std::int64_t> sizes_;
    std::vector<std::int64_t> strides_;
    std::int64_t indexOffset(std::span<const std::int64_t> index) const;
    void requireDefined() const;
};

/// Device-resident float32 tensor (contiguous allocation + view). Owns its buffer
/// through a shared handle, so views share it like Tensor views share Storage.
class DeviceTensor {
public:
    DeviceTensor() = default;
    static DeviceTensor empty(std::vector<std::int64_t> sizes);
    static DeviceTensor upload(const Tensor& host, void* stream = nullptr);
    Tensor download(void* stream = nullptr) const;

    bool defined() const { return buf_ != nullptr; }
    float* data() const;  // first logical element
    float* base() const { return static_cast<float*>(buf_.get()); }
    const std::vector<std::int64_t>& sizes() const { return sizes_; }
    const std::vector<std::int64_t>& strides() const { return strides_; }
    std::int64_t storageOffset() const { return offset_; }
    std::int64_t numel() const;
    bool isContiguous() const;
    int dim() const { return static_cast<int>(sizes_.size()); }
    DeviceTensor narrow(int dim, std::int64_t start, std::int64_t length) const;
    DeviceTensor select(int dim, std::int64_t index) const;
    pt_view view() const;

private:
    std::shared_ptr<void> buf_;
    std::int64_t capacity_ = 0;
    std::int64_t offset_ = 0;
    std::vector<std::int64_t> sizes_;
    std::vector<std::int64_t> strides_;
};

}  // namespace portten
