// nnc/tensor.hpp -- owned host tensor, the boundary I/O type.
// Mirrors reference core/include/nnc/tensor.hpp:10-62 (f32/f64, row-major).
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <utility>
#include <string>
#include <vector>

namespace nnc {

// Byte storage whose resize() leaves new bytes uninitialised (value-init is
// skipped), so buffers that are about to be overwritten by a copy are not
// zero-filled first; assign(n, 0) still zero-fills explicitly.
template <typename T>
struct DefaultInitAllocator : std::allocator<T> {
    template <typename U>
    struct rebind { using other = DefaultInitAllocator<U>; };
    DefaultInitAllocator() = default;
    template <typename U>
    DefaultInitAllocator(const DefaultInitAllocator<U>&) noexcept {}
    template <typename U>
    void construct(U* p) noexcept { ::new (static_cast<void*>(p)) U; }
    template <typename U, typename... Args>
    void construct(U* p, Args&&... args) { ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...); }
};

enum class DType : uint8_t { F32 = 0, F64 = 1 };
inline size_t dtype_size(DType dt) { return dt == DType::F32 ? 4 : 8; }

int64_t element_count(const std::vector<int64_t>& dims);
std::string dims_to_string(const std::vector<int64_t>& dims);

class Tensor {
public:
    Tensor() = default;
    Tensor(DType dt, std::vector<int64_t> dims);   // zero-filled (as the reference's)
    static Tensor from_f32(std::vector<int64_t> dims, std::vector<float> values);
    static Tensor from_f64(std::vector<int64_t> dims, std::vector<double> values);
    bool bitwise_equal(const Tensor& other) const;
    // storage left uninitialised: only for tensors fully overwritten right away
    static Tensor uninitialized(DType dt, std::vector<int64_t> dims);

    DType dtype() const { return dtype_; }
    const std::vector<int64_t>& dims() const { return dims_; }
    size_t rank() const { return dims_.size(); }
    int64_t elements() const { return element_count(dims_); }
    // read-only view of caller memory (not owned; must outlive every use).
    // Writing through a view first copies it into owned storage.
    static Tensor view(DType dt, std::vector<int64_t> dims, const void* data);
    bool is_view() const { return view_ != nullptr; }

    size_t byte_size() const { return view_ ? view_bytes_ : data_.size(); }
    const uint8_t* data() const { return view_ ? view_ : data_.data(); }
    uint8_t* data() {
        if (view_) own();
        return data_.data();
    }
    const float* f32() const { return reinterpret_cast<const float*>(data()); }
    float* f32() { return reinterpret_cast<float*>(data()); }
    double get(int64_t i) const;
    void set(int64_t i, double v);

private:
    void own();
    DType dtype_ = DType::F32;
    std::vector<int64_t> dims_;
    std::vector<uint8_t, DefaultInitAllocator<uint8_t>> data_;
    const uint8_t* view_ = nullptr;
    size_t view_bytes_ = 0;
};

}  // namespace nnc
