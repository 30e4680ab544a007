// nnc/tensor.hpp -- owned host tensor, the boundary I/O type.
// Mirrors reference core/include/nnc/tensor.hpp:10-62 (f32/f64, row-major).
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace nnc {

enum class DType : uint8_t { F32 = 0, F64 = 1 };
inline size_t dtype_size(DType dt) { return dt == DType::F32 ? 4 : 8; }

int64_t element_count(const std::vector<int64_t>& dims);
std::string dims_to_string(const std::vector<int64_t>& dims);

class Tensor {
public:
    Tensor() = default;
    Tensor(DType dt, std::vector<int64_t> dims);
    static Tensor from_f32(std::vector<int64_t> dims, std::vector<float> values);

    DType dtype() const { return dtype_; }
    const std::vector<int64_t>& dims() const { return dims_; }
    size_t rank() const { return dims_.size(); }
    int64_t elements() const { return element_count(dims_); }
    size_t byte_size() const { return data_.size(); }
    const uint8_t* data() const { return data_.data(); }
    uint8_t* data() { return data_.data(); }
    const float* f32() const { return reinterpret_cast<const float*>(data_.data()); }
    float* f32() { return reinterpret_cast<float*>(data_.data()); }
    double get(int64_t i) const;
    void set(int64_t i, double v);

private:
    DType dtype_ = DType::F32;
    std::vector<int64_t> dims_;
    std::vector<uint8_t> data_;
};

}  // namespace nnc
