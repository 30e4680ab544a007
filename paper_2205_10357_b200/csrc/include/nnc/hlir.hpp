// nnc/hlir.hpp -- graph IR of the B200 backend.
//
// Mirrors the reference IR so reference callers port unchanged:
//   Dim/Shape/TensorType      reference core/include/nnc/hlir.hpp:24-76
//   OpKind                    reference core/include/nnc/hlir.hpp:79-103
//   Attrs/Node/Graph          reference core/include/nnc/hlir.hpp:110-180
//   GraphBuilder              reference core/include/nnc/hlir.hpp:196-219
// Extension (not in the reference, parity unpinned -> oracle/nnc_oracle.c):
//   BatchNorm (+ two grad kernels), Gelu (+grad), LayerNorm (+ two grad kernels).
// Shapes in this backend are fully bound at optimize time (the batch symbol is
// pinned to its seed); symbolic dims are parsed and collapsed by passes::optimize.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "nnc/error.hpp"
#include "nnc/tensor.hpp"

namespace nnc::hlir {

class Dim {
public:
    static Dim fixed(int64_t extent) { Dim d; d.extent_ = extent; return d; }
    static Dim sym(int32_t id, int64_t seed) { Dim d; d.extent_ = seed; d.sym_id_ = id; return d; }
    bool is_sym() const { return sym_id_ >= 0; }
    int32_t sym_id() const { return sym_id_; }
    int64_t seed_extent() const { return extent_; }
    friend bool operator==(const Dim& a, const Dim& b) {
        if (a.is_sym() != b.is_sym()) return false;
        return a.is_sym() ? a.sym_id_ == b.sym_id_ : a.extent_ == b.extent_;
    }
private:
    int64_t extent_ = 1;
    int32_t sym_id_ = -1;
};

/// Layout tag of the reference's Shape::fixed (hlir.hpp:46); this backend's
/// tensors are NHWC / flat by construction, so the tag is accepted and ignored.
enum class Layout : uint8_t { NHWC = 0, FLAT = 1, SCALAR = 2, RAW = 3 };

struct Shape {
    std::vector<Dim> dims;
    size_t rank() const { return dims.size(); }
    std::vector<int64_t> seed_dims() const {
        std::vector<int64_t> o;
        for (const Dim& d : dims) o.push_back(d.seed_extent());
        return o;
    }
    int64_t seed_elements() const { return element_count(seed_dims()); }
    static Shape fixed(const std::vector<int64_t>& e, Layout = Layout::RAW) {
        Shape s;
        for (int64_t x : e) s.dims.push_back(Dim::fixed(x));
        return s;
    }
    friend bool operator==(const Shape& a, const Shape& b) { return a.dims == b.dims; }
};

struct TensorType {
    Shape shape;
    DType dtype = DType::F32;
};

enum class OpKind : uint8_t {
    Input, Const, Conv2D, MaxPool2D, AdaptiveAvgPool2D, Dense, ReLU, Flatten, Add, Mul, CumSum,
    Identity,
    DenseGradInput, DenseGradWeight, SumCols, Conv2DGradInput, Conv2DGradWeight, SumNHW, ReluGrad,
    MaxPool2DGrad, AdaptiveAvgPool2DGrad, Unflatten,
    // ---- extensions (B200 backend; CPU restatement in oracle/nnc_oracle.c) ----
    BatchNorm,            // training: batch statistics over all axes but the last
    BatchNormGradInput,   // (x, stats, g; gamma) -> dx
    BatchNormGradGamma,   // (x, stats, g) -> dgamma
    Gelu,                 // exact (erf) GELU
    GeluGrad,             // (x, g) -> dx
    LayerNorm,            // over the last axis
    LayerNormGradInput,   // (x, g; gamma) -> dx
    LayerNormGradGamma,   // (x, g) -> dgamma
};

const char* op_name(OpKind op);

enum class Padding : uint8_t { Same = 0, Valid = 1 };

struct Attrs {
    int64_t out_channels = 0;
    std::array<int64_t, 2> kernel{0, 0};
    std::array<int64_t, 2> stride{1, 1};
    Padding padding = Padding::Valid;
    bool has_bias = false;
    std::array<int64_t, 2> out_hw{0, 0};
    int64_t out_features = 0;
    int64_t axis = 0;
    bool exclusive = false;
    bool reverse = false;
    std::vector<int64_t> fwd_dims;
    double eps = 1e-3;     // BatchNorm / LayerNorm
    bool inference = false;  // BatchNorm: use moving statistics (inference version)
    bool batch_stats = false;  // BatchNorm: batch statistics in every version (DLB "training": true)
};

struct Node {
    std::string name;
    OpKind op = OpKind::Identity;
    Attrs attrs;
    std::vector<std::string> inputs;
    std::vector<std::string> outputs;
    std::vector<std::string> weights;
};

struct GraphInput {
    std::string name;
    TensorType type;
};

struct Graph {
    DType dtype = DType::F32;
    std::vector<Node> nodes;
    std::vector<GraphInput> inputs;
    std::vector<std::string> outputs;
    std::map<std::string, Tensor> initializers;
    std::map<std::string, TensorType> value_types;
    int32_t next_sym_id = 0;

    const Node* find_node(const std::string& name) const;
    int producer_of(const std::string& value) const;
    bool is_graph_input(const std::string& value) const;
    const TensorType* type_of(const std::string& value) const;
};

/// Deterministic topological order (ties by insertion index), as the
/// reference's topo_order (hlir.cpp:298-326).
std::vector<std::string> topo_order(const Graph& g);

class GraphBuilder {
public:
    explicit GraphBuilder(DType dt = DType::F32) { g_.dtype = dt; }
    GraphBuilder& input(const std::string& name, TensorType type, bool materialize_node = false);
    GraphBuilder& initializer(const std::string& name, Tensor value);
    GraphBuilder& node(const std::string& name, OpKind op, std::vector<std::string> inputs,
                       Attrs attrs = {}, std::vector<std::string> weights = {});
    GraphBuilder& output(const std::string& value);
    Graph build() const { return g_; }
    Graph& graph() { return g_; }
private:
    Graph g_;
};

}  // namespace nnc::hlir
