// core.cpp -- Tensor and HLIR basics of the B200 host (reference tensor.cpp,
// hlir.cpp:150-361 restated for this backend's IR).
#include <cstring>
#include <set>
#include <sstream>
#include <unordered_map>

#include "nnc/hlir.hpp"
#include "nnc/tensor.hpp"

namespace nnc {

int64_t element_count(const std::vector<int64_t>& dims) {
    int64_t n = 1;
    for (int64_t d : dims) n *= d;
    return n;
}

std::string dims_to_string(const std::vector<int64_t>& dims) {
    std::ostringstream os;
    os << "[";
    for (size_t i = 0; i < dims.size(); ++i) os << (i ? ", " : "") << dims[i];
    os << "]";
    return os.str();
}

Tensor::Tensor(DType dt, std::vector<int64_t> dims) : dtype_(dt), dims_(std::move(dims)) {
    data_.assign(static_cast<size_t>(element_count(dims_)) * dtype_size(dt), 0);
}

Tensor Tensor::uninitialized(DType dt, std::vector<int64_t> dims) {
    Tensor t;
    t.dtype_ = dt;
    t.dims_ = std::move(dims);
    t.data_.resize(static_cast<size_t>(element_count(t.dims_)) * dtype_size(dt));
    return t;
}

Tensor Tensor::view(DType dt, std::vector<int64_t> dims, const void* data) {
    Tensor t;
    t.dtype_ = dt;
    t.dims_ = std::move(dims);
    t.view_ = static_cast<const uint8_t*>(data);
    t.view_bytes_ = static_cast<size_t>(element_count(t.dims_)) * dtype_size(dt);
    return t;
}

void Tensor::own() {
    data_.resize(view_bytes_);
    std::memcpy(data_.data(), view_, view_bytes_);
    view_ = nullptr;
    view_bytes_ = 0;
}

Tensor Tensor::from_f64(std::vector<int64_t> dims, std::vector<double> values) {
    Tensor t(DType::F64, std::move(dims));
    if (static_cast<int64_t>(values.size()) != t.elements())
        throw Error(Error::Code::ShapeMismatch, "from_f64: value count does not match the dims");
    std::memcpy(t.data(), values.data(), values.size() * sizeof(double));
    return t;
}

bool Tensor::bitwise_equal(const Tensor& o) const {
    return dtype_ == o.dtype_ && dims_ == o.dims_ && byte_size() == o.byte_size() &&
           std::memcmp(data(), o.data(), byte_size()) == 0;
}

Tensor Tensor::from_f32(std::vector<int64_t> dims, std::vector<float> values) {
    Tensor t(DType::F32, std::move(dims));
    std::memcpy(t.data(), values.data(), t.byte_size());
    return t;
}

double Tensor::get(int64_t i) const {
    if (dtype_ == DType::F32) return reinterpret_cast<const float*>(data())[i];
    return reinterpret_cast<const double*>(data())[i];
}

void Tensor::set(int64_t i, double v) {
    if (dtype_ == DType::F32)
        reinterpret_cast<float*>(data())[i] = static_cast<float>(v);
    else
        reinterpret_cast<double*>(data())[i] = v;
}

}  // namespace nnc

namespace nnc::hlir {

const char* op_name(OpKind op) {
    switch (op) {
        case OpKind::Input: return "Input";
        case OpKind::Const: return "Const";
        case OpKind::Conv2D: return "Conv2D";
        case OpKind::MaxPool2D: return "MaxPool2D";
        case OpKind::AdaptiveAvgPool2D: return "AdaptiveAvgPool2D";
        case OpKind::Dense: return "Dense";
        case OpKind::ReLU: return "ReLU";
        case OpKind::Flatten: return "Flatten";
        case OpKind::Add: return "Add";
        case OpKind::Mul: return "Mul";
        case OpKind::CumSum: return "CumSum";
        case OpKind::Identity: return "Identity";
        case OpKind::DenseGradInput: return "DenseGradInput";
        case OpKind::DenseGradWeight: return "DenseGradWeight";
        case OpKind::SumCols: return "SumCols";
        case OpKind::Conv2DGradInput: return "Conv2DGradInput";
        case OpKind::Conv2DGradWeight: return "Conv2DGradWeight";
        case OpKind::SumNHW: return "SumNHW";
        case OpKind::ReluGrad: return "ReluGrad";
        case OpKind::MaxPool2DGrad: return "MaxPool2DGrad";
        case OpKind::AdaptiveAvgPool2DGrad: return "AdaptiveAvgPool2DGrad";
        case OpKind::Unflatten: return "Unflatten";
        case OpKind::BatchNorm: return "BatchNorm";
        case OpKind::BatchNormGradInput: return "BatchNormGradInput";
        case OpKind::BatchNormGradGamma: return "BatchNormGradGamma";
        case OpKind::Gelu: return "Gelu";
        case OpKind::GeluGrad: return "GeluGrad";
        case OpKind::LayerNorm: return "LayerNorm";
        case OpKind::LayerNormGradInput: return "LayerNormGradInput";
        case OpKind::LayerNormGradGamma: return "LayerNormGradGamma";
    }
    return "?";
}

const Node* Graph::find_node(const std::string& name) const {
    for (const Node& n : nodes)
        if (n.name == name) return &n;
    return nullptr;
}

int Graph::producer_of(const std::string& value) const {
    for (size_t i = 0; i < nodes.size(); ++i)
        for (const std::string& o : nodes[i].outputs)
            if (o == value) return static_cast<int>(i);
    return -1;
}

bool Graph::is_graph_input(const std::string& value) const {
    for (const GraphInput& gi : inputs)
        if (gi.name == value) return true;
    return false;
}

const TensorType* Graph::type_of(const std::string& value) const {
    auto it = value_types.find(value);
    return it == value_types.end() ? nullptr : &it->second;
}

std::vector<std::string> topo_order(const Graph& g) {
    std::unordered_map<std::string, int> producers;
    for (size_t i = 0; i < g.nodes.size(); ++i)
        for (const std::string& out : g.nodes[i].outputs) producers[out] = static_cast<int>(i);
    std::vector<int> indeg(g.nodes.size(), 0);
    std::vector<std::vector<int>> succ(g.nodes.size());
    for (size_t i = 0; i < g.nodes.size(); ++i)
        for (const std::string& in : g.nodes[i].inputs) {
            auto it = producers.find(in);
            if (it != producers.end()) {
                succ[it->second].push_back(static_cast<int>(i));
                ++indeg[i];
            }
        }
    std::set<int> ready;
    for (size_t i = 0; i < indeg.size(); ++i)
        if (indeg[i] == 0) ready.insert(static_cast<int>(i));
    std::vector<std::string> order;
    while (!ready.empty()) {
        int v = *ready.begin();
        ready.erase(ready.begin());
        order.push_back(g.nodes[v].name);
        for (int s : succ[v])
            if (--indeg[s] == 0) ready.insert(s);
    }
    if (order.size() != g.nodes.size())
        throw Error(Error::Code::BadDocument, "topo_order: cycle detected");
    return order;
}

GraphBuilder& GraphBuilder::input(const std::string& name, TensorType type, bool materialize) {
    type.dtype = g_.dtype;
    g_.inputs.push_back({name, type});
    if (materialize) {
        Node n;
        n.name = name;
        n.op = OpKind::Input;
        n.outputs = {name};
        g_.nodes.push_back(std::move(n));
    }
    return *this;
}

GraphBuilder& GraphBuilder::initializer(const std::string& name, Tensor value) {
    g_.initializers.emplace(name, std::move(value));
    return *this;
}

GraphBuilder& GraphBuilder::node(const std::string& name, OpKind op, std::vector<std::string> inputs,
                                 Attrs attrs, std::vector<std::string> weights) {
    Node n;
    n.name = name;
    n.op = op;
    n.attrs = std::move(attrs);
    n.inputs = std::move(inputs);
    n.outputs = {name};
    n.weights = std::move(weights);
    g_.nodes.push_back(std::move(n));
    return *this;
}

GraphBuilder& GraphBuilder::output(const std::string& value) {
    g_.outputs.push_back(value);
    return *this;
}

}  // namespace nnc::hlir
