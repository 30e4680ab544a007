// ingest.cpp -- DLB model documents -> canonical NHWC graph.
// Follows reference ingest.cpp:43-70 (initializer stream), :143-300 (conv/dense
// lowering), :301-409 (node ops), :411-500 (document) for the DLB dialect.
#include "nnc/ingest.hpp"

#include <cmath>
#include <optional>

#include <json.hpp>

#include "nnc/geometry.hpp"

namespace nnc::ingest {

using hlir::Attrs;
using hlir::Dim;
using hlir::OpKind;
using hlir::Padding;
using json = nlohmann::json;

uint64_t fnv1a64(const std::string& text) {
    uint64_t h = 14695981039346656037ull;
    for (unsigned char c : text) {
        h ^= c;
        h *= 1099511628211ull;
    }
    return h;
}

InitStream::InitStream(uint64_t seed, const std::string& name) : state_(seed ^ fnv1a64(name)) {
    state_ = state_ * 6364136223846793005ull + 1442695040888963407ull;
}

double InitStream::uniform(double lo, double hi) {
    state_ = state_ * 6364136223846793005ull + 1442695040888963407ull;
    double u = static_cast<double>(state_ >> 11) * 0x1.0p-53;
    return lo + u * (hi - lo);
}

namespace {

[[noreturn]] void bad(const std::string& m) { throw Error(Error::Code::BadDocument, m); }

Tensor random_init(DType dt, const std::vector<int64_t>& dims, int64_t fan_in, uint64_t seed,
                   const std::string& name) {
    Tensor t(dt, dims);
    InitStream rng(seed, name);
    double bound = 1.0 / std::sqrt(static_cast<double>(fan_in));
    for (int64_t i = 0; i < t.elements(); ++i) {
        double v = rng.uniform(-bound, bound);
        if (dt == DType::F32)
            t.set(i, static_cast<double>(static_cast<float>(v)));
        else
            t.set(i, v);
    }
    return t;
}

Tensor filled(DType dt, const std::vector<int64_t>& dims, double v) {
    Tensor t(dt, dims);
    for (int64_t i = 0; i < t.elements(); ++i) t.set(i, v);
    return t;
}

std::array<int64_t, 2> pair_attr(const json& a, const char* key, bool required,
                                 std::array<int64_t, 2> fb = {0, 0}) {
    if (!a.contains(key)) {
        if (required) bad(std::string("missing attribute ") + key);
        return fb;
    }
    const json& v = a.at(key);
    if (v.is_number_integer()) return {v.get<int64_t>(), v.get<int64_t>()};
    if (v.is_array() && v.size() == 2) return {v[0].get<int64_t>(), v[1].get<int64_t>()};
    bad(std::string(key) + " must be an integer or a pair");
}

struct Converter {
    DType dtype;
    uint64_t seed;
    const std::map<std::string, Tensor>* store;
    hlir::GraphBuilder b;
    std::map<std::string, std::vector<int64_t>> dims;

    Converter(DType dt, uint64_t s, const std::map<std::string, Tensor>* w)
        : dtype(dt), seed(s), store(w), b(dt) {}

    const std::vector<int64_t>& in_dims(const std::string& node, const std::string& v) {
        auto it = dims.find(v);
        if (it == dims.end()) bad(node + ": unknown input " + v);
        return it->second;
    }

    Tensor weight(const std::string& name, const std::vector<int64_t>& shape, int64_t fan_in,
                  std::optional<double> fill = std::nullopt) {
        if (store) {
            auto it = store->find(name);
            if (it != store->end()) {
                if (it->second.dims() != shape)
                    throw Error(Error::Code::ShapeMismatch, name + ": expected " +
                                                                dims_to_string(shape));
                Tensor t(dtype, shape);
                for (int64_t i = 0; i < t.elements(); ++i) t.set(i, it->second.get(i));
                return t;
            }
        }
        if (fill) return filled(dtype, shape, *fill);
        return random_init(dtype, shape, fan_in, seed, name);
    }

    void add_node(const json& jn) {
        std::string name = jn.at("name").get<std::string>();
        std::string op = jn.at("op").get<std::string>();
        std::vector<std::string> ins = jn.value("inputs", std::vector<std::string>{});
        json at = jn.value("attrs", json::object());
        if (dims.count(name)) bad("duplicate node name " + name);
        auto one = [&]() -> const std::string& {
            if (ins.size() != 1) bad(name + ": " + op + " takes exactly one input");
            return ins[0];
        };
        if (op == "conv2d") {
            const auto& xd = in_dims(name, one());
            if (xd.size() != 4) bad(name + ": conv2d input must be rank 4");
            Attrs a;
            a.out_channels = at.at("filters").get<int64_t>();
            a.kernel = pair_attr(at, "kernel_size", true);
            a.stride = pair_attr(at, "strides", false, {1, 1});
            std::string pad = at.value("padding", "valid");
            if (pad != "same" && pad != "valid") bad("padding must be \"same\" or \"valid\"");
            a.padding = pad == "same" ? Padding::Same : Padding::Valid;
            a.has_bias = at.value("use_bias", true);
            int64_t ci = xd[3];
            int64_t fan_in = a.kernel[0] * a.kernel[1] * ci;
            b.initializer(name + ".weight",
                          weight(name + ".weight", {a.kernel[0], a.kernel[1], ci, a.out_channels}, fan_in));
            std::vector<std::string> w{name + ".weight"};
            if (a.has_bias) {
                b.initializer(name + ".bias", weight(name + ".bias", {a.out_channels}, fan_in));
                w.push_back(name + ".bias");
            }
            b.node(name, OpKind::Conv2D, {ins[0]}, a, w);
            nncb_gemm_desc d{};
            geom::conv_geometry(d, xd, a);
            dims[name] = {d.n, d.oh, d.ow, d.co};
        } else if (op == "max_pooling2d") {
            const auto& xd = in_dims(name, one());
            if (xd.size() != 4) bad(name + ": pooling input must be rank 4");
            Attrs a;
            a.kernel = pair_attr(at, "pool_size", true);
            a.stride = pair_attr(at, "strides", false, a.kernel);
            b.node(name, OpKind::MaxPool2D, {ins[0]}, a);
            auto g = geom::pool_geometry(xd, a);
            dims[name] = {g.n, g.oh, g.ow, g.c};
        } else if (op == "global_avg_pool2d") {
            const auto& xd = in_dims(name, one());
            if (xd.size() != 4) bad(name + ": pooling input must be rank 4");
            Attrs a;
            a.out_hw = {1, 1};
            b.node(name, OpKind::AdaptiveAvgPool2D, {ins[0]}, a);
            dims[name] = {xd[0], 1, 1, xd[3]};
        } else if (op == "dense") {
            const auto& xd = in_dims(name, one());
            if (xd.size() != 2) bad(name + ": dense input must be rank 2");
            Attrs a;
            a.out_features = at.at("units").get<int64_t>();
            a.has_bias = at.value("use_bias", true);
            b.initializer(name + ".weight", weight(name + ".weight", {xd[1], a.out_features}, xd[1]));
            std::vector<std::string> w{name + ".weight"};
            if (a.has_bias) {
                b.initializer(name + ".bias", weight(name + ".bias", {a.out_features}, xd[1]));
                w.push_back(name + ".bias");
            }
            b.node(name, OpKind::Dense, {ins[0]}, a, w);
            dims[name] = {xd[0], a.out_features};
        } else if (op == "relu" || op == "identity" || op == "flatten" || op == "gelu") {
            const auto xd = in_dims(name, one());
            OpKind k = op == "relu" ? OpKind::ReLU
                       : op == "identity" ? OpKind::Identity
                       : op == "gelu" ? OpKind::Gelu : OpKind::Flatten;
            b.node(name, k, {ins[0]});
            if (k == OpKind::Flatten) {
                if (xd.size() < 2) bad(name + ": flatten input must be rank >= 2");
                int64_t rest = 1;
                for (size_t i = 1; i < xd.size(); ++i) rest *= xd[i];
                dims[name] = {xd[0], rest};
            } else {
                dims[name] = xd;
            }
        } else if (op == "add" || op == "mul") {
            if (ins.size() != 2) bad(name + ": " + op + " takes exactly two inputs");
            if (in_dims(name, ins[0]) != in_dims(name, ins[1])) bad(name + ": operand shapes differ");
            b.node(name, op == "add" ? OpKind::Add : OpKind::Mul, ins);
            dims[name] = in_dims(name, ins[0]);
        } else if (op == "cumsum") {
            const auto xd = in_dims(name, one());
            int64_t rank = static_cast<int64_t>(xd.size());
            Attrs a;
            int64_t axis = at.at("axis").get<int64_t>();
            if (axis < 0) axis += rank;
            if (axis < 0 || axis >= rank) bad(name + ": cumsum axis out of range");
            a.axis = axis;
            a.exclusive = at.value("exclusive", false);
            a.reverse = at.value("reverse", false);
            b.node(name, OpKind::CumSum, {ins[0]}, a);
            dims[name] = xd;
        } else if (op == "batch_normalization" || op == "layer_normalization") {
            const auto xd = in_dims(name, one());
            int64_t c = xd.back();
            Attrs a;
            a.eps = at.value("epsilon", 1e-3);
            bool bn = op == "batch_normalization";
            a.batch_stats = bn && at.value("training", false);
            std::vector<std::string> w{name + ".gamma", name + ".beta"};
            b.initializer(name + ".gamma", weight(name + ".gamma", {c}, c, 1.0));
            b.initializer(name + ".beta", weight(name + ".beta", {c}, c, 0.0));
            if (bn) {
                b.initializer(name + ".moving_mean", weight(name + ".moving_mean", {c}, c, 0.0));
                b.initializer(name + ".moving_variance", weight(name + ".moving_variance", {c}, c, 1.0));
                w.push_back(name + ".moving_mean");
                w.push_back(name + ".moving_variance");
            }
            b.node(name, bn ? OpKind::BatchNorm : OpKind::LayerNorm, {ins[0]}, a, w);
            dims[name] = xd;
        } else if (op == "const") {
            if (!ins.empty()) bad(name + ": const takes no inputs");
            std::vector<int64_t> d = at.at("shape").get<std::vector<int64_t>>();
            std::string wn = name + ".value";
            b.initializer(wn, weight(wn, d, std::max<int64_t>(element_count(d), 1)));
            b.node(name, OpKind::Const, {}, {}, {wn});
            dims[name] = d;
        } else {
            throw Error(Error::Code::UnknownOp, name + ": unknown op \"" + op + "\" in dialect dlb");
        }
    }
};

}  // namespace

Model parse_model(const std::string& document, const std::map<std::string, Tensor>* weights) {
    json j;
    try {
        j = json::parse(document);
    } catch (const json::exception& e) {
        bad(std::string("invalid JSON: ") + e.what());
    }
    if (!j.contains("dialect")) bad("missing dialect tag");
    if (j.at("dialect").get<std::string>() != "dlb")
        bad("this backend ingests the dlb dialect (got \"" + j.at("dialect").get<std::string>() + "\")");
    if (!j.contains("inputs") || j.at("inputs").empty()) bad("model declares no inputs");
    DType dtype = DType::F32;
    std::string dt = j.at("inputs")[0].value("dtype", "f32");
    if (dt == "f64")
        dtype = DType::F64;
    else if (dt != "f32")
        bad("dtype must be f32 or f64");
    if (dtype != DType::F32)
        throw Error(Error::Code::BadDocument, "the B200 backend executes f32 graphs");

    Model m;
    m.seed = j.value("seed", 0ull);
    m.name = j.value("name", "model");
    Converter cv(dtype, m.seed, weights);
    int32_t next_sym = 0;
    for (const json& ji : j.at("inputs")) {
        std::string in_name = ji.at("name").get<std::string>();
        std::vector<int64_t> seed;
        if (ji.contains("seed_shape")) seed = ji.at("seed_shape").get<std::vector<int64_t>>();
        hlir::Shape s;
        std::vector<int64_t> sd;
        const json& shape = ji.at("shape");
        for (size_t i = 0; i < shape.size(); ++i) {
            if (shape[i].is_null()) {
                if (i >= seed.size())
                    throw Error(Error::Code::MissingSeed,
                                in_name + ": axis " + std::to_string(i) + " is dynamic but seed_shape is missing");
                s.dims.push_back(Dim::sym(next_sym++, seed[i]));
                sd.push_back(seed[i]);
            } else {
                s.dims.push_back(Dim::fixed(shape[i].get<int64_t>()));
                sd.push_back(shape[i].get<int64_t>());
            }
        }
        cv.b.input(in_name, hlir::TensorType{s, dtype}, true);
        cv.dims[in_name] = sd;
    }
    cv.b.graph().next_sym_id = next_sym;
    for (const json& jn : j.value("nodes", json::array())) cv.add_node(jn);
    if (!j.contains("outputs") || j.at("outputs").empty()) bad("model declares no outputs");
    for (const json& jo : j.at("outputs")) cv.b.output(jo.get<std::string>());
    m.graph = cv.b.build();
    return m;
}

}  // namespace nnc::ingest
