// passes.cpp -- shape inference, dead-layer elimination, canonicalization.
// Shape rules follow reference passes.cpp:209-391 (fixed-extent case); the
// extension ops keep their input shape (BatchNorm/Gelu/LayerNorm) or reduce to
// [C] (grad-gamma kernels). DCE follows passes.cpp:574-620, canonicalize
// passes.cpp:704-781.
#include "nnc/passes.hpp"

#include <algorithm>
#include <unordered_map>
#include <unordered_set>

#include "nnc/geometry.hpp"

namespace nnc::passes {

using hlir::Dim;
using hlir::Graph;
using hlir::Node;
using hlir::OpKind;
using hlir::Shape;
using hlir::TensorType;

namespace {
[[noreturn]] void rank_error(const Node& n, const std::string& m) {
    throw Error(Error::Code::RankError, n.name + ": " + m);
}
[[noreturn]] void extent_error(const Node& n, const std::string& m) {
    throw Error(Error::Code::ExtentMismatch, n.name + ": " + m);
}
}  // namespace

ShapeInfo infer_shapes(const Graph& input) {
    ShapeInfo info;
    info.graph = input;
    Graph& g = info.graph;
    g.value_types.clear();
    for (const auto& gi : g.inputs) g.value_types[gi.name] = gi.type;
    for (const auto& [name, t] : g.initializers)
        g.value_types[name] = TensorType{Shape::fixed(t.dims()), g.dtype};

    std::unordered_map<std::string, const Node*> by_name;
    for (const Node& n : g.nodes) by_name[n.name] = &n;
    for (const std::string& name : hlir::topo_order(g)) {
        const Node& n = *by_name.at(name);
        auto in = [&](size_t i) -> std::vector<int64_t> {
            if (i >= n.inputs.size()) rank_error(n, "missing input " + std::to_string(i));
            auto it = g.value_types.find(n.inputs[i]);
            if (it == g.value_types.end())
                throw Error(Error::Code::ShapeMismatch, n.name + ": untyped input " + n.inputs[i]);
            return it->second.shape.seed_dims();
        };
        auto need_rank = [&](size_t i, size_t r) {
            auto d = in(i);
            if (d.size() != r)
                rank_error(n, "input " + std::to_string(i) + " must be rank " + std::to_string(r) +
                                  ", got " + std::to_string(d.size()));
            return d;
        };
        auto w = [&](size_t i) -> const Tensor& {
            if (i >= n.weights.size())
                throw Error(Error::Code::ShapeMismatch, n.name + ": missing weight " + std::to_string(i));
            auto it = g.initializers.find(n.weights[i]);
            if (it == g.initializers.end())
                throw Error(Error::Code::ShapeMismatch, n.name + ": unknown initializer " + n.weights[i]);
            return it->second;
        };
        auto set_out = [&](size_t i, std::vector<int64_t> d) {
            g.value_types[n.outputs[i]] = TensorType{Shape::fixed(d), g.dtype};
        };
        const hlir::Attrs& a = n.attrs;
        switch (n.op) {
            case OpKind::Input: break;
            case OpKind::Const: set_out(0, w(0).dims()); break;
            case OpKind::Identity:
            case OpKind::ReLU:
            case OpKind::Gelu: set_out(0, in(0)); break;
            case OpKind::CumSum: {
                auto d = in(0);
                if (a.axis < 0 || a.axis >= static_cast<int64_t>(d.size())) rank_error(n, "cumsum axis out of range");
                set_out(0, d);
                break;
            }
            case OpKind::Add:
            case OpKind::Mul:
            case OpKind::ReluGrad:
            case OpKind::GeluGrad: {
                auto x = in(0), y = in(1);
                if (x.size() != y.size()) rank_error(n, "operand ranks differ");
                for (size_t i = 0; i < x.size(); ++i)
                    if (x[i] != y[i])
                        extent_error(n, "axis " + std::to_string(i) + ": " + std::to_string(x[i]) + " vs " +
                                            std::to_string(y[i]));
                set_out(0, x);
                break;
            }
            case OpKind::Flatten: {
                auto d = in(0);
                if (d.size() < 2) rank_error(n, "flatten requires rank >= 2");
                int64_t rest = 1;
                for (size_t i = 1; i < d.size(); ++i) rest *= d[i];
                set_out(0, {d[0], rest});
                break;
            }
            case OpKind::Unflatten: {
                auto d = need_rank(0, 2);
                std::vector<int64_t> o{d[0]};
                o.insert(o.end(), a.fwd_dims.begin(), a.fwd_dims.end());
                set_out(0, o);
                break;
            }
            case OpKind::Dense: {
                auto d = need_rank(0, 2);
                const Tensor& wt = w(0);
                if (wt.rank() != 2) throw Error(Error::Code::ShapeMismatch, n.name + ": dense weight must be rank 2");
                if (wt.dims()[1] != a.out_features)
                    throw Error(Error::Code::ShapeMismatch, n.name + ": weight out_features mismatch");
                if (d[1] != wt.dims()[0])
                    extent_error(n, "in_features: expected " + std::to_string(wt.dims()[0]) + ", got " +
                                        std::to_string(d[1]));
                if (a.has_bias && (w(1).rank() != 1 || w(1).dims()[0] != a.out_features))
                    throw Error(Error::Code::ShapeMismatch, n.name + ": bias shape mismatch");
                set_out(0, {d[0], a.out_features});
                break;
            }
            case OpKind::DenseGradInput: {
                auto d = need_rank(0, 2);
                if (d[1] != w(0).dims()[1]) extent_error(n, "grad out_features");
                set_out(0, {d[0], w(0).dims()[0]});
                break;
            }
            case OpKind::DenseGradWeight: {
                auto x = need_rank(0, 2), gr = need_rank(1, 2);
                if (x[0] != gr[0]) extent_error(n, "axis 0");
                set_out(0, {x[1], gr[1]});
                break;
            }
            case OpKind::SumCols: set_out(0, {need_rank(0, 2)[1]}); break;
            case OpKind::SumNHW: set_out(0, {need_rank(0, 4)[3]}); break;
            case OpKind::Conv2D: {
                auto d = need_rank(0, 4);
                const Tensor& k = w(0);
                if (k.rank() != 4) throw Error(Error::Code::ShapeMismatch, n.name + ": conv kernel must be rank 4");
                if (k.dims()[0] != a.kernel[0] || k.dims()[1] != a.kernel[1] || k.dims()[3] != a.out_channels)
                    throw Error(Error::Code::ShapeMismatch, n.name + ": kernel attrs mismatch");
                if (d[3] != k.dims()[2])
                    extent_error(n, "in_channels: expected " + std::to_string(k.dims()[2]) + ", got " +
                                        std::to_string(d[3]));
                if (a.has_bias && (w(1).rank() != 1 || w(1).dims()[0] != a.out_channels))
                    throw Error(Error::Code::ShapeMismatch, n.name + ": bias shape mismatch");
                nncb_gemm_desc gd{};
                geom::conv_geometry(gd, d, a);
                set_out(0, {gd.n, gd.oh, gd.ow, gd.co});
                break;
            }
            case OpKind::Conv2DGradInput: {
                auto d = need_rank(0, 4);
                if (a.fwd_dims.size() != 3) rank_error(n, "fwd_dims must be [ih,iw,ci]");
                set_out(0, {d[0], a.fwd_dims[0], a.fwd_dims[1], a.fwd_dims[2]});
                break;
            }
            case OpKind::Conv2DGradWeight: {
                auto x = need_rank(0, 4), gr = need_rank(1, 4);
                if (x[0] != gr[0]) extent_error(n, "axis 0");
                set_out(0, {a.kernel[0], a.kernel[1], x[3], a.out_channels});
                break;
            }
            case OpKind::MaxPool2D: {
                auto d = need_rank(0, 4);
                auto pg = geom::pool_geometry(d, a);
                set_out(0, {pg.n, pg.oh, pg.ow, pg.c});
                if (n.outputs.size() == 2) set_out(1, {pg.n, pg.oh, pg.ow, pg.c});
                break;
            }
            case OpKind::MaxPool2DGrad: {
                auto idx = need_rank(0, 4), gr = need_rank(1, 4);
                if (idx[0] != gr[0]) extent_error(n, "axis 0");
                if (a.fwd_dims.size() != 2) rank_error(n, "fwd_dims must be [ih,iw]");
                set_out(0, {gr[0], a.fwd_dims[0], a.fwd_dims[1], gr[3]});
                break;
            }
            case OpKind::AdaptiveAvgPool2D: {
                auto d = need_rank(0, 4);
                set_out(0, {d[0], a.out_hw[0], a.out_hw[1], d[3]});
                break;
            }
            case OpKind::AdaptiveAvgPool2DGrad: {
                auto d = need_rank(0, 4);
                if (a.fwd_dims.size() != 2) rank_error(n, "fwd_dims must be [ih,iw]");
                set_out(0, {d[0], a.fwd_dims[0], a.fwd_dims[1], d[3]});
                break;
            }
            case OpKind::BatchNorm:
            case OpKind::LayerNorm: {
                auto d = in(0);
                if (d.size() < 2) rank_error(n, "normalization input must be rank >= 2");
                if (w(0).elements() != d.back() || w(1).elements() != d.back())
                    throw Error(Error::Code::ShapeMismatch, n.name + ": gamma/beta must be [C]");
                set_out(0, d);
                if (n.outputs.size() == 2) set_out(1, {2, d.back()});
                break;
            }
            case OpKind::BatchNormGradInput: set_out(0, in(0)); break;
            case OpKind::LayerNormGradInput: set_out(0, in(0)); break;
            case OpKind::BatchNormGradGamma:
            case OpKind::LayerNormGradGamma: set_out(0, {in(0).back()}); break;
        }
    }
    for (const std::string& out : g.outputs)
        if (!g.value_types.count(out))
            throw Error(Error::Code::ShapeMismatch, "graph output untyped: " + out);
    return info;
}

Graph eliminate_dead(const Graph& g) {
    std::unordered_map<std::string, int> producers;
    for (size_t i = 0; i < g.nodes.size(); ++i)
        for (const std::string& o : g.nodes[i].outputs) producers[o] = static_cast<int>(i);
    std::vector<bool> keep(g.nodes.size(), false);
    std::vector<std::string> work(g.outputs.begin(), g.outputs.end());
    while (!work.empty()) {
        std::string v = work.back();
        work.pop_back();
        auto it = producers.find(v);
        if (it == producers.end() || keep[it->second]) continue;
        keep[it->second] = true;
        for (const std::string& in : g.nodes[it->second].inputs) work.push_back(in);
    }
    Graph out = g;
    out.nodes.clear();
    for (size_t i = 0; i < g.nodes.size(); ++i)
        if (keep[i]) out.nodes.push_back(g.nodes[i]);
    std::unordered_set<std::string> consumed(g.outputs.begin(), g.outputs.end());
    for (const Node& n : out.nodes) {
        for (const std::string& v : n.inputs) consumed.insert(v);
        for (const std::string& v : n.weights) consumed.insert(v);
    }
    for (auto it = out.initializers.begin(); it != out.initializers.end();)
        it = consumed.count(it->first) ? std::next(it) : out.initializers.erase(it);
    out.value_types.clear();
    return out;
}

Graph canonicalize(const Graph& g) {
    Graph out = g;
    out.value_types.clear();
    std::unordered_set<std::string> output_set(out.outputs.begin(), out.outputs.end());
    bool changed = true;
    while (changed) {
        changed = false;
        for (size_t i = 0; i < out.nodes.size(); ++i) {
            Node& n = out.nodes[i];
            if (n.op != OpKind::Identity || output_set.count(n.outputs[0])) continue;
            const std::string from = n.outputs[0], to = n.inputs[0];
            for (Node& m : out.nodes)
                for (std::string& in : m.inputs)
                    if (in == from) in = to;
            out.nodes.erase(out.nodes.begin() + static_cast<long>(i));
            changed = true;
            break;
        }
    }
    std::unordered_set<std::string> bypassed;
    changed = true;
    while (changed) {
        changed = false;
        std::unordered_map<std::string, const Node*> producer;
        for (const Node& n : out.nodes)
            for (const std::string& o : n.outputs) producer[o] = &n;
        for (Node& n : out.nodes) {
            if (n.op != OpKind::Flatten) continue;
            auto it = producer.find(n.inputs[0]);
            if (it != producer.end() && it->second->op == OpKind::Flatten && it->second != &n) {
                bypassed.insert(n.inputs[0]);
                n.inputs[0] = it->second->inputs[0];
                changed = true;
            }
        }
    }
    changed = true;
    while (changed) {
        changed = false;
        std::unordered_set<std::string> referenced(out.outputs.begin(), out.outputs.end());
        for (const Node& n : out.nodes)
            for (const std::string& v : n.inputs) referenced.insert(v);
        for (size_t i = 0; i < out.nodes.size(); ++i) {
            const Node& n = out.nodes[i];
            if (n.op == OpKind::Flatten && bypassed.count(n.outputs[0]) && !referenced.count(n.outputs[0])) {
                out.nodes.erase(out.nodes.begin() + static_cast<long>(i));
                changed = true;
                break;
            }
        }
    }
    return out;
}

VdimBinding VdimBinding::enable(std::initializer_list<int32_t> ids) {
    VdimBinding b;
    for (int32_t id : ids) b.items[id] = {Action::Enable, 0};
    return b;
}

VdimReport infer_vdims(const Graph& g) {
    VdimReport r;
    for (const auto& gi : g.inputs)
        for (const Dim& d : gi.type.shape.dims)
            if (d.is_sym() && !r.report_id.count(d.sym_id())) {
                const int32_t id = static_cast<int32_t>(r.free_syms.size());
                r.report_id[d.sym_id()] = id;
                r.free_syms.push_back({id, d.seed_extent()});
            }
    return r;
}

Graph bind_vdims(const Graph& g, const VdimReport& report, const VdimBinding& binding) {
    for (const auto& [id, item] : binding.items) {
        const bool known = std::any_of(report.free_syms.begin(), report.free_syms.end(),
                                       [&](const VdimReport::FreeSym& f) { return f.id == id; });
        if (!known) throw Error(Error::Code::UnknownSymbol, "unknown vdim #" + std::to_string(id));
        if (item.action == VdimBinding::Action::Override && item.extent < 1)
            throw Error(Error::Code::IllegalOverride, "#" + std::to_string(id) + ": override extent must be >= 1");
    }
    Graph out = g;
    out.value_types.clear();
    out.next_sym_id = 0;
    for (auto& gi : out.inputs)
        for (Dim& d : gi.type.shape.dims) {
            if (!d.is_sym()) continue;
            auto it = report.report_id.find(d.sym_id());
            if (it == report.report_id.end()) {
                d = Dim::fixed(d.seed_extent());
                continue;
            }
            const int32_t rid = it->second;
            auto bit = binding.items.find(rid);
            const VdimBinding::Action a = bit == binding.items.end() ? VdimBinding::Action::Disable : bit->second.action;
            if (a == VdimBinding::Action::Disable) {
                d = Dim::fixed(d.seed_extent());
            } else if (a == VdimBinding::Action::Override) {
                d = Dim::fixed(bit->second.extent);
            } else {
                d = Dim::sym(rid, d.seed_extent());
                out.next_sym_id = std::max(out.next_sym_id, rid + 1);
            }
        }
    try {
        return infer_shapes(out).graph;
    } catch (const Error& e) {
        if (e.code() == Error::Code::ExtentMismatch)
            throw Error(Error::Code::IllegalOverride, std::string("binding failed: ") + e.what());
        throw;
    }
}

OptimizeResult optimize(const Graph& g, const VdimBinding& binding) {
    Graph cur = eliminate_dead(canonicalize(g));
    OptimizeResult r;
    r.report = infer_vdims(cur);
    r.graph = bind_vdims(cur, r.report, binding);
    return r;
}

}  // namespace nnc::passes
