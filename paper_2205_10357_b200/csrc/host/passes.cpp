// passes.cpp -- shape inference, dead-layer elimination, canonicalization.
// Shape rules follow reference passes.cpp:209-391 (fixed-extent case); the
// extension ops keep their input shape (BatchNorm/Gelu/LayerNorm) or reduce to
// [C] (grad-gamma kernels). Dead-layer elimination and canonicalization give
// the results of reference passes.cpp:574-620 / 704-781 (same kept nodes,
// order and initializers) by their own algorithms (backward liveness sweeps,
// alias resolution, chain roots with reader counts).
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

// Liveness by backward sweeps over the node list: a node is live when one of
// its outputs is needed, and its inputs become needed. A graph whose nodes
// are topologically ordered settles in one sweep; the sweep repeats until
// nothing changes, so any order is handled. Initializers survive when a live
// node reads them (input or weight) or the graph returns them.
Graph eliminate_dead(const Graph& g) {
    std::unordered_set<std::string> needed(g.outputs.begin(), g.outputs.end());
    std::vector<char> live(g.nodes.size(), 0);
    for (bool grew = true; grew;) {
        grew = false;
        for (size_t i = g.nodes.size(); i-- > 0;) {
            if (live[i]) continue;
            const Node& n = g.nodes[i];
            if (std::none_of(n.outputs.begin(), n.outputs.end(), [&](const std::string& v) { return needed.count(v) > 0; }))
                continue;
            live[i] = 1;
            grew = true;
            needed.insert(n.inputs.begin(), n.inputs.end());
        }
    }
    Graph out = g;
    out.nodes.clear();
    std::unordered_set<std::string> read(g.outputs.begin(), g.outputs.end());
    for (size_t i = 0; i < g.nodes.size(); ++i) {
        if (!live[i]) continue;
        out.nodes.push_back(g.nodes[i]);
        read.insert(g.nodes[i].inputs.begin(), g.nodes[i].inputs.end());
        read.insert(g.nodes[i].weights.begin(), g.nodes[i].weights.end());
    }
    std::erase_if(out.initializers, [&](const auto& kv) { return read.count(kv.first) == 0; });
    out.value_types.clear();   // re-inferred by the caller
    return out;
}

namespace {

/// Follows an alias map to the value at the end of the chain (bounded, so a
/// malformed cyclic graph cannot hang the pass).
std::string resolve_alias(const std::unordered_map<std::string, std::string>& alias, std::string v) {
    for (size_t hops = 0; hops <= alias.size(); ++hops) {
        auto it = alias.find(v);
        if (it == alias.end()) break;
        v = it->second;
    }
    return v;
}

}  // namespace

// Canonical form: (1) an Identity whose result is not a graph output is
// removed and its readers read its source (chains resolve through an alias
// map); (2) a Flatten fed by a Flatten reads the chain's first input instead,
// and the bypassed inner Flattens are dropped once nothing reads them.
Graph canonicalize(const Graph& g) {
    const std::unordered_set<std::string> returned(g.outputs.begin(), g.outputs.end());
    Graph out = g;
    out.value_types.clear();

    std::unordered_map<std::string, std::string> alias;   // removed Identity result -> its source
    for (const Node& n : g.nodes)
        if (n.op == OpKind::Identity && !returned.count(n.outputs[0])) alias.emplace(n.outputs[0], n.inputs[0]);
    out.nodes.clear();
    for (const Node& n : g.nodes) {
        if (n.op == OpKind::Identity && alias.count(n.outputs[0])) continue;
        Node m = n;
        for (std::string& in : m.inputs) in = resolve_alias(alias, in);
        out.nodes.push_back(std::move(m));
    }

    // Flatten chains, judged on the producers as they stand after (1)
    std::unordered_map<std::string, size_t> made_by;
    for (size_t i = 0; i < out.nodes.size(); ++i)
        for (const std::string& o : out.nodes[i].outputs) made_by[o] = i;
    auto flatten_source = [&](size_t self, const std::string& v) -> const Node* {
        auto it = made_by.find(v);
        if (it == made_by.end() || it->second == self || out.nodes[it->second].op != OpKind::Flatten) return nullptr;
        return &out.nodes[it->second];
    };
    std::vector<std::string> root(out.nodes.size());
    std::unordered_set<std::string> bypassed;
    for (size_t i = 0; i < out.nodes.size(); ++i) {
        if (out.nodes[i].op != OpKind::Flatten) continue;
        std::string v = out.nodes[i].inputs[0];
        for (size_t hops = 0; hops <= out.nodes.size(); ++hops) {
            const Node* f = flatten_source(i, v);
            if (!f) break;
            bypassed.insert(v);
            v = f->inputs[0];
        }
        root[i] = v;
    }
    for (size_t i = 0; i < out.nodes.size(); ++i)
        if (out.nodes[i].op == OpKind::Flatten) out.nodes[i].inputs[0] = root[i];

    // drop bypassed Flattens nobody reads; a removal can orphan the next one
    std::unordered_map<std::string, int> readers;
    for (const std::string& v : g.outputs) ++readers[v];
    for (const Node& n : out.nodes)
        for (const std::string& v : n.inputs) ++readers[v];
    std::vector<char> drop(out.nodes.size(), 0);
    std::vector<size_t> work;
    for (size_t i = 0; i < out.nodes.size(); ++i)
        if (out.nodes[i].op == OpKind::Flatten && bypassed.count(out.nodes[i].outputs[0]) &&
            readers[out.nodes[i].outputs[0]] == 0)
            work.push_back(i);
    while (!work.empty()) {
        const size_t i = work.back();
        work.pop_back();
        if (drop[i]) continue;
        drop[i] = 1;
        const std::string& src = out.nodes[i].inputs[0];
        if (--readers[src] == 0) {
            auto it = made_by.find(src);
            if (it != made_by.end() && out.nodes[it->second].op == OpKind::Flatten && bypassed.count(src))
                work.push_back(it->second);
        }
    }
    std::vector<Node> kept;
    for (size_t i = 0; i < out.nodes.size(); ++i)
        if (!drop[i]) kept.push_back(std::move(out.nodes[i]));
    out.nodes = std::move(kept);
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
