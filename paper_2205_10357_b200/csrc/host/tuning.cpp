// tuning.cpp -- measured layer-wise tuning (reference backends.cpp:73-176).
//
// The reference times each compute node in isolation on seed-shaped random
// inputs for every backend that supports it (median of `trials` after
// `warmup`, wall clock on the CPU) and assigns the cheapest. On the B200 each
// op has exactly one device backend, so the measured choice that matters is
// the tensor-core TILE of every contraction: a GEMM node is timed once per
// tile candidate of its shape (nncb_gemm_candidates / nncb_gemm_time_tile,
// CUDA events on the compute stream) and the fastest code is recorded in the
// report (TuningReport::tiles) and persisted into the plan's launch
// descriptors (plan::attach_tuning -> SOLP). Other nodes are timed as their
// one-node fused lowering (runtime::profile_run). Injected costs bypass the
// device, as in the reference.
#include <algorithm>
#include <cstdio>
#include <sstream>

#include "nncb.h"
#include "nnc/backends.hpp"
#include "nnc/error.hpp"
#include "nnc/geometry.hpp"
#include "nnc/ingest.hpp"
#include "nnc/passes.hpp"
#include "nnc/plan.hpp"
#include "nnc/runtime.hpp"

namespace nnc::backends {

using hlir::Graph;
using hlir::Node;
using hlir::OpKind;

CostModel CostModel::injected_from(std::map<std::pair<std::string, BackendId>, double> costs) {
    CostModel c;
    c.kind = Kind::Injected;
    c.injected = std::move(costs);
    return c;
}

namespace {

void check(int rc) {
    if (rc) throw Error(Error::Code::DeviceError, std::string("tuning: ") + nncb_last_error());
}

/// Seed-shaped random contents, as the reference's measure_node
/// (InitStream(1, "tune." + value), uniform in [-1, 1]).
Tensor random_tensor(const Graph& g, const std::string& v) {
    const hlir::TensorType* t = g.type_of(v);
    if (!t) throw Error(Error::Code::ShapeMismatch, "tuning: untyped value " + v);
    Tensor x(DType::F32, t->shape.seed_dims());
    ingest::InitStream rng(1, "tune." + v);
    for (int64_t i = 0; i < x.elements(); ++i) x.set(i, rng.uniform(-1.0, 1.0));
    return x;
}

struct DeviceBuffer {
    nncb_ctx* ctx;
    void* p = nullptr;
    DeviceBuffer(nncb_ctx* c, const Tensor* host, int64_t bytes) : ctx(c) {
        check(nncb_malloc(ctx, static_cast<size_t>(std::max<int64_t>(bytes, 16)), &p));
        if (host) check(nncb_h2d(ctx, p, host->data(), host->byte_size()));
        else check(nncb_memset(ctx, p, 0, static_cast<size_t>(std::max<int64_t>(bytes, 16))));
    }
    ~DeviceBuffer() { nncb_free(ctx, p); }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    float* f() const { return static_cast<float*>(p); }
};

const std::vector<int64_t>& seed_dims_of(const Graph& g, const std::string& v, std::vector<int64_t>& keep) {
    const hlir::TensorType* t = g.type_of(v);
    if (!t) throw Error(Error::Code::ShapeMismatch, "tuning: untyped value " + v);
    keep = t->shape.seed_dims();
    return keep;
}

/// The contraction descriptor of a GEMM node at its seed shape (the same
/// mapping the runtime binds, runtime.cpp resolve()).
nncb_gemm_desc gemm_desc(const Graph& g, const Node& n, int precision) {
    nncb_gemm_desc d{};
    d.precision = precision;
    std::vector<int64_t> a, b;
    switch (n.op) {
        case OpKind::Conv2D:
            d.kind = NNCB_CONV_FWD;
            geom::conv_geometry(d, seed_dims_of(g, n.inputs[0], a), n.attrs);
            d.epilogue = n.attrs.has_bias ? NNCB_EPI_BIAS : 0;
            break;
        case OpKind::Conv2DGradInput:
            d.kind = NNCB_CONV_DGRAD;
            geom::conv_geometry(d, seed_dims_of(g, n.outputs[0], a), n.attrs);
            break;
        case OpKind::Conv2DGradWeight:
            d.kind = NNCB_CONV_WGRAD;
            geom::conv_geometry(d, seed_dims_of(g, n.inputs[0], a), n.attrs);
            break;
        case OpKind::Dense:
            d.kind = NNCB_DENSE_FWD;
            seed_dims_of(g, n.inputs[0], a);
            d.batch = a[0]; d.in_f = a[1]; d.out_f = n.attrs.out_features;
            d.epilogue = n.attrs.has_bias ? NNCB_EPI_BIAS : 0;
            break;
        case OpKind::DenseGradInput:
            d.kind = NNCB_DENSE_DGRAD;
            seed_dims_of(g, n.inputs[0], a);
            seed_dims_of(g, n.outputs[0], b);
            d.batch = a[0]; d.out_f = a[1]; d.in_f = b[1];
            break;
        case OpKind::DenseGradWeight:
            d.kind = NNCB_DENSE_WGRAD;
            seed_dims_of(g, n.inputs[0], a);
            seed_dims_of(g, n.inputs[1], b);
            d.batch = a[0]; d.in_f = a[1]; d.out_f = b[1];
            break;
        default: throw Error(Error::Code::UnsupportedInGroup, "tuning: not a GEMM op: " + n.name);
    }
    return d;
}

int64_t out_elems(const nncb_gemm_desc& d) {
    switch (d.kind) {
        case NNCB_DENSE_FWD: return d.batch * d.out_f;
        case NNCB_DENSE_DGRAD: return d.batch * d.in_f;
        case NNCB_DENSE_WGRAD: return d.in_f * d.out_f;
        case NNCB_CONV_FWD: return d.n * d.oh * d.ow * d.co;
        case NNCB_CONV_DGRAD: return d.n * d.ih * d.iw * d.ci;
        default: return d.kh * d.kw * d.ci * d.co;
    }
}

/// GEMM node: (tile code, median us) per candidate.
std::vector<std::pair<int32_t, double>> measure_gemm(const Graph& g, const Node& n, const CostModel& cm) {
    nncb_ctx* ctx = runtime::default_device().ctx();
    const nncb_gemm_desc d = gemm_desc(g, n, cm.gemm_precision);
    // operands: the node's two data inputs (weights count as inputs here)
    std::vector<std::string> ops = n.inputs;
    ops.insert(ops.end(), n.weights.begin(), n.weights.end());
    std::vector<Tensor> host;
    for (size_t i = 0; i < 2 && i < ops.size(); ++i)
        host.push_back(g.initializers.count(ops[i]) ? g.initializers.at(ops[i]) : random_tensor(g, ops[i]));
    if (host.size() < 2) throw Error(Error::Code::UnsupportedInGroup, "tuning: GEMM node without two operands: " + n.name);
    DeviceBuffer A(ctx, &host[0], host[0].byte_size()), B(ctx, &host[1], host[1].byte_size());
    const bool bias = (d.epilogue & NNCB_EPI_BIAS) && ops.size() > 2;
    Tensor bias_host = bias ? (g.initializers.count(ops[2]) ? g.initializers.at(ops[2]) : random_tensor(g, ops[2]))
                            : Tensor();
    DeviceBuffer C(ctx, bias ? &bias_host : nullptr, bias ? bias_host.byte_size() : 16);
    DeviceBuffer O(ctx, nullptr, out_elems(d) * 4);
    int n_c = 0;
    check(nncb_gemm_candidates(&d, nullptr, 0, &n_c));
    std::vector<int32_t> codes(static_cast<size_t>(std::max(n_c, 1)), 0);
    if (n_c) check(nncb_gemm_candidates(&d, codes.data(), n_c, &n_c));
    std::vector<std::pair<int32_t, double>> out;
    for (int32_t code : codes) {
        float ms = 0.f;
        check(nncb_gemm_time_tile(ctx, &d, A.f(), B.f(), bias ? C.f() : nullptr, O.f(), code,
                                  std::max(cm.warmup, 0), std::max(cm.trials, 1), &ms));
        out.push_back({code, 1000.0 * ms});
    }
    return out;
}

/// Any other node: its fused lowering as a one-node plan on the device; the
/// median over trials of the summed launch times.
double measure_fused(const Graph& g, const Node& n, const CostModel& cm) {
    hlir::GraphBuilder b(g.dtype);
    std::map<std::string, Tensor> feed;
    for (const std::string& v : n.inputs) {
        if (g.initializers.count(v)) {
            b.initializer(v, g.initializers.at(v));
            continue;
        }
        const hlir::TensorType* t = g.type_of(v);
        if (!t) throw Error(Error::Code::ShapeMismatch, "tuning: untyped value " + v);
        hlir::TensorType ft = *t;
        ft.shape = hlir::Shape::fixed(t->shape.seed_dims());
        b.input(v, ft);
        feed[v] = random_tensor(g, v);
    }
    for (const std::string& w : n.weights) b.initializer(w, g.initializers.at(w));
    b.graph().nodes.push_back(n);   // as is: every output (e.g. BatchNorm's statistics) and attribute
    for (const std::string& o : n.outputs) b.output(o);
    Graph one = passes::infer_shapes(b.build()).graph;
    const plan::ExecutionPlan p =
        plan::compile_plan(one, group_layers(one, default_assignment(one)), plan::PlanRole::Inference);
    runtime::HostModel model = runtime::HostModel::from_graph(one);
    runtime::ExecOptions opts;
    opts.gemm_precision = cm.gemm_precision;
    std::vector<double> samples;
    for (int t = 0; t < std::max(cm.warmup, 0) + std::max(cm.trials, 1); ++t) {
        double us = 0;
        for (const auto& l : runtime::profile_run(p, feed, model, nullptr, opts)) us += 1000.0 * l.ms;
        if (t >= cm.warmup) samples.push_back(us);
    }
    std::sort(samples.begin(), samples.end());
    return samples[samples.size() / 2];
}

}  // namespace

TuningReport tune_with_report(const Graph& g0, const CostModel& cost) {
    TuningReport report;
    Graph annotated;
    const Graph* gp = &g0;
    if (g0.value_types.empty() && !g0.nodes.empty()) {
        annotated = passes::infer_shapes(g0).graph;
        gp = &annotated;
    }
    const Graph& g = *gp;
    for (const std::string& name : hlir::topo_order(g)) {
        const Node& n = *g.find_node(name);
        if (!is_compute(n.op)) continue;
        const size_t first = report.records.size();
        bool have = false;
        double best_cost = 0;
        BackendId best = BackendId::B200_FUSED;
        int32_t best_tile = 0;
        for (BackendId bk : {BackendId::B200_FUSED, BackendId::B200_GEMM}) {
            if (!supports(bk, n.op)) continue;
            std::vector<std::pair<int32_t, double>> costs;
            if (cost.kind == CostModel::Kind::Injected) {
                auto it = cost.injected.find({n.name, bk});
                if (it == cost.injected.end())
                    throw Error(Error::Code::BadDocument,
                                "injected cost model misses (" + n.name + ", " + backend_name(bk) + ")");
                costs.push_back({0, it->second});
            } else if (bk == BackendId::B200_GEMM) {
                costs = measure_gemm(g, n, cost);
            } else {
                costs.push_back({0, measure_fused(g, n, cost)});
            }
            for (const auto& [tile, c] : costs) {
                report.records.push_back({n.name, bk, c, false, tile});
                if (!have || c < best_cost) {   // strict: ties keep the first (lowest id, first tile)
                    have = true;
                    best_cost = c;
                    best = bk;
                    best_tile = tile;
                }
            }
        }
        if (!have) throw Error(Error::Code::NoBackend, n.name + ": no supporting backend");
        for (size_t i = first; i < report.records.size(); ++i)
            report.records[i].chosen = report.records[i].backend == best && report.records[i].tile == best_tile &&
                                       report.records[i].cost == best_cost;
        report.assignment[n.name] = best;
        if (best == BackendId::B200_GEMM && best_tile) report.tiles[n.name] = best_tile;
    }
    return report;
}

BackendAssignment tune(const Graph& g, const CostModel& cost) { return tune_with_report(g, cost).assignment; }

std::string TuningReport::render_text() const {
    std::ostringstream os;
    os << "node                                     backend     tile        cost_us  chosen\n";
    char line[256];
    for (const TuningRecord& r : records) {
        snprintf(line, sizeof(line), "%-40s %-11s 0x%06x %10.3f  %s\n", r.node.c_str(), backend_name(r.backend),
                 static_cast<unsigned>(r.tile), r.cost, r.chosen ? "*" : "");
        os << line;
    }
    return os.str();
}

std::string TuningReport::render_csv() const {
    std::ostringstream os;
    os << "node,backend,tile,cost_us,chosen\n";
    for (const TuningRecord& r : records)
        os << r.node << "," << backend_name(r.backend) << "," << r.tile << "," << r.cost << "," << (r.chosen ? 1 : 0)
           << "\n";
    return os.str();
}

}  // namespace nnc::backends

namespace nnc::plan {

size_t attach_tuning(ExecutionPlan& p, const backends::TuningReport& report) {
    size_t n = 0;
    for (GroupKernel& gk : p.groups)
        for (Launch& L : gk.launches) {
            if (L.kind != LaunchKind::Gemm) continue;
            auto it = report.tiles.find(L.label);
            if (it == report.tiles.end()) continue;
            L.tile = it->second;
            ++n;
        }
    if (n) p.uid = next_plan_uid();   // a new identity: runtime caches never serve the untuned binding
    return n;
}

size_t attach_tuning(VersionPlans& v, const backends::TuningReport& report) {
    return attach_tuning(v.inference, report) + attach_tuning(v.train_fwd, report) + attach_tuning(v.train_bwd, report);
}

}  // namespace nnc::plan
