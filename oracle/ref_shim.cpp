// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A small extern "C" shim over the *reference* nnc library (compiled from
// /root/reference/proj by oracle/Makefile, namespace renamed nnc -> nncref).
// It lets the Python tests and bench.py's CPU-baseline leg drive the reference
// exactly through its public C++ API:
//   ingest::parse_model        (ingest.cpp:411-500)
//   passes::optimize           (passes.cpp:785-793)
//   autodiff::derive_versions  (autodiff.cpp:89-319)
//   plan::compile_version_set  (plan.cpp:441-457)
//   runtime::execute           (runtime.cpp:314-462)
//   runtime::train_step        (runtime.cpp:498-537)
//   backends::group_layers     (backends.cpp:321-400)
//   schedule::estimate_peak    (schedule.cpp:157-204)
// All numeric I/O crosses the ABI as double and is cast to the graph dtype.
#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "nnc/autodiff.hpp"
#include "nnc/backends.hpp"
#include "nnc/error.hpp"
#include "nnc/ingest.hpp"
#include "nnc/kernels.hpp"
#include "nnc/passes.hpp"
#include "nnc/plan.hpp"
#include "nnc/runtime.hpp"
#include "nnc/schedule.hpp"
#include "oracles.hpp"

#include <json.hpp>

using namespace nnc;  // == nncref via -Dnnc=nncref

namespace {

thread_local std::string g_err;
thread_local std::string g_desc;

struct RefModel {
    ingest::Model model;
    hlir::Graph optimized;
    autodiff::VersionSet versions;
    plan::VersionPlans plans;
    runtime::HostModel host;
    std::map<std::string, Tensor> feed;
    std::map<std::string, Tensor> outputs;   // last run's values
    std::map<std::string, Tensor> grads;     // last grads() call, by weight name
    int policy = 0;
};

// 0: the reference's default_assignment (backends.cpp:179-191).
// 1: the B200 policy encoded in reference backends: Conv2D/Dense -> GEMM_TILED,
//    every other compute op -> REF.
backends::BackendAssignment assign(const hlir::Graph& g, int policy) {
    if (policy == 0) return backends::default_assignment(g);
    backends::BackendAssignment a;
    for (const hlir::Node& n : g.nodes) {
        if (!backends::is_compute(n.op)) continue;
        a[n.name] = backends::supports(backends::BackendId::GEMM_TILED, n.op)
                        ? backends::BackendId::GEMM_TILED
                        : backends::BackendId::REF;
    }
    return a;
}

std::string jstr(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') o += '\\';
        o += c;
    }
    return o + "\"";
}

void describe_plan(std::ostringstream& os, const plan::ExecutionPlan& p) {
    os << "{\"groups\":[";
    for (size_t i = 0; i < p.groups.size(); ++i) {
        const auto& g = p.groups[i];
        os << (i ? "," : "") << "{\"backend\":" << jstr(backends::backend_name(g.backend))
           << ",\"label\":" << jstr(g.label) << ",\"members\":[";
        for (size_t k = 0; k < g.members.size(); ++k) os << (k ? "," : "") << jstr(g.members[k]);
        os << "],\"ew_program_len\":" << g.ew_program.size() << "}";
    }
    os << "],\"exec_steps\":[";
    for (size_t i = 0; i < p.exec_steps.size(); ++i)
        os << (i ? "," : "") << jstr(p.exec_steps[i].label);
    os << "],\"values\":[";
    for (size_t i = 0; i < p.values.size(); ++i) {
        const auto& v = p.values[i];
        os << (i ? "," : "") << "{\"name\":" << jstr(v.name) << ",\"category\":"
           << jstr(schedule::category_name(v.category))
           << ",\"storage\":" << (v.storage == plan::StorageClass::Buffer ? "\"buffer\"" : "\"register\"")
           << ",\"resident\":" << (v.resident ? "true" : "false") << ",\"dims\":[";
        for (size_t d = 0; d < v.dims.size(); ++d) os << (d ? "," : "") << v.dims[d].seed_extent();
        os << "]}";
    }
    os << "],\"events\":[";
    for (size_t i = 0; i < p.events.size(); ++i)
        os << (i ? "," : "") << "[" << p.events[i].step << "," << (p.events[i].alloc ? 1 : 0) << ","
           << p.events[i].slot << "]";
    os << "]}";
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        g_err = std::string("nnc::Error(") + std::to_string(static_cast<int>(e.code())) + "): " + e.what();
        return 1 + static_cast<int>(e.code());
    } catch (const std::exception& e) {
        g_err = e.what();
        return 100;
    }
}

Tensor make_tensor(DType dt, const double* data, const int64_t* dims, int rank) {
    Tensor t(dt, std::vector<int64_t>(dims, dims + rank));
    for (int64_t i = 0; i < t.elements(); ++i) t.set(i, data[i]);
    return t;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Parses a DLB/DLA document, runs optimize -> derive_versions -> compile_version_set.
void* ref_model_load(const char* doc, int policy) {
    RefModel* m = new RefModel;
    m->policy = policy;
    int rc = guarded([&] {
        m->model = ingest::parse_model(doc);
        m->optimized = passes::optimize(m->model.graph).graph;
        m->versions = autodiff::derive_versions(m->optimized);
        m->plans = plan::compile_version_set(
            m->versions, [policy](const hlir::Graph& g) { return assign(g, policy); });
        m->host = runtime::HostModel::from_graph(m->optimized);
    });
    if (rc) {
        delete m;
        return nullptr;
    }
    return m;
}

void ref_model_free(void* h) { delete static_cast<RefModel*>(h); }

const char* ref_model_describe(void* h) {
    RefModel* m = static_cast<RefModel*>(h);
    std::ostringstream os;
    os << "{\"inference\":";
    describe_plan(os, m->plans.inference);
    os << ",\"train_fwd\":";
    describe_plan(os, m->plans.train_fwd);
    os << ",\"train_bwd\":";
    describe_plan(os, m->plans.train_bwd);
    os << ",\"save_set\":[";
    for (size_t i = 0; i < m->plans.save_set.size(); ++i)
        os << (i ? "," : "") << jstr(m->plans.save_set[i]);
    os << "],\"output_grads\":[";
    for (size_t i = 0; i < m->plans.output_grads.size(); ++i)
        os << (i ? "," : "") << jstr(m->plans.output_grads[i]);
    os << "],\"weight_grads\":{";
    size_t k = 0;
    for (const auto& [w, v] : m->plans.weight_grads) os << (k++ ? "," : "") << jstr(w) << ":" << jstr(v);
    os << "},\"weights\":{";
    k = 0;
    for (const auto& [w, t] : m->host.weights) {
        os << (k++ ? "," : "") << jstr(w) << ":[";
        for (size_t d = 0; d < t.dims().size(); ++d) os << (d ? "," : "") << t.dims()[d];
        os << "]";
    }
    auto peak = schedule::estimate_peak(m->plans, 64);
    os << "},\"peak\":{\"inference\":" << peak.inference_bytes
       << ",\"training\":" << peak.training_bytes << "}}";
    g_desc = os.str();
    return g_desc.c_str();
}

int ref_feed(void* h, const char* name, const double* data, const int64_t* dims, int rank) {
    RefModel* m = static_cast<RefModel*>(h);
    return guarded([&] {
        m->feed[name] = make_tensor(m->optimized.dtype, data, dims, rank);
    });
}

// Inference through runtime::execute on the compiled inference plan.
int ref_run_inference(void* h) {
    RefModel* m = static_cast<RefModel*>(h);
    return guarded([&] { m->outputs = runtime::execute(m->plans.inference, m->feed, m->host); });
}

// Every value of the inference graph through kernels::eval_graph (REF kernels).
int ref_eval_all(void* h) {
    RefModel* m = static_cast<RefModel*>(h);
    return guarded([&] {
        std::map<std::string, Tensor> w = m->host.weights;
        m->outputs = kernels::eval_graph(m->optimized, m->feed, &w);
    });
}

int ref_value_rank(void* h, const char* name, int64_t* dims) {
    RefModel* m = static_cast<RefModel*>(h);
    auto it = m->outputs.find(name);
    if (it == m->outputs.end()) {
        g_err = std::string("no value ") + name;
        return -1;
    }
    for (size_t i = 0; i < it->second.dims().size(); ++i) dims[i] = it->second.dims()[i];
    return static_cast<int>(it->second.dims().size());
}

int ref_value(void* h, const char* name, double* out, int64_t n) {
    RefModel* m = static_cast<RefModel*>(h);
    auto it = m->outputs.find(name);
    if (it == m->outputs.end()) {
        g_err = std::string("no value ") + name;
        return 1;
    }
    if (it->second.elements() != n) {
        g_err = "size mismatch";
        return 2;
    }
    for (int64_t i = 0; i < n; ++i) out[i] = it->second.get(i);
    return 0;
}

int ref_weight(void* h, const char* name, double* out, int64_t n) {
    RefModel* m = static_cast<RefModel*>(h);
    return guarded([&] {
        const Tensor& t = m->host.tensor(name);
        if (t.elements() != n) throw std::invalid_argument("size mismatch");
        for (int64_t i = 0; i < n; ++i) out[i] = t.get(i);
    });
}

int ref_set_weight(void* h, const char* name, const double* in, int64_t n) {
    RefModel* m = static_cast<RefModel*>(h);
    return guarded([&] {
        Tensor t = m->host.tensor(name);
        if (t.elements() != n) throw std::invalid_argument("size mismatch");
        for (int64_t i = 0; i < n; ++i) t.set(i, in[i]);
        m->host.set(name, std::move(t));
    });
}

// Forward (train_fwd plan) + L1 + backward (train_bwd plan), no update: the
// first three of train_step's four phases (runtime.cpp:498-527). Gradients are
// kept by weight name; the forward outputs/SaveSet in `outputs`.
int ref_grads(void* h, const double* target, const int64_t* dims, int rank, double* loss) {
    RefModel* m = static_cast<RefModel*>(h);
    return guarded([&] {
        const auto& p = m->plans;
        std::string pred = p.inference.values[p.inference.output_slots[0]].name;
        runtime::ExecutionContext ctx(64);
        runtime::ExecOptions opts;
        auto fwd = runtime::execute(p.train_fwd, m->feed, m->host, nullptr, opts, &ctx);
        Tensor t = make_tensor(m->optimized.dtype, target, dims, rank);
        auto l1 = runtime::l1_loss(fwd.at(pred), t);
        *loss = l1.loss;
        std::map<std::string, Tensor> feed;
        feed.emplace("d." + pred, l1.grad);
        auto bwd = runtime::execute(p.train_bwd, feed, m->host, nullptr, opts, &ctx);
        m->outputs = fwd;
        m->outputs.emplace("d." + pred, l1.grad);
        m->grads.clear();
        for (const auto& [w, v] : p.weight_grads) {
            m->grads.emplace(w, bwd.at(v));
            m->outputs.emplace(v, bwd.at(v));
        }
    });
}

int ref_grad(void* h, const char* weight, double* out, int64_t n) {
    RefModel* m = static_cast<RefModel*>(h);
    auto it = m->grads.find(weight);
    if (it == m->grads.end() || it->second.elements() != n) {
        g_err = std::string("no gradient for ") + weight;
        return 1;
    }
    for (int64_t i = 0; i < n; ++i) out[i] = it->second.get(i);
    return 0;
}

// The reference's train_step (forward, loss, backward, SGD update).
int ref_train_step(void* h, const double* target, const int64_t* dims, int rank, double lr,
                   double* loss) {
    RefModel* m = static_cast<RefModel*>(h);
    return guarded([&] {
        Tensor t = make_tensor(m->optimized.dtype, target, dims, rank);
        *loss = runtime::train_step(m->plans, m->feed, t, m->host, lr);
    });
}

// Partition of an arbitrary graph given as a DLB/DLA document: the optimized
// inference graph grouped under `policy`. Returns JSON [[members...],...].
const char* ref_group_document(const char* doc, int policy) {
    g_desc.clear();
    int rc = guarded([&] {
        auto model = ingest::parse_model(doc);
        auto g = passes::optimize(model.graph).graph;
        auto groups = backends::group_layers(g, assign(g, policy));
        std::ostringstream os;
        os << "[";
        for (size_t i = 0; i < groups.size(); ++i) {
            os << (i ? "," : "") << "{\"backend\":" << jstr(backends::backend_name(groups[i].backend))
               << ",\"members\":[";
            for (size_t k = 0; k < groups[i].members.size(); ++k)
                os << (k ? "," : "") << jstr(groups[i].members[k]);
            os << "]}";
        }
        os << "]";
        g_desc = os.str();
    });
    return rc ? nullptr : g_desc.c_str();
}

// The deterministic initializer stream (ingest.cpp:43-52), for pinning.
double ref_init_uniform(uint64_t seed, const char* name, int64_t index, double lo, double hi) {
    ingest::InitStream s(seed, name);
    double v = 0;
    for (int64_t i = 0; i <= index; ++i) v = s.uniform(lo, hi);
    return v;
}

// The reference harness's partition oracles (tests/harness/oracle_groups.cpp:
// 117-150) applied to a partition of one role graph of the document's version
// set: bit 0 = oracle_valid_partition, bit 1 = oracle_maximal_partition; -1 on
// error. partition_json: [{"backend": int, "members": [...]}] (any backend ids).
int ref_check_partition(const char* doc, int role, const char* partition_json) {
    int result = 0;
    int rc = guarded([&] {
        auto model = ingest::parse_model(doc);
        auto g = passes::optimize(model.graph).graph;
        auto vs = autodiff::derive_versions(g);
        const hlir::Graph& rg = role == 2 ? vs.train_bwd : role == 1 ? vs.train_fwd : vs.inference;
        auto j = nlohmann::json::parse(partition_json);
        std::map<std::string, int> backend_of;
        testing::Partition part;
        for (const auto& grp : j) {
            std::vector<std::string> members = grp.at("members").get<std::vector<std::string>>();
            for (const auto& m : members) backend_of[m] = grp.at("backend").get<int>();
            part.push_back(members);
        }
        result = (testing::oracle_valid_partition(rg, backend_of, part) ? 1 : 0) |
                 (testing::oracle_maximal_partition(rg, backend_of, part) ? 2 : 0);
    });
    return rc ? -1 : result;
}

}  // extern "C"
