// capi.cpp -- extern "C" surface of libnnc_b200.so (include/nnc_b200.h).
#include "nnc_b200.h"
#include "nncb.h"

#include <cstring>
#include <memory>
#include <sstream>

#include <json.hpp>

#include "nnc/autodiff.hpp"
#include "nnc/backends.hpp"
#include "nnc/ingest.hpp"
#include "nnc/passes.hpp"
#include "nnc/plan.hpp"
#include "nnc/runtime.hpp"

using namespace nnc;

struct nnc_model {
    ingest::Model model;
    hlir::Graph optimized;
    autodiff::VersionSet versions;
    plan::VersionPlans plans;
    std::unique_ptr<runtime::HostModel> host;
    runtime::ExecOptions opts;
    std::map<std::string, Tensor> inputs;
    std::map<std::string, Tensor> outputs;
    std::map<std::string, Tensor> grads;
    runtime::Trainer* trainer = nullptr;   // runtime::shared_trainer's, owned by the runtime cache
    std::string desc;
};

namespace {

thread_local std::string g_err;
thread_local std::string g_buf;
thread_local int g_status = 0;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return g_status = 0;
    } catch (const Error& e) {
        g_err = e.what();
        return g_status = 1 + static_cast<int>(e.code());
    } catch (const std::exception& e) {
        g_err = e.what();
        return g_status = 100;
    }
}

std::string jstr(const std::string& s) { return nlohmann::json(s).dump(); }

void describe_plan(std::ostringstream& os, const plan::ExecutionPlan& p) {
    os << "{\"groups\":[";
    for (size_t i = 0; i < p.groups.size(); ++i) {
        const auto& g = p.groups[i];
        os << (i ? "," : "") << "{\"backend\":" << jstr(backends::backend_name(g.backend)) << ",\"label\":" << jstr(g.label)
           << ",\"members\":[";
        for (size_t k = 0; k < g.members.size(); ++k) os << (k ? "," : "") << jstr(g.members[k]);
        os << "],\"launches\":[";
        for (size_t k = 0; k < g.launches.size(); ++k) {
            const auto& L = g.launches[k];
            os << (k ? "," : "") << "{\"kind\":" << jstr(plan::launch_kind_name(L.kind)) << ",\"label\":" << jstr(L.label)
               << ",\"instrs\":" << L.ew.size() << ",\"tile\":" << L.tile << ",\"args\":[";
            for (size_t a = 0; a < L.args.size(); ++a)
                os << (a ? "," : "") << "[" << jstr(p.values[L.args[a].slot].name) << "," << L.args[a].offset << ","
                   << (L.is_out[a] ? 1 : 0) << "]";
            os << "]}";
        }
        os << "]}";
    }
    os << "],\"exec_steps\":[";
    for (size_t i = 0; i < p.exec_steps.size(); ++i) os << (i ? "," : "") << jstr(p.exec_steps[i].label);
    os << "],\"values\":[";
    for (size_t i = 0; i < p.values.size(); ++i) {
        const auto& v = p.values[i];
        os << (i ? "," : "") << "{\"name\":" << jstr(v.name) << ",\"category\":" << jstr(plan::category_name(v.category))
           << ",\"storage\":" << (v.storage == plan::StorageClass::Buffer ? "\"buffer\"" : "\"register\"")
           << ",\"resident\":" << (v.resident ? "true" : "false") << ",\"dims\":[";
        for (size_t d = 0; d < v.dims.size(); ++d) os << (d ? "," : "") << v.dims[d];
        os << "]}";
    }
    os << "],\"events\":[";
    for (size_t i = 0; i < p.events.size(); ++i)
        os << (i ? "," : "") << "[" << p.events[i].step << "," << (p.events[i].alloc ? 1 : 0) << "," << p.events[i].slot
           << "]";
    os << "],\"launch_count\":" << p.launch_count() << "}";
}

const plan::ExecutionPlan& pred_plan(nnc_model* m) { return m->plans.inference; }

Tensor target_tensor(nnc_model* m, const float* target, int64_t n) {
    // the prediction's shape for the fed inputs (a dynamic batch re-specialises the plans)
    const auto& p = runtime::plan_for_inputs(pred_plan(m), m->inputs, m->opts.bindings);
    const auto& v = p.values[p.output_slots.at(0)];
    if (element_count(v.dims) != n) throw Error(Error::Code::ShapeMismatch, "target size mismatch");
    // borrowed: every consumer (train_step, gradients, stage, trainer_prepare)
    // has uploaded it before the C-ABI call returns
    return Tensor::view(DType::F32, v.dims, target);
}

}  // namespace

extern "C" {

const char* nnc_last_error(void) { return g_err.c_str(); }
int nnc_last_status(void) { return g_status; }

nnc_model* nnc_model_compile(const char* doc, int precision) { return nnc_model_compile_ex(doc, precision, nullptr, 0); }

nnc_model* nnc_model_compile_ex(const char* doc, int precision, const int32_t* enable_vdims, int n_enable) {
    auto m = std::make_unique<nnc_model>();
    int rc = guarded([&] {
        m->model = ingest::parse_model(doc);
        passes::VdimBinding binding;
        for (int i = 0; i < n_enable; ++i) binding.items[enable_vdims[i]] = {passes::VdimBinding::Action::Enable, 0};
        m->optimized = passes::optimize(m->model.graph, binding).graph;
        m->versions = autodiff::derive_versions(m->optimized);
        m->plans = plan::compile_version_set(m->versions, [](const hlir::Graph& g) { return backends::default_assignment(g); });
        m->host = std::make_unique<runtime::HostModel>(runtime::HostModel::from_graph(m->optimized));
        m->opts.gemm_precision = precision;
    });
    return rc ? nullptr : m.release();
}

void nnc_model_free(nnc_model* m) {
    if (!m) return;
    try {
        m->trainer = nullptr;
        runtime::release(m->plans);
        runtime::default_device().evict_model(*m->host);
    } catch (...) {
    }
    delete m;
}

const char* nnc_model_describe(nnc_model* m) {
    std::ostringstream os;
    os << "{\"inference\":";
    describe_plan(os, m->plans.inference);
    os << ",\"train_fwd\":";
    describe_plan(os, m->plans.train_fwd);
    os << ",\"train_bwd\":";
    describe_plan(os, m->plans.train_bwd);
    os << ",\"save_set\":" << nlohmann::json(m->plans.save_set).dump();
    os << ",\"output_grads\":" << nlohmann::json(m->plans.output_grads).dump();
    os << ",\"weight_grads\":" << nlohmann::json(m->plans.weight_grads).dump();
    os << ",\"weights\":{";
    size_t k = 0;
    for (const auto& name : m->host->names()) os << (k++ ? "," : "") << jstr(name) << ":" << nlohmann::json(m->optimized.initializers.at(name).dims()).dump();
    auto peak = plan::estimate_peak(m->plans, 64);
    os << "},\"peak\":{\"inference\":" << peak.inference_bytes << ",\"training\":" << peak.training_bytes << "}}";
    m->desc = os.str();
    return m->desc.c_str();
}

int nnc_model_set_weight(nnc_model* m, const char* name, const float* data, int64_t n) {
    return guarded([&] {
        Tensor t = m->host->tensor(name);
        if (t.elements() != n) throw Error(Error::Code::ShapeMismatch, std::string(name) + ": size mismatch");
        std::memcpy(t.data(), data, t.byte_size());
        m->host->set(name, std::move(t));
    });
}

int nnc_model_get_weight(nnc_model* m, const char* name, float* out, int64_t n) {
    return guarded([&] {
        const Tensor& t = m->host->tensor(name);
        if (t.elements() != n) throw Error(Error::Code::ShapeMismatch, std::string(name) + ": size mismatch");
        std::memcpy(out, t.data(), t.byte_size());
    });
}

int nnc_model_set_input(nnc_model* m, const char* name, const float* data, const int64_t* dims, int rank) {
    return guarded([&] {
        // steady-state steps feed the same shapes: copy into the existing
        // storage on the copy threads instead of allocating (and zero-filling)
        // a fresh tensor every call
        std::vector<int64_t> d(dims, dims + rank);
        auto it = m->inputs.find(name);
        if (it == m->inputs.end() || it->second.dims() != d || it->second.is_view()) {
            it = m->inputs.insert_or_assign(name, Tensor::uninitialized(DType::F32, d)).first;
        }
        nncb_host_copy(it->second.data(), data, it->second.byte_size());
    });
}

// borrowed inputs are valid only for the call that consumes them
void drop_views(nnc_model* m) {
    for (auto it = m->inputs.begin(); it != m->inputs.end();)
        it = it->second.is_view() ? m->inputs.erase(it) : std::next(it);
}

int nnc_model_set_input_borrowed(nnc_model* m, const char* name, const float* data, const int64_t* dims, int rank) {
    // no copy: the next run / train_step streams straight from `data`
    return guarded([&] { m->inputs.insert_or_assign(name, Tensor::view(DType::F32, std::vector<int64_t>(dims, dims + rank), data)); });
}

int nnc_model_save_plans(nnc_model* m, uint8_t* out, uint64_t capacity, uint64_t* size) {
    return guarded([&] {
        // SOLP stream of the three role plans (ref plan.cpp:633-848 plus B200 launch descriptors);
        // call with out == nullptr to query the size
        std::vector<uint8_t> b = plan::serialize_version_plans(m->plans);
        *size = b.size();
        if (out) {
            if (capacity < b.size()) throw Error(Error::Code::ShapeMismatch, "save_plans: buffer too small");
            std::memcpy(out, b.data(), b.size());
        }
    });
}

int nnc_model_load_plans(nnc_model* m, const uint8_t* bytes, uint64_t n) {
    return guarded([&] {
        plan::VersionPlans v = plan::load_version_plans(std::vector<uint8_t>(bytes, bytes + n));
        for (const std::string& w : v.inference.weight_names)
            if (!m->host->has(w)) throw Error(Error::Code::BadDocument, "load_plans: plan weight " + w + " is not in the model");
        m->trainer = nullptr;
        runtime::release(m->plans);
        m->plans = std::move(v);
    });
}

int nnc_model_run(nnc_model* m, int role) {
    const int rc = guarded([&] {
        const plan::ExecutionPlan& p = role == 1 ? m->plans.train_fwd : m->plans.inference;
        m->outputs = runtime::execute_on(p, m->inputs, *m->host, nullptr, m->opts);
    });
    drop_views(m);
    return rc;
}

int nnc_model_run_outputs(nnc_model* m, int role, const char* names) {
    const int rc = guarded([&] {
        // ExecOptions::materialize: only the named outputs are copied back
        std::set<std::string> want;
        std::string cur;
        for (const char* c = names; c && *c; ++c) {
            if (*c == ',') {
                if (!cur.empty()) want.insert(cur);
                cur.clear();
            } else {
                cur += *c;
            }
        }
        if (!cur.empty()) want.insert(cur);
        runtime::ExecOptions o = m->opts;
        o.materialize = &want;
        const plan::ExecutionPlan& p = role == 1 ? m->plans.train_fwd : m->plans.inference;
        m->outputs = runtime::execute_on(p, m->inputs, *m->host, nullptr, o);
    });
    drop_views(m);
    return rc;
}

// Pipelined runs from host buffers (runtime::execute_stage / execute_launch_staged /
// execute_staged_outputs). names: comma-separated outputs to bring back (NULL or "" = all).
int nnc_model_stage_run(nnc_model* m, int role) {
    const int rc = guarded([&] {
        const plan::ExecutionPlan& p = role == 1 ? m->plans.train_fwd : m->plans.inference;
        runtime::execute_stage(p, m->inputs, nullptr);
    });
    drop_views(m);
    return rc;
}

int nnc_model_run_staged(nnc_model* m, int role, const char* names) {
    return guarded([&] {
        std::set<std::string> want;
        std::string cur;
        for (const char* c = names; c && *c; ++c) {
            if (*c == ',') {
                if (!cur.empty()) want.insert(cur);
                cur.clear();
            } else {
                cur += *c;
            }
        }
        if (!cur.empty()) want.insert(cur);
        runtime::ExecOptions o = m->opts;
        if (!want.empty()) o.materialize = &want;
        const plan::ExecutionPlan& p = role == 1 ? m->plans.train_fwd : m->plans.inference;
        runtime::execute_launch_staged(p, *m->host, nullptr, o);
    });
}

int nnc_model_staged_outputs(nnc_model* m, int role) {
    return guarded([&] {
        const plan::ExecutionPlan& p = role == 1 ? m->plans.train_fwd : m->plans.inference;
        m->outputs = runtime::execute_staged_outputs(p, nullptr);
    });
}

int nnc_model_output_dims(nnc_model* m, const char* name, int64_t* dims, int* rank) {
    return guarded([&] {
        auto it = m->outputs.find(name);
        if (it == m->outputs.end()) throw Error(Error::Code::ShapeMismatch, std::string("no output ") + name);
        *rank = static_cast<int>(it->second.dims().size());
        for (int i = 0; i < *rank && i < 8; ++i) dims[i] = it->second.dims()[i];
    });
}

int nnc_model_output(nnc_model* m, const char* name, float* out, int64_t n) {
    return guarded([&] {
        auto it = m->outputs.find(name);
        if (it == m->outputs.end()) throw Error(Error::Code::ShapeMismatch, std::string("no output ") + name);
        if (it->second.elements() != n) throw Error(Error::Code::ShapeMismatch, "output size mismatch");
        nncb_host_copy(out, it->second.data(), it->second.byte_size());
    });
}

int nnc_model_train_step(nnc_model* m, const float* target, int64_t n, double lr, double* loss) {
    const int rc = guarded([&] { *loss = runtime::train_step_on(m->plans, m->inputs, target_tensor(m, target, n), *m->host, lr, nullptr, m->opts); });
    drop_views(m);
    return rc;
}

// Pipelined training from host buffers (runtime::Trainer::stage / launch_staged /
// staged_loss): stage step i + 1 while step i computes.
int nnc_model_stage_step(nnc_model* m, const float* target, int64_t n) {
    const int rc = guarded([&] {
        runtime::Trainer& t = runtime::shared_trainer(m->plans, *m->host, runtime::default_device(), m->opts);
        t.stage(m->inputs, target_tensor(m, target, n));
    });
    drop_views(m);
    return rc;
}

int nnc_model_train_step_staged(nnc_model* m, double lr) {
    return guarded([&] { runtime::shared_trainer(m->plans, *m->host, runtime::default_device(), m->opts).launch_staged(lr); });
}

int nnc_model_staged_loss(nnc_model* m, double* loss) {
    return guarded([&] { *loss = runtime::shared_trainer(m->plans, *m->host, runtime::default_device(), m->opts).staged_loss(); });
}

int nnc_model_gradients(nnc_model* m, const float* target, int64_t n, double* loss) {
    const int rc = guarded([&] { m->grads = runtime::gradients(m->plans, m->inputs, target_tensor(m, target, n), *m->host, loss, nullptr, m->opts); });
    drop_views(m);
    return rc;
}

int nnc_model_set_loss(nnc_model* m, int kind) {
    return guarded([&] {
        if (kind != runtime::LOSS_L1 && kind != runtime::LOSS_SOFTMAX_CE)
            throw Error(Error::Code::BadDocument, "unknown loss kind " + std::to_string(kind));
        runtime::release(m->plans);   // trainers are bound with their loss
        m->trainer = nullptr;
        m->opts.loss = kind;
    });
}

int nnc_model_debug_keep_values(nnc_model* m, int on) {
    return guarded([&] {
        runtime::release(m->plans);   // the next training call binds afresh
        m->trainer = nullptr;
        m->opts.keep_values = on != 0;
    });
}

int nnc_model_run_value(nnc_model* m, int role, const char* name, float* out, int64_t n, int64_t* dims, int* rank) {
    return guarded([&] {
        const plan::ExecutionPlan& p0 = role == 1 ? m->plans.train_fwd : m->plans.inference;
        Tensor v = runtime::last_run_value(runtime::plan_for_inputs(p0, m->inputs, m->opts.bindings), name);
        if (rank) {
            *rank = static_cast<int>(v.dims().size());
            for (size_t i = 0; i < v.dims().size() && i < 8; ++i) dims[i] = v.dims()[i];
        }
        if (!out) return;
        if (v.elements() != n) throw Error(Error::Code::ShapeMismatch, std::string("value size mismatch: ") + name);
        std::memcpy(out, v.data(), v.byte_size());
    });
}
int nnc_model_trainer_value(nnc_model* m, const char* name, float* out, int64_t n, int64_t* dims, int* rank) {
    return guarded([&] {
        runtime::Trainer& t = runtime::shared_trainer(m->plans, *m->host, runtime::default_device(), m->opts);
        Tensor v = t.value(name);
        if (rank) {
            *rank = static_cast<int>(v.dims().size());
            for (size_t i = 0; i < v.dims().size() && i < 8; ++i) dims[i] = v.dims()[i];
        }
        if (!out) return;
        if (v.elements() != n) throw Error(Error::Code::ShapeMismatch, std::string("value size mismatch: ") + name);
        std::memcpy(out, v.data(), v.byte_size());
    });
}

int nnc_model_grad(nnc_model* m, const char* weight, float* out, int64_t n) {
    return guarded([&] {
        auto it = m->grads.find(weight);
        if (it == m->grads.end()) throw Error(Error::Code::MissingGrad, std::string("no gradient for ") + weight);
        if (it->second.elements() != n) throw Error(Error::Code::ShapeMismatch, "gradient size mismatch");
        std::memcpy(out, it->second.data(), it->second.byte_size());
    });
}

int nnc_model_trainer_prepare(nnc_model* m, const float* target, int64_t n) {
    const int rc = guarded([&] {
        auto& dev = runtime::default_device();
        m->trainer = &runtime::shared_trainer(m->plans, *m->host, dev, m->opts);
        Tensor t = target_tensor(m, target, n);
        // one full host step uploads inputs + target and warms every kernel
        m->trainer->step(m->inputs, t, 0.0);
    });
    drop_views(m);
    return rc;
}

int nnc_model_trainer_step_device(nnc_model* m, double lr) {
    return guarded([&] {
        if (!m->trainer) throw Error(Error::Code::BadDocument, "trainer not prepared");
        m->trainer->step_device(lr);
    });
}

int nnc_model_trainer_loss(nnc_model* m, double* loss) {
    return guarded([&] {
        if (!m->trainer) throw Error(Error::Code::BadDocument, "trainer not prepared");
        *loss = m->trainer->last_loss();
    });
}

// Data-parallel region layout and bucket schedule (runtime::dp_layout) as
// JSON; host-only (no device needed).
const char* nnc_model_dp_schedule(nnc_model* m, int64_t bucket_bytes) {
    int rc = guarded([&] {
        runtime::DpLayout L = runtime::dp_layout(m->plans, *m->host, std::max<int64_t>(bucket_bytes / 4, 64));
        nlohmann::json w = nlohmann::json::array(), b = nlohmann::json::array();
        for (const std::string& n : L.weights)
            w.push_back({{"name", n}, {"offset", L.offset[n]}, {"elements", L.elements[n]}, {"grad_launch", L.grad_launch[n]}});
        for (const auto& x : L.buckets)
            b.push_back({{"offset", x.offset}, {"count", x.count}, {"close_launch", x.close_launch},
                         {"update_launch", x.update_launch}});
        g_buf = nlohmann::json{{"region_elems", L.region_elems}, {"bwd_launches", L.bwd_launches}, {"weights", w},
                               {"buckets", b}}.dump();
    });
    return rc ? nullptr : g_buf.c_str();
}

const char* nnc_model_step_schedule(nnc_model* m, int64_t bucket_bytes, int comm, int do_sgd) {
    int rc = guarded([&] {
        runtime::DpLayout L = runtime::dp_layout(m->plans, *m->host, std::max<int64_t>(bucket_bytes / 4, 64));
        nlohmann::json acts = nlohmann::json::array();
        static const char* kinds[] = {"fork", "allreduce", "update", "join"};
        for (const auto& a : runtime::step_schedule(L, comm != 0, do_sgd != 0))
            acts.push_back({{"after", a.after}, {"kind", kinds[a.kind]}, {"bucket", a.bucket}});
        // what each backward launch writes (weight gradients) and reads (weights)
        std::map<std::string, std::string> weight_of_grad;
        for (const auto& [w, gv] : m->plans.weight_grads) weight_of_grad[gv] = w;
        nlohmann::json writes = nlohmann::json::array(), reads = nlohmann::json::array();
        const plan::ExecutionPlan& bwd = m->plans.train_bwd;
        for (const auto& es : bwd.exec_steps)
            for (uint32_t li : es.launches) {
                const auto& Lc = bwd.groups[es.group].launches[li];
                nlohmann::json wr = nlohmann::json::array(), rd = nlohmann::json::array();
                for (size_t a = 0; a < Lc.args.size(); ++a) {
                    const plan::ValueEntry& v = bwd.values[Lc.args[a].slot];
                    if (Lc.is_out[a]) {
                        auto it = weight_of_grad.find(v.name);
                        if (it != weight_of_grad.end()) wr.push_back(it->second);
                    } else if (v.category == plan::MemCategory::Parameter) {
                        rd.push_back(v.source_weight);
                    }
                }
                writes.push_back(wr);
                reads.push_back(rd);
            }
        nlohmann::json b = nlohmann::json::array();
        for (const auto& x : L.buckets)
            b.push_back({{"offset", x.offset}, {"count", x.count}, {"close_launch", x.close_launch},
                         {"update_launch", x.update_launch}});
        nlohmann::json w = nlohmann::json::array();
        for (const std::string& n : L.weights)
            w.push_back({{"name", n}, {"offset", L.offset[n]}, {"elements", L.elements[n]}});
        g_buf = nlohmann::json{{"bwd_launches", L.bwd_launches}, {"region_elems", L.region_elems}, {"actions", acts},
                               {"launch_writes", writes}, {"launch_reads", reads}, {"buckets", b}, {"weights", w}}
                    .dump();
    });
    return rc ? nullptr : g_buf.c_str();
}

const char* nnc_model_profile_run(nnc_model* m, int role) {
    int rc = guarded([&] {
        const plan::ExecutionPlan& p = role == 1 ? m->plans.train_fwd : m->plans.inference;
        auto t = runtime::profile_run(p, m->inputs, *m->host, nullptr, m->opts);
        nlohmann::json j = nlohmann::json::array();
        for (const auto& x : t)
            j.push_back({{"label", x.label}, {"kind", x.kind}, {"ms", x.ms}, {"bytes", x.bytes}, {"flops", x.flops}});
        g_buf = j.dump();
    });
    drop_views(m);
    return rc ? nullptr : g_buf.c_str();
}

const char* nnc_model_profile_step(nnc_model* m, double lr) {
    int rc = guarded([&] {
        if (!m->trainer) throw Error(Error::Code::BadDocument, "trainer not prepared");
        auto t = m->trainer->profile_step(lr);
        nlohmann::json j = nlohmann::json::array();
        for (const auto& x : t)
            j.push_back({{"label", x.label}, {"kind", x.kind}, {"ms", x.ms}, {"bytes", x.bytes}, {"flops", x.flops}});
        g_buf = j.dump();
    });
    return rc ? nullptr : g_buf.c_str();
}

int nnc_model_memory(nnc_model* m, int role, uint64_t* arena, uint64_t* live_high, uint64_t* estimate) {
    return guarded([&] {
        runtime::MemoryReport r;
        if (role == 2) {
            if (!m->trainer) throw Error(Error::Code::BadDocument, "trainer not prepared");
            r = m->trainer->memory_report();
        } else {
            r = runtime::memory_report(role == 1 ? m->plans.train_fwd : m->plans.inference);
        }
        *arena = static_cast<uint64_t>(r.arena_bytes);
        *live_high = static_cast<uint64_t>(r.live_high_water);
        *estimate = static_cast<uint64_t>(r.estimate);
    });
}

uint64_t nnc_model_launches_per_step(nnc_model* m) { return m->trainer ? m->trainer->launches_per_step() : 0; }
uint64_t nnc_model_arena_bytes(nnc_model* m) { return m->trainer ? m->trainer->arena_bytes() : 0; }

int nnc_model_run_device(nnc_model* m, int role) {
    return guarded([&] {
        std::set<std::string> none;
        runtime::ExecOptions o = m->opts;
        o.materialize = &none;
        o.inputs_resident = true;
        runtime::execute_on(role == 1 ? m->plans.train_fwd : m->plans.inference, m->inputs, *m->host, nullptr, o);
    });
}

int nnc_model_infer_device(nnc_model* m) { return nnc_model_run_device(m, 0); }

int nnc_model_check_kernels(nnc_model* m) {
    return guarded([&] {
        for (const auto* p : {&m->plans.inference, &m->plans.train_fwd, &m->plans.train_bwd})
            for (const auto& g : p->groups)
                for (const auto& L : g.launches) {
                    if (L.kind != plan::LaunchKind::Ew) continue;
                    nncb_ew_program prog{static_cast<int32_t>(L.ew.size()), L.ew.data(), L.ew_regs,
                                         static_cast<int32_t>(L.args.size())};
                    if (nncb_ew_compile_check(&prog))
                        throw Error(Error::Code::DeviceError, L.label + ": " + nncb_last_error());
                }
    });
}

int nnc_device_sync_stats(int reset, uint64_t* h2d_bytes, uint64_t* d2h_bytes, uint64_t* weight_bytes) {
    return guarded([&] {
        runtime::SyncStats st = runtime::default_device().sync_stats(reset != 0);
        if (h2d_bytes) *h2d_bytes = st.h2d_bytes;
        if (d2h_bytes) *d2h_bytes = st.d2h_bytes;
        if (weight_bytes) *weight_bytes = st.weight_bytes;
    });
}

void* nnc_device_ctx(void) {
    try {
        return runtime::default_device().ctx();
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

int nnc_comm_unique_id(uint8_t id[128]) {
    if (nncb_comm_unique_id(id)) {
        g_err = nncb_last_error();
        return 100;
    }
    return 0;
}

int nnc_init_comm(int nranks, int rank, const uint8_t id[128]) {
    return guarded([&] { runtime::default_device().init_comm(nranks, rank, id); });
}

const char* nnc_model_tune(nnc_model* m, int warmup, int trials, const char* injected_json) {
    const char* out = nullptr;
    int rc = guarded([&] {
        backends::CostModel cm;
        cm.warmup = warmup;
        cm.trials = trials;
        cm.gemm_precision = m->opts.gemm_precision;
        if (injected_json && *injected_json) {   // {"node": {"b200_gemm": us, "b200_fused": us}, ...}
            std::map<std::pair<std::string, backends::BackendId>, double> costs;
            const nlohmann::json spec = nlohmann::json::parse(injected_json);
            for (const auto& [node, per] : spec.items())
                for (const auto& [bk, c] : per.items())
                    costs[{node, bk == "b200_gemm" ? backends::BackendId::B200_GEMM : backends::BackendId::B200_FUSED}] =
                        c.get<double>();
            cm = backends::CostModel::injected_from(std::move(costs));
        }
        nlohmann::json j;
        size_t attached = 0;
        runtime::release(m->plans);   // bound programs / trainers of the untuned plans
        m->trainer = nullptr;
        for (const auto& [role, g] : {std::pair<const char*, const hlir::Graph*>{"inference", &m->versions.inference},
                                      {"train_fwd", &m->versions.train_fwd},
                                      {"train_bwd", &m->versions.train_bwd}}) {
            backends::TuningReport r = backends::tune_with_report(*g, cm);
            nlohmann::json recs = nlohmann::json::array();
            for (const auto& x : r.records)
                recs.push_back({{"node", x.node}, {"backend", backends::backend_name(x.backend)}, {"tile", x.tile},
                                {"cost_us", x.cost}, {"chosen", x.chosen}});
            j[role] = {{"records", recs}, {"tiles", r.tiles}, {"text", r.render_text()}};
            plan::ExecutionPlan& p = std::string(role) == "inference" ? m->plans.inference
                                     : std::string(role) == "train_fwd" ? m->plans.train_fwd
                                                                        : m->plans.train_bwd;
            attached += plan::attach_tuning(p, r);
        }
        j["attached_launches"] = attached;
        m->trainer = nullptr;   // rebinds with the tuned plans
        m->desc = j.dump();
        out = m->desc.c_str();
    });
    return rc ? nullptr : out;
}

const char* nnc_group_document(const char* doc, const char* assignment_json) {
    int rc = guarded([&] {
        auto model = ingest::parse_model(doc);
        auto g = passes::optimize(model.graph).graph;
        std::vector<std::vector<std::string>> groups;
        if (assignment_json) {
            std::map<std::string, int> a = nlohmann::json::parse(assignment_json).get<std::map<std::string, int>>();
            groups = backends::group_layers_ints(g, a);
        } else {
            for (const auto& fg : backends::group_layers(g, backends::default_assignment(g))) groups.push_back(fg.members);
        }
        g_buf = nlohmann::json(groups).dump();
    });
    return rc ? nullptr : g_buf.c_str();
}

const char* nnc_group_document_role(const char* doc, int role) {
    int rc = guarded([&] {
        auto model = ingest::parse_model(doc);
        auto g = passes::optimize(model.graph).graph;
        auto vs = autodiff::derive_versions(g);
        const hlir::Graph& rg = role == 2 ? vs.train_bwd : role == 1 ? vs.train_fwd : vs.inference;
        nlohmann::json out = nlohmann::json::array();
        for (const auto& fg : backends::group_layers(rg, backends::default_assignment(rg)))
            out.push_back({{"backend", static_cast<int>(fg.backend)}, {"members", fg.members}});
        g_buf = out.dump();
    });
    return rc ? nullptr : g_buf.c_str();
}

}  // extern "C"
