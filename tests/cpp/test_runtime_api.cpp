// tests/cpp/test_runtime_api.cpp -- the reference's C++ runtime API, called
// exactly as a reference caller does (reference tests/test_runtime.cpp), linked
// against libnnc_b200.so and run on the B200 (tests/test_cpp_api.py, -m gpu).
//
// Covered (reference file:line):
//   identity plan                              test_runtime.cpp:46-55
//   l1_loss / sgd_step known answers, errors   test_runtime.cpp:67-127
//   offload stamp protocol (OffloadDevice)     test_runtime.cpp:129-193
//   ExecutionContext high water == estimate    test_runtime.cpp:195-240
//   training loop: converge, trace, lr = 0     test_runtime.cpp:242-287
//   enabled batch dim (VdimBinding::enable)    test_runtime.cpp:289-303
//   tune_with_report / CostModel / attach      backends.hpp:35-73, backends.cpp:73-176
#include <execinfo.h>
#include <signal.h>
#include <unistd.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "nnc/autodiff.hpp"
#include "nnc/backends.hpp"
#include "nnc/error.hpp"
#include "nnc/ingest.hpp"
#include "nnc/passes.hpp"
#include "nnc/plan.hpp"
#include "nnc/runtime.hpp"
#include "nnc/schedule.hpp"

using namespace nnc;
using namespace nnc::hlir;
using namespace nnc::runtime;

namespace {

int g_failures = 0, g_checks = 0;
#define CHECK(cond)                                                                      \
    do {                                                                                 \
        ++g_checks;                                                                      \
        if (!(cond)) {                                                                   \
            std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #cond); \
            ++g_failures;                                                                \
        }                                                                                \
    } while (0)
#define CHECK_THROWS_AS(expr, type)              \
    do {                                         \
        bool thrown = false;                     \
        try {                                    \
            (void)(expr);                        \
        } catch (const type&) {                  \
            thrown = true;                       \
        }                                        \
        CHECK(thrown && "throws " #type);        \
    } while (0)

plan::VersionPlans compile_versions(const Graph& g) {
    auto versions = autodiff::derive_versions(passes::infer_shapes(g).graph);
    return plan::compile_version_set(versions, [](const Graph& gg) { return backends::default_assignment(gg); });
}

Graph dense1d() {
    GraphBuilder b;
    b.input("x", TensorType{Shape::fixed({2, 1}, Layout::FLAT), DType::F32});
    Attrs d;
    d.out_features = 1;
    d.has_bias = false;
    b.initializer("fit.weight", Tensor::from_f32({1, 1}, {0.0f}));
    b.node("fit", OpKind::Dense, {"x"}, d, {"fit.weight"});
    b.output("fit");
    return b.build();
}

// C1 small CNN (conv -> ReLU -> max-pool x2, flatten, dense), optionally with a dynamic batch
std::string c1_doc(const char* batch_shape) {
    return std::string(R"({"dialect":"dlb","name":"c1","seed":7,"inputs":[{"name":"x","dtype":"f32",)") + batch_shape +
           R"(}],"outputs":["fc"],"nodes":[
{"name":"c1","op":"conv2d","inputs":["x"],"attrs":{"filters":16,"kernel_size":3,"padding":"same","use_bias":true}},
{"name":"r1","op":"relu","inputs":["c1"]},
{"name":"p1","op":"max_pooling2d","inputs":["r1"],"attrs":{"pool_size":2}},
{"name":"c2","op":"conv2d","inputs":["p1"],"attrs":{"filters":32,"kernel_size":3,"padding":"same","use_bias":true}},
{"name":"bn2","op":"batch_normalization","inputs":["c2"],"attrs":{"epsilon":0.001}},
{"name":"r2","op":"relu","inputs":["bn2"]},
{"name":"p2","op":"max_pooling2d","inputs":["r2"],"attrs":{"pool_size":2}},
{"name":"f","op":"flatten","inputs":["p2"]},
{"name":"fc","op":"dense","inputs":["f"],"attrs":{"units":16}}]})";
}

Tensor uniform(std::vector<int64_t> dims, uint64_t seed) {
    Tensor t(DType::F32, dims);
    uint64_t s = seed * 6364136223846793005ull + 1442695040888963407ull;
    for (int64_t i = 0; i < t.elements(); ++i) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        t.set(i, static_cast<double>(s >> 11) * 0x1.0p-53 * 2.0 - 1.0);
    }
    return t;
}

void identity_plan_returns_its_input() {
    GraphBuilder b;
    b.input("x", TensorType{Shape::fixed({3}), DType::F32});
    b.node("i", OpKind::Identity, {"x"});
    b.output("i");
    auto plans = compile_versions(b.build());
    HostModel host;
    auto out = execute(plans.inference, {{"x", Tensor::from_f32({3}, {1, 2, 3})}}, host);
    CHECK(out.at("i").bitwise_equal(Tensor::from_f32({3}, {1, 2, 3})));
}

void loss_and_update_known_answers() {
    // l1: p = 2, t = 0 -> loss 2, grad 1; zero case
    L1Result r = l1_loss(Tensor::from_f32({1}, {2}), Tensor::from_f32({1}, {0}));
    CHECK(r.loss == 2.0);
    CHECK(r.grad.get(0) == 1.0);
    L1Result z = l1_loss(Tensor::from_f32({2}, {1, 1}), Tensor::from_f32({2}, {1, 1}));
    CHECK(z.loss == 0.0 && z.grad.get(0) == 0.0 && z.grad.get(1) == 0.0);
    CHECK_THROWS_AS(l1_loss(Tensor::from_f32({2}, {1, 1}), Tensor::from_f32({1}, {1})), Error);
    // sgd: w = 1, g = 2, lr = .5 -> 0; stamps bump even at lr = 0
    HostModel m;
    m.weights.emplace("w", Tensor::from_f32({1}, {1}));
    m.stamps["w"] = 0;
    sgd_step(m, {{"w", Tensor::from_f32({1}, {2})}}, 0.5);
    CHECK(m.tensor("w").get(0) == 0.0);
    CHECK(m.stamp("w") == 1);
    sgd_step(m, {{"w", Tensor::from_f32({1}, {2})}}, 0.0);
    CHECK(m.stamp("w") == 2 && m.weights.at("w").get(0) == 0.0);
    CHECK_THROWS_AS(sgd_step(m, {{"missing", Tensor::from_f32({1}, {1})}}, 0.1), Error);
    try {
        sgd_step(m, {{"missing", Tensor::from_f32({1}, {1})}}, 0.1);
    } catch (const Error& e) {
        CHECK(e.code() == Error::Code::MissingGrad);
    }
}

void offload_stamp_protocol() {
    auto model = ingest::parse_model(c1_doc(R"("shape":[4,32,32,3])"));
    auto opt = passes::optimize(model.graph, {});
    auto plans = compile_versions(opt.graph);
    HostModel host = HostModel::from_graph(opt.graph);
    std::map<std::string, Tensor> feed{{"x", uniform({4, 32, 32, 3}, 5)}};

    OffloadDevice device;
    CHECK(device.sync_stats().h2d_bytes == 0);
    CHECK(device.sync_stats().d2h_bytes == 0);
    ExecOptions opts;
    opts.alignment = 64;
    auto host_out = execute(plans.inference, feed, host, nullptr, opts);
    auto dev_out = execute(plans.inference, feed, host, &device, opts);
    for (const auto& [name, t] : host_out) CHECK(t.bitwise_equal(dev_out.at(name)));

    auto stats1 = device.sync_stats();
    int64_t full = 0;
    for (const std::string& w : plans.inference.weight_names)
        full += schedule::align_bytes(static_cast<int64_t>(host.tensor(w).byte_size()), 64);
    CHECK(stats1.weight_bytes == static_cast<uint64_t>(full));
    (void)execute(plans.inference, feed, host, &device, opts);   // nothing stale
    auto stats2 = device.sync_stats();
    CHECK(stats2.weight_bytes == stats1.weight_bytes);
    Tensor b0 = host.tensor("c1.bias");
    host.set("c1.bias", b0);   // one mutation: exactly its aligned bytes move
    auto out3 = execute(plans.inference, feed, host, &device, opts);
    auto stats3 = device.sync_stats();
    CHECK(stats3.weight_bytes - stats2.weight_bytes ==
          static_cast<uint64_t>(schedule::align_bytes(static_cast<int64_t>(b0.byte_size()), 64)));
    CHECK(stats3.weight_transfers.at("c1.bias") == 2);
    CHECK(stats3.weight_transfers.at("c1.weight") == 1);
    for (const auto& [name, t] : host_out) CHECK(t.bitwise_equal(out3.at(name)));
    (void)device.sync_stats(true);
    CHECK(device.sync_stats().h2d_bytes == 0);
    CHECK(device.cache().size() == plans.inference.weight_names.size());
}

void arena_instrumentation_equals_estimate() {
    for (const char* shape : {R"("shape":[2,32,32,3])", R"("shape":[5,32,32,3])"}) {
        auto model = ingest::parse_model(c1_doc(shape));
        Graph g = passes::optimize(model.graph, {}).graph;
        auto plans = compile_versions(g);
        HostModel host = HostModel::from_graph(g);
        const int64_t n = g.inputs[0].type.shape.dims[0].seed_extent();
        std::map<std::string, Tensor> feed{{"x", uniform({n, 32, 32, 3}, 9)}};
        for (int64_t align : {int64_t(1), int64_t(64)}) {
            ExecOptions opts;
            opts.alignment = align;
            ExecutionContext ctx(align);
            (void)execute(plans.inference, feed, host, nullptr, opts, &ctx);
            CHECK(ctx.high_water() == schedule::plan_timeline(plans.inference, align).peak_bytes);
            ExecutionContext tctx(align);
            Tensor target(DType::F32, {n, 16});
            (void)train_step(plans, feed, target, host, 0.1, nullptr, opts, &tctx);
            CHECK(tctx.high_water() == schedule::training_timeline(plans, align).peak_bytes);
            CHECK(tctx.high_water() == schedule::estimate_peak(plans, align).training_bytes);
        }
    }
}

void training_loop_converges_and_traces() {
    Graph g = passes::infer_shapes(dense1d()).graph;
    auto plans = compile_versions(g);
    HostModel host = HostModel::from_graph(g);
    std::map<std::string, Tensor> feed{{"x", Tensor::from_f32({2, 1}, {1, 1})}};
    Tensor target = Tensor::from_f32({2, 1}, {2.005f, 1.995f});
    std::vector<std::string> trace;
    ExecOptions opts;
    opts.trace = &trace;
    std::vector<double> losses;
    for (int step = 0; step < 100; ++step) losses.push_back(train_step(plans, feed, target, host, 0.1, nullptr, opts));
    CHECK(losses.back() < 0.01);
    int non_increasing = 0;
    for (size_t i = 1; i < losses.size(); ++i) non_increasing += losses[i] <= losses[i - 1];
    CHECK(non_increasing >= 90);
    std::vector<std::string> phases;
    for (const std::string& line : trace)
        if (line == "forward" || line == "loss" || line == "backward" || line == "update") phases.push_back(line);
    CHECK(phases.size() == 400);
    CHECK(phases.size() >= 4 && phases[0] == "forward" && phases[1] == "loss" && phases[2] == "backward" &&
          phases[3] == "update");
    // the host weights are the updated ones after each step (public map)
    CHECK(std::fabs(host.weights.at("fit.weight").get(0) - 2.0) < 0.02);
    // lr = 0: identical losses
    HostModel frozen = HostModel::from_graph(g);
    double l1 = train_step(plans, feed, target, frozen, 0.0);
    double l2 = train_step(plans, feed, target, frozen, 0.0);
    CHECK(l1 == l2);
    // the returned loss equals an external recomputation at the pre-step weights
    HostModel snap = HostModel::from_graph(g);
    auto out = execute(plans.inference, feed, snap);
    double external = l1_loss(out.at("fit"), target).loss;
    HostModel stepper = HostModel::from_graph(g);
    double returned = train_step(plans, feed, target, stepper, 0.1);
    CHECK(returned == external);
}

void enabled_batch_dim() {
    Graph g = ingest::parse_model(c1_doc(R"("shape":[null,32,32,3],"seed_shape":[2,32,32,3])")).graph;
    auto opt = passes::optimize(g, passes::VdimBinding::enable({0}));
    CHECK(opt.report.free_syms.size() == 1 && opt.report.free_syms[0].seed == 2);
    auto plans = compile_versions(opt.graph);
    HostModel host = HostModel::from_graph(opt.graph);
    for (int64_t batch : {int64_t(1), int64_t(3), int64_t(2)}) {
        Tensor x = uniform({batch, 32, 32, 3}, 11);
        auto out = execute(plans.inference, {{"x", x}}, host);
        CHECK((out.at("fc").dims() == std::vector<int64_t>{batch, 16}));
    }
    // the batch-3 specialisation computes what a batch-3 compile computes, bit for bit
    {
        Graph g3 = ingest::parse_model(c1_doc(R"("shape":[3,32,32,3])")).graph;
        auto p3 = compile_versions(passes::optimize(g3, {}).graph);
        Tensor x = uniform({3, 32, 32, 3}, 11);
        auto a = execute(plans.inference, {{"x", x}}, host);
        auto b = execute(p3.inference, {{"x", x}}, host);
        CHECK(a.at("fc").bitwise_equal(b.at("fc")));
    }
    // mismatched fixed axis rejected
    Tensor bad(DType::F32, {1, 31, 32, 3});
    CHECK_THROWS_AS(execute(plans.inference, {{"x", bad}}, host), Error);
    // explicit binding conflicting with the fed extent
    ExecOptions conflict;
    conflict.bindings[0] = 4;
    CHECK_THROWS_AS(execute(plans.inference, {{"x", uniform({3, 32, 32, 3}, 1)}}, host, nullptr, conflict), Error);
    // training at two batches through the same plans
    for (int64_t batch : {int64_t(4), int64_t(2)}) {
        Tensor target(DType::F32, {batch, 16});
        double loss = train_step(plans, {{"x", uniform({batch, 32, 32, 3}, 3)}}, target, host, 0.01);
        CHECK(std::isfinite(loss) && loss > 0);
    }
    // a disabled vdim collapses to its seed; unknown ids are rejected
    auto fixed = passes::optimize(g, {});
    CHECK(fixed.graph.inputs[0].type.shape.dims[0].seed_extent() == 2 && !fixed.graph.inputs[0].type.shape.dims[0].is_sym());
    CHECK_THROWS_AS(passes::optimize(g, passes::VdimBinding::enable({3})), Error);
}

}  // namespace

void on_fatal(int sig) {
    void* frames[64];
    const int n = backtrace(frames, 64);
    std::fprintf(stderr, "fatal signal %d; backtrace:\n", sig);
    backtrace_symbols_fd(frames, n, STDERR_FILENO);
    _exit(128 + sig);
}

// measured layer-wise tuning as a reference caller uses it (backends.hpp:35-73):
// injected costs are total and deterministic; measured tuning times every GEMM
// tile, and the tuned plans (tiles attached) compute what the untuned ones do
void tuning_report_and_tuned_plans() {
    auto model = ingest::parse_model(c1_doc(R"("shape":[8,16,16,3])"));
    Graph g = passes::optimize(model.graph).graph;
    std::map<std::pair<std::string, backends::BackendId>, double> costs;
    for (const Node& n : g.nodes)
        for (backends::BackendId b : {backends::BackendId::B200_FUSED, backends::BackendId::B200_GEMM})
            if (backends::supports(b, n.op)) costs[{n.name, b}] = 1.0;
    backends::TuningReport inj = backends::tune_with_report(g, backends::CostModel::injected_from(costs));
    CHECK(inj.assignment == backends::default_assignment(g));
    CHECK(inj.render_csv().rfind("node,backend,tile,cost_us,chosen\n", 0) == 0);
    costs.erase(costs.begin());
    {
        bool bad_document = false;
        try {
            backends::tune_with_report(g, backends::CostModel::injected_from(costs));
        } catch (const Error& e) {
            bad_document = e.code() == Error::Code::BadDocument;
        }
        CHECK(bad_document);
    }

    backends::TuningReport rep = backends::tune_with_report(g, backends::CostModel::measured());
    size_t gemm_records = 0;
    for (const auto& r : rep.records) gemm_records += r.backend == backends::BackendId::B200_GEMM;
    CHECK(gemm_records > 2);   // c1, c2, fc: several tile candidates each
    auto versions = autodiff::derive_versions(g);
    auto plans = plan::compile_version_set(versions, [](const Graph& gg) { return backends::default_assignment(gg); });
    auto tuned = plans;
    CHECK(plan::attach_tuning(tuned.inference, rep) > 0);
    HostModel host = HostModel::from_graph(g);
    std::map<std::string, Tensor> in{{"x", uniform({8, 16, 16, 3}, 3)}};
    auto a = execute(plans.inference, in, host);
    auto b = execute(tuned.inference, in, host);
    const Tensor& ya = a.at("fc");
    const Tensor& yb = b.at("fc");
    double num = 0, den = 0;
    for (int64_t i = 0; i < ya.elements(); ++i) {
        num += (ya.get(i) - yb.get(i)) * (ya.get(i) - yb.get(i));
        den += ya.get(i) * ya.get(i);
    }
    CHECK(std::sqrt(num / den) < 1e-2);
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    signal(SIGSEGV, on_fatal);
    signal(SIGABRT, on_fatal);
    struct Case {
        const char* name;
        void (*fn)();
    } cases[] = {
        {"identity plan returns its input", identity_plan_returns_its_input},
        {"l1_loss / sgd_step known answers", loss_and_update_known_answers},
        {"offload: outputs bitwise equal, transfers follow the stamp protocol", offload_stamp_protocol},
        {"arena instrumentation equals the schedule estimate", arena_instrumentation_equals_estimate},
        {"training loop: dense(1->1) converges and traces the four steps", training_loop_converges_and_traces},
        {"enabled batch dim: any batch accepted, fixed axes enforced", enabled_batch_dim},
        {"layer-wise tuning: injected report, measured tiles, tuned plans", tuning_report_and_tuned_plans},
    };
    for (const Case& c : cases) {
        std::printf("[ RUN ] %s\n", c.name);
        const int before = g_failures;
        try {
            c.fn();
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s: unexpected exception: %s\n", c.name, e.what());
            ++g_failures;
        }
        std::printf("[%s] %s\n", g_failures == before ? "PASS" : "FAIL", c.name);
    }
    std::printf("%d checks, %d failures\n", g_checks, g_failures);
    return g_failures == 0 ? 0 : 1;
}
