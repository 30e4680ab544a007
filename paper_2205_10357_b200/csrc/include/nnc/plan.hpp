// nnc/plan.hpp -- lowering of a grouped graph into a B200 execution plan.
//
// Mirrors reference core/include/nnc/plan.hpp:24-182: the same value table
// (names, MemCategory, StorageClass, resident flags), the same static
// alloc/free event schedule and ExecStep structure (one step per member of a
// GEMM group, one step per fused group), and compile_version_set. What differs
// is the lowering of a group: the reference emits one CPU KernelStep per member
// or a per-element register program (plan.cpp:296-353); here a fused group is
// lowered to a short list of device launches -- generated elementwise kernels
// (register programs compiled to sm_100a) plus reduction / pooling kernels --
// and a GEMM member to one tensor-core launch.
#pragma once

#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "nncb.h"
#include "nnc/autodiff.hpp"
#include "nnc/backends.hpp"
#include "nnc/hlir.hpp"

namespace nnc::plan {

enum class MemCategory : uint8_t { Parameter = 0, Input = 1, Output = 2, Intermediate = 3, Saved = 4 };
const char* category_name(MemCategory c);
inline int64_t align_bytes(int64_t b, int64_t a) { return (b + a - 1) / a * a; }

enum class StorageClass : uint8_t { Buffer = 0, FusedRegister = 1 };

struct ValueEntry {
    std::string name;
    MemCategory category = MemCategory::Intermediate;
    StorageClass storage = StorageClass::Buffer;
    bool resident = false;
    std::string source_weight;
    std::vector<int64_t> dims;
};

enum class LaunchKind : uint8_t {
    Ew, Gemm, MaxPool, MaxPoolGrad, AvgPool, AvgPoolGrad, SumRows, CumSum, BnStats,
    BnGradReduce, LnFwd, LnBwd, LnDgamma,
};
const char* launch_kind_name(LaunchKind k);

/// A kernel argument: value-table slot plus an element offset into it.
struct Arg {
    uint32_t slot = 0;
    int64_t offset = 0;
};

struct Launch {
    LaunchKind kind = LaunchKind::Ew;
    std::string label;
    std::vector<Arg> args;
    std::vector<bool> is_out;      // per arg: written by the launch
    // Ew: register program whose slot fields index `args`.
    std::vector<nncb_ew_instr> ew;
    int32_t ew_regs = 0;
    uint32_t elem_slot = 0;        // value whose dims define the iteration space
    // Gemm / pooling / reductions: the originating op and attributes.
    hlir::OpKind op = hlir::OpKind::Identity;
    hlir::Attrs attrs;
    bool relu_epilogue = false;
    // Gemm: the tensor-core tile chosen by measured layer-wise tuning
    // (backends::tune_with_report, attached with attach_tuning); 0 = the
    // kernel library's deterministic table / static rule
    int32_t tile = 0;
};

struct GroupKernel {
    uint32_t id = 0;
    backends::BackendId backend = backends::BackendId::B200_FUSED;
    std::string label;
    std::vector<std::string> members;
    std::vector<Launch> launches;
};

struct PlanEvent {
    int32_t step = 0;
    bool alloc = true;
    uint32_t slot = 0;
};

/// One schedule step: a member of a GEMM group (kernel = member index) or a
/// whole fused group (kernel = -1). Step s >= 1 is exec_steps[s-1].
struct ExecStep {
    uint32_t group = 0;
    int32_t kernel = -1;
    std::string label;
    std::vector<uint32_t> launches;   // indices into groups[group].launches
};

enum class PlanRole : uint8_t { Inference = 0, TrainFwd = 1, TrainBwd = 2 };

/// An enabled (dynamic) dim of a plan input (reference plan.hpp VdimSlot):
/// vdim `sym` is axis `axis` of input value `slot`; the plan is compiled at `extent`.
struct VdimSlot {
    int32_t sym = 0;
    uint32_t slot = 0;
    uint32_t axis = 0;
    int64_t extent = 0;
};

class Specializer;

struct ExecutionPlan {
    uint64_t uid = 0;   // process-unique id (runtime caches key on it, never on addresses)
    DType dtype = DType::F32;
    PlanRole role = PlanRole::Inference;
    std::vector<ValueEntry> values;
    std::vector<GroupKernel> groups;
    std::vector<ExecStep> exec_steps;
    std::vector<PlanEvent> events;
    std::vector<uint32_t> input_slots;
    std::vector<uint32_t> output_slots;
    std::vector<std::string> weight_names;
    // dynamic dims: the runtime re-specialises the plan for other extents
    // (per call, cached) through `spec`; empty for fixed-shape plans
    std::vector<VdimSlot> vdims;
    std::shared_ptr<const Specializer> spec;

    int find_value(const std::string& name) const;
    size_t launch_count() const;
};

ExecutionPlan compile_plan(const hlir::Graph& g, const std::vector<backends::FusionGroup>& groups,
                           PlanRole role = PlanRole::Inference,
                           const autodiff::VersionSet* versions = nullptr);

struct VersionPlans {
    ExecutionPlan inference;
    ExecutionPlan train_fwd;
    ExecutionPlan train_bwd;
    std::vector<std::string> save_set;
    std::vector<std::string> output_grads;
    std::map<std::string, std::string> weight_grads;
};

VersionPlans compile_version_set(
    const autodiff::VersionSet& versions,
    const std::function<backends::BackendAssignment(const hlir::Graph&)>& assign);

/// Persists measured tile choices into a plan: every GEMM launch whose node
/// the report tuned carries the chosen tile code (Launch::tile, saved in SOLP).
/// Returns the number of launches updated.
size_t attach_tuning(ExecutionPlan& p, const backends::TuningReport& report);
size_t attach_tuning(VersionPlans& v, const backends::TuningReport& report);

/// Per-binding re-specialisation of plans compiled with enabled vdims: the
/// source graph with the bound extents substituted runs through the same
/// infer_shapes -> derive_versions -> compile_version_set pipeline once per
/// distinct binding; the result is cached (thread-safe) for the plans' lifetime.
class Specializer {
public:
    using Assign = std::function<backends::BackendAssignment(const hlir::Graph&)>;
    Specializer(hlir::Graph source, Assign assign) : source_(std::move(source)), assign_(std::move(assign)) {}
    const VersionPlans& plans_for(const std::map<int32_t, int64_t>& binding) const;
    static const ExecutionPlan& role_plan(const VersionPlans& v, PlanRole r);

private:
    hlir::Graph source_;
    Assign assign_;
    mutable std::mutex mu_;
    mutable std::map<std::map<int32_t, int64_t>, std::unique_ptr<VersionPlans>> cache_;
};

// Process-unique plan id (runtime caches key on it).
uint64_t next_plan_uid();

/* ------------------------------------------------------------------ */
/*  Serialization (SOLP; ref plan.hpp:154-160) with B200 descriptors    */
/* ------------------------------------------------------------------ */
std::vector<uint8_t> serialize_plan(const ExecutionPlan& p);
ExecutionPlan load_plan(const std::vector<uint8_t>& bytes);
ExecutionPlan load_plan_file(const std::string& path);
void save_plan_file(const ExecutionPlan& p, const std::string& path);
// The three role plans plus the version-set maps, one stream.
std::vector<uint8_t> serialize_version_plans(const VersionPlans& v);
VersionPlans load_version_plans(const std::vector<uint8_t>& bytes);

struct PeakEstimate {
    int64_t inference_bytes = 0;
    int64_t training_bytes = 0;
};
/// Static peak of the event schedule (reference schedule.cpp:157-204 semantics:
/// training carries SaveSet + parameters across the fwd/bwd boundary).
PeakEstimate estimate_peak(const VersionPlans& plans, int64_t alignment = 64);
int64_t plan_peak(const ExecutionPlan& p, int64_t alignment = 64);

}  // namespace nnc::plan
