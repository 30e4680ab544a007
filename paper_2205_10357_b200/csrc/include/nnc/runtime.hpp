// nnc/runtime.hpp -- the B200 executor behind the reference runtime API.
//
// Reference API kept (core/include/nnc/runtime.hpp):
//   HostModel (:21-34), SyncStats (:40-45), ExecOptions (:81-87),
//   execute (:126-130), l1_loss/sgd_step (:141-144), train_step (:149-152).
// B200 design: a Device owns one nncb context (one GPU), a version-stamped device
// weight cache with the OffloadDevice protocol (runtime.cpp:71-102), and one
// BoundProgram per (plan, role): arena offsets from the static event schedule,
// compiled kernels, and a CUDA graph replayed per call. Training keeps weights
// device-authoritative: SGD runs on the device and HostModel tensors are
// refreshed lazily (HostModel::tensor() pulls stale weights back).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "nnc/plan.hpp"
#include "nnc/tensor.hpp"

struct nncb_ctx;

namespace nnc::runtime {

class Device;

/// Host weights with per-tensor version stamps (reference runtime.hpp:21-34):
/// `weights` and `stamps` are public maps, as the reference's. Training keeps
/// weights device-authoritative; tensor() (and sync()) pull a device-newer
/// weight back before it is read, and the reference-signature train_step
/// syncs after its update, so `weights` reads fresh there too.
class HostModel {
public:
    HostModel();
    HostModel(const HostModel& o);
    HostModel& operator=(const HostModel& o);
    /// Drops the runtime state tied to this model (its cached trainers and
    /// device weight copies) -- a HostModel may die before the plans it ran.
    ~HostModel();
    uint64_t uid() const { return uid_; }
    static HostModel from_graph(const hlir::Graph& g);
    bool has(const std::string& name) const { return weights.count(name) != 0; }
    const Tensor& tensor(const std::string& name) const;   // pulls if device-newer
    uint64_t stamp(const std::string& name) const;
    void set(const std::string& name, Tensor value);      // bumps the stamp
    void bump(const std::string& name);
    std::vector<std::string> names() const;
    /// Pulls every device-newer weight back into `weights`.
    void sync() const;

    mutable std::map<std::string, Tensor> weights;
    std::map<std::string, uint64_t> stamps;

    // Device-authoritative bookkeeping (B200 training).
    mutable Device* device_owner = nullptr;
    mutable std::set<std::string> device_newer;

private:
    uint64_t uid_ = 0;
};

struct SyncStats {
    uint64_t h2d_bytes = 0;
    uint64_t d2h_bytes = 0;
    uint64_t weight_bytes = 0;
    std::map<std::string, uint64_t> weight_transfers;
};

struct ExecOptions {
    int64_t alignment = 64;
    std::map<int32_t, int64_t> bindings;            // vdim id -> extent (explicit wins)
    std::vector<std::string>* trace = nullptr;
    const std::set<std::string>* materialize = nullptr;
    bool use_graphs = true;           // capture each bound program into a CUDA graph
    int gemm_precision = NNCB_PREC_TF32;
    // inputs already on the device from a previous execute of this plan:
    // skip the host->device input copies (device-resident replay)
    bool inputs_resident = false;
    // parity debugging: every Buffer value of a training step gets its own
    // arena bytes (no reuse), so after a step every forward and backward
    // value can be read back (Trainer::value) and checked launch by launch
    bool keep_values = false;
    // the training loss: L1 (the reference's, runtime.cpp:468-483) or softmax
    // cross-entropy over the prediction's last axis (extension; targets are
    // probability vectors)
    int loss = 0;   // LossKind
};

enum LossKind : int { LOSS_L1 = 0, LOSS_SOFTMAX_CE = 1 };

struct L1Result {
    double loss = 0;
    Tensor grad;
};

struct Program;   // a bound plan (internal)

class Device {
public:
    explicit Device(int ordinal = 0);
    ~Device();
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;

    nncb_ctx* ctx() const { return ctx_; }
    SyncStats sync_stats(bool reset = false);

    /// Data parallelism: one process per GPU, NCCL over NVLink/NVSwitch.
    void init_comm(int nranks, int rank, const uint8_t id[128]);
    int nranks() const { return nranks_; }
    int rank() const { return rank_; }

    // --- internals used by execute/train_step -------------------------
    // The cache is keyed by (HostModel uid, weight name): two models never share entries.
    void* weight_buffer(const HostModel& m, const std::string& name, const Tensor& host, uint64_t stamp);
    void* weight_ptr(const HostModel& m, const std::string& name) const;
    void pull_weight(const HostModel& m, const std::string& name, Tensor& host);
    void mark_device_newer(HostModel& m, const std::string& name, uint64_t new_stamp);
    /// Makes `ptr` (a trainer's flat parameter region) the device home of a weight.
    void adopt_weight(const HostModel& m, const std::string& name, void* ptr, size_t bytes, uint64_t stamp);
    /// Pulls device-newer weights of `m` back to the host and drops its cache entries.
    void evict_model(HostModel& m);
    /// Drops the cache entries of a model that is being destroyed (no pull).
    void forget_model(uint64_t model_uid);
    uint64_t cached_stamp(const HostModel& m, const std::string& name) const;
    std::map<const void*, std::unique_ptr<Program>>& programs() { return programs_; }
    SyncStats& stats() { return stats_; }

private:
    struct CachedWeight {
        void* ptr = nullptr;
        size_t bytes = 0;
        uint64_t stamp = 0;
        bool external = false;
    };
    nncb_ctx* ctx_ = nullptr;
    std::map<std::pair<uint64_t, std::string>, CachedWeight> cache_;
    std::map<const void*, std::unique_ptr<Program>> programs_;
    SyncStats stats_;
    int nranks_ = 1, rank_ = 0;
};

/// Process-wide default device (cuda:0 unless NNC_DEVICE is set).
Device& default_device();

/// The reference's offload device (runtime.hpp:40-75), on a B200: a
/// version-stamped weight cache in device memory. sync_weight copies a weight
/// only when its cached stamp is stale, counting h2d / weight bytes (aligned,
/// as the reference) and per-weight transfers; execute / train_step route
/// weights through it and count their input / output copies. Each
/// OffloadDevice has its own cache (a fresh one re-uploads everything).
class OffloadDevice {
public:
    struct CachedWeight {
        void* device = nullptr;   // device bytes (the reference keeps a host byte vector)
        int64_t bytes = 0;
        uint64_t stamp = 0;
    };
    explicit OffloadDevice(Device* device = nullptr);
    ~OffloadDevice();
    OffloadDevice(const OffloadDevice&) = delete;
    OffloadDevice& operator=(const OffloadDevice&) = delete;

    uint8_t* sync_weight(const std::string& name, const Tensor& host, uint64_t stamp, int64_t aligned_bytes);
    void count_h2d(int64_t bytes) { stats_.h2d_bytes += static_cast<uint64_t>(bytes); }
    void count_d2h(int64_t bytes) { stats_.d2h_bytes += static_cast<uint64_t>(bytes); }
    SyncStats sync_stats(bool reset = false);
    /// Marks a weight as already device-resident (persisted cache state): its
    /// bytes are placed without counting a transfer.
    void preseed(const std::string& name, const Tensor& host, uint64_t stamp, int64_t aligned_bytes);
    const std::map<std::string, CachedWeight>& cache() const { return cache_; }
    /// Records that the device copy of `name` is current at `stamp` (training
    /// updates weights on the device; nothing moves).
    void note_device_current(const std::string& name, uint64_t stamp);
    Device& device() const { return *dev_; }

private:
    Device* dev_;
    std::map<std::string, CachedWeight> cache_;
    SyncStats stats_;
};

/// Live values of a run plus exact byte accounting (reference runtime.hpp:92-121).
/// execute / train_step replay the plan's alloc/free events into a context at
/// its alignment, so high_water() equals the static planner's estimate
/// (schedule::plan_timeline / training_timeline); data() is the DEVICE address
/// of a live value. alloc() reserves device memory the context owns.
class ExecutionContext {
public:
    explicit ExecutionContext(int64_t alignment = 64) : alignment_(alignment) {}
    ~ExecutionContext();
    ExecutionContext(const ExecutionContext&) = delete;
    ExecutionContext& operator=(const ExecutionContext&) = delete;

    int64_t current_bytes() const { return current_; }
    int64_t high_water() const { return high_; }
    int64_t alignment() const { return alignment_; }
    /// Arena capacity; checked when >= 0 (ArenaOverflow).
    int64_t capacity = -1;

    bool live(const std::string& name) const { return buffers_.count(name) != 0; }
    uint8_t* data(const std::string& name);
    uint8_t* alloc(const std::string& name, int64_t bytes);
    /// Accounts for an externally owned buffer (device weight cache, arena).
    void adopt(const std::string& name, uint8_t* ptr, int64_t bytes);
    void release(const std::string& name);
    void release_all();

private:
    struct Buffer {
        uint8_t* ptr = nullptr;
        int64_t bytes = 0;
        bool owned = false;
    };
    std::map<std::string, Buffer> buffers_;
    int64_t alignment_;
    int64_t current_ = 0;
    int64_t high_ = 0;
};

/// Runs a plan on the B200 (reference runtime.hpp:126-130, same semantics):
/// inputs bind free vdims (a plan compiled with an enabled vdim accepts any
/// extent on that axis: it is re-specialised per binding, and the arena and
/// CUDA graph are cached per binding; explicit bindings win, conflicts and
/// fixed-axis mismatches throw ShapeMismatch); weights come from the model,
/// through `device`'s cache when given. Returns the materialized outputs.
std::map<std::string, Tensor> execute(const plan::ExecutionPlan& p,
                                      const std::map<std::string, Tensor>& inputs,
                                      const HostModel& model, OffloadDevice* device = nullptr,
                                      const ExecOptions& opts = {},
                                      ExecutionContext* shared_ctx = nullptr);

/// B200-native execute on an explicit Device (no offload accounting).
std::map<std::string, Tensor> execute_on(const plan::ExecutionPlan& p,
                                         const std::map<std::string, Tensor>& inputs,
                                         const HostModel& model, Device* device,
                                         const ExecOptions& opts = {});

/// A value of the last execute of `p` on `device` (parity debugging; the
/// program must be bound with ExecOptions::keep_values, i.e. no arena reuse).
Tensor last_run_value(const plan::ExecutionPlan& p, const std::string& name, Device* device = nullptr);

struct LaunchProfile {
    std::string label, kind;
    double ms = 0, bytes = 0, flops = 0;
};
/// One eager execute of `p` with CUDA events around every launch on the
/// compute stream: (label, kind, ms, algorithmic bytes, algorithmic flops).
std::vector<LaunchProfile> profile_run(const plan::ExecutionPlan& p, const std::map<std::string, Tensor>& inputs,
                                       const HostModel& model, Device* device = nullptr, const ExecOptions& opts = {});

/// The plan `p` specialised for the vdim binding these inputs (and explicit
/// bindings) imply -- `p` itself when they match its compiled extents.
const plan::ExecutionPlan& plan_for_inputs(const plan::ExecutionPlan& p,
                                           const std::map<std::string, Tensor>& inputs,
                                           const std::map<int32_t, int64_t>& bindings = {});
const plan::VersionPlans& plans_for_inputs(const plan::VersionPlans& plans,
                                           const std::map<std::string, Tensor>& inputs,
                                           const std::map<int32_t, int64_t>& bindings = {});

/// Pipelined execute from host buffers. execute_stage uploads the next run's
/// inputs into one of two device staging slots on the copy stream (the host
/// bytes are consumed on return); execute_launch_staged makes the compute
/// stream wait for the oldest staged slot, copies it into the plan's inputs
/// (device to device), runs the plan and starts the output downloads into
/// pinned buffers; execute_staged_outputs waits for them. Calling
/// execute_stage for run i + 1 between the launch and the collection of run i
/// overlaps its upload with run i. Outputs equal execute()'s.
void execute_stage(const plan::ExecutionPlan& p, const std::map<std::string, Tensor>& inputs,
                   Device* device = nullptr);
void execute_launch_staged(const plan::ExecutionPlan& p, const HostModel& model, Device* device = nullptr,
                           const ExecOptions& opts = {});
std::map<std::string, Tensor> execute_staged_outputs(const plan::ExecutionPlan& p, Device* device = nullptr);

/// Framework-side kernels (reference runtime.hpp:141-144), run on the device:
/// loss = sum|p - t|/N in double, grad = sign(p - t)/N; w <- (float)((double)w
/// - lr*(double)g) with the stamp bumped even at lr = 0 (F32 tensors).
L1Result l1_loss(const Tensor& pred, const Tensor& target);
void sgd_step(HostModel& model, const std::map<std::string, Tensor>& grads, double lr);
L1Result l1_loss_on(const Tensor& pred, const Tensor& target, Device* device);
/// Softmax cross-entropy (extension loss) with the same result layout: loss
/// = -(1/rows) sum t log softmax(pred) over the last axis, grad = (softmax - t)/rows.
L1Result softmax_ce_loss(const Tensor& pred, const Tensor& target, Device* device = nullptr);
void sgd_step_on(HostModel& model, const std::map<std::string, Tensor>& grads, double lr, Device* device);

/// One forward / loss / backward / update cycle (reference runtime.hpp:149-152):
/// the whole step runs as one CUDA graph on the device (runtime::Trainer);
/// afterwards `model.weights` holds the updated weights (stamps bumped), the
/// four trace phases are logged, a caller-owned context carries the shared
/// forward + backward byte accounting, and `device` (if given) counts the
/// weight / input / loss traffic of its cache protocol.
double train_step(const plan::VersionPlans& plans, const std::map<std::string, Tensor>& inputs,
                  const Tensor& target, HostModel& model, double lr, OffloadDevice* device = nullptr,
                  const ExecOptions& opts = {}, ExecutionContext* shared_ctx = nullptr);

/// B200-native training step on an explicit Device: weights stay
/// device-authoritative (HostModel::tensor pulls lazily).
double train_step_on(const plan::VersionPlans& plans, const std::map<std::string, Tensor>& inputs,
                     const Tensor& target, HostModel& model, double lr, Device* device,
                     const ExecOptions& opts = {});

/// Drops every device program / CUDA graph / trainer cached for these plans.
// Device memory of a bound program against the static planner: arena_bytes is
// the arena's address span (best-fit offsets), live_high_water the live-bytes
// high water of every buffer value replayed over the plan events, estimate
// plan::estimate_peak at the arena alignment (256 B). live == estimate is the
// reference's runtime high_water == estimate invariant (test_runtime.cpp:195-240).
struct MemoryReport {
    int64_t arena_bytes = 0, live_high_water = 0, estimate = 0;
};
MemoryReport memory_report(const plan::ExecutionPlan& inference_plan, Device* device = nullptr);

class Trainer;
void release(const plan::VersionPlans& plans);

// The Trainer that train_step / gradients use for (plans, model) on `device`,
// created on first use and kept until release(plans). Device-resident
// stepping (Trainer::step_device) through it shares the same arena and graph.
Trainer& shared_trainer(const plan::VersionPlans& plans, HostModel& model, Device& device, const ExecOptions& opts = {});

/// Forward + loss + backward without the update (for gradient parity tests).
std::map<std::string, Tensor> gradients(const plan::VersionPlans& plans,
                                        const std::map<std::string, Tensor>& inputs,
                                        const Tensor& target, HostModel& model, double* loss,
                                        Device* device = nullptr, const ExecOptions& opts = {});

/// Data-parallel layout of the flat parameter / gradient regions: trainable
/// weights in the order their gradients are produced by the backward plan
/// (so all-reduce buckets close early), then the remaining parameters; 256-byte
/// aligned. Buckets of ~bucket_elems cover the trainable prefix; close_launch
/// is the index (flattened exec_steps x launches order of train_bwd) of the
/// launch after which every gradient in the bucket has been written: its
/// all-reduce can start there, overlapping the rest of the backward pass.
struct DpBucket {
    int64_t offset = 0, count = 0, close_launch = -1;
    // the launch after which the bucket's weights may be updated: its
    // gradients are final AND no later backward launch reads its weights
    int64_t update_launch = -1;
};
struct DpLayout {
    std::vector<std::string> weights;              // region order
    std::map<std::string, int64_t> offset, elements, grad_launch;   // grad_launch: -1 for non-trainable
    std::map<std::string, int64_t> read_launch;    // last backward launch reading the weight (-1: none)
    int64_t region_elems = 0;
    int64_t bwd_launches = 0;
    std::vector<DpBucket> buckets;
};
DpLayout dp_layout(const plan::VersionPlans& plans, HostModel& model, int64_t bucket_elems = int64_t(8) << 20);

/// The backward half of a training step as the Trainer issues it (host-only,
/// so the exchange / update ordering is testable without a GPU): after
/// backward launch `after`, fork the comm stream off the compute stream,
/// all-reduce bucket `bucket` on it (only with a communicator) and apply the
/// bucket's SGD there once its gradients are final and no later backward
/// launch reads its weights; the compute stream joins the comm stream after
/// the last launch.
struct StepAction {
    enum Kind : int { Fork = 0, AllReduce = 1, Update = 2, Join = 3 };
    int64_t after = -1;   // backward launch index the action follows
    Kind kind = Fork;
    int64_t bucket = -1;
};
std::vector<StepAction> step_schedule(const DpLayout& layout, bool comm, bool do_sgd);

/// Device-resident training step for benchmarking: inputs/target already on the
/// device (pointers), everything stays on the device; returns nothing (the loss
/// is left in a device double readable with last_loss()).
struct Trainer {
    Trainer(const plan::VersionPlans& plans, HostModel& model, Device& device,
            const ExecOptions& opts = {});
    ~Trainer();
    /// H2D of host inputs+target, one graph replay, D2H of the loss.
    double step(const std::map<std::string, Tensor>& inputs, const Tensor& target, double lr);
    /// Device-resident variant (no host copies): enqueue one step.
    void step_device(double lr);
    double last_loss();
    /// Pipelined stepping from host buffers. stage() uploads the next step's
    /// inputs + target into one of two device staging slots on the copy
    /// stream (the host bytes are consumed on return); launch_staged() makes
    /// the compute stream wait for the oldest staged slot, copies it into the
    /// step's input values (device to device), replays the step and reads the
    /// loss back asynchronously; staged_loss() waits for that loss. Calling
    /// stage(i + 1) between launch_staged() and staged_loss() of step i
    /// overlaps the upload of step i + 1 with the compute of step i.
    void stage(const std::map<std::string, Tensor>& inputs, const Tensor& target);
    void launch_staged(double lr);
    double staged_loss();
    /// One eager step with CUDA events around every launch on the compute
    /// stream: (label, kind, ms, algorithmic bytes, algorithmic flops) per launch.
    struct LaunchTiming {
        std::string label, kind;
        double ms = 0, bytes = 0, flops = 0;
    };
    std::vector<LaunchTiming> profile_step(double lr);
    void* input_device_ptr(const std::string& name);
    /// Replays the step's alloc/free events into `ctx` (byte accounting of a
    /// caller-owned ExecutionContext; reference train_step's shared context).
    void account(ExecutionContext& ctx) const;
    /// Device bytes of any Buffer value of the bound step (meaningful for
    /// every value only when the trainer was built with keep_values).
    Tensor value(const std::string& name);
    void* target_device_ptr();
    size_t arena_bytes() const;
    uint64_t launches_per_step() const;
    MemoryReport memory_report() const;
    struct Impl;
    std::unique_ptr<Impl> impl;
};

}  // namespace nnc::runtime
