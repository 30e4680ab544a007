/* include/nnc_b200.h -- C-ABI of the B200 host library (libnnc_b200.so).
 *
 * The drop-in boundary for non-C++ callers (Python ctypes in this repo; cgo /
 * JNI / N-API stubs in INTEGRATION.md). Each entry point wraps the C++ API that
 * mirrors the reference (namespace nnc, include paths nnc/<module>.hpp):
 *
 *   nnc_model_compile     ingest::parse_model (ref ingest.cpp:411-500) ->
 *                         passes::optimize (ref passes.cpp:785-793) ->
 *                         autodiff::derive_versions (ref autodiff.cpp:89-319) ->
 *                         plan::compile_version_set (ref plan.cpp:441-457)
 *   nnc_model_run         runtime::execute (ref runtime.cpp:314-462)
 *   nnc_model_train_step  runtime::train_step (ref runtime.cpp:498-537)
 *   nnc_group_document    backends::group_layers (ref backends.cpp:321-400)
 *   nnc_model_tune        backends::tune_with_report (ref backends.cpp:73-176)
 *
 * Conventions: int status (0 = OK; otherwise 1 + nnc::Error::Code, or 100 for
 * other failures) with nnc_last_error(); tensors are float32, row-major NHWC;
 * no exceptions cross the ABI. A model is used by one host thread at a time.
 */
#ifndef NNC_B200_H
#define NNC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nnc_model nnc_model;

const char* nnc_last_error(void);
int         nnc_last_status(void);   /* status of the last failed call (for NULL-returning calls) */

/* Parse + optimize + derive versions + compile plans. gemm_precision:
 * 0 = tcgen05 tf32 (default), 1 = exact fp32 (bit-exact with the reference). */
nnc_model*  nnc_model_compile(const char* dlb_document, int gemm_precision);
/* As nnc_model_compile, with the listed free vdims (#k of the document's
 * dynamic input axes: "shape": null + "seed_shape") ENABLED
 * (passes::VdimBinding::enable): the model then accepts any extent on those
 * axes per call; plans are re-specialised and cached per binding.          */
nnc_model*  nnc_model_compile_ex(const char* dlb_document, int gemm_precision, const int32_t* enable_vdims,
                                 int n_enable);
void        nnc_model_free(nnc_model* m);
const char* nnc_model_describe(nnc_model* m);          /* JSON: plans, groups, launches, save set */

int nnc_model_set_weight(nnc_model* m, const char* name, const float* data, int64_t n);
int nnc_model_get_weight(nnc_model* m, const char* name, float* out, int64_t n);
int nnc_model_set_input(nnc_model* m, const char* name, const float* data, const int64_t* dims, int rank);
/* Like nnc_model_set_input but without a copy: `data` is borrowed and must stay
   valid and unchanged until the next run / gradients / train_step call returns. */
int nnc_model_set_input_borrowed(nnc_model* m, const char* name, const float* data, const int64_t* dims, int rank);

/* role: 0 = inference plan, 1 = train_fwd plan (outputs include the SaveSet). */
/* SOLP serialization of the compiled plans (ref plan.hpp:154-160: serialize_plan / load_plan), carrying
   the B200 launch descriptors. save: out == NULL queries *size. load replaces the model's plans. */
int nnc_model_save_plans(nnc_model* m, uint8_t* out, uint64_t capacity, uint64_t* size);
int nnc_model_load_plans(nnc_model* m, const uint8_t* bytes, uint64_t n);
int nnc_model_run(nnc_model* m, int role);
/* nnc_model_run copying back only the comma-separated outputs `names` (ExecOptions::materialize). */
int nnc_model_run_outputs(nnc_model* m, int role, const char* names);
/* Dims of a materialized output of the last run (rank <= 8).              */
int nnc_model_output_dims(nnc_model* m, const char* name, int64_t* dims, int* rank);
int nnc_model_output(nnc_model* m, const char* name, float* out, int64_t n);
/* Pipelined runs from host buffers: nnc_model_run_staged launches the oldest
 * staged run (names: comma-separated outputs, NULL or "" = all),
 * nnc_model_stage_run stages the current inputs of the next one (the upload
 * overlaps the launched run), nnc_model_staged_outputs waits for the launched
 * run and makes its outputs readable with nnc_model_output.                */
int nnc_model_stage_run(nnc_model* m, int role);
int nnc_model_run_staged(nnc_model* m, int role, const char* names);
int nnc_model_staged_outputs(nnc_model* m, int role);

int nnc_model_train_step(nnc_model* m, const float* target, int64_t n, double lr, double* loss);
/* Pipelined training from host buffers: stage the current inputs + target of
 * step i + 1 (host bytes are consumed on return; the upload runs on the copy
 * stream) while step i computes. Order per step: train_step_staged (launch the
 * oldest staged step), stage_step (the next one), staged_loss (wait for the
 * launched step's loss). Same result as nnc_model_train_step per step.     */
int nnc_model_stage_step(nnc_model* m, const float* target, int64_t n);
int nnc_model_train_step_staged(nnc_model* m, double lr);
int nnc_model_staged_loss(nnc_model* m, double* loss);
int nnc_model_gradients(nnc_model* m, const float* target, int64_t n, double* loss);
int nnc_model_grad(nnc_model* m, const char* weight, float* out, int64_t n);
/* Parity debugging: with keep_values on, the training step binds every value
 * to its own device bytes (no arena reuse), so after gradients() any forward
 * or backward value can be read back by name (nnc_model_trainer_value; out
 * NULL returns only dims/rank). Not for production: the arena grows to the
 * sum of all values. Values living in fused-group registers have no bytes.  */
int nnc_model_debug_keep_values(nnc_model* m, int on);
/* Training loss of the model's steps: 0 = L1 (the reference's), 1 = softmax
 * cross-entropy over the prediction's last axis (targets: probability rows). */
int nnc_model_set_loss(nnc_model* m, int kind);
int nnc_model_trainer_value(nnc_model* m, const char* name, float* out, int64_t n, int64_t* dims, int* rank);
/* The same for runs (nnc_model_run with keep_values on): a value of the last
 * run of a plan (0 inference, 1 train_fwd), for launch-by-launch parity of
 * inference plans.                                                        */
int nnc_model_run_value(nnc_model* m, int role, const char* name, float* out, int64_t n,
                        int64_t* dims, int* rank);

/* Data-parallel layout (runtime::dp_layout) as JSON: region order, ~bucket_bytes
 * all-reduce buckets and the backward launch after which each can start.
 * Host-only. Returns NULL on error. The string is valid until the next call. */
const char* nnc_model_dp_schedule(nnc_model* m, int64_t bucket_bytes);
/* The backward half of the training step as issued (runtime::step_schedule),
 * host-only, as JSON: {"actions": [{"after": k, "kind": fork|allreduce|update|
 * join, "bucket": b}], "launch_writes"/"launch_reads": per backward launch the
 * weights whose gradient it writes / whose value it reads, "buckets",
 * "weights", "region_elems", "bwd_launches"}. comm: with a communicator;
 * do_sgd: with the update. NULL on error; valid until the next call.        */
const char* nnc_model_step_schedule(nnc_model* m, int64_t bucket_bytes, int comm, int do_sgd);

/* Device-resident stepping for benchmarks: inputs/target stay on the device. */
int      nnc_model_trainer_prepare(nnc_model* m, const float* target, int64_t n);
int      nnc_model_trainer_step_device(nnc_model* m, double lr);
int      nnc_model_trainer_loss(nnc_model* m, double* loss);
uint64_t nnc_model_launches_per_step(nnc_model* m);
/* One eager step with CUDA events around each launch; JSON list of
 * {label, kind, ms, bytes, flops} (algorithmic bytes / flops per launch). */
/* One eager run of a plan (0 inference, 1 train_fwd) on the fed inputs with CUDA
 * events around every launch (runtime::profile_run), as JSON
 * [{label, kind, ms, bytes, flops}] (algorithmic bytes/flops). NULL on error. */
const char* nnc_model_profile_run(nnc_model* m, int role);
const char* nnc_model_profile_step(nnc_model* m, double lr);
/* Measured layer-wise tuning (backends::tune_with_report, ref backends.cpp:
 * 73-176) of the model's three role graphs before first execution: every
 * compute node timed in isolation on seed-shaped random inputs (median of
 * `trials` after `warmup`; GEMM nodes once per tensor-core tile candidate),
 * the chosen tiles attached to the plans (plan::attach_tuning, saved with
 * them in SOLP). injected_json (optional) {"node": {"b200_gemm"|"b200_fused":
 * cost}} skips the device (CostModel::injected_from). Returns the report as
 * JSON {role: {records, tiles, text}, attached_launches}; NULL on error.   */
const char* nnc_model_tune(nnc_model* m, int warmup, int trials, const char* injected_json);
uint64_t nnc_model_arena_bytes(nnc_model* m);
/* Device memory of a bound program (role 0 inference / 1 train_fwd after a run, 2 the trainer):
   arena address span, live-bytes high water and plan::estimate_peak at the same 256-byte alignment. */
int      nnc_model_memory(nnc_model* m, int role, uint64_t* arena, uint64_t* live_high, uint64_t* estimate);
int      nnc_model_infer_device(nnc_model* m);         /* replay inference, no host copies */
/* Replays plan `role` (0 inference, 1 train_fwd) with the inputs already on the device
   (from the last nnc_model_run of that role): no host<->device copies. */
int      nnc_model_run_device(nnc_model* m, int role);

/* NVRTC-compiles every generated fused-group kernel of the model's three plans
 * for sm_100a (no device needed). */
int nnc_model_check_kernels(nnc_model* m);

/* The device context (nncb_ctx*) for stream events / timing via nncb.h. */
/* Device transfer counters (runtime::OffloadDevice::sync_stats, ref runtime.hpp:50-75): weight_bytes
   counts each stamp-triggered weight upload at 64-byte alignment; reset zeroes them after reading. */
int nnc_device_sync_stats(int reset, uint64_t* h2d_bytes, uint64_t* d2h_bytes, uint64_t* weight_bytes);
void* nnc_device_ctx(void);

/* Data parallelism (one process per GPU). */
int nnc_comm_unique_id(uint8_t id[128]);
int nnc_init_comm(int nranks, int rank, const uint8_t id[128]);

/* Partition of the optimized inference graph of a document under the B200
 * default assignment (policy 0) or an explicit {"node": backend_int} JSON map
 * (assignment_json != NULL). Returns JSON [[members...], ...]. */
const char* nnc_group_document(const char* dlb_document, const char* assignment_json);
/* backends::group_layers with the B200 default assignment on one role graph
 * of the document's version set (0 inference, 1 train_fwd, 2 train_bwd), as
 * JSON [{"backend": int, "members": [...]}]. NULL on error.                */
const char* nnc_group_document_role(const char* doc, int role);

#ifdef __cplusplus
}
#endif
#endif /* NNC_B200_H */
