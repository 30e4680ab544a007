// runtime.cpp -- the B200 executor behind runtime::execute / train_step.
//
// Reference semantics kept (runtime.cpp:314-537): inputs bind by name and must
// match the plan's shapes (ShapeMismatch), parameters come from the HostModel
// through a version-stamped device cache (the OffloadDevice protocol,
// runtime.cpp:71-102: a weight crosses to the device only when its stamp is
// stale, counted in SyncStats), outputs are materialized by name (optionally a
// subset), train_step runs forward -> L1 loss -> backward -> SGD with the four
// trace phases (runtime.cpp:506-527).
//
// B200 design:
//  * Bind once per plan: every Buffer value gets an arena offset from a replay
//    of the plan's static alloc/free events (best-fit, 256-byte aligned), so
//    the whole plan runs out of ONE device allocation; kernels (generated
//    fused-group kernels, GEMM descriptors, pool geometry) are resolved to raw
//    pointers at bind time.
//  * Run: the launch list is captured once into a CUDA graph and replayed.
//  * Training: parameters live in one flat device region and weight gradients
//    in a second flat region with the same layout; backward GEMM/reduction
//    kernels write gradients straight into it, the data-parallel all-reduce
//    (NCCL) runs over it in buckets, and SGD is one kernel over the region.
//    Forward, loss, backward, all-reduce and update are one CUDA graph.
#include "nnc/runtime.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <set>
#include <list>
#include <mutex>
#include <unordered_map>

#include "nnc/geometry.hpp"

namespace nnc::runtime {

using plan::ExecutionPlan;
using plan::Launch;
using plan::LaunchKind;
using plan::MemCategory;
using plan::StorageClass;

namespace {

[[noreturn]] void device_fail(const std::string& what) {
    throw Error(Error::Code::DeviceError, what + ": " + nncb_last_error());
}
#define NNC_CHECK(expr)                                         \
    do {                                                        \
        if ((expr) != 0) device_fail(#expr);                    \
    } while (0)

constexpr int64_t kAlign = 256;

int64_t value_bytes(const ExecutionPlan& p, uint32_t s) {
    return static_cast<int64_t>(element_count(p.values[s].dims)) * static_cast<int64_t>(dtype_size(p.dtype));
}

/// Best-fit offset allocator over a static schedule (free blocks coalesce).
class OffsetPlanner {
public:
    int64_t alloc(int64_t bytes) {
        bytes = plan::align_bytes(std::max<int64_t>(bytes, 1), kAlign);
        auto best = free_.end();
        for (auto it = free_.begin(); it != free_.end(); ++it)
            if (it->second >= bytes && (best == free_.end() || it->second < best->second)) best = it;
        int64_t off;
        if (best != free_.end()) {
            off = best->first;
            int64_t rest = best->second - bytes;
            free_.erase(best);
            if (rest > 0) free_[off + bytes] = rest;
        } else {
            off = top_;
            top_ += bytes;
            high_ = std::max(high_, top_);
        }
        sizes_[off] = bytes;
        return off;
    }
    void release(int64_t off) {
        auto sz = sizes_.find(off);
        if (sz == sizes_.end()) return;
        auto it = free_.emplace(off, sz->second).first;
        sizes_.erase(sz);
        auto nx = std::next(it);
        if (nx != free_.end() && it->first + it->second == nx->first) {
            it->second += nx->second;
            free_.erase(nx);
        }
        if (it != free_.begin()) {
            auto pv = std::prev(it);
            if (pv->first + pv->second == it->first) {
                pv->second += it->second;
                free_.erase(it);
                it = pv;
            }
        }
        if (it->first + it->second == top_) {
            top_ = it->first;
            free_.erase(it);
        }
    }
    int64_t high() const { return high_; }
    void note() {}

private:
    std::map<int64_t, int64_t> free_;
    std::map<int64_t, int64_t> sizes_;
    int64_t top_ = 0, high_ = 0;
};

struct BoundLaunch {
    LaunchKind kind;
    bool bn_finalize = false;      // BnStats rewritten to read GEMM-epilogue column sums
    double* colstats = nullptr;
    std::vector<void*> ptrs;
    nncb_ew_kernel* ew = nullptr;
    int64_t n = 0, c = 0;
    nncb_gemm_desc gemm{};
    nncb_pool_geom pool{};
    int64_t d0 = 0, d1 = 0, d2 = 0, d3 = 0, d4 = 0, d5 = 0;
    double eps = 0;
    int flag0 = 0, flag1 = 0;
    bool skip = false;                      // work absorbed by another launch (fused reduction)
    // Gemm with NNCB_EPI_RELU_GRAD: the dy sums (2C doubles) -> the group's sum_g / sum_gx
    float* eg_sg = nullptr;
    float* eg_sgx = nullptr;
    std::vector<nncb_ew_instr> ew_prog;     // rewritten Ew program (empty: the plan's own)
    int ew_regs = 0;
    // weight gradient whose weights the training step updates in the same
    // call (nncb_gemm_desc::sgd_w, the update fused into the split-K fold)
    float* sgd_w = nullptr;
    // device bytes bound beyond the plan arguments by a fusion pass (folded
    // reductions' operands and results): what the launch additionally reads
    // or writes, for the producer / hazard checks of later passes
    struct Extra {
        const void* p;
        int64_t bytes;
        bool out;
    };
    std::vector<Extra> extra;
};

void enqueue(nncb_ctx* ctx, const BoundLaunch& b, const double* sgd_lr = nullptr, double sgd_scale = 1.0) {
    if (b.skip) return;
    auto P = [&](size_t i) { return static_cast<float*>(b.ptrs.at(i)); };
    switch (b.kind) {
        case LaunchKind::Ew: NNC_CHECK(nncb_ew_launch(ctx, b.ew, b.ptrs.data(), b.n, b.c)); break;
        case LaunchKind::Gemm:
            if (b.sgd_w && sgd_lr) {   // the training step's update of these weights, fused into the call
                nncb_gemm_desc d = b.gemm;
                d.sgd_w = b.sgd_w;
                d.sgd_lr = sgd_lr;
                d.sgd_scale = sgd_scale;
                NNC_CHECK(nncb_gemm(ctx, &d, P(0), P(1), b.flag0 ? P(2) : nullptr, P(b.ptrs.size() - 1)));
                break;
            }
            NNC_CHECK(nncb_gemm(ctx, &b.gemm, P(0), P(1), b.flag0 ? P(2) : nullptr, P(b.ptrs.size() - 1)));
            if (b.eg_sg)
                NNC_CHECK(nncb_colsums_to_float(ctx, b.gemm.eg_sums, b.eg_sg, b.eg_sgx,
                                                b.gemm.kind == NNCB_DENSE_DGRAD ? b.gemm.in_f : b.gemm.ci));
            break;
        case LaunchKind::MaxPool:
            NNC_CHECK(nncb_maxpool_fwd(ctx, &b.pool, P(0), P(1), b.ptrs.size() > 2 ? P(2) : nullptr));
            break;
        case LaunchKind::MaxPoolGrad: NNC_CHECK(nncb_maxpool_bwd(ctx, &b.pool, P(0), P(1), P(2))); break;
        case LaunchKind::AvgPool: NNC_CHECK(nncb_avgpool_fwd(ctx, b.d0, b.d1, b.d2, b.d3, b.d4, b.d5, P(0), P(1))); break;
        case LaunchKind::AvgPoolGrad:
            NNC_CHECK(nncb_avgpool_bwd(ctx, b.d0, b.d1, b.d2, b.d3, b.d4, b.d5, P(0), P(1)));
            break;
        case LaunchKind::SumRows: NNC_CHECK(nncb_sum_rows(ctx, P(0), P(1), b.d0, b.d1, b.flag0)); break;
        case LaunchKind::CumSum: NNC_CHECK(nncb_cumsum(ctx, P(0), P(1), b.d0, b.d1, b.d2, b.flag0, b.flag1)); break;
        case LaunchKind::BnStats:
            if (b.bn_finalize)
                NNC_CHECK(nncb_bn_finalize(ctx, b.colstats, P(1), b.d0, b.d1, b.eps));
            else
                NNC_CHECK(nncb_bn_stats(ctx, P(0), P(1), b.d0, b.d1, b.eps));
            break;
        case LaunchKind::BnGradReduce:
            NNC_CHECK(nncb_bn_grad_reduce(ctx, P(0), P(1), P(2), P(3), P(4), b.d0, b.d1));
            break;
        case LaunchKind::LnFwd: NNC_CHECK(nncb_layernorm_fwd(ctx, P(0), P(1), P(2), P(3), b.d0, b.d1, b.eps)); break;
        case LaunchKind::LnBwd:
            if (b.ptrs.size() >= 6)   // parameter gradients folded in (fuse_ln_param_grads)
                NNC_CHECK(nncb_layernorm_bwd_params(ctx, P(0), P(1), P(2), P(3), P(4), P(5), b.d0, b.d1, b.eps));
            else
                NNC_CHECK(nncb_layernorm_bwd(ctx, P(0), P(1), P(2), P(3), b.d0, b.d1, b.eps));
            break;
        case LaunchKind::LnDgamma: NNC_CHECK(nncb_layernorm_dgamma(ctx, P(0), P(1), P(2), b.d0, b.d1, b.eps)); break;
    }
}

// Algorithmic (minimum) HBM bytes and flops of one launch: every operand read
// once and every result written once; GEMMs count 2*M*N*K flops.
void launch_cost(const BoundLaunch& b, const Launch& L, const ExecutionPlan& p, double& bytes, double& flops) {
    bytes = flops = 0;
    auto elems = [&](size_t arg) { return static_cast<double>(element_count(p.values[L.args[arg].slot].dims)); };
    switch (b.kind) {
        case LaunchKind::Ew: {
            // element loads / stores move n floats; per-channel operands C
            // floats; a folded BatchNorm backward reduction writes 2C floats
            const double n = static_cast<double>(b.n);
            const double c = static_cast<double>(std::max<int64_t>(b.c, 1));
            for (const auto& in : b.ew_prog.empty() ? L.ew : b.ew_prog) {
                if (in.op == NNCB_EW_LOAD || in.op == NNCB_EW_STORE) bytes += 4.0 * n;
                if (in.op == NNCB_EW_LOAD_CH) bytes += 4.0 * c;
                if (in.op == NNCB_EW_REDUCE_BN_GRAD || in.op == NNCB_EW_REDUCE_STATS) bytes += 8.0 * c;
                if (in.op == NNCB_EW_REDUCE_SUM) bytes += 4.0 * c;
            }
            break;
        }
        case LaunchKind::BnStats:
            if (b.bn_finalize) {   // reads the GEMM epilogue's 2C double sums, writes 2C floats
                bytes = 16.0 * b.d1 + 8.0 * b.d1;
                break;
            }
            bytes = 4.0 * elems(0) + 8.0 * b.d1;
            break;
        case LaunchKind::BnGradReduce:   // reads x, g (rows*C) and the 2C stats; writes 2C sums
            bytes = 8.0 * elems(0) + 16.0 * b.d1;
            break;
        case LaunchKind::LnBwd:   // x, gamma, g read, gx written; folded dgamma / dbeta written
            for (size_t a = 0; a < L.args.size(); ++a) bytes += 4.0 * elems(a);
            for (size_t a = L.args.size(); a < b.ptrs.size(); ++a)
                if (b.ptrs[a]) bytes += 4.0 * b.d1;
            break;
        case LaunchKind::Gemm: {
            const nncb_gemm_desc& d = b.gemm;
            double M, N, K;
            switch (d.kind) {
                case NNCB_DENSE_FWD: M = d.batch; N = d.out_f; K = d.in_f; break;
                case NNCB_DENSE_DGRAD: M = d.batch; N = d.in_f; K = d.out_f; break;
                case NNCB_DENSE_WGRAD: M = d.in_f; N = d.out_f; K = d.batch; break;
                // all three contractions of a convolution perform the forward's
                // 2*N*OH*OW*CO*KH*KW*CI useful flops (strided dgrad skips zeros)
                default: M = double(d.n) * d.oh * d.ow; N = d.co; K = double(d.kh) * d.kw * d.ci; break;
            }
            flops = 2.0 * M * N * K;
            for (size_t a = 0; a < L.args.size(); ++a) bytes += 4.0 * elems(a);
            break;
        }
        default:
            for (size_t a = 0; a < L.args.size(); ++a) bytes += 4.0 * elems(a);
            break;
    }
}

}  // namespace

/* ------------------------------------------------------------------ */
/*  Program: one or more plans bound to device memory                  */
/* ------------------------------------------------------------------ */

struct Program {
    Device* dev = nullptr;
    std::vector<const ExecutionPlan*> plans;
    void* arena = nullptr;
    int64_t arena_bytes = 0;
    // live bytes (every Buffer value, wherever it is stored: arena, weight
    // cache, gradient region) replayed over the plan events at kAlign: the
    // high water equals plan::estimate_peak at the same alignment
    int64_t live_high = 0;
    void* side = nullptr;          // fused BatchNorm column-sum accumulators
    void* side_eg = nullptr;       // dgrad-epilogue BatchNorm backward sums
    // K-major copies of the forward conv weights, refreshed by one batched
    // transpose at the head of each plan (nncb_transpose_batch)
    void* wt_region = nullptr;
    struct KmajorSet {
        void* jobs = nullptr;      // device nncb_transpose_job[n]
        int n = 0;
        int64_t tiles = 0;
    };
    std::vector<KmajorSet> kmajor;   // per plan
    std::unordered_map<std::string, void*> where;   // value name -> device pointer
    std::vector<std::vector<BoundLaunch>> steps;     // per plan, flattened launches
    std::vector<std::vector<const Launch*>> sources; // per plan, the plan launch of each bound launch
    std::vector<std::vector<std::pair<size_t, std::string>>> step_labels;  // per plan: (launch idx, label)
    int precision = NNCB_PREC_TF32;

    ~Program() {
        if (arena) nncb_free(dev->ctx(), arena);
        if (side) nncb_free(dev->ctx(), side);
        if (side_eg) nncb_free(dev->ctx(), side_eg);
        if (wt_region) nncb_free(dev->ctx(), wt_region);
        for (const KmajorSet& k : kmajor)
            if (k.jobs) nncb_free(dev->ctx(), k.jobs);
    }

    /// tf32 forward convolutions on the implicit-GEMM path read K-major
    /// weights: instead of each GEMM transposing its weights per call, the
    /// copies live in one region and a single launch at the head of the plan
    /// refreshes them all (after the previous step's SGD in training).
    void prepare_kmajor_weights() {
        kmajor.assign(steps.size(), KmajorSet{});
        std::vector<std::vector<std::pair<size_t, nncb_transpose_job>>> jobs(steps.size());
        int64_t elems = 0;
        for (size_t pi = 0; pi < steps.size(); ++pi)
            for (size_t k = 0; k < steps[pi].size(); ++k) {
                const BoundLaunch& b = steps[pi][k];
                if (b.kind != LaunchKind::Gemm || b.skip || b.gemm.kind != NNCB_CONV_FWD) continue;
                const int64_t K = b.gemm.kh * b.gemm.kw * b.gemm.ci, co = b.gemm.co;
                if (b.gemm.ci % 32 != 0 || K % 4 != 0 || K >= (int64_t(1) << 31) || co >= (int64_t(1) << 31)) continue;
                nncb_transpose_job j{};
                j.src = static_cast<const float*>(b.ptrs[1]);
                j.rows = static_cast<int32_t>(K);
                j.cols = static_cast<int32_t>(co);
                j.tile0 = elems;   // element offset for now
                jobs[pi].push_back({k, j});
                elems += (K * co + 63) / 64 * 64;
            }
        if (elems == 0) return;
        NNC_CHECK(nncb_malloc(dev->ctx(), static_cast<size_t>(elems) * sizeof(float), &wt_region));
        for (size_t pi = 0; pi < steps.size(); ++pi) {
            if (jobs[pi].empty()) continue;
            std::vector<nncb_transpose_job> table;
            int64_t tiles = 0;
            for (auto& [k, j] : jobs[pi]) {
                j.dst = static_cast<float*>(wt_region) + j.tile0;
                j.tile0 = tiles;
                tiles += static_cast<int64_t>((j.rows + 31) / 32) * ((j.cols + 31) / 32);
                steps[pi][k].gemm.b_kmajor = j.dst;
                table.push_back(j);
            }
            KmajorSet& s = kmajor[pi];
            s.n = static_cast<int>(table.size());
            s.tiles = tiles;
            NNC_CHECK(nncb_malloc(dev->ctx(), table.size() * sizeof(nncb_transpose_job), &s.jobs));
            NNC_CHECK(nncb_h2d(dev->ctx(), s.jobs, table.data(), table.size() * sizeof(nncb_transpose_job)));
        }
        NNC_CHECK(nncb_sync(dev->ctx()));
    }

    /// Work every plan execution starts with: the K-major weight refresh.
    void plan_prologue(size_t pi) const {
        if (pi < kmajor.size() && kmajor[pi].n)
            NNC_CHECK(nncb_transpose_batch(dev->ctx(), static_cast<const nncb_transpose_job*>(kmajor[pi].jobs),
                                           kmajor[pi].n, kmajor[pi].tiles));
    }

    void* ptr(const std::string& name) const {
        auto it = where.find(name);
        if (it == where.end()) throw Error(Error::Code::ShapeMismatch, "no device buffer for " + name);
        return it->second;
    }

    /// `param_ptr(name)` supplies Parameter buffers; `fixed(name)` may pin other
    /// values (flat gradient region) -- return nullptr to arena-allocate.
    bool keep_values = false;   // no arena reuse (parity debugging)

    void bind(const std::function<void*(const std::string&)>& param_ptr,
              const std::function<void*(const std::string&)>& fixed) {
        OffsetPlanner pl;
        std::unordered_map<std::string, int64_t> offset;
        std::unordered_map<std::string, bool> live;
        std::unordered_map<std::string, int64_t> live_bytes;
        int64_t live_cur = 0;
        for (const ExecutionPlan* p : plans)
            for (const plan::PlanEvent& ev : p->events) {
                const plan::ValueEntry& v = p->values[ev.slot];
                if (v.storage != StorageClass::Buffer) continue;
                if (ev.alloc && !live_bytes.count(v.name)) {
                    const int64_t b = plan::align_bytes(value_bytes(*p, ev.slot), kAlign);
                    live_bytes[v.name] = b;
                    live_cur += b;
                    live_high = std::max(live_high, live_cur);
                } else if (!ev.alloc) {
                    auto lb = live_bytes.find(v.name);
                    if (lb != live_bytes.end()) {
                        live_cur -= lb->second;
                        live_bytes.erase(lb);
                    }
                }
                if (v.category == MemCategory::Parameter) {
                    if (!where.count(v.name)) where[v.name] = param_ptr(v.source_weight);
                    continue;
                }
                if (ev.alloc) {
                    if (live[v.name] || where.count(v.name)) continue;
                    if (void* f = fixed(v.name)) {
                        where[v.name] = f;
                        continue;
                    }
                    offset[v.name] = pl.alloc(value_bytes(*p, ev.slot));
                    live[v.name] = true;
                    pl.note();
                } else {
                    auto it = offset.find(v.name);
                    if (it != offset.end() && live[v.name] && !keep_values) {
                        pl.release(it->second);
                        live[v.name] = false;
                    }
                }
            }
        arena_bytes = std::max<int64_t>(pl.high(), kAlign);
        NNC_CHECK(nncb_malloc(dev->ctx(), static_cast<size_t>(arena_bytes), &arena));
        for (auto& [name, off] : offset) where[name] = static_cast<char*>(arena) + off;
        // every referenced Buffer value must have storage (values produced but
        // never in an alloc event, e.g. scratch, get arena space too)
        for (const ExecutionPlan* p : plans)
            for (const auto& v : p->values)
                if (v.storage == StorageClass::Buffer && !where.count(v.name))
                    throw Error(Error::Code::ArenaOverflow, "value " + v.name + " has no schedule entry");
        // resolve launches
        for (const ExecutionPlan* p : plans) {
            steps.emplace_back();
            step_labels.emplace_back();
            sources.emplace_back();
            for (const plan::ExecStep& es : p->exec_steps) {
                step_labels.back().push_back({steps.back().size(), es.label});
                for (uint32_t li : es.launches) {
                    steps.back().push_back(resolve(*p, p->groups[es.group].launches[li]));
                    sources.back().push_back(&p->groups[es.group].launches[li]);
                }
            }
        }
        if (precision != NNCB_PREC_FP32) {   // tensor-core modes (tf32, bf16)
            fuse_bn_statistics();
            fuse_bn_grad_reduce();
            fuse_relu_grad_epilogue();
            fuse_bn_infer_epilogue();
            fuse_ln_param_grads();
            fuse_bias_grad_reduce();
            // (the 3xTF32 route builds its own split weight copies)
            if (!std::getenv("NNC_NO_KMAJOR_BATCH") && precision != NNCB_PREC_TF32X3) prepare_kmajor_weights();
        }
        hint_unchanged_activations();
    }

    /// A weight gradient whose activation is a value an earlier forward conv
    /// of the same step already read (values are written once per step, so
    /// its bytes are unchanged) may reuse that call's lowered copy of it
    /// (NNCB_EPI_A_UNCHANGED; the space-to-depth input of the stem).
    void hint_unchanged_activations() {
        std::set<std::string> fwd_inputs;
        for (size_t pi = 0; pi < steps.size(); ++pi)
            for (size_t k = 0; k < steps[pi].size(); ++k) {
                BoundLaunch& b = steps[pi][k];
                const Launch& L = *sources[pi][k];
                if (b.kind != LaunchKind::Gemm || b.skip || L.args.empty()) continue;
                const std::string& an = plans[pi]->values[L.args[0].slot].name;
                if (b.gemm.kind == NNCB_CONV_FWD)
                    fwd_inputs.insert(an);
                else if (b.gemm.kind == NNCB_CONV_WGRAD && fwd_inputs.count(an))
                    b.gemm.epilogue |= NNCB_EPI_A_UNCHANGED;
            }
    }

    /// Device byte ranges a bound launch reads or writes. Arena offsets are
    /// shared between values with disjoint lifetimes, so producer/consumer
    /// matching must go by byte overlap, never by pointer identity alone.
    struct Range {
        const char* p;
        int64_t n;
        bool overlaps(const char* q, int64_t m) const { return p < q + m && q < p + n; }
    };
    std::vector<Range> launch_ranges(size_t pi, size_t k, bool outputs) const {
        std::vector<Range> r;
        const BoundLaunch& b = steps[pi][k];
        if (b.skip) return r;   // its work (if any) runs inside the absorbing launch
        const Launch& L = *sources[pi][k];
        const ExecutionPlan& p = *plans[pi];
        for (size_t a = 0; a < L.args.size() && a < b.ptrs.size(); ++a) {
            const bool out = a < L.is_out.size() && L.is_out[a];
            if (out != outputs) continue;
            const int64_t bytes = (element_count(p.values[L.args[a].slot].dims) - L.args[a].offset) *
                                  static_cast<int64_t>(dtype_size(p.dtype));
            r.push_back({static_cast<const char*>(b.ptrs[a]), std::max<int64_t>(bytes, 1)});
        }
        // operands bound beyond the plan arguments
        for (const BoundLaunch::Extra& e : b.extra)
            if (e.out == outputs && e.p) r.push_back({static_cast<const char*>(e.p), std::max<int64_t>(e.bytes, 1)});
        if (b.kind == LaunchKind::Gemm && b.eg_sg) {
            const int64_t C = (b.gemm.kind == NNCB_DENSE_DGRAD ? b.gemm.in_f : b.gemm.ci) * 4;
            if (outputs) {
                r.push_back({reinterpret_cast<const char*>(b.eg_sg), C});
                r.push_back({reinterpret_cast<const char*>(b.eg_sgx), C});
            }
        }
        return r;
    }
    /// Whether a launch of plan `pi` writes any byte of [q, q+m) (fusion passes
    /// may redirect or absorb a value's producer: a plan value whose producer
    /// was folded away is never written).
    bool written_by_plan(size_t pi, const char* q, int64_t m) const {
        for (size_t k = 0; k < steps[pi].size(); ++k)
            if (launch_touches(pi, k, q, m, true)) return true;
        return false;
    }
    bool launch_touches(size_t pi, size_t k, const char* q, int64_t m, bool outputs) const {
        for (const Range& r : launch_ranges(pi, k, outputs))
            if (r.overlaps(q, m)) return true;
        return false;
    }
    int64_t arg_bytes(size_t pi, size_t k, size_t a) const {
        const Launch& L = *sources[pi][k];
        const ExecutionPlan& p = *plans[pi];
        return (element_count(p.values[L.args[a].slot].dims) - L.args[a].offset) *
               static_cast<int64_t>(dtype_size(p.dtype));
    }
    /// The nearest launch before `j` that writes any byte of [q, q+m), or -1.
    int64_t last_writer(size_t pi, size_t j, const char* q, int64_t m) const {
        for (size_t i = j; i-- > 0;)
            if (launch_touches(pi, i, q, m, true)) return static_cast<int64_t>(i);
        return -1;
    }

    /// The BatchNorm backward reduction (sum g, sum g*xhat per channel) of a
    /// gradient g that the immediately preceding fused elementwise group
    /// stores is folded into that group (NNCB_EW_REDUCE_BN_GRAD): g is reduced
    /// from registers as it is written instead of being read back by a
    /// separate pass. Applies when the group can run channel-stationary.
    /// A fused group that only turns a dgrad's output g into the gradient at
    /// the input of the following ReLU, dy = relu_grad(mask, g [+ residual]),
    /// and reduces dy for BatchNorm (REDUCE_BN_GRAD), moves into that dgrad's
    /// epilogue (NNCB_EPI_RELU_GRAD): g is never written or read back. The
    /// group's program is checked symbolically, and g must have no other reader.
    void fuse_relu_grad_epilogue() {
        // opt-in: the fused epilogue is correct but measured slower than the
        // separate pass (relu-grad epilogue)
        if (!std::getenv("NNC_RELU_GRAD_EPILOGUE")) return;
        const bool debug = std::getenv("NNC_EG_DEBUG") != nullptr;
        struct Fused { BoundLaunch* g; int64_t C; };
        std::vector<Fused> fused;
        for (size_t pi = 0; pi < steps.size(); ++pi)
            for (size_t j = 1; j < steps[pi].size(); ++j) {
                BoundLaunch& e = steps[pi][j];
                if (e.kind != LaunchKind::Ew || e.skip) continue;
                // the dgrad producing a value this group loads (the layer's wgrad
                // usually sits in between)
                size_t gi = j;
                for (size_t i = j; i-- > 0 && j - i <= 6;) {
                    const BoundLaunch& c = steps[pi][i];
                    if (c.kind != LaunchKind::Gemm || c.skip || c.eg_sg) continue;
                    if (c.gemm.kind != NNCB_CONV_DGRAD) continue;   // the epilogue exists in the conv path
                    // strided dgrads store sub-pixel phases directly: no TMA side
                    // tiles, and the per-row side loads measured 2-6x slower
                    if (c.gemm.sh != 1 || c.gemm.sw != 1) continue;
                    if (std::find(e.ptrs.begin(), e.ptrs.end(), c.ptrs.back()) != e.ptrs.end()) {
                        gi = i;
                        break;
                    }
                }
                if (gi == j) {
                    if (debug && sources[pi][j]->label.find("relu") != std::string::npos)
                        std::fprintf(stderr, "relu_grad_epilogue: %s: no dgrad producer\n", sources[pi][j]->label.c_str());
                    continue;
                }
                BoundLaunch& g = steps[pi][gi];
                void* gout = g.ptrs.back();
                const std::vector<nncb_ew_instr>& prog = e.ew_prog.empty() ? sources[pi][j]->ew : e.ew_prog;
                // symbolic registers: kind 0 unknown, 1 LOAD(ptr), 2 LOAD_CH(ptr), 3 g (+res) sum, 4 dy
                struct Sym { int kind = 0; void* ptr = nullptr; void* res = nullptr; void* mask = nullptr; };
                std::map<int, Sym> r;
                void *dy = nullptr, *x = nullptr, *mean = nullptr, *inv = nullptr, *sg = nullptr, *sgx = nullptr,
                     *res = nullptr, *mask = nullptr;
                int stores = 0, reduces = 0;
                bool ok = true;
                for (const nncb_ew_instr& in : prog) {
                    switch (in.op) {
                        case NNCB_EW_LOAD: r[in.dst] = {1, e.ptrs[in.slot]}; break;
                        case NNCB_EW_LOAD_CH: r[in.dst] = {2, e.ptrs[in.slot]}; break;
                        case NNCB_EW_ADD: {
                            const Sym &a = r[in.a], &b = r[in.b];
                            if (a.kind == 1 && b.kind == 1 && (a.ptr == gout) != (b.ptr == gout))
                                r[in.dst] = {3, gout, a.ptr == gout ? b.ptr : a.ptr};
                            else
                                ok = false;
                            break;
                        }
                        case NNCB_EW_RELU_GRAD: {   // relu_grad(x = mask, g)
                            const Sym &m = r[in.a], &gg = r[in.b];
                            const bool plain = gg.kind == 1 && gg.ptr == gout;
                            if (m.kind == 1 && m.ptr != gout && (plain || gg.kind == 3)) {
                                Sym d;
                                d.kind = 4;
                                d.res = plain ? nullptr : gg.res;
                                d.mask = m.ptr;
                                r[in.dst] = d;
                            } else {
                                ok = false;
                            }
                            break;
                        }
                        case NNCB_EW_STORE:
                            ++stores;
                            if (r[in.a].kind != 4) ok = false;
                            dy = e.ptrs[in.slot];
                            res = r[in.a].res;
                            mask = r[in.a].mask;
                            break;
                        case NNCB_EW_REDUCE_BN_GRAD: {
                            ++reduces;
                            const Sym &a = r[in.a], &b = r[in.b], &c = r[in.c], &dd = r[in.d];
                            if (a.kind != 4 || b.kind != 1 || c.kind != 2 || dd.kind != 2) ok = false;
                            x = b.ptr;
                            mean = c.ptr;
                            inv = dd.ptr;
                            sg = e.ptrs[in.slot];
                            sgx = e.ptrs[in.e];
                            break;
                        }
                        default: ok = false; break;
                    }
                    if (!ok) break;
                }
                const int64_t C = g.gemm.ci;
                if (!ok || stores != 1 || reduces != 1 || !dy || dy == gout ||
                    static_cast<float*>(inv) != static_cast<float*>(mean) + C) {
                    if (debug)
                        std::fprintf(stderr, "relu_grad_epilogue: %s: program (ok %d stores %d reduces %d)\n",
                                     sources[pi][j]->label.c_str(), ok, stores, reduces);
                    continue;
                }
                // g (a value of this plan; arena addresses are shared between
                // values with disjoint lifetimes) must have no other reader
                const Launch& gl = *sources[pi][gi];
                bool other = gl.args.empty() || !gl.is_out.back();
                const uint32_t gslot = other ? 0 : gl.args.back().slot;
                for (uint32_t o : plans[pi]->output_slots) other = other || o == gslot;
                for (size_t k = 0; k < sources[pi].size() && !other; ++k) {
                    if (k == j || k == gi) continue;
                    const Launch& L = *sources[pi][k];
                    for (size_t a = 0; a < L.args.size(); ++a)
                        other = other || (L.args[a].slot == gslot && !(a < L.is_out.size() && L.is_out[a]));
                }
                // values are shared between the bound plans by name
                const std::string& gname = plans[pi]->values[gslot].name;
                for (size_t pk = 0; pk < plans.size() && !other; ++pk)
                    if (pk != pi && plans[pk]->find_value(gname) >= 0) other = true;
                if (other) {
                    if (debug) std::fprintf(stderr, "relu_grad_epilogue: %s: g has another reader\n", sources[pi][j]->label.c_str());
                    continue;
                }
                // dy is now written at the dgrad, before the launches in between
                // (the layer's wgrad): none of them may touch dy's arena bytes
                // (the planner may share them with a value that dies there), and
                // none may write a side input the epilogue reads
                {
                    auto overlaps = [](const char* a0, int64_t an, const char* b0, int64_t bn) {
                        return a0 < b0 + bn && b0 < a0 + an;
                    };
                    const int64_t B = e.n * static_cast<int64_t>(sizeof(float));
                    const char* dyc = static_cast<const char*>(dy);
                    const char* side_in[4] = {static_cast<const char*>(mask), static_cast<const char*>(x),
                                              static_cast<const char*>(res), static_cast<const char*>(mean)};
                    const int64_t side_n[4] = {B, B, B, 2 * C * static_cast<int64_t>(sizeof(float))};
                    bool clash = false;
                    for (size_t k = gi; k < j && !clash; ++k) {   // k == gi: the dgrad's own inputs
                        const Launch& L = *sources[pi][k];
                        for (size_t a = 0; a < L.args.size() && !clash; ++a) {
                            if (k == gi && a < L.is_out.size() && L.is_out[a]) continue;
                            const plan::ValueEntry& v = plans[pi]->values[L.args[a].slot];
                            const char* b0 = static_cast<const char*>(ptr(v.name));
                            const int64_t bn = element_count(v.dims) * static_cast<int64_t>(sizeof(float));
                            clash = overlaps(b0, bn, dyc, B);
                            if (a < L.is_out.size() && L.is_out[a])
                                for (int q = 0; q < 4 && !clash; ++q)
                                    clash = side_in[q] && overlaps(b0, bn, side_in[q], side_n[q]);
                        }
                        // pointers bound beyond the plan arguments (a folded reduction's sums)
                        for (size_t a = L.args.size(); a < steps[pi][k].ptrs.size() && !clash; ++a)
                            clash = overlaps(static_cast<const char*>(steps[pi][k].ptrs[a]), 1, dyc, B);
                    }
                    if (clash) {
                        if (debug)
                            std::fprintf(stderr, "relu_grad_epilogue: %s: dy / side inputs alias a value live in between\n",
                                         sources[pi][j]->label.c_str());
                        continue;
                    }
                }
                if (debug) std::fprintf(stderr, "relu_grad_epilogue: %s: fused\n", sources[pi][j]->label.c_str());
                g.gemm.epilogue |= NNCB_EPI_RELU_GRAD;
                g.gemm.eg_mask = static_cast<const float*>(mask);
                g.gemm.eg_res = static_cast<const float*>(res);
                g.gemm.eg_x = static_cast<const float*>(x);
                g.gemm.eg_stats = static_cast<const float*>(mean);
                g.ptrs.back() = dy;
                g.eg_sg = static_cast<float*>(sg);
                g.eg_sgx = static_cast<float*>(sgx);
                e.skip = true;
                fused.push_back({&g, C});
            }
        if (fused.empty()) return;
        int64_t doubles = 0;
        for (const Fused& f : fused) doubles += 2 * f.C;
        NNC_CHECK(nncb_malloc(dev->ctx(), static_cast<size_t>(doubles) * sizeof(double), &side_eg));
        int64_t off = 0;
        for (const Fused& f : fused) {
            f.g->gemm.eg_sums = static_cast<double*>(side_eg) + off;
            off += 2 * f.C;
        }
    }

    /// An inference BatchNorm (+ ReLU) group that only transforms a forward
    /// GEMM's output y -- program exactly LOAD y, 4 x LOAD_CH, BN_INFER,
    /// [RELU], STORE z -- moves into that GEMM's epilogue (NNCB_EPI_BN_AFFINE
    /// [| NNCB_EPI_RELU], the same fp32 operation sequence): the GEMM writes z
    /// and the pass over y disappears. y must have no other reader, and no
    /// launch between the two may touch z's bytes (z is now written earlier).
    void fuse_bn_infer_epilogue() {
        if (std::getenv("NNC_NO_BN_INFER_EPILOGUE")) return;
        const bool debug = std::getenv("NNC_BN_INFER_DEBUG") != nullptr;
        auto why = [&](const Launch& L, const char* r) {
            if (debug) std::fprintf(stderr, "bn_infer_epilogue: %s: %s\n", L.label.c_str(), r);
        };
        for (size_t pi = 0; pi < steps.size(); ++pi)
            for (size_t j = 1; j < steps[pi].size(); ++j) {
                BoundLaunch& e = steps[pi][j];
                if (e.kind != LaunchKind::Ew || e.skip || !e.ew_prog.empty()) continue;
                const Launch& L = *sources[pi][j];
                // program: LOAD y, 4 x LOAD_CH, BN_INFER(y) [, LOAD r, ADD(bn, r)] [, RELU], STORE z
                int n_ch = 0, n_bn = 0, n_relu = 0, n_store = 0, n_add = 0, other = 0;
                int z_slot = -1, bn_reg = -1, relu_reg = -1, store_reg = -1, add_reg = -1;
                std::map<int, int> load_slot, ch_slot;   // register -> slot of a LOAD / LOAD_CH
                nncb_ew_instr bn{}, add{};
                for (const nncb_ew_instr& in : L.ew) {
                    switch (in.op) {
                        case NNCB_EW_LOAD: load_slot[in.dst] = in.slot; break;
                        case NNCB_EW_LOAD_CH: ++n_ch; ch_slot[in.dst] = in.slot; break;
                        case NNCB_EW_BN_INFER: ++n_bn; bn = in; bn_reg = in.dst; break;
                        case NNCB_EW_ADD: ++n_add; add = in; add_reg = in.dst; break;
                        case NNCB_EW_RELU: ++n_relu; relu_reg = in.dst; if (in.a != (n_add ? add_reg : bn_reg)) ++other; break;
                        case NNCB_EW_STORE: ++n_store; z_slot = in.slot; store_reg = in.a; break;
                        default: ++other; break;
                    }
                }
                if (other || n_ch != 4 || n_bn != 1 || n_add > 1 || n_relu > 1 || n_store != 1 ||
                    load_slot.size() != static_cast<size_t>(1 + n_add)) {
                    if (n_bn) why(L, "program shape");
                    continue;
                }
                if (!load_slot.count(bn.a) || !ch_slot.count(bn.b) || !ch_slot.count(bn.c) || !ch_slot.count(bn.d) ||
                    !ch_slot.count(bn.e)) {
                    why(L, "operands");
                    continue;
                }
                const int y_slot = load_slot[bn.a];
                int r_slot = -1;
                if (n_add) {   // ADD(bn, r) in either order, r an element load
                    const int other_reg = add.a == bn_reg ? add.b : add.b == bn_reg ? add.a : -1;
                    if (other_reg < 0 || !load_slot.count(other_reg) || other_reg == bn.a) { why(L, "add operands"); continue; }
                    r_slot = load_slot[other_reg];
                }
                if (store_reg != (n_relu ? relu_reg : n_add ? add_reg : bn_reg)) { why(L, "store"); continue; }
                const char* y = static_cast<const char*>(e.ptrs[y_slot]);
                const int64_t ybytes = arg_bytes(pi, j, static_cast<size_t>(y_slot));
                const int64_t w = last_writer(pi, j, y, ybytes);
                if (w < 0) { why(L, "no producer"); continue; }
                BoundLaunch& g = steps[pi][static_cast<size_t>(w)];
                if (g.kind != LaunchKind::Gemm || g.skip || g.ptrs.back() != e.ptrs[y_slot]) { why(L, "producer not a GEMM"); continue; }
                if (g.gemm.kind != NNCB_CONV_FWD && g.gemm.kind != NNCB_DENSE_FWD) { why(L, "not forward"); continue; }
                if (g.gemm.epilogue & (NNCB_EPI_COLSTATS | NNCB_EPI_RELU_GRAD | NNCB_EPI_BN_AFFINE)) { why(L, "epilogue taken"); continue; }
                // y has no other reader in any bound plan, and is not an output
                const std::string& yname = plans[pi]->values[L.args[y_slot].slot].name;
                bool busy = false;
                for (size_t pk = 0; pk < plans.size() && !busy; ++pk) {
                    const ExecutionPlan& pp = *plans[pk];
                    for (uint32_t o : pp.output_slots) busy = busy || pp.values[o].name == yname;
                    for (size_t k = 0; k < sources[pk].size() && !busy; ++k) {
                        if (pk == pi && (k == j || k == static_cast<size_t>(w))) continue;
                        const Launch& Lk = *sources[pk][k];
                        for (size_t a = 0; a < Lk.args.size(); ++a)
                            busy = busy || (!Lk.is_out[a] && pp.values[Lk.args[a].slot].name == yname);
                    }
                }
                // z is written earlier now: nothing in between may read or write its
                // bytes; the residual is read earlier: nothing in between may write it
                const char* z = static_cast<const char*>(e.ptrs[z_slot]);
                const int64_t zbytes = arg_bytes(pi, j, static_cast<size_t>(z_slot));
                for (size_t k = static_cast<size_t>(w) + 1; k < j && !busy; ++k) {
                    busy = launch_touches(pi, k, z, zbytes, true) || launch_touches(pi, k, z, zbytes, false);
                    if (r_slot >= 0)
                        busy = busy || launch_touches(pi, k, static_cast<const char*>(e.ptrs[r_slot]),
                                                      arg_bytes(pi, j, static_cast<size_t>(r_slot)), true);
                }
                if (r_slot >= 0 && (g.gemm.kind != NNCB_CONV_FWD || g.gemm.sh != 1 || g.gemm.sw != 1) &&
                    g.gemm.kind != NNCB_DENSE_FWD)
                    busy = true;   // the residual must be laid out like the output
                // the residual join in the epilogue is opt-in: its per-row residual
                // loads ran the output-bound 1x1 convs at ~1 TB/s (a TMA side tile,
                // as the gradient epilogue uses, is the way to make it pay)
                static const bool residual_on = std::getenv("NNC_BN_INFER_RESIDUAL") != nullptr;
                if (r_slot >= 0 && !residual_on) {
                    why(L, "residual join (opt-in: NNC_BN_INFER_RESIDUAL=1)");
                    continue;
                }
                if (busy) { why(L, "y read elsewhere / z touched in between"); continue; }
                why(L, "fused");
                g.gemm.epilogue |= NNCB_EPI_BN_AFFINE | (n_relu ? NNCB_EPI_RELU : 0) | (n_add ? NNCB_EPI_RESIDUAL : 0);
                g.gemm.residual = n_add ? static_cast<const float*>(e.ptrs[r_slot]) : nullptr;
                g.gemm.bn_mean = static_cast<const float*>(e.ptrs[ch_slot[bn.b]]);
                g.gemm.bn_var = static_cast<const float*>(e.ptrs[ch_slot[bn.c]]);
                g.gemm.bn_gamma = static_cast<const float*>(e.ptrs[ch_slot[bn.d]]);
                g.gemm.bn_beta = static_cast<const float*>(e.ptrs[ch_slot[bn.e]]);
                g.gemm.bn_eps = bn.imm;
                g.ptrs.back() = e.ptrs[z_slot];
                e.skip = true;
            }
    }

    void fuse_bn_grad_reduce() {
        if (std::getenv("NNC_NO_FUSED_BN_GRAD")) return;
        for (size_t pi = 0; pi < steps.size(); ++pi)
            for (size_t j = 1; j < steps[pi].size(); ++j) {
                BoundLaunch& r = steps[pi][j];
                if (r.kind != LaunchKind::BnGradReduce || r.skip) continue;
                // the launch that last wrote g's bytes must be a fused group
                // storing exactly g (arena bytes are shared between values with
                // disjoint lifetimes: an older launch that stored a dead value
                // at the same address is not the producer)
                const char* gp = static_cast<const char*>(r.ptrs[2]);
                const int64_t gbytes = arg_bytes(pi, j, 2);
                const int64_t w = last_writer(pi, j, gp, gbytes);
                if (w < 0) continue;
                const size_t pj = static_cast<size_t>(w);
                if (steps[pi][pj].kind != LaunchKind::Ew) continue;
                {
                    bool stores_g = false;
                    const BoundLaunch& c = steps[pi][pj];
                    for (const auto& in : c.ew_prog.empty() ? sources[pi][pj]->ew : c.ew_prog)
                        stores_g = stores_g || (in.op == NNCB_EW_STORE && c.ptrs[in.slot] == r.ptrs[2]);
                    if (!stores_g) continue;
                }
                // the reduction moves from j up to pj: x and the statistics must
                // hold their final bytes there already (no writer in [pj, j)),
                // and the sums it writes early must not be read or written by
                // any launch in between (their bytes may belong to a value that
                // is live there)
                {
                    const int64_t C0 = r.d1;
                    const Range xr{static_cast<const char*>(r.ptrs[0]), arg_bytes(pi, j, 0)};
                    const Range sr{static_cast<const char*>(r.ptrs[1]), 2 * C0 * 4};
                    const Range o0{static_cast<const char*>(r.ptrs[3]), C0 * 4}, o1{static_cast<const char*>(r.ptrs[4]), C0 * 4};
                    bool clash = false;
                    for (size_t k = pj; k < j && !clash; ++k) {
                        clash = launch_touches(pi, k, xr.p, xr.n, true) || launch_touches(pi, k, sr.p, sr.n, true);
                        if (k > pj)
                            for (const Range& q : {o0, o1})
                                clash = clash || launch_touches(pi, k, q.p, q.n, true) || launch_touches(pi, k, q.p, q.n, false);
                    }
                    if (clash) continue;
                }
                BoundLaunch& e = steps[pi][pj];
                const int64_t rows = r.d0, C = r.d1;
                if (C < 4 || C > 2048 || (C & (C - 1)) || (rows * C) % 4 || e.n != rows * C) continue;
                if (e.c > 0 && e.c != C) continue;
                const Launch& L = *sources[pi][pj];
                std::vector<nncb_ew_instr> prog = e.ew_prog.empty() ? L.ew : e.ew_prog;
                int regs = e.ew_prog.empty() ? L.ew_regs : e.ew_regs;
                int n_reduce = 0;
                int at = -1;
                for (size_t k = 0; k < prog.size(); ++k) {
                    n_reduce += prog[k].op == NNCB_EW_REDUCE_BN_GRAD;
                    if (prog[k].op == NNCB_EW_STORE && e.ptrs[prog[k].slot] == r.ptrs[2]) at = static_cast<int>(k);
                }
                // at most two reductions per group: the second one (the residual
                // join of a projection block, both BatchNorms fed the same
                // gradient) puts the group on the 2-block register budget; with
                // its loads staged through the cp.async ring it beats the
                // standalone pass (C4 +1%; it measured neutral before the ring).
                // NNC_BN_GRAD_REDUCE_MAX=1 keeps one.
                static const int max_reduce = std::getenv("NNC_BN_GRAD_REDUCE_MAX") ? std::atoi(std::getenv("NNC_BN_GRAD_REDUCE_MAX")) : 2;
                if (n_reduce >= max_reduce || at < 0 || e.ptrs.size() + 5 > 48) continue;
                const int s0 = static_cast<int>(e.ptrs.size());
                std::vector<void*> ptrs = e.ptrs;
                ptrs.push_back(r.ptrs[0]);                                  // x
                ptrs.push_back(r.ptrs[1]);                                  // mean   = stats[0:C]
                ptrs.push_back(static_cast<float*>(r.ptrs[1]) + C);         // invstd = stats[C:2C]
                ptrs.push_back(r.ptrs[3]);                                  // sum_g
                ptrs.push_back(r.ptrs[4]);                                  // sum_gx
                const int rx = regs, rm = regs + 1, rs = regs + 2;
                auto mk = [](int op, int dst, int slot) {
                    nncb_ew_instr in{};
                    in.op = op;
                    in.dst = dst;
                    in.slot = slot;
                    return in;
                };
                nncb_ew_instr red{};
                red.op = NNCB_EW_REDUCE_BN_GRAD;
                red.a = prog[at].a;
                red.b = rx;
                red.c = rm;
                red.d = rs;
                red.slot = s0 + 3;
                red.e = s0 + 4;
                prog.insert(prog.begin() + at + 1, {mk(NNCB_EW_LOAD, rx, s0), mk(NNCB_EW_LOAD_CH, rm, s0 + 1),
                                                    mk(NNCB_EW_LOAD_CH, rs, s0 + 2), red});
                nncb_ew_program ep{static_cast<int32_t>(prog.size()), prog.data(), regs + 3,
                                   static_cast<int32_t>(ptrs.size())};
                nncb_ew_kernel* k = nullptr;
                NNC_CHECK(nncb_ew_compile(dev->ctx(), &ep, &k));
                e.ew = k;
                e.ptrs = std::move(ptrs);
                e.ew_prog = std::move(prog);
                e.ew_regs = regs + 3;
                e.c = C;
                e.extra.push_back({r.ptrs[0], rows * C * 4, false});   // x
                e.extra.push_back({r.ptrs[1], 2 * C * 4, false});      // mean, invstd
                e.extra.push_back({r.ptrs[3], C * 4, true});           // sum_g
                e.extra.push_back({r.ptrs[4], C * 4, true});           // sum_gx
                r.skip = true;
            }
    }

    /// A column sum (the Dense bias gradient, SumRows over the [rows, C]
    /// gradient g) is folded into the fused elementwise group that stores g
    /// (NNCB_EW_REDUCE_SUM): g is summed from registers as it is written
    /// instead of being read back. Tensor-core modes only (the fp32 mode keeps
    /// the exact SumRows order). Same producer / hazard rules as the BatchNorm
    /// gradient reduction above.
    void fuse_bias_grad_reduce() {
        if (std::getenv("NNC_NO_FUSED_BIAS_GRAD")) return;
        for (size_t pi = 0; pi < steps.size(); ++pi)
            for (size_t j = 1; j < steps[pi].size(); ++j) {
                BoundLaunch& r = steps[pi][j];
                if (r.kind != LaunchKind::SumRows || r.skip || r.flag0) continue;
                const int64_t rows = r.d0, C = r.d1;
                if (C < 4 || C > 8192 || (C & (C - 1)) || (rows * C) % 4) continue;
                const char* gp = static_cast<const char*>(r.ptrs[0]);
                const int64_t gbytes = arg_bytes(pi, j, 0);
                const int64_t w = last_writer(pi, j, gp, gbytes);
                if (w < 0) continue;
                const size_t pj = static_cast<size_t>(w);
                BoundLaunch& e = steps[pi][pj];
                if (e.kind != LaunchKind::Ew || e.n != rows * C || (e.c > 0 && e.c != C)) continue;
                const Launch& L = *sources[pi][pj];
                std::vector<nncb_ew_instr> prog = e.ew_prog.empty() ? L.ew : e.ew_prog;
                const int regs = e.ew_prog.empty() ? L.ew_regs : e.ew_regs;
                int n_reduce = 0, at = -1;
                for (size_t k = 0; k < prog.size(); ++k) {
                    n_reduce += prog[k].op == NNCB_EW_REDUCE_BN_GRAD || prog[k].op == NNCB_EW_REDUCE_STATS ||
                                prog[k].op == NNCB_EW_REDUCE_SUM;
                    if (prog[k].op == NNCB_EW_STORE && e.ptrs[prog[k].slot] == r.ptrs[0]) at = static_cast<int>(k);
                }
                if (at < 0 || n_reduce >= 2 || e.ptrs.size() + 1 > 48) continue;
                // the sum moves from j up to pj: its output must be neither
                // read nor written in between
                const Range o{static_cast<const char*>(r.ptrs[1]), C * 4};
                bool clash = false;
                for (size_t k = pj + 1; k < j && !clash; ++k)
                    clash = launch_touches(pi, k, o.p, o.n, true) || launch_touches(pi, k, o.p, o.n, false);
                if (clash) continue;
                nncb_ew_instr red{};
                red.op = NNCB_EW_REDUCE_SUM;
                red.a = prog[at].a;
                red.slot = static_cast<int32_t>(e.ptrs.size());
                prog.insert(prog.begin() + at + 1, red);
                std::vector<void*> ptrs = e.ptrs;
                ptrs.push_back(r.ptrs[1]);
                nncb_ew_program ep{static_cast<int32_t>(prog.size()), prog.data(), regs, static_cast<int32_t>(ptrs.size())};
                nncb_ew_kernel* k = nullptr;
                NNC_CHECK(nncb_ew_compile(dev->ctx(), &ep, &k));
                e.ew = k;
                e.ptrs = std::move(ptrs);
                e.ew_prog = std::move(prog);
                e.ew_regs = regs;
                e.c = C;
                e.extra.push_back({r.ptrs[1], C * 4, true});
                r.skip = true;
            }
    }

    /// The LayerNorm parameter gradients (LnDgamma: sum g*xhat, and the beta
    /// gradient's SumRows: sum g) of the same x and g as a LayerNorm input
    /// gradient move into that launch (nncb_layernorm_bwd_params), which has
    /// x and g in registers already: two passes over x and g disappear.
    /// Tensor-core modes only (the fp32 mode keeps the exact SumRows order).
    void fuse_ln_param_grads() {
        if (std::getenv("NNC_NO_FUSED_LN_PARAMS")) return;
        for (size_t pi = 0; pi < steps.size(); ++pi)
            for (size_t j = 0; j < steps[pi].size(); ++j) {
                BoundLaunch& b = steps[pi][j];
                if (b.kind != LaunchKind::LnBwd || b.skip || b.ptrs.size() != 4) continue;
                const int64_t rows = b.d0, C = b.d1;
                const Range xr{static_cast<const char*>(b.ptrs[0]), arg_bytes(pi, j, 0)};
                const Range gr{static_cast<const char*>(b.ptrs[2]), arg_bytes(pi, j, 2)};
                // a candidate at m may move to j when x and g keep their bytes
                // and its output is neither read nor written in between
                auto movable = [&](size_t m, const Range& o) {
                    const size_t lo = std::min(m, j), hi = std::max(m, j);
                    for (size_t k = lo + 1; k < hi; ++k)
                        if (launch_touches(pi, k, xr.p, xr.n, true) || launch_touches(pi, k, gr.p, gr.n, true) ||
                            launch_touches(pi, k, o.p, o.n, true) || launch_touches(pi, k, o.p, o.n, false))
                            return false;
                    // the output must not alias the operands of the fused launch
                    return !(o.overlaps(xr.p, xr.n) || o.overlaps(gr.p, gr.n) ||
                             o.overlaps(static_cast<const char*>(b.ptrs[3]), arg_bytes(pi, j, 3)));
                };
                int64_t dg = -1, db = -1;
                for (size_t m = 0; m < steps[pi].size(); ++m) {
                    const BoundLaunch& c = steps[pi][m];
                    if (m == j || c.skip || c.d0 != rows || c.d1 != C) continue;
                    if (dg < 0 && c.kind == LaunchKind::LnDgamma && c.ptrs[0] == b.ptrs[0] && c.ptrs[1] == b.ptrs[2] &&
                        movable(m, Range{static_cast<const char*>(c.ptrs[2]), C * 4}))
                        dg = static_cast<int64_t>(m);
                    else if (db < 0 && c.kind == LaunchKind::SumRows && c.ptrs[0] == b.ptrs[2] &&
                             movable(m, Range{static_cast<const char*>(c.ptrs[1]), C * 4}))
                        db = static_cast<int64_t>(m);
                }
                if (dg < 0 && db < 0) continue;
                b.ptrs.push_back(dg >= 0 ? steps[pi][dg].ptrs[2] : nullptr);
                b.ptrs.push_back(db >= 0 ? steps[pi][db].ptrs[1] : nullptr);
                b.extra.push_back({b.ptrs[4], C * 4, true});
                b.extra.push_back({b.ptrs[5], C * 4, true});
                if (dg >= 0) steps[pi][dg].skip = true;
                if (db >= 0) steps[pi][db].skip = true;
            }
    }

    /// BatchNorm statistics of a tensor-core GEMM's output are accumulated in
    /// that GEMM's epilogue (column sum / sum of squares), so the separate
    /// statistics pass over the activation disappears; the BN launch only
    /// finalizes mean / invstd from 2*C doubles.
    void fuse_bn_statistics() {
        std::vector<BoundLaunch*> fused;
        int64_t doubles = 0;
        for (auto& plan_steps : steps)
            for (size_t j = 0; j < plan_steps.size(); ++j) {
                BoundLaunch& bn = plan_steps[j];
                if (bn.kind != LaunchKind::BnStats) continue;
                // the launch that last wrote the BatchNorm input's bytes; fuse
                // only if it is a forward GEMM whose output is exactly that
                // input (an older GEMM that wrote a dead value at a reused
                // arena address must never be matched)
                const size_t pi = static_cast<size_t>(&plan_steps - steps.data());
                const int64_t w = last_writer(pi, j, static_cast<const char*>(bn.ptrs[0]), arg_bytes(pi, j, 0));
                for (int64_t once = w; once >= 0; once = -1) {   // `break` = do not fuse
                    BoundLaunch& g = plan_steps[static_cast<size_t>(once)];
                    if (g.kind != LaunchKind::Gemm || g.ptrs.back() != bn.ptrs[0]) break;
                    if (g.gemm.kind != NNCB_CONV_FWD && g.gemm.kind != NNCB_DENSE_FWD) break;
                    // measured per ResNet-50 shape (tools/gemm_bench.py --colstats vs
                    // tools/stats_bench.py): the epilogue statistics cost less than a
                    // separate pass over the output on every shape
                    if (std::getenv("NNC_NO_FUSED_BN_STATS")) break;
                    static const int64_t min_k = std::getenv("NNC_BN_STATS_FUSE_MIN_K")
                                                     ? std::atoll(std::getenv("NNC_BN_STATS_FUSE_MIN_K")) : 0;
                    const int64_t K = g.gemm.kind == NNCB_DENSE_FWD ? g.gemm.in_f
                                                                    : g.gemm.kh * g.gemm.kw * g.gemm.ci;
                    if (K < min_k) break;
                    g.gemm.epilogue |= NNCB_EPI_COLSTATS;
                    g.gemm.colstats = reinterpret_cast<double*>(static_cast<uintptr_t>(doubles));  // offset for now
                    bn.bn_finalize = true;
                    bn.colstats = g.gemm.colstats;
                    doubles += 2 * bn.d1;
                    fused.push_back(&g);
                    fused.push_back(&bn);
                    // the finalize itself folds into the GEMM (its last CTA) when the
                    // statistics' bytes are untouched between the two launches
                    {
                        const Range st{static_cast<const char*>(bn.ptrs[1]), 2 * bn.d1 * 4};
                        bool clash = std::getenv("NNC_NO_FUSED_BN_FINALIZE") != nullptr;
                        for (size_t k = static_cast<size_t>(once) + 1; k < j && !clash; ++k)
                            clash = launch_touches(pi, k, st.p, st.n, true) || launch_touches(pi, k, st.p, st.n, false);
                        if (!clash) {
                            g.gemm.colstats_finalize = static_cast<float*>(bn.ptrs[1]);
                            g.gemm.colstats_eps = bn.eps;
                            g.extra.push_back({bn.ptrs[1], 2 * bn.d1 * 4, true});
                            bn.skip = true;
                        }
                    }
                    break;
                }
            }
        if (!doubles) return;
        NNC_CHECK(nncb_malloc(dev->ctx(), static_cast<size_t>(doubles) * sizeof(double), &side));
        auto rebase = [&](double* off) { return static_cast<double*>(side) + reinterpret_cast<uintptr_t>(off); };
        for (BoundLaunch* b : fused) {
            if (b->kind == LaunchKind::Gemm)
                b->gemm.colstats = rebase(b->gemm.colstats);
            else
                b->colstats = rebase(b->colstats);
        }
    }

    BoundLaunch resolve(const ExecutionPlan& p, const Launch& L) {
        BoundLaunch b;
        b.kind = L.kind;
        for (const plan::Arg& a : L.args)
            b.ptrs.push_back(static_cast<float*>(ptr(p.values[a.slot].name)) + a.offset);
        auto dims = [&](size_t arg) -> const std::vector<int64_t>& { return p.values[L.args.at(arg).slot].dims; };
        const hlir::Attrs& at = L.attrs;
        switch (L.kind) {
            case LaunchKind::Ew: {
                nncb_ew_program prog{static_cast<int32_t>(L.ew.size()), L.ew.data(), L.ew_regs,
                                     static_cast<int32_t>(L.args.size())};
                // tf32 mode: the BatchNorm input gradient takes per-channel
                // quotients instead of a per-element IEEE division, and GELU
                // is evaluated in fp32 instead of double
                bool fast = false;
                for (const auto& in : L.ew)
                    fast = fast || in.op == NNCB_EW_BN_GRAD || in.op == NNCB_EW_GELU || in.op == NNCB_EW_GELU_GRAD;
                if (fast && (precision == NNCB_PREC_TF32 || precision == NNCB_PREC_BF16) &&
                    !std::getenv("NNC_EXACT_BN_GRAD")) {
                    b.ew_prog = L.ew;
                    for (auto& in : b.ew_prog) {
                        if (in.op == NNCB_EW_BN_GRAD) in.op = NNCB_EW_BN_GRAD_FAST;
                        if (in.op == NNCB_EW_GELU) in.op = NNCB_EW_GELU_FAST;
                        if (in.op == NNCB_EW_GELU_GRAD) in.op = NNCB_EW_GELU_GRAD_FAST;
                    }
                    b.ew_regs = L.ew_regs;
                    prog.instr = b.ew_prog.data();
                }
                NNC_CHECK(nncb_ew_compile(dev->ctx(), &prog, &b.ew));
                b.n = element_count(p.values[L.elem_slot].dims);
                b.c = at.out_channels;
                break;
            }
            case LaunchKind::Gemm: {
                nncb_gemm_desc& d = b.gemm;
                d.precision = precision;
                d.tile = L.tile;
                switch (L.op) {
                    case hlir::OpKind::Conv2D:
                        d.kind = NNCB_CONV_FWD;
                        geom::conv_geometry(d, dims(0), at);
                        b.flag0 = at.has_bias ? 1 : 0;
                        d.epilogue = at.has_bias ? NNCB_EPI_BIAS : 0;
                        break;
                    case hlir::OpKind::Conv2DGradInput:
                        d.kind = NNCB_CONV_DGRAD;
                        geom::conv_geometry(d, dims(L.args.size() - 1), at);
                        break;
                    case hlir::OpKind::Conv2DGradWeight:
                        d.kind = NNCB_CONV_WGRAD;
                        geom::conv_geometry(d, dims(0), at);
                        break;
                    case hlir::OpKind::Dense:
                        d.kind = NNCB_DENSE_FWD;
                        d.batch = dims(0)[0];
                        d.in_f = dims(0)[1];
                        d.out_f = at.out_features;
                        b.flag0 = at.has_bias ? 1 : 0;
                        d.epilogue = at.has_bias ? NNCB_EPI_BIAS : 0;
                        break;
                    case hlir::OpKind::DenseGradInput:
                        d.kind = NNCB_DENSE_DGRAD;
                        d.batch = dims(0)[0];
                        d.out_f = dims(0)[1];
                        d.in_f = dims(1)[0];
                        break;
                    case hlir::OpKind::DenseGradWeight:
                        d.kind = NNCB_DENSE_WGRAD;
                        d.batch = dims(0)[0];
                        d.in_f = dims(0)[1];
                        d.out_f = dims(1)[1];
                        break;
                    default: throw Error(Error::Code::UnsupportedInGroup, "not a GEMM op");
                }
                break;
            }
            case LaunchKind::MaxPool: b.pool = geom::pool_geometry(dims(0), at); break;
            case LaunchKind::MaxPoolGrad: b.pool = geom::pool_geometry(dims(2), at); break;
            case LaunchKind::AvgPool: {
                const auto& x = dims(0);
                b.d0 = x[0]; b.d1 = x[1]; b.d2 = x[2]; b.d3 = x[3]; b.d4 = at.out_hw[0]; b.d5 = at.out_hw[1];
                break;
            }
            case LaunchKind::AvgPoolGrad: {
                const auto& gx = dims(1);
                const auto& gy = dims(0);
                b.d0 = gx[0]; b.d1 = gx[1]; b.d2 = gx[2]; b.d3 = gx[3]; b.d4 = gy[1]; b.d5 = gy[2];
                break;
            }
            case LaunchKind::SumRows: {
                const auto& x = dims(0);
                b.d1 = x.back();
                b.d0 = element_count(x) / std::max<int64_t>(b.d1, 1);
                b.flag0 = precision == NNCB_PREC_FP32 ? 1 : 0;
                break;
            }
            case LaunchKind::CumSum: {
                const auto& x = dims(0);
                int64_t outer = 1, inner = 1;
                for (int64_t i = 0; i < at.axis; ++i) outer *= x[i];
                for (size_t i = at.axis + 1; i < x.size(); ++i) inner *= x[i];
                b.d0 = outer; b.d1 = x.empty() ? 1 : x[at.axis]; b.d2 = inner;
                b.flag0 = at.exclusive; b.flag1 = at.reverse;
                break;
            }
            case LaunchKind::BnStats:
            case LaunchKind::BnGradReduce:
            case LaunchKind::LnFwd:
            case LaunchKind::LnBwd:
            case LaunchKind::LnDgamma: {
                const auto& x = dims(0);
                b.d1 = x.back();
                b.d0 = element_count(x) / b.d1;
                b.eps = at.eps;
                break;
            }
        }
        return b;
    }

    void enqueue_plan(size_t pi, std::vector<std::string>* trace, const std::function<void(size_t)>& after = nullptr,
                      const double* sgd_lr = nullptr, double sgd_scale = 1.0) const {
        const auto& labels = step_labels[pi];
        size_t li = 0;
        plan_prologue(pi);
        for (size_t k = 0; k < steps[pi].size(); ++k) {
            while (trace && li < labels.size() && labels[li].first == k) trace->push_back("exec:" + labels[li++].second);
            enqueue(dev->ctx(), steps[pi][k], sgd_lr, sgd_scale);
            if (after) after(k);
        }
        while (trace && li < labels.size()) trace->push_back("exec:" + labels[li++].second);
    }
};

/* ------------------------------------------------------------------ */
/*  HostModel                                                          */
/* ------------------------------------------------------------------ */

HostModel::HostModel() {
    static std::atomic<uint64_t> next{1};
    uid_ = next.fetch_add(1);
}

HostModel::HostModel(const HostModel& o) : HostModel() { *this = o; }

void forget_trainers_of(uint64_t model_uid);   // (below, with the trainer cache)

HostModel::~HostModel() {
    try {
        forget_trainers_of(uid_);
        if (device_owner) device_owner->forget_model(uid_);
    } catch (...) {
    }
}

HostModel& HostModel::operator=(const HostModel& o) {
    if (this == &o) return *this;
    o.sync();   // a copy is a value: device-newer weights come with it
    weights = o.weights;
    stamps = o.stamps;
    device_owner = nullptr;   // the copy has its own identity (uid) in device caches
    device_newer.clear();
    return *this;
}

HostModel HostModel::from_graph(const hlir::Graph& g) {
    HostModel m;
    for (const auto& [name, t] : g.initializers) {
        m.weights.emplace(name, t);
        m.stamps[name] = 0;
    }
    return m;
}

const Tensor& HostModel::tensor(const std::string& name) const {
    auto it = weights.find(name);
    if (it == weights.end()) throw Error(Error::Code::ShapeMismatch, "model has no weight " + name);
    if (device_owner && device_newer.count(name)) {
        device_owner->pull_weight(*this, name, it->second);
        device_newer.erase(name);
    }
    return it->second;
}

void HostModel::sync() const {
    for (const std::string& name : std::vector<std::string>(device_newer.begin(), device_newer.end()))
        (void)tensor(name);
}

uint64_t HostModel::stamp(const std::string& name) const {
    auto it = stamps.find(name);
    return it == stamps.end() ? 0 : it->second;
}

void HostModel::set(const std::string& name, Tensor value) {
    weights[name] = std::move(value);
    device_newer.erase(name);
    ++stamps[name];
}

void HostModel::bump(const std::string& name) { ++stamps[name]; }

std::vector<std::string> HostModel::names() const {
    std::vector<std::string> out;
    for (const auto& [k, v] : weights) out.push_back(k);
    return out;
}

/* ------------------------------------------------------------------ */
/*  Device                                                             */
/* ------------------------------------------------------------------ */

Device::Device(int ordinal) { NNC_CHECK(nncb_create(ordinal, &ctx_)); }

Device::~Device() {
    programs_.clear();
    for (auto& [name, cw] : cache_)
        if (cw.ptr && !cw.external) nncb_free(ctx_, cw.ptr);
    nncb_destroy(ctx_);
}

SyncStats Device::sync_stats(bool reset) {
    SyncStats s = stats_;
    if (reset) stats_ = {};
    return s;
}

void Device::init_comm(int nranks, int rank, const uint8_t id[128]) {
    NNC_CHECK(nncb_comm_init(ctx_, nranks, rank, id));
    nranks_ = nranks;
    rank_ = rank;
}

void* Device::weight_buffer(const HostModel& m, const std::string& name, const Tensor& host, uint64_t stamp) {
    auto key = std::make_pair(m.uid(), name);
    auto it = cache_.find(key);
    size_t bytes = host.byte_size();
    if (it == cache_.end()) {
        CachedWeight cw;
        cw.bytes = bytes;
        NNC_CHECK(nncb_malloc(ctx_, std::max<size_t>(bytes, 4), &cw.ptr));
        cw.stamp = stamp + 1;  // force upload below
        it = cache_.emplace(key, cw).first;
    }
    CachedWeight& cw = it->second;
    if (cw.bytes != bytes) throw Error(Error::Code::ShapeMismatch, name + ": stored weight does not match plan");
    if (cw.stamp != stamp) {
        NNC_CHECK(nncb_h2d(ctx_, cw.ptr, host.data(), bytes));
        cw.stamp = stamp;
        stats_.h2d_bytes += bytes;
        stats_.weight_bytes += plan::align_bytes(static_cast<int64_t>(bytes), 64);   // aligned, as the reference counts
        ++stats_.weight_transfers[name];
    }
    return cw.ptr;
}

void* Device::weight_ptr(const HostModel& m, const std::string& name) const {
    auto it = cache_.find({m.uid(), name});
    return it == cache_.end() ? nullptr : it->second.ptr;
}

void Device::pull_weight(const HostModel& m, const std::string& name, Tensor& host) {
    void* p = weight_ptr(m, name);
    if (!p) return;
    NNC_CHECK(nncb_d2h(ctx_, host.data(), p, host.byte_size()));
    NNC_CHECK(nncb_sync(ctx_));
    stats_.d2h_bytes += host.byte_size();
}

void Device::adopt_weight(const HostModel& m, const std::string& name, void* ptr, size_t bytes, uint64_t stamp) {
    auto key = std::make_pair(m.uid(), name);
    auto it = cache_.find(key);
    if (it != cache_.end() && !it->second.external && it->second.ptr) nncb_free(ctx_, it->second.ptr);
    cache_[key] = CachedWeight{ptr, bytes, stamp, true};
}

void Device::evict_model(HostModel& m) {
    for (const std::string& name : std::vector<std::string>(m.device_newer.begin(), m.device_newer.end()))
        (void)m.tensor(name);   // pulls and clears device_newer
    for (auto it = cache_.begin(); it != cache_.end();) {
        if (it->first.first != m.uid()) {
            ++it;
            continue;
        }
        if (!it->second.external && it->second.ptr) nncb_free(ctx_, it->second.ptr);
        it = cache_.erase(it);
    }
}

void Device::forget_model(uint64_t model_uid) {
    for (auto it = cache_.begin(); it != cache_.end();) {
        if (it->first.first != model_uid) {
            ++it;
            continue;
        }
        if (!it->second.external && it->second.ptr) nncb_free(ctx_, it->second.ptr);
        it = cache_.erase(it);
    }
}

uint64_t Device::cached_stamp(const HostModel& m, const std::string& name) const {
    auto it = cache_.find({m.uid(), name});
    return it == cache_.end() ? ~0ull : it->second.stamp;
}

void Device::mark_device_newer(HostModel& m, const std::string& name, uint64_t new_stamp) {
    auto it = cache_.find({m.uid(), name});
    if (it != cache_.end()) it->second.stamp = new_stamp;
    m.device_owner = this;
    m.device_newer.insert(name);
}

Device& default_device() {
    static std::unique_ptr<Device> dev;
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    if (!dev) {
        const char* env = std::getenv("NNC_DEVICE");
        dev = std::make_unique<Device>(env ? std::atoi(env) : 0);
    }
    return *dev;
}

/* ------------------------------------------------------------------ */
/*  OffloadDevice / ExecutionContext (reference runtime.hpp:40-121)    */
/* ------------------------------------------------------------------ */

OffloadDevice::OffloadDevice(Device* device) : dev_(device ? device : &default_device()) {}

OffloadDevice::~OffloadDevice() {
    for (auto& [n, c] : cache_)
        if (c.device) nncb_free(dev_->ctx(), c.device);
}

uint8_t* OffloadDevice::sync_weight(const std::string& name, const Tensor& host, uint64_t stamp, int64_t aligned_bytes) {
    auto it = cache_.find(name);
    if (it == cache_.end() || it->second.bytes != aligned_bytes) {
        if (it != cache_.end() && it->second.device) nncb_free(dev_->ctx(), it->second.device);
        CachedWeight c;
        c.bytes = aligned_bytes;
        NNC_CHECK(nncb_malloc(dev_->ctx(), static_cast<size_t>(std::max<int64_t>(aligned_bytes, 256)), &c.device));
        c.stamp = ~stamp;   // stale: forces the copy below
        it = cache_.insert_or_assign(name, c).first;
    }
    CachedWeight& c = it->second;
    if (c.stamp != stamp) {
        NNC_CHECK(nncb_h2d(dev_->ctx(), c.device, host.data(), host.byte_size()));
        c.stamp = stamp;
        stats_.h2d_bytes += static_cast<uint64_t>(aligned_bytes);
        stats_.weight_bytes += static_cast<uint64_t>(aligned_bytes);
        ++stats_.weight_transfers[name];
    }
    return static_cast<uint8_t*>(c.device);
}

void OffloadDevice::preseed(const std::string& name, const Tensor& host, uint64_t stamp, int64_t aligned_bytes) {
    const SyncStats keep = stats_;
    (void)sync_weight(name, host, ~stamp, aligned_bytes);   // place the bytes ...
    cache_[name].stamp = stamp;                              // ... as current at `stamp`
    stats_ = keep;                                           // without counting a transfer
}

void OffloadDevice::note_device_current(const std::string& name, uint64_t stamp) {
    auto it = cache_.find(name);
    if (it != cache_.end()) it->second.stamp = stamp;
}

SyncStats OffloadDevice::sync_stats(bool reset) {
    SyncStats s = stats_;
    if (reset) stats_ = {};
    return s;
}

ExecutionContext::~ExecutionContext() { release_all(); }

uint8_t* ExecutionContext::data(const std::string& name) {
    auto it = buffers_.find(name);
    if (it == buffers_.end()) throw Error(Error::Code::ShapeMismatch, "no live buffer " + name);
    return it->second.ptr;
}

uint8_t* ExecutionContext::alloc(const std::string& name, int64_t bytes) {
    if (buffers_.count(name)) throw Error(Error::Code::ArenaOverflow, "double allocation of " + name);
    Buffer b;
    b.bytes = bytes;
    if (bytes > 0) {
        void* p = nullptr;
        NNC_CHECK(nncb_malloc(default_device().ctx(), static_cast<size_t>(bytes), &p));
        b.ptr = static_cast<uint8_t*>(p);
        b.owned = true;
    }
    adopt(name, b.ptr, bytes);
    buffers_[name].owned = b.owned;
    return b.ptr;
}

void ExecutionContext::adopt(const std::string& name, uint8_t* ptr, int64_t bytes) {
    if (buffers_.count(name)) throw Error(Error::Code::ArenaOverflow, "double allocation of " + name);
    buffers_[name] = Buffer{ptr, bytes, false};
    current_ += bytes;
    high_ = std::max(high_, current_);
    if (capacity >= 0 && current_ > capacity)
        throw Error(Error::Code::ArenaOverflow, "context capacity exceeded by " + name);
}

void ExecutionContext::release(const std::string& name) {
    auto it = buffers_.find(name);
    if (it == buffers_.end()) return;
    current_ -= it->second.bytes;
    if (it->second.owned && it->second.ptr) nncb_free(default_device().ctx(), it->second.ptr);
    buffers_.erase(it);
}

void ExecutionContext::release_all() {
    while (!buffers_.empty()) release(buffers_.begin()->first);
}

/* ------------------------------------------------------------------ */
/*  execute                                                            */
/* ------------------------------------------------------------------ */

namespace {

struct ExecCache {
    std::unique_ptr<Program> prog;
    void* graph = nullptr;
    std::map<std::string, void*> weight_ptrs;   // pointers baked into the graph
    int runs = 0;
    ~ExecCache() {
        if (graph) nncb_graph_destroy(graph);
    }
};

std::map<std::pair<const Device*, uint64_t>, std::unique_ptr<ExecCache>>& exec_caches() {
    static std::map<std::pair<const Device*, uint64_t>, std::unique_ptr<ExecCache>> m;
    return m;
}

void check_inputs(const ExecutionPlan& p, const std::map<std::string, Tensor>& inputs) {
    for (uint32_t slot : p.input_slots) {
        const auto& v = p.values[slot];
        auto fed = inputs.find(v.name);
        if (fed == inputs.end()) throw Error(Error::Code::ShapeMismatch, "missing input " + v.name);
        if (fed->second.dims().size() != v.dims.size())
            throw Error(Error::Code::ShapeMismatch, v.name + ": rank " + std::to_string(fed->second.dims().size()) +
                                                        ", plan expects " + std::to_string(v.dims.size()));
        if (fed->second.dims() != v.dims)
            throw Error(Error::Code::ShapeMismatch,
                        v.name + ": expected " + dims_to_string(v.dims) + ", got " + dims_to_string(fed->second.dims()));
        if (fed->second.dtype() != p.dtype) throw Error(Error::Code::ShapeMismatch, v.name + ": dtype mismatch");
    }
}

}  // namespace

namespace {

// The bound program of `p` on `dev` with the current weights (stamp-checked
// device cache; a changed weight pointer rebinds).
using WeightSource = std::function<void*(const std::string&)>;

ExecCache& bound_cache(const ExecutionPlan& p, const HostModel& model, Device& dev, const ExecOptions& opts,
                       const WeightSource* weights = nullptr) {
    auto& slot = exec_caches()[{&dev, p.uid}];
    std::map<std::string, void*> wptrs;
    for (const std::string& w : p.weight_names)
        wptrs[w] = weights ? (*weights)(w) : dev.weight_buffer(model, w, model.tensor(w), model.stamp(w));
    if (!slot || slot->weight_ptrs != wptrs || slot->prog->precision != opts.gemm_precision ||
        slot->prog->keep_values != opts.keep_values) {
        slot = std::make_unique<ExecCache>();
        slot->prog = std::make_unique<Program>();
        slot->prog->dev = &dev;
        slot->prog->plans = {&p};
        slot->prog->precision = opts.gemm_precision;
        slot->prog->keep_values = opts.keep_values;
        slot->prog->bind([&](const std::string& w) { return wptrs.at(w); },
                         [](const std::string&) -> void* { return nullptr; });
        slot->weight_ptrs = wptrs;
    }
    return *slot;
}

}  // namespace

/// A value of the last execute of `p` on `device` (parity debugging): the
/// program must have been bound with ExecOptions::keep_values, so no later
/// launch of the run reused the value's arena bytes.
Tensor last_run_value(const ExecutionPlan& p, const std::string& name, Device* device) {
    Device& dev = device ? *device : default_device();
    auto it = exec_caches().find({&dev, p.uid});
    if (it == exec_caches().end() || !it->second)
        throw Error(Error::Code::ShapeMismatch, "last_run_value: the plan has not run on this device");
    Program& prog = *it->second->prog;
    if (!prog.keep_values)
        throw Error(Error::Code::ShapeMismatch, "last_run_value: bind with ExecOptions::keep_values");
    const int s = p.find_value(name);
    if (s < 0) throw Error(Error::Code::ShapeMismatch, "no value " + name + " in the plan");
    const plan::ValueEntry& v = p.values[s];
    if (v.storage != StorageClass::Buffer)
        throw Error(Error::Code::ShapeMismatch, name + " lives in registers of a fused group");
    Tensor t(p.dtype, v.dims);
    bool fed = false;
    for (uint32_t is : p.input_slots) fed = fed || p.values[is].name == name;
    if (!fed && v.category != plan::MemCategory::Input && v.category != plan::MemCategory::Parameter &&
        !prog.written_by_plan(0, static_cast<const char*>(prog.ptr(name)), static_cast<int64_t>(t.byte_size())))
        throw Error(Error::Code::ShapeMismatch, name + " is never written: its producer was fused into another launch");
    NNC_CHECK(nncb_sync(dev.ctx()));
    NNC_CHECK(nncb_d2h(dev.ctx(), t.data(), prog.ptr(name), t.byte_size()));
    NNC_CHECK(nncb_sync(dev.ctx()));
    return t;
}

namespace {

// first run eagerly (sizes scratch, compiles kernels); later runs replay a graph
void run_bound(ExecCache& c, const ExecutionPlan& p, const ExecOptions& opts) {
    nncb_ctx* ctx = c.prog->dev->ctx();
    if (!opts.use_graphs || c.runs == 0) {
        c.prog->enqueue_plan(0, opts.trace);
    } else {
        if (!c.graph) {
            NNC_CHECK(nncb_capture_begin(ctx));
            c.prog->enqueue_plan(0, nullptr);
            NNC_CHECK(nncb_capture_end(ctx, &c.graph));
        }
        if (opts.trace)
            for (const auto& es : p.exec_steps) opts.trace->push_back("exec:" + es.label);
        NNC_CHECK(nncb_graph_launch(ctx, c.graph));
    }
    ++c.runs;
}

// Pipelined execute (execute_stage / execute_launch_staged / execute_staged_outputs)
struct StagedIO {
    struct Slot {
        std::vector<void*> in;   // per input slot of the plan
        void* ready = nullptr;
        void* consumed = nullptr;
        bool used = false;
    };
    Device* dev = nullptr;
    Slot slots[2];
    uint64_t n_staged = 0, n_launched = 0;
    std::vector<std::string> out_names;
    std::vector<void*> out_pinned;
    std::vector<std::vector<int64_t>> out_dims;
    void* done = nullptr;
    bool pending = false;
    ~StagedIO() {
        try {
            nncb_ctx* ctx = dev->ctx();
            nncb_sync(ctx);
            for (Slot& s : slots) {
                for (void* q : s.in) nncb_free(ctx, q);
                for (void* e : {s.ready, s.consumed})
                    if (e) nncb_event_destroy(e);
            }
            for (void* h : out_pinned) nncb_host_free(h);
            if (done) nncb_event_destroy(done);
        } catch (...) {
        }
    }
};

std::map<std::pair<const Device*, uint64_t>, std::unique_ptr<StagedIO>>& staged_ios() {
    static std::map<std::pair<const Device*, uint64_t>, std::unique_ptr<StagedIO>> m;
    return m;
}

}  // namespace

namespace {

// Runs the (already specialised) plan `p`; `od` routes weights through an
// offload cache and counts the copies.
std::map<std::string, Tensor> run_plan(const ExecutionPlan& p, const std::map<std::string, Tensor>& inputs,
                                       const HostModel& model, Device& dev, const ExecOptions& opts,
                                       OffloadDevice* od, ExecutionContext* ctx_acc) {
    {
        auto it = exec_caches().find({&dev, p.uid});
        const bool reuse = opts.inputs_resident && it != exec_caches().end() && it->second && it->second->runs > 0;
        if (!reuse) check_inputs(p, inputs);
    }
    const bool had_runs = [&] {
        auto it = exec_caches().find({&dev, p.uid});
        return it != exec_caches().end() && it->second && it->second->runs > 0;
    }();
    const int64_t A = std::max<int64_t>(opts.alignment, 1);
    WeightSource via_offload = [&](const std::string& w) -> void* {
        const Tensor& t = model.tensor(w);
        return od->sync_weight(w, t, model.stamp(w), plan::align_bytes(static_cast<int64_t>(t.byte_size()), A));
    };
    ExecCache& c = bound_cache(p, model, dev, opts, od ? &via_offload : nullptr);
    Program& prog = *c.prog;
    nncb_ctx* ctx = dev.ctx();
    const bool reuse_inputs = opts.inputs_resident && had_runs && c.runs > 0;
    if (!reuse_inputs)   // (a rebound program starts with runs == 0)
        for (uint32_t s : p.input_slots) {
            const Tensor& t = inputs.at(p.values[s].name);
            NNC_CHECK(nncb_h2d(ctx, prog.ptr(p.values[s].name), t.data(), t.byte_size()));
            dev.stats().h2d_bytes += t.byte_size();
            if (od) od->count_h2d(plan::align_bytes(static_cast<int64_t>(t.byte_size()), A));
        }
    run_bound(c, p, opts);
    std::map<std::string, Tensor> out;
    for (uint32_t s : p.output_slots) {
        const auto& v = p.values[s];
        if (opts.materialize && !opts.materialize->count(v.name)) continue;
        Tensor t = Tensor::uninitialized(p.dtype, v.dims);   // the download overwrites every byte
        NNC_CHECK(nncb_d2h(ctx, t.data(), prog.ptr(v.name), t.byte_size()));
        dev.stats().d2h_bytes += t.byte_size();
        if (od) od->count_d2h(plan::align_bytes(static_cast<int64_t>(t.byte_size()), A));
        out.emplace(v.name, std::move(t));
    }
    NNC_CHECK(nncb_sync(ctx));
    if (ctx_acc) {
        // the plan's alloc/free events replayed at the context's alignment
        // (reference runtime.cpp:365-437): values carried in from an earlier
        // plan of the same step stay; data() addresses the device buffers
        const int64_t CA = std::max<int64_t>(ctx_acc->alignment(), 1);
        for (const plan::PlanEvent& ev : p.events) {
            const plan::ValueEntry& v = p.values[ev.slot];
            if (!ev.alloc) {
                ctx_acc->release(v.name);
                continue;
            }
            if (ctx_acc->live(v.name)) continue;
            const int64_t bytes = v.storage == StorageClass::Buffer
                                      ? plan::align_bytes(element_count(v.dims) * static_cast<int64_t>(dtype_size(p.dtype)), CA)
                                      : 0;
            auto w = prog.where.find(v.name);
            ctx_acc->adopt(v.name, w == prog.where.end() ? nullptr : static_cast<uint8_t*>(w->second), bytes);
        }
    }
    return out;
}

std::map<int32_t, int64_t> call_binding(const ExecutionPlan& p, const std::map<std::string, Tensor>& inputs,
                                        const std::map<int32_t, int64_t>& explicit_bindings) {
    // reference runtime.cpp:318-360
    std::map<int32_t, int64_t> bindings = explicit_bindings;
    for (uint32_t slot : p.input_slots) {
        const plan::ValueEntry& e = p.values[slot];
        auto fed = inputs.find(e.name);
        if (fed == inputs.end()) continue;
        const auto& got = fed->second.dims();
        if (got.size() != e.dims.size())
            throw Error(Error::Code::ShapeMismatch, e.name + ": rank " + std::to_string(got.size()) +
                                                        ", plan expects " + std::to_string(e.dims.size()));
        for (size_t i = 0; i < got.size(); ++i) {
            const plan::VdimSlot* vs = nullptr;
            for (const plan::VdimSlot& d : p.vdims)
                if (d.slot == slot && d.axis == i) vs = &d;
            if (!vs) {
                if (e.dims[i] != got[i])
                    throw Error(Error::Code::ShapeMismatch, e.name + ": axis " + std::to_string(i) + " expected " +
                                                                std::to_string(e.dims[i]) + ", got " + std::to_string(got[i]));
                continue;
            }
            auto [it, fresh] = bindings.emplace(vs->sym, got[i]);
            if (!fresh && it->second != got[i])
                throw Error(Error::Code::ShapeMismatch,
                            e.name + ": conflicting extents for vdim #" + std::to_string(vs->sym));
        }
    }
    for (auto it = bindings.begin(); it != bindings.end();) {   // only this plan's vdims matter
        const bool mine = std::any_of(p.vdims.begin(), p.vdims.end(), [&](const plan::VdimSlot& d) { return d.sym == it->first; });
        if (it->second < 1) throw Error(Error::Code::ShapeMismatch, "vdim #" + std::to_string(it->first) + " bound to " + std::to_string(it->second));
        it = mine ? std::next(it) : bindings.erase(it);
    }
    return bindings;
}

bool at_compiled_extents(const ExecutionPlan& p, const std::map<int32_t, int64_t>& b) {
    for (const plan::VdimSlot& d : p.vdims) {
        auto it = b.find(d.sym);
        if (it != b.end() && it->second != d.extent) return false;
    }
    return true;
}

}  // namespace

std::vector<LaunchProfile> profile_run(const ExecutionPlan& p0, const std::map<std::string, Tensor>& inputs,
                                       const HostModel& model, Device* device, const ExecOptions& opts) {
    Device& dev = device ? *device : default_device();
    const ExecutionPlan& p = plan_for_inputs(p0, inputs, opts.bindings);
    check_inputs(p, inputs);
    ExecCache& c = bound_cache(p, model, dev, opts);
    Program& prog = *c.prog;
    nncb_ctx* ctx = dev.ctx();
    for (uint32_t s : p.input_slots) {
        const Tensor& t = inputs.at(p.values[s].name);
        NNC_CHECK(nncb_h2d(ctx, prog.ptr(p.values[s].name), t.data(), t.byte_size()));
    }
    if (c.runs == 0) {   // first use: compiles kernels (and, in live tuning mode, times GEMM tiles)
        prog.enqueue_plan(0, nullptr);
        NNC_CHECK(nncb_sync(ctx));
        ++c.runs;
    }
    std::vector<LaunchProfile> out;
    std::vector<void*> evs;
    auto ev = [&]() {
        void* e = nullptr;
        NNC_CHECK(nncb_event_create(&e));
        NNC_CHECK(nncb_event_record(ctx, e));
        evs.push_back(e);
    };
    ev();
    if (!prog.kmajor.empty() && prog.kmajor[0].n) {
        prog.plan_prologue(0);
        ev();
        out.push_back({"kmajor_weights", "transpose", 0, 8.0 * 1024 * static_cast<double>(prog.kmajor[0].tiles), 0});
    }
    for (size_t k = 0; k < prog.steps[0].size(); ++k) {
        const BoundLaunch& b = prog.steps[0][k];
        const Launch& L = *prog.sources[0][k];
        if (b.skip) continue;
        enqueue(ctx, b);
        ev();
        LaunchProfile t;
        t.label = b.ew_prog.empty() ? L.label : L.label + "+bn_grad_reduce";
        t.kind = L.kind == LaunchKind::Gemm ? std::string("gemm:") + hlir::op_name(L.op) : plan::launch_kind_name(L.kind);
        launch_cost(b, L, p, t.bytes, t.flops);
        out.push_back(t);
    }
    NNC_CHECK(nncb_sync(ctx));
    for (size_t i = 0; i < out.size(); ++i) {
        float ms = 0;
        NNC_CHECK(nncb_event_elapsed_ms(evs[i], evs[i + 1], &ms));
        out[i].ms = ms;
    }
    for (void* e : evs) nncb_event_destroy(e);
    return out;
}

const ExecutionPlan& plan_for_inputs(const ExecutionPlan& p, const std::map<std::string, Tensor>& inputs,
                                     const std::map<int32_t, int64_t>& bindings) {
    if (p.vdims.empty() || !p.spec) return p;
    const auto b = call_binding(p, inputs, bindings);
    if (at_compiled_extents(p, b)) return p;
    return plan::Specializer::role_plan(p.spec->plans_for(b), p.role);
}

const plan::VersionPlans& plans_for_inputs(const plan::VersionPlans& plans, const std::map<std::string, Tensor>& inputs,
                                           const std::map<int32_t, int64_t>& bindings) {
    const ExecutionPlan& f = plans.train_fwd;
    if (f.vdims.empty() || !f.spec) return plans;
    const auto b = call_binding(f, inputs, bindings);
    if (at_compiled_extents(f, b)) return plans;
    return f.spec->plans_for(b);
}

std::map<std::string, Tensor> execute_on(const ExecutionPlan& p, const std::map<std::string, Tensor>& inputs,
                                         const HostModel& model, Device* device, const ExecOptions& opts) {
    Device& dev = device ? *device : default_device();
    const ExecutionPlan& q = opts.inputs_resident ? p : plan_for_inputs(p, inputs, opts.bindings);
    return run_plan(q, inputs, model, dev, opts, nullptr, nullptr);
}

std::map<std::string, Tensor> execute(const ExecutionPlan& p, const std::map<std::string, Tensor>& inputs,
                                      const HostModel& model, OffloadDevice* device, const ExecOptions& opts,
                                      ExecutionContext* shared_ctx) {
    Device& dev = device ? device->device() : default_device();
    const ExecutionPlan& q = plan_for_inputs(p, inputs, opts.bindings);
    return run_plan(q, inputs, model, dev, opts, device, shared_ctx);
}

void execute_stage(const ExecutionPlan& p, const std::map<std::string, Tensor>& inputs, Device* device) {
    Device& dev = device ? *device : default_device();
    check_inputs(p, inputs);
    auto& io = staged_ios()[{&dev, p.uid}];
    if (!io) {
        io = std::make_unique<StagedIO>();
        io->dev = &dev;
    }
    nncb_ctx* ctx = dev.ctx();
    StagedIO::Slot& S = io->slots[io->n_staged % 2];
    if (!S.ready) {
        for (uint32_t s : p.input_slots) {
            void* b = nullptr;
            NNC_CHECK(nncb_malloc(ctx, static_cast<size_t>(element_count(p.values[s].dims)) * dtype_size(p.dtype), &b));
            S.in.push_back(b);
        }
        NNC_CHECK(nncb_event_create(&S.ready));
        NNC_CHECK(nncb_event_create(&S.consumed));
    }
    if (S.used) NNC_CHECK(nncb_stream_wait(ctx, NNCB_STREAM_COPY, S.consumed));
    for (size_t k = 0; k < p.input_slots.size(); ++k) {
        const Tensor& t = inputs.at(p.values[p.input_slots[k]].name);
        NNC_CHECK(nncb_h2d_async(ctx, S.in[k], t.data(), t.byte_size()));
        dev.stats().h2d_bytes += t.byte_size();
    }
    NNC_CHECK(nncb_event_record_on(ctx, NNCB_STREAM_COPY, S.ready));
    ++io->n_staged;
}

void execute_launch_staged(const ExecutionPlan& p, const HostModel& model, Device* device, const ExecOptions& opts) {
    Device& dev = device ? *device : default_device();
    auto it = staged_ios().find({&dev, p.uid});
    if (it == staged_ios().end() || it->second->n_launched >= it->second->n_staged)
        throw Error(Error::Code::BadDocument, "execute_launch_staged: no staged inputs");
    StagedIO& io = *it->second;
    if (io.pending) throw Error(Error::Code::BadDocument, "execute_launch_staged: collect the previous outputs first");
    ExecCache& c = bound_cache(p, model, dev, opts);
    nncb_ctx* ctx = dev.ctx();
    StagedIO::Slot& S = io.slots[io.n_launched % 2];
    NNC_CHECK(nncb_stream_wait(ctx, NNCB_STREAM_COMPUTE, S.ready));
    for (size_t k = 0; k < p.input_slots.size(); ++k) {
        const auto& v = p.values[p.input_slots[k]];
        NNC_CHECK(nncb_d2d(ctx, c.prog->ptr(v.name), S.in[k], static_cast<size_t>(element_count(v.dims)) * dtype_size(p.dtype)));
    }
    NNC_CHECK(nncb_event_record_on(ctx, NNCB_STREAM_COMPUTE, S.consumed));
    S.used = true;
    run_bound(c, p, opts);
    // the outputs come back into pinned buffers asynchronously
    std::vector<std::string> names;
    std::vector<std::vector<int64_t>> dims;
    for (uint32_t s : p.output_slots) {
        const auto& v = p.values[s];
        if (opts.materialize && !opts.materialize->count(v.name)) continue;
        names.push_back(v.name);
        dims.push_back(v.dims);
    }
    if (names != io.out_names) {
        NNC_CHECK(nncb_sync(ctx));
        for (void* h : io.out_pinned) nncb_host_free(h);
        io.out_pinned.clear();
        for (const auto& d : dims) {
            void* h = nullptr;
            NNC_CHECK(nncb_host_alloc(std::max<size_t>(static_cast<size_t>(element_count(d)) * dtype_size(p.dtype), 16), &h));
            io.out_pinned.push_back(h);
        }
        io.out_names = names;
        io.out_dims = dims;
    }
    for (size_t k = 0; k < names.size(); ++k) {
        const size_t bytes = static_cast<size_t>(element_count(dims[k])) * dtype_size(p.dtype);
        NNC_CHECK(nncb_d2h_async(ctx, io.out_pinned[k], c.prog->ptr(names[k]), bytes));
        dev.stats().d2h_bytes += bytes;
    }
    if (!io.done) NNC_CHECK(nncb_event_create(&io.done));
    NNC_CHECK(nncb_event_record_on(ctx, NNCB_STREAM_COMPUTE, io.done));
    io.pending = true;
    ++io.n_launched;
}

std::map<std::string, Tensor> execute_staged_outputs(const ExecutionPlan& p, Device* device) {
    Device& dev = device ? *device : default_device();
    auto it = staged_ios().find({&dev, p.uid});
    if (it == staged_ios().end() || !it->second->pending)
        throw Error(Error::Code::BadDocument, "execute_staged_outputs: no launched run");
    StagedIO& io = *it->second;
    NNC_CHECK(nncb_event_sync(io.done));
    std::map<std::string, Tensor> out;
    for (size_t k = 0; k < io.out_names.size(); ++k) {
        Tensor t = Tensor::uninitialized(p.dtype, io.out_dims[k]);
        nncb_host_copy(t.data(), io.out_pinned[k], t.byte_size());
        out.emplace(io.out_names[k], std::move(t));
    }
    io.pending = false;
    return out;
}

/* ------------------------------------------------------------------ */
/*  Loss and update (host-tensor API, run on the device)               */
/* ------------------------------------------------------------------ */

L1Result l1_loss(const Tensor& pred, const Tensor& target) { return l1_loss_on(pred, target, nullptr); }

void sgd_step(HostModel& model, const std::map<std::string, Tensor>& grads, double lr) {
    sgd_step_on(model, grads, lr, nullptr);
}

L1Result l1_loss_on(const Tensor& pred, const Tensor& target, Device* device) {
    if (pred.dims() != target.dims() || pred.dtype() != target.dtype())
        throw Error(Error::Code::ShapeMismatch, "l1_loss: operand shapes differ");
    if (pred.dtype() != DType::F32) throw Error(Error::Code::ShapeMismatch, "l1_loss: the device computes f32 tensors");
    Device& dev = device ? *device : default_device();
    nncb_ctx* ctx = dev.ctx();
    size_t bytes = pred.byte_size();
    void *p = nullptr, *t = nullptr, *g = nullptr, *loss = nullptr;
    NNC_CHECK(nncb_malloc(ctx, std::max<size_t>(bytes, 16), &p));
    NNC_CHECK(nncb_malloc(ctx, std::max<size_t>(bytes, 16), &t));
    NNC_CHECK(nncb_malloc(ctx, std::max<size_t>(bytes, 16), &g));
    NNC_CHECK(nncb_malloc(ctx, 16, &loss));
    NNC_CHECK(nncb_h2d(ctx, p, pred.data(), bytes));
    NNC_CHECK(nncb_h2d(ctx, t, target.data(), bytes));
    NNC_CHECK(nncb_l1_loss(ctx, static_cast<float*>(p), static_cast<float*>(t), static_cast<float*>(g),
                           static_cast<double*>(loss), pred.elements()));
    L1Result r;
    r.grad = Tensor(pred.dtype(), pred.dims());
    NNC_CHECK(nncb_d2h(ctx, r.grad.data(), g, bytes));
    NNC_CHECK(nncb_d2h(ctx, &r.loss, loss, sizeof(double)));
    NNC_CHECK(nncb_sync(ctx));
    for (void* b : {p, t, g, loss}) nncb_free(ctx, b);
    return r;
}

L1Result softmax_ce_loss(const Tensor& pred, const Tensor& target, Device* device) {
    if (pred.dims() != target.dims() || pred.dtype() != target.dtype() || pred.dims().empty())
        throw Error(Error::Code::ShapeMismatch, "softmax_ce_loss: operand shapes differ");
    if (pred.dtype() != DType::F32) throw Error(Error::Code::ShapeMismatch, "softmax_ce_loss: the device computes f32 tensors");
    Device& dev = device ? *device : default_device();
    nncb_ctx* ctx = dev.ctx();
    const size_t bytes = pred.byte_size();
    void *p = nullptr, *t = nullptr, *g = nullptr, *loss = nullptr;
    NNC_CHECK(nncb_malloc(ctx, std::max<size_t>(bytes, 16), &p));
    NNC_CHECK(nncb_malloc(ctx, std::max<size_t>(bytes, 16), &t));
    NNC_CHECK(nncb_malloc(ctx, std::max<size_t>(bytes, 16), &g));
    NNC_CHECK(nncb_malloc(ctx, 16, &loss));
    NNC_CHECK(nncb_h2d(ctx, p, pred.data(), bytes));
    NNC_CHECK(nncb_h2d(ctx, t, target.data(), bytes));
    const int64_t C = pred.dims().back();
    NNC_CHECK(nncb_softmax_ce(ctx, static_cast<float*>(p), static_cast<float*>(t), static_cast<float*>(g),
                              static_cast<double*>(loss), pred.elements() / C, C));
    L1Result r;
    r.grad = Tensor(pred.dtype(), pred.dims());
    NNC_CHECK(nncb_d2h(ctx, r.grad.data(), g, bytes));
    NNC_CHECK(nncb_d2h(ctx, &r.loss, loss, sizeof(double)));
    NNC_CHECK(nncb_sync(ctx));
    for (void* b : {p, t, g, loss}) nncb_free(ctx, b);
    return r;
}

void sgd_step_on(HostModel& model, const std::map<std::string, Tensor>& grads, double lr, Device* device) {
    Device& dev = device ? *device : default_device();
    nncb_ctx* ctx = dev.ctx();
    for (const auto& [name, g] : grads) {
        if (!model.has(name)) throw Error(Error::Code::MissingGrad, "gradient for unknown weight " + name);
        Tensor w = model.tensor(name);
        if (w.dims() != g.dims()) throw Error(Error::Code::ShapeMismatch, name + ": gradient shape mismatch");
        if (w.dtype() != DType::F32 || g.dtype() != DType::F32)
            throw Error(Error::Code::ShapeMismatch, name + ": the device updates f32 tensors");
        size_t bytes = w.byte_size();
        void *wd = nullptr, *gd = nullptr;
        NNC_CHECK(nncb_malloc(ctx, std::max<size_t>(bytes, 16), &wd));
        NNC_CHECK(nncb_malloc(ctx, std::max<size_t>(bytes, 16), &gd));
        NNC_CHECK(nncb_h2d(ctx, wd, w.data(), bytes));
        NNC_CHECK(nncb_h2d(ctx, gd, g.data(), bytes));
        NNC_CHECK(nncb_sgd(ctx, static_cast<float*>(wd), static_cast<float*>(gd), w.elements(), lr, 1.0));
        NNC_CHECK(nncb_d2h(ctx, w.data(), wd, bytes));
        NNC_CHECK(nncb_sync(ctx));
        nncb_free(ctx, wd);
        nncb_free(ctx, gd);
        model.set(name, std::move(w));
    }
}

/* ------------------------------------------------------------------ */
/*  Trainer: the fused training step                                   */
/* ------------------------------------------------------------------ */

struct Trainer::Impl {
    const plan::VersionPlans* plans = nullptr;
    HostModel* model = nullptr;
    Device* dev = nullptr;
    ExecOptions opts;
    std::unique_ptr<Program> prog;
    std::string pred, dpred;
    std::vector<std::string> weights;                 // all parameters, region order
    std::map<std::string, int64_t> w_off, w_elems;    // element offsets in the flat regions
    int64_t region_elems = 0;
    void *params = nullptr, *grads = nullptr, *target = nullptr, *loss = nullptr;
    double* lr_dev = nullptr;                 // the learning rate the update kernels read
    double lr_written = std::nan("");
    void* graph = nullptr;
    void* graph_nosgd = nullptr;
    DpLayout layout;                                      // region order and all-reduce buckets
    // weights updated inside their weight-gradient call at G = 1 (the
    // reference's update fused into the backward, runtime.cpp:485-496), and
    // per bucket the element ranges the bucket update still covers
    std::set<std::string> fused_sgd;
    std::vector<std::vector<std::pair<int64_t, int64_t>>> bucket_rest;
    void* rest_ranges = nullptr;                 // device [offset, count] pairs of every bucket's rest
    std::vector<int64_t> rest_first, rest_max;   // per bucket: first pair index, largest count
    bool fused_planned = false;
    uint64_t launches_per_step = 0;
    bool warmed = false;
    // pipelined stepping (stage / launch_staged / staged_loss): two staging slots
    struct Slot {
        std::vector<void*> in;            // per train_fwd input slot, in input_slots order
        void* tgt = nullptr;
        void* ready = nullptr;            // copy stream: slot filled
        void* consumed = nullptr;         // compute stream: slot copied into the step's inputs
        bool used = false;
    };
    Slot slots[2];
    uint64_t n_staged = 0, n_launched = 0;
    double* loss_host = nullptr;          // pinned
    void* loss_ev = nullptr;

    bool model_dying = false;

    ~Impl() {
        try {
            if (!model_dying)
                dev->evict_model(*model);   // device-newer weights back to the host before the region goes
            else
                dev->forget_model(model->uid());
        } catch (...) {
        }
        if (graph) nncb_graph_destroy(graph);
        if (graph_nosgd) nncb_graph_destroy(graph_nosgd);
        nncb_ctx* ctx = dev->ctx();
        nncb_sync(ctx);
        for (Slot& s : slots) {
            for (void* p : s.in) nncb_free(ctx, p);
            if (s.tgt) nncb_free(ctx, s.tgt);
            for (void* e : {s.ready, s.consumed})
                if (e) nncb_event_destroy(e);
        }
        if (loss_ev) nncb_event_destroy(loss_ev);
        if (loss_host) nncb_host_free(loss_host);
        for (void* p : {params, grads, target, loss, static_cast<void*>(lr_dev), rest_ranges})
            if (p) nncb_free(ctx, p);
    }

    /// One training step on the compute stream. The update is issued per
    /// all-reduce bucket as soon as it is legal -- the bucket's gradients are
    /// final and no later backward launch reads its weights (DpBucket::
    /// update_launch) -- on the comm stream, so it overlaps the rest of the
    /// backward pass: at G > 1 it directly follows the bucket's all-reduce
    /// (a per-bucket post-all-reduce epilogue), at G = 1 it forks off the
    /// compute stream. The compute stream joins the comm stream at the end
    /// (before the next step's forward reads the weights). The learning rate
    /// is read from device memory, so the captured graph survives lr changes.
    /// G = 1: a weight whose gradient is written last by a weight-gradient
    /// GEMM, after every backward launch that reads the weight, is updated by
    /// that call (the update fused into its split-K fold); the bucket updates
    /// cover the remaining weights. NNC_NO_FUSED_SGD=1 keeps bucket updates only.
    void plan_fused_sgd() {
        fused_planned = true;
        fused_sgd.clear();
        if (!std::getenv("NNC_NO_FUSED_SGD") && prog->steps.size() > 1) {
            auto& bwd = prog->steps[1];
            for (const std::string& w : layout.weights) {
                const int64_t k = layout.grad_launch.count(w) ? layout.grad_launch.at(w) : -1;
                if (k < 0 || k >= static_cast<int64_t>(bwd.size())) continue;
                BoundLaunch& b = bwd[static_cast<size_t>(k)];
                if (b.skip || b.kind != LaunchKind::Gemm ||
                    (b.gemm.kind != NNCB_CONV_WGRAD && b.gemm.kind != NNCB_DENSE_WGRAD))
                    continue;
                float* g = static_cast<float*>(grads) + layout.offset.at(w);
                if (b.ptrs.back() != g) continue;   // the call writes this weight's final gradient
                auto rd = layout.read_launch.find(w);
                if (rd != layout.read_launch.end() && rd->second >= k) continue;   // a later launch reads the weights
                b.sgd_w = static_cast<float*>(params) + layout.offset.at(w);
                fused_sgd.insert(w);
            }
        }
        if (std::getenv("NNC_FUSED_SGD_DEBUG")) {
            int64_t fe = 0, te = 0;
            for (const std::string& w : layout.weights)
                if (layout.grad_launch.at(w) >= 0) {
                    te += layout.elements.at(w);
                    if (fused_sgd.count(w)) fe += layout.elements.at(w);
                }
            std::fprintf(stderr, "[fused sgd] %zu of %zu weights (%lld of %lld elements) updated in their weight-gradient call\n",
                         fused_sgd.size(), layout.weights.size(), (long long)fe, (long long)te);
        }
        bucket_rest.assign(layout.buckets.size(), {});
        for (size_t bi = 0; bi < layout.buckets.size(); ++bi) {
            const DpBucket& bk = layout.buckets[bi];
            int64_t cur = bk.offset;
            const int64_t end = bk.offset + bk.count;
            std::vector<std::pair<int64_t, int64_t>> gaps;   // fused weights' ranges inside the bucket
            for (const std::string& w : fused_sgd) {
                const int64_t o = layout.offset.at(w), n = (layout.elements.at(w) + 63) / 64 * 64;
                if (o < end && bk.offset < o + n) gaps.push_back({std::max(o, bk.offset), std::min(o + n, end)});
            }
            std::sort(gaps.begin(), gaps.end());
            for (const auto& [a, e] : gaps) {
                if (a > cur) bucket_rest[bi].push_back({cur, a - cur});
                cur = std::max(cur, e);
            }
            if (cur < end) bucket_rest[bi].push_back({cur, end - cur});
        }
        // one multi-range update launch per bucket: the ranges live on the device
        std::vector<int64_t> flat;
        rest_first.assign(layout.buckets.size(), 0);
        rest_max.assign(layout.buckets.size(), 0);
        for (size_t bi = 0; bi < bucket_rest.size(); ++bi) {
            rest_first[bi] = static_cast<int64_t>(flat.size() / 2);
            for (const auto& [o, n] : bucket_rest[bi]) {
                flat.push_back(o);
                flat.push_back(n);
                rest_max[bi] = std::max(rest_max[bi], n);
            }
        }
        nncb_ctx* ctx = dev->ctx();
        if (rest_ranges) nncb_free(ctx, rest_ranges);
        rest_ranges = nullptr;
        if (!flat.empty()) {
            NNC_CHECK(nncb_malloc(ctx, flat.size() * sizeof(int64_t), &rest_ranges));
            NNC_CHECK(nncb_h2d(ctx, rest_ranges, flat.data(), flat.size() * sizeof(int64_t)));
            NNC_CHECK(nncb_sync(ctx));
        }
    }

    void enqueue_step(bool do_sgd) {
        nncb_ctx* ctx = dev->ctx();
        prog->enqueue_plan(0, nullptr);
        enqueue_loss();
        const bool comm = nncb_comm_active(ctx) != 0;
        const double scale = 1.0 / static_cast<double>(dev->nranks());
        const bool fused = do_sgd && !comm && fused_planned;
        std::map<int64_t, std::vector<StepAction>> after;
        for (const StepAction& a : step_schedule(layout, comm, do_sgd)) after[a.after].push_back(a);
        auto issue = [&](const StepAction& a) {
            switch (a.kind) {
                case StepAction::Fork: NNC_CHECK(nncb_fork(ctx, NNCB_STREAM_COMM)); break;
                case StepAction::Join: NNC_CHECK(nncb_join(ctx, NNCB_STREAM_COMM)); break;
                case StepAction::AllReduce: {
                    const DpBucket& bk = layout.buckets[a.bucket];
                    NNC_CHECK(nncb_allreduce_sum_on_comm(ctx, static_cast<float*>(grads) + bk.offset, bk.count));
                    break;
                }
                case StepAction::Update: {
                    const DpBucket& bk = layout.buckets[a.bucket];
                    if (fused) {   // the weights not updated by their weight-gradient call, one launch
                        const size_t bi = static_cast<size_t>(a.bucket);
                        if (!bucket_rest[bi].empty())
                            NNC_CHECK(nncb_sgd_dev_ranges(
                                ctx, NNCB_STREAM_COMM, static_cast<float*>(params), static_cast<float*>(grads),
                                static_cast<const int64_t*>(rest_ranges) + 2 * rest_first[bi],
                                static_cast<int>(bucket_rest[bi].size()), rest_max[bi], lr_dev, scale));
                        break;
                    }
                    NNC_CHECK(nncb_sgd_dev(ctx, NNCB_STREAM_COMM, static_cast<float*>(params) + bk.offset,
                                           static_cast<float*>(grads) + bk.offset, bk.count, lr_dev, scale));
                    break;
                }
            }
        };
        prog->enqueue_plan(
            1, nullptr,
            [&](size_t k) {
                auto it = after.find(static_cast<int64_t>(k));
                if (it != after.end())
                    for (const StepAction& a : it->second) issue(a);
            },
            fused && !fused_sgd.empty() ? lr_dev : nullptr, scale);
    }

    /// The loss launch(es): prediction + target -> d.pred and the device loss.
    void enqueue_loss() {
        nncb_ctx* ctx = dev->ctx();
        const auto& pd = plans->train_fwd.values[plans->train_fwd.find_value(pred)].dims;
        const int64_t n = element_count(pd);
        if (opts.loss == LOSS_SOFTMAX_CE) {
            const int64_t C = pd.empty() ? 1 : pd.back();
            NNC_CHECK(nncb_softmax_ce(ctx, static_cast<float*>(prog->ptr(pred)), static_cast<float*>(target),
                                      static_cast<float*>(prog->ptr(dpred)), static_cast<double*>(loss), n / C, C));
        } else {
            NNC_CHECK(nncb_l1_loss(ctx, static_cast<float*>(prog->ptr(pred)), static_cast<float*>(target),
                                   static_cast<float*>(prog->ptr(dpred)), static_cast<double*>(loss), n));
        }
    }

    void sync_params() {
        // host-side edits (HostModel::set) since the last step: re-upload in place
        for (const std::string& w : weights)
            if (!model->device_newer.count(w) && dev->cached_stamp(*model, w) != model->stamp(w))
                dev->weight_buffer(*model, w, model->tensor(w), model->stamp(w));
    }

    void run(double lr, bool do_sgd) {
        nncb_ctx* ctx = dev->ctx();
        sync_params();
        if (do_sgd && !(lr == lr_written)) {   // stream-ordered before the step that reads it
            NNC_CHECK(nncb_set_f64(ctx, lr_dev, lr));
            lr_written = lr;
        }
        if (!opts.use_graphs || !warmed) {
            uint64_t before = nncb_launch_count(ctx);
            enqueue_step(do_sgd);
            NNC_CHECK(nncb_sync(ctx));
            if (do_sgd) launches_per_step = nncb_launch_count(ctx) - before;
            warmed = true;
        } else {
            void*& g = do_sgd ? graph : graph_nosgd;
            if (!g) {
                // the captured kernels are exactly what every replay launches
                // (the first eager step also ran the GEMM tile autotuner)
                const uint64_t before = nncb_launch_count(ctx);
                NNC_CHECK(nncb_capture_begin(ctx));
                enqueue_step(do_sgd);
                NNC_CHECK(nncb_capture_end(ctx, &g));
                if (do_sgd) launches_per_step = nncb_launch_count(ctx) - before;
            }
            NNC_CHECK(nncb_graph_launch(ctx, g));
        }
        if (do_sgd)
            for (const std::string& w : weights) {
                model->bump(w);
                dev->mark_device_newer(*model, w, model->stamp(w));
            }
    }
};

DpLayout dp_layout(const plan::VersionPlans& plans, HostModel& model, int64_t bucket_elems) {
    DpLayout L;
    std::map<std::string, std::string> grad_to_weight;
    for (const auto& [w, gv] : plans.weight_grads) grad_to_weight[gv] = w;
    const ExecutionPlan& bwd = plans.train_bwd;
    int64_t k = 0;
    for (const auto& es : bwd.exec_steps)
        for (uint32_t li : es.launches) {
            const auto& Lc = bwd.groups[es.group].launches[li];
            for (size_t a = 0; a < Lc.args.size(); ++a) {
                const plan::ValueEntry& v = bwd.values[Lc.args[a].slot];
                if (!Lc.is_out[a] && v.category == MemCategory::Parameter) L.read_launch[v.source_weight] = k;
                if (!Lc.is_out[a]) continue;
                auto it = grad_to_weight.find(v.name);
                if (it == grad_to_weight.end()) continue;
                if (!L.grad_launch.count(it->second)) L.weights.push_back(it->second);   // first production order
                L.grad_launch[it->second] = k;                                          // last write
            }
            ++k;
        }
    L.bwd_launches = k;
    for (const auto* p : {&plans.train_fwd, &plans.train_bwd})
        for (const std::string& w : p->weight_names)
            if (std::find(L.weights.begin(), L.weights.end(), w) == L.weights.end()) {
                L.weights.push_back(w);
                L.grad_launch[w] = -1;
            }
    int64_t trainable_end = 0;
    for (const std::string& w : L.weights) {
        const int64_t n = model.tensor(w).elements();
        L.offset[w] = L.region_elems;
        L.elements[w] = n;
        if (L.grad_launch[w] >= 0) trainable_end = L.region_elems + n;
        L.region_elems += (n + 63) / 64 * 64;   // 256-byte aligned tensors
    }
    for (int64_t off = 0; off < trainable_end; off += bucket_elems) {
        DpBucket b;
        b.offset = off;
        b.count = std::min(bucket_elems, trainable_end - off);
        for (const std::string& w : L.weights)
            if (L.grad_launch[w] >= 0 && L.offset[w] < off + b.count && off < L.offset[w] + L.elements[w]) {
                b.close_launch = std::max(b.close_launch, L.grad_launch[w]);
                auto rd = L.read_launch.find(w);
                b.update_launch = std::max(b.update_launch, rd == L.read_launch.end() ? int64_t(-1) : rd->second);
            }
        b.update_launch = std::max(b.update_launch, b.close_launch);
        L.buckets.push_back(b);
    }
    return L;
}

std::vector<StepAction> step_schedule(const DpLayout& layout, bool comm, bool do_sgd) {
    const int64_t last = std::max<int64_t>(layout.bwd_launches - 1, 0);
    auto at = [&](int64_t k) { return (k < 0 || k > last) ? last : k; };
    std::map<int64_t, std::vector<StepAction>> by;
    for (size_t b = 0; b < layout.buckets.size(); ++b) {
        const DpBucket& bk = layout.buckets[b];
        if (comm) by[at(bk.close_launch)].push_back({at(bk.close_launch), StepAction::AllReduce, static_cast<int64_t>(b)});
        if (do_sgd) by[at(bk.update_launch)].push_back({at(bk.update_launch), StepAction::Update, static_cast<int64_t>(b)});
    }
    std::vector<StepAction> out;
    for (auto& [k, acts] : by) {
        // all-reduces of a launch before its updates (a bucket's update follows
        // its own all-reduce on the in-order comm stream)
        std::stable_sort(acts.begin(), acts.end(), [](const StepAction& x, const StepAction& y) { return x.kind < y.kind; });
        out.push_back({k, StepAction::Fork, -1});
        out.insert(out.end(), acts.begin(), acts.end());
    }
    if (!out.empty()) out.push_back({last, StepAction::Join, -1});
    return out;
}

Trainer::Trainer(const plan::VersionPlans& plans, HostModel& model, Device& dev, const ExecOptions& opts)
    : impl(std::make_unique<Impl>()) {
    Impl& I = *impl;
    I.plans = &plans;
    I.model = &model;
    I.dev = &dev;
    I.opts = opts;
    if (plans.inference.output_slots.size() != 1)
        throw Error(Error::Code::BadDocument, "train_step expects exactly one prediction output");
    I.pred = plans.inference.values[plans.inference.output_slots[0]].name;
    I.dpred = "d." + I.pred;
    nncb_ctx* ctx = dev.ctx();
    // flat parameter / gradient regions and all-reduce buckets (dp_layout)
    I.layout = dp_layout(plans, model);
    I.weights = I.layout.weights;
    I.w_off = I.layout.offset;
    I.w_elems = I.layout.elements;
    I.region_elems = I.layout.region_elems;
    size_t region_bytes = static_cast<size_t>(std::max<int64_t>(I.region_elems, 64)) * 4;
    NNC_CHECK(nncb_malloc(ctx, region_bytes, &I.params));
    NNC_CHECK(nncb_malloc(ctx, region_bytes, &I.grads));
    NNC_CHECK(nncb_memset(ctx, I.params, 0, region_bytes));
    NNC_CHECK(nncb_memset(ctx, I.grads, 0, region_bytes));
    for (const std::string& w : I.weights) {
        const Tensor& t = model.tensor(w);
        void* home = static_cast<float*>(I.params) + I.w_off[w];
        NNC_CHECK(nncb_h2d(ctx, home, t.data(), t.byte_size()));
        dev.stats().h2d_bytes += t.byte_size();
        dev.stats().weight_bytes += t.byte_size();
        dev.adopt_weight(model, w, home, t.byte_size(), model.stamp(w));
    }
    const int64_t pred_elems = element_count(plans.train_fwd.values[plans.train_fwd.find_value(I.pred)].dims);
    NNC_CHECK(nncb_malloc(ctx, static_cast<size_t>(std::max<int64_t>(pred_elems, 4)) * 4, &I.target));
    NNC_CHECK(nncb_malloc(ctx, 64, &I.loss));
    {
        void* p = nullptr;
        NNC_CHECK(nncb_malloc(ctx, 64, &p));
        I.lr_dev = static_cast<double*>(p);
    }
    I.prog = std::make_unique<Program>();
    I.prog->dev = &dev;
    I.prog->plans = {&plans.train_fwd, &plans.train_bwd};
    I.prog->precision = opts.gemm_precision;
    I.prog->keep_values = opts.keep_values;
    std::map<std::string, std::string> weight_of_grad;
    for (const auto& [w, gv] : plans.weight_grads) weight_of_grad[gv] = w;
    I.prog->bind([&](const std::string& w) { return static_cast<void*>(static_cast<float*>(I.params) + I.w_off.at(w)); },
                 [&](const std::string& v) -> void* {
                     auto it = weight_of_grad.find(v);
                     if (it == weight_of_grad.end()) return nullptr;
                     return static_cast<float*>(I.grads) + I.w_off.at(it->second);
                 });
    I.plan_fused_sgd();   // before any capture (it uploads the bucket ranges); used only at G = 1
}

Trainer::~Trainer() = default;

std::vector<Trainer::LaunchTiming> Trainer::profile_step(double lr) {
    Impl& I = *impl;
    nncb_ctx* ctx = I.dev->ctx();
    I.sync_params();
    std::vector<LaunchTiming> out;
    std::vector<void*> evs;
    auto ev = [&]() {
        void* e = nullptr;
        NNC_CHECK(nncb_event_create(&e));
        NNC_CHECK(nncb_event_record(ctx, e));
        evs.push_back(e);
    };
    ev();
    for (size_t pi = 0; pi < 2; ++pi) {
        const ExecutionPlan& p = *I.prog->plans[pi];
        if (pi < I.prog->kmajor.size() && I.prog->kmajor[pi].n) {
            I.prog->plan_prologue(pi);
            ev();
            out.push_back({"kmajor_weights", "transpose", 0, 8.0 * 1024 * static_cast<double>(I.prog->kmajor[pi].tiles), 0});
        }
        for (size_t k = 0; k < I.prog->steps[pi].size(); ++k) {
            const BoundLaunch& b = I.prog->steps[pi][k];
            const Launch& L = *I.prog->sources[pi][k];
            if (b.skip) continue;
            enqueue(ctx, b);
            ev();
            LaunchTiming t;
            t.label = b.ew_prog.empty() ? L.label : L.label + "+bn_grad_reduce";
            t.kind = L.kind == LaunchKind::Gemm ? std::string("gemm:") + hlir::op_name(L.op) : plan::launch_kind_name(L.kind);
            launch_cost(b, L, p, t.bytes, t.flops);
            out.push_back(t);
        }
        if (pi == 0) {
            int64_t n = element_count(I.plans->train_fwd.values[I.plans->train_fwd.find_value(I.pred)].dims);
            I.enqueue_loss();
            ev();
            const char* lk = I.opts.loss == LOSS_SOFTMAX_CE ? "softmax_ce_loss" : "l1_loss";
            out.push_back({lk, lk, 0, 12.0 * n, 0});
        }
    }
    NNC_CHECK(nncb_sgd(ctx, static_cast<float*>(I.params), static_cast<float*>(I.grads), I.region_elems, lr,
                       1.0 / static_cast<double>(I.dev->nranks())));
    ev();
    out.push_back({"sgd", "sgd", 0, 12.0 * static_cast<double>(I.region_elems), 0});
    NNC_CHECK(nncb_sync(ctx));
    for (size_t i = 0; i < out.size(); ++i) {
        float ms = 0;
        NNC_CHECK(nncb_event_elapsed_ms(evs[i], evs[i + 1], &ms));
        out[i].ms = ms;
    }
    for (void* e : evs) nncb_event_destroy(e);
    for (const std::string& w : I.weights) {
        I.model->bump(w);
        I.dev->mark_device_newer(*I.model, w, I.model->stamp(w));
    }
    return out;
}

void Trainer::account(ExecutionContext& ctx) const {
    // train_fwd then train_bwd events at the context's alignment, values
    // carried across the boundary (reference train_step's shared context)
    const int64_t CA = std::max<int64_t>(ctx.alignment(), 1);
    for (const ExecutionPlan* p : impl->prog->plans)
        for (const plan::PlanEvent& ev : p->events) {
            const plan::ValueEntry& v = p->values[ev.slot];
            if (!ev.alloc) {
                ctx.release(v.name);
                continue;
            }
            if (ctx.live(v.name)) continue;
            const int64_t bytes = v.storage == StorageClass::Buffer
                                      ? plan::align_bytes(element_count(v.dims) * static_cast<int64_t>(dtype_size(p->dtype)), CA)
                                      : 0;
            auto w = impl->prog->where.find(v.name);
            ctx.adopt(v.name, w == impl->prog->where.end() ? nullptr : static_cast<uint8_t*>(w->second), bytes);
        }
}

void* Trainer::input_device_ptr(const std::string& name) { return impl->prog->ptr(name); }

Tensor Trainer::value(const std::string& name) {
    Impl& I = *impl;
    for (size_t pi = 0; pi < I.prog->plans.size(); ++pi) {
        const ExecutionPlan* p = I.prog->plans[pi];
        const int s = p->find_value(name);
        if (s < 0) continue;
        const plan::ValueEntry& v = p->values[s];
        if (v.storage != StorageClass::Buffer)
            throw Error(Error::Code::ShapeMismatch, name + " lives in registers of a fused group");
        Tensor t(p->dtype, v.dims);
        bool fed = false;   // a graph input (also when the plan saves it for backward)
        for (uint32_t is : p->input_slots) fed = fed || p->values[is].name == name;
        if (!fed && v.category != plan::MemCategory::Input && v.category != plan::MemCategory::Parameter) {
            bool written = false;
            for (size_t q = 0; q < I.prog->plans.size() && !written; ++q)
                written = I.prog->written_by_plan(q, static_cast<const char*>(I.prog->ptr(name)),
                                                  static_cast<int64_t>(t.byte_size()));
            if (!written)
                throw Error(Error::Code::ShapeMismatch, name + " is never written: its producer was fused into another launch");
        }
        NNC_CHECK(nncb_sync(I.dev->ctx()));
        NNC_CHECK(nncb_d2h(I.dev->ctx(), t.data(), I.prog->ptr(name), t.byte_size()));
        NNC_CHECK(nncb_sync(I.dev->ctx()));
        return t;
    }
    throw Error(Error::Code::ShapeMismatch, "no value " + name + " in the training step");
}
void* Trainer::target_device_ptr() { return impl->target; }
size_t Trainer::arena_bytes() const { return static_cast<size_t>(impl->prog->arena_bytes); }
uint64_t Trainer::launches_per_step() const { return impl->launches_per_step; }

MemoryReport Trainer::memory_report() const {
    MemoryReport r;
    r.arena_bytes = impl->prog->arena_bytes;
    r.live_high_water = impl->prog->live_high;
    r.estimate = plan::estimate_peak(*impl->plans, kAlign).training_bytes;
    return r;
}

MemoryReport memory_report(const ExecutionPlan& p, Device* device) {
    Device& dev = device ? *device : default_device();
    auto it = exec_caches().find({&dev, p.uid});
    if (it == exec_caches().end() || !it->second)
        throw Error(Error::Code::BadDocument, "memory_report: the plan has not been executed on this device");
    MemoryReport r;
    r.arena_bytes = it->second->prog->arena_bytes;
    r.live_high_water = it->second->prog->live_high;
    r.estimate = plan::plan_peak(p, kAlign);
    return r;
}

double Trainer::step(const std::map<std::string, Tensor>& inputs, const Tensor& target, double lr) {
    Impl& I = *impl;
    check_inputs(I.plans->train_fwd, inputs);
    nncb_ctx* ctx = I.dev->ctx();
    for (uint32_t s : I.plans->train_fwd.input_slots) {
        const std::string& name = I.plans->train_fwd.values[s].name;
        const Tensor& t = inputs.at(name);
        NNC_CHECK(nncb_h2d(ctx, I.prog->ptr(name), t.data(), t.byte_size()));
    }
    NNC_CHECK(nncb_h2d(ctx, I.target, target.data(), target.byte_size()));
    I.run(lr, true);
    double loss = 0;
    NNC_CHECK(nncb_d2h(ctx, &loss, I.loss, sizeof(double)));
    NNC_CHECK(nncb_sync(ctx));
    return loss;
}

void Trainer::step_device(double lr) { impl->run(lr, true); }

void Trainer::stage(const std::map<std::string, Tensor>& inputs, const Tensor& target) {
    Impl& I = *impl;
    const ExecutionPlan& p = I.plans->train_fwd;
    check_inputs(p, inputs);
    nncb_ctx* ctx = I.dev->ctx();
    Impl::Slot& S = I.slots[I.n_staged % 2];
    if (!S.ready) {
        for (uint32_t s : p.input_slots) {
            void* b = nullptr;
            NNC_CHECK(nncb_malloc(ctx, static_cast<size_t>(element_count(p.values[s].dims)) * 4, &b));
            S.in.push_back(b);
        }
        NNC_CHECK(nncb_malloc(ctx, std::max<size_t>(target.byte_size(), 16), &S.tgt));
        NNC_CHECK(nncb_event_create(&S.ready));
        NNC_CHECK(nncb_event_create(&S.consumed));
    }
    if (target.elements() != element_count(p.values[p.find_value(I.pred)].dims))
        throw Error(Error::Code::ShapeMismatch, "stage: target size differs from the prediction");
    if (S.used) NNC_CHECK(nncb_stream_wait(ctx, NNCB_STREAM_COPY, S.consumed));   // the step reading it has copied it out
    for (size_t k = 0; k < p.input_slots.size(); ++k) {
        const Tensor& t = inputs.at(p.values[p.input_slots[k]].name);
        NNC_CHECK(nncb_h2d_async(ctx, S.in[k], t.data(), t.byte_size()));
    }
    NNC_CHECK(nncb_h2d_async(ctx, S.tgt, target.data(), target.byte_size()));
    NNC_CHECK(nncb_event_record_on(ctx, NNCB_STREAM_COPY, S.ready));
    ++I.n_staged;
}

void Trainer::launch_staged(double lr) {
    Impl& I = *impl;
    if (I.n_launched >= I.n_staged) throw Error(Error::Code::BadDocument, "launch_staged: no staged step");
    const ExecutionPlan& p = I.plans->train_fwd;
    nncb_ctx* ctx = I.dev->ctx();
    Impl::Slot& S = I.slots[I.n_launched % 2];
    NNC_CHECK(nncb_stream_wait(ctx, NNCB_STREAM_COMPUTE, S.ready));
    for (size_t k = 0; k < p.input_slots.size(); ++k) {
        const std::string& name = p.values[p.input_slots[k]].name;
        NNC_CHECK(nncb_d2d(ctx, I.prog->ptr(name), S.in[k], static_cast<size_t>(element_count(p.values[p.input_slots[k]].dims)) * 4));
    }
    const int64_t n = element_count(p.values[p.find_value(I.pred)].dims);
    NNC_CHECK(nncb_d2d(ctx, I.target, S.tgt, static_cast<size_t>(n) * 4));
    NNC_CHECK(nncb_event_record_on(ctx, NNCB_STREAM_COMPUTE, S.consumed));
    S.used = true;
    I.run(lr, true);
    if (!I.loss_host) {
        void* h = nullptr;
        NNC_CHECK(nncb_host_alloc(sizeof(double), &h));
        I.loss_host = static_cast<double*>(h);
        NNC_CHECK(nncb_event_create(&I.loss_ev));
    }
    NNC_CHECK(nncb_d2h_async(ctx, I.loss_host, I.loss, sizeof(double)));
    NNC_CHECK(nncb_event_record_on(ctx, NNCB_STREAM_COMPUTE, I.loss_ev));
    ++I.n_launched;
}

double Trainer::staged_loss() {
    Impl& I = *impl;
    if (!I.loss_ev) throw Error(Error::Code::BadDocument, "staged_loss: no step launched");
    NNC_CHECK(nncb_event_sync(I.loss_ev));
    return *I.loss_host;
}

double Trainer::last_loss() {
    double loss = 0;
    NNC_CHECK(nncb_d2h(impl->dev->ctx(), &loss, impl->loss, sizeof(double)));
    NNC_CHECK(nncb_sync(impl->dev->ctx()));
    return loss;
}

namespace {
std::map<std::pair<uint64_t, uint64_t>, std::unique_ptr<Trainer>>& trainers() {
    static std::map<std::pair<uint64_t, uint64_t>, std::unique_ptr<Trainer>> m;
    return m;
}
}  // namespace

void forget_trainers_of(uint64_t model_uid) {
    for (auto it = trainers().begin(); it != trainers().end();) {
        if (it->first.second != model_uid) {
            ++it;
            continue;
        }
        if (it->second) it->second->impl->model_dying = true;
        it = trainers().erase(it);
    }
}

Trainer& shared_trainer(const plan::VersionPlans& plans, HostModel& model, Device& dev, const ExecOptions& opts) {
    auto& t = trainers()[{plans.train_fwd.uid, model.uid()}];
    if (!t || t->impl->dev != &dev) t = std::make_unique<Trainer>(plans, model, dev, opts);
    return *t;
}

void release(const plan::VersionPlans& plans) {
    for (auto it = exec_caches().begin(); it != exec_caches().end();) {
        uint64_t u = it->first.second;
        bool drop = u == plans.inference.uid || u == plans.train_fwd.uid || u == plans.train_bwd.uid;
        it = drop ? exec_caches().erase(it) : std::next(it);
    }
    for (auto it = trainers().begin(); it != trainers().end();)
        it = it->first.first == plans.train_fwd.uid ? trainers().erase(it) : std::next(it);
}

double train_step_on(const plan::VersionPlans& plans0, const std::map<std::string, Tensor>& inputs,
                     const Tensor& target, HostModel& model, double lr, Device* device, const ExecOptions& opts) {
    Device& dev = device ? *device : default_device();
    const plan::VersionPlans& plans = plans_for_inputs(plans0, inputs, opts.bindings);
    if (opts.trace)
        for (const char* ph : {"forward", "loss", "backward", "update"}) opts.trace->push_back(ph);
    return shared_trainer(plans, model, dev, opts).step(inputs, target, lr);
}

double train_step(const plan::VersionPlans& plans0, const std::map<std::string, Tensor>& inputs, const Tensor& target,
                  HostModel& model, double lr, OffloadDevice* device, const ExecOptions& opts,
                  ExecutionContext* shared_ctx) {
    Device& dev = device ? device->device() : default_device();
    const plan::VersionPlans& plans = plans_for_inputs(plans0, inputs, opts.bindings);
    if (plans.inference.output_slots.size() != 1)
        throw Error(Error::Code::BadDocument, "train_step expects exactly one prediction output");
    const int64_t A = std::max<int64_t>(opts.alignment, 1);
    auto aligned = [&](const Tensor& t) { return plan::align_bytes(static_cast<int64_t>(t.byte_size()), A); };
    if (device) {
        // the reference's cache protocol (runtime.cpp:388-397): every weight
        // whose cached stamp is stale crosses (after an update: all of them)
        for (const std::string& w : plans.train_fwd.weight_names)
            (void)device->sync_weight(w, model.tensor(w), model.stamp(w), aligned(model.tensor(w)));
        for (const auto& [k, t] : inputs) device->count_h2d(aligned(t));
    }
    if (opts.trace)
        for (const char* ph : {"forward", "loss", "backward", "update"}) opts.trace->push_back(ph);
    Trainer& tr = shared_trainer(plans, model, dev, opts);
    const double loss = tr.step(inputs, target, lr);
    if (device) {
        const std::string pred = plans.inference.values[plans.inference.output_slots[0]].name;
        device->count_d2h(aligned(target));   // the prediction (materialize = {pred})
        device->count_h2d(aligned(target));   // d.pred into the backward plan
        for (const auto& [w, gv] : plans.weight_grads) device->count_d2h(aligned(model.weights.at(w)));
    }
    model.sync();   // reference semantics: the host weights are the updated ones
    if (shared_ctx) tr.account(*shared_ctx);
    return loss;
}

std::map<std::string, Tensor> gradients(const plan::VersionPlans& plans0, const std::map<std::string, Tensor>& inputs,
                                        const Tensor& target, HostModel& model, double* loss, Device* device,
                                        const ExecOptions& opts) {
    Device& dev = device ? *device : default_device();
    const plan::VersionPlans& plans = plans_for_inputs(plans0, inputs, opts.bindings);
    Trainer& tr = shared_trainer(plans, model, dev, opts);
    Trainer::Impl& I = *tr.impl;
    check_inputs(plans.train_fwd, inputs);
    nncb_ctx* ctx = dev.ctx();
    for (uint32_t s : plans.train_fwd.input_slots) {
        const std::string& name = plans.train_fwd.values[s].name;
        const Tensor& t = inputs.at(name);
        NNC_CHECK(nncb_h2d(ctx, I.prog->ptr(name), t.data(), t.byte_size()));
    }
    NNC_CHECK(nncb_h2d(ctx, I.target, target.data(), target.byte_size()));
    I.run(0.0, false);
    std::map<std::string, Tensor> out;
    for (const auto& [w, gv] : plans.weight_grads) {
        Tensor t(DType::F32, model.tensor(w).dims());
        NNC_CHECK(nncb_d2h(ctx, t.data(), static_cast<float*>(I.grads) + I.w_off.at(w), t.byte_size()));
        out.emplace(w, std::move(t));
    }
    if (loss) NNC_CHECK(nncb_d2h(ctx, loss, I.loss, sizeof(double)));
    NNC_CHECK(nncb_sync(ctx));
    return out;
}

}  // namespace nnc::runtime
