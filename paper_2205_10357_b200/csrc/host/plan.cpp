// plan.cpp -- grouped graph -> B200 execution plan.
//
// Structure follows reference plan.cpp:133-439: group execution order is the
// topological order of the group quotient DAG with ties broken by the smallest
// member position (order_groups, plan.cpp:38-83); the value table lists
// parameters, graph inputs, then node outputs in group order with the same
// MemCategory/resident rules (plan.cpp:185-283); one ExecStep per GEMM-group
// member and one per fused group (plan.cpp:357-370); allocs at production,
// frees at max(last use, production) (plan.cpp:372-437).
//
// The B200 lowering of a fused group (replacing plan.cpp:296-337) is
// depth-first: members run in topo order; maximal runs of elementwise members
// over one iteration space become ONE generated kernel whose interior values
// stay in registers (StorageClass::FusedRegister); BatchNorm statistics,
// pooling, row/column reductions and LayerNorm are reduction launches between
// runs. BatchNorm backward members that share (x, stats, g) are bundled: one
// reduction launch produces sum(g) and sum(g*xhat) straight into the dbeta /
// dgamma gradient buffers and the dx kernel reads them.
#include "nnc/plan.hpp"

#include <algorithm>
#include <atomic>
#include <set>
#include <unordered_map>
#include <unordered_set>

#include "nnc/geometry.hpp"
#include "nnc/passes.hpp"

namespace nnc::plan {

using backends::BackendId;
using backends::FusionGroup;
using hlir::Graph;
using hlir::Node;
using hlir::OpKind;

const char* category_name(MemCategory c) {
    switch (c) {
        case MemCategory::Parameter: return "parameter";
        case MemCategory::Input: return "input";
        case MemCategory::Output: return "output";
        case MemCategory::Intermediate: return "intermediate";
        case MemCategory::Saved: return "saved";
    }
    return "?";
}

const char* launch_kind_name(LaunchKind k) {
    switch (k) {
        case LaunchKind::Ew: return "ew";
        case LaunchKind::Gemm: return "gemm";
        case LaunchKind::MaxPool: return "maxpool";
        case LaunchKind::MaxPoolGrad: return "maxpool_grad";
        case LaunchKind::AvgPool: return "avgpool";
        case LaunchKind::AvgPoolGrad: return "avgpool_grad";
        case LaunchKind::SumRows: return "sum_rows";
        case LaunchKind::CumSum: return "cumsum";
        case LaunchKind::BnStats: return "bn_stats";
        case LaunchKind::BnGradReduce: return "bn_grad_reduce";
        case LaunchKind::LnFwd: return "ln_fwd";
        case LaunchKind::LnBwd: return "ln_bwd";
        case LaunchKind::LnDgamma: return "ln_dgamma";
    }
    return "?";
}

int ExecutionPlan::find_value(const std::string& name) const {
    for (size_t i = 0; i < values.size(); ++i)
        if (values[i].name == name) return static_cast<int>(i);
    return -1;
}

size_t ExecutionPlan::launch_count() const {
    size_t n = 0;
    for (const auto& g : groups) n += g.launches.size();
    return n;
}

namespace {

bool is_elementwise(const Node& n) {
    switch (n.op) {
        case OpKind::ReLU:
        case OpKind::ReluGrad:
        case OpKind::Add:
        case OpKind::Mul:
        case OpKind::Identity:
        case OpKind::Flatten:
        case OpKind::Unflatten:
        case OpKind::Gelu:
        case OpKind::GeluGrad:
        case OpKind::BatchNorm:            // apply part (stats launch precedes it)
        case OpKind::BatchNormGradInput:   // dx part (reduction launch precedes it)
            return true;
        default: return false;
    }
}

std::vector<size_t> order_groups(const Graph& g, const std::vector<FusionGroup>& groups) {
    std::unordered_map<std::string, size_t> member_group, node_pos, producer_group;
    auto topo = hlir::topo_order(g);
    for (size_t i = 0; i < topo.size(); ++i) node_pos[topo[i]] = i;
    for (size_t gi = 0; gi < groups.size(); ++gi)
        for (const std::string& m : groups[gi].members) member_group[m] = gi;
    for (const auto& fg : groups)
        for (const std::string& m : fg.members)
            for (const std::string& o : g.find_node(m)->outputs) producer_group[o] = member_group[m];
    size_t n = groups.size();
    std::vector<std::set<size_t>> succ(n);
    std::vector<int> indeg(n, 0);
    for (size_t gi = 0; gi < n; ++gi)
        for (const std::string& m : groups[gi].members)
            for (const std::string& in : g.find_node(m)->inputs) {
                auto it = producer_group.find(in);
                if (it != producer_group.end() && it->second != gi && succ[it->second].insert(gi).second) ++indeg[gi];
            }
    auto first_pos = [&](size_t gi) {
        size_t best = SIZE_MAX;
        for (const std::string& m : groups[gi].members) best = std::min(best, node_pos[m]);
        return best;
    };
    std::set<std::pair<size_t, size_t>> ready;
    for (size_t gi = 0; gi < n; ++gi)
        if (indeg[gi] == 0) ready.insert({first_pos(gi), gi});
    std::vector<size_t> order;
    while (!ready.empty()) {
        auto [pos, gi] = *ready.begin();
        ready.erase(ready.begin());
        order.push_back(gi);
        for (size_t s : succ[gi])
            if (--indeg[s] == 0) ready.insert({first_pos(s), s});
    }
    if (order.size() != n) throw Error(Error::Code::UnsupportedInGroup, "group DAG has a cycle (non-convex groups?)");
    return order;
}

struct Lowering {
    const Graph& g;
    ExecutionPlan& plan;
    std::unordered_map<std::string, uint32_t>& slot_of;
    std::unordered_map<std::string, std::vector<std::string>> consumers;   // value -> nodes
    std::unordered_set<std::string> keep;   // outputs / saved / grads: always stored

    uint32_t slot(const std::string& v) const {
        auto it = slot_of.find(v);
        if (it == slot_of.end()) throw Error(Error::Code::ShapeMismatch, "plan: unknown value " + v);
        return it->second;
    }
    const std::vector<int64_t>& dims(const std::string& v) const { return plan.values[slot(v)].dims; }

    uint32_t scratch(const std::string& name, std::vector<int64_t> d) {
        auto it = slot_of.find(name);
        if (it != slot_of.end()) return it->second;
        ValueEntry e;
        e.name = name;
        e.category = MemCategory::Intermediate;
        e.dims = std::move(d);
        uint32_t s = static_cast<uint32_t>(plan.values.size());
        plan.values.push_back(std::move(e));
        slot_of[name] = s;
        return s;
    }

    // ---- elementwise segment builder ------------------------------------
    struct Segment {
        std::vector<const Node*> members;
        int64_t elems = -1;
        int64_t channels = -1;
    };

    // stats_bn: instead of the segment's pass, emit a STATISTICS pass for the
    // training BatchNorm stats_bn whose input the segment computes: the chain
    // is evaluated from the group's inputs, nothing is stored, and
    // REDUCE_STATS writes mean / invstd into stats_slot; the segment stays open
    // (its values are recomputed by the pass that finally stores them).
    void flush(Segment& seg, GroupKernel& gk, const Node* stats_bn = nullptr, uint32_t stats_slot = 0) {
        if (seg.members.empty()) return;
        std::unordered_set<std::string> in_seg;
        for (const Node* n : seg.members) in_seg.insert(n->name);
        Launch L;
        L.kind = LaunchKind::Ew;
        L.elem_slot = slot(seg.members.front()->outputs[0]);
        std::map<std::pair<uint32_t, int64_t>, int32_t> arg_of;
        std::map<std::tuple<uint32_t, int64_t, int>, int32_t> reg_of_load;
        std::unordered_map<std::string, int32_t> reg_of_value;
        int32_t next_reg = 0;
        auto arg = [&](uint32_t s, int64_t off, bool out) {
            auto key = std::make_pair(s, off);
            auto it = arg_of.find(key);
            if (it != arg_of.end()) return it->second;
            int32_t a = static_cast<int32_t>(L.args.size());
            L.args.push_back({s, off});
            L.is_out.push_back(out);
            arg_of[key] = a;
            return a;
        };
        auto load = [&](uint32_t s, int64_t off, bool per_channel) {
            auto key = std::make_tuple(s, off, per_channel ? 1 : 0);
            auto it = reg_of_load.find(key);
            if (it != reg_of_load.end()) return it->second;
            nncb_ew_instr in{};
            in.op = per_channel ? NNCB_EW_LOAD_CH : NNCB_EW_LOAD;
            in.slot = arg(s, off, false);
            in.dst = next_reg++;
            L.ew.push_back(in);
            reg_of_load[key] = in.dst;
            return in.dst;
        };
        auto value = [&](const std::string& v) {
            auto it = reg_of_value.find(v);
            if (it != reg_of_value.end()) return it->second;
            int32_t r = load(slot(v), 0, false);
            reg_of_value[v] = r;
            return r;
        };
        auto weight_ch = [&](const std::string& w, int64_t off = 0) { return load(slot(w), off, true); };
        std::string label;
        for (const Node* n : seg.members) {
            label += (label.empty() ? "" : "+") + n->name;
            nncb_ew_instr in{};
            in.a = in.b = in.c = in.d = in.e = in.f = in.h = -1;
            switch (n->op) {
                case OpKind::ReLU: in.op = NNCB_EW_RELU; in.a = value(n->inputs[0]); break;
                case OpKind::ReluGrad:
                    in.op = NNCB_EW_RELU_GRAD; in.a = value(n->inputs[0]); in.b = value(n->inputs[1]);
                    break;
                case OpKind::Add: in.op = NNCB_EW_ADD; in.a = value(n->inputs[0]); in.b = value(n->inputs[1]); break;
                case OpKind::Mul: in.op = NNCB_EW_MUL; in.a = value(n->inputs[0]); in.b = value(n->inputs[1]); break;
                case OpKind::Identity:
                case OpKind::Flatten:
                case OpKind::Unflatten: in.op = NNCB_EW_COPY; in.a = value(n->inputs[0]); break;
                case OpKind::Gelu: in.op = NNCB_EW_GELU; in.a = value(n->inputs[0]); break;
                case OpKind::GeluGrad: in.op = NNCB_EW_GELU_GRAD; in.a = value(n->inputs[0]); in.b = value(n->inputs[1]); break;
                case OpKind::BatchNorm: {
                    int64_t C = dims(n->inputs[0]).back();
                    in.a = value(n->inputs[0]);
                    in.d = weight_ch(n->weights[0]);
                    in.e = weight_ch(n->weights[1]);
                    if (n->attrs.inference) {
                        in.op = NNCB_EW_BN_INFER;
                        in.b = weight_ch(n->weights[2]);
                        in.c = weight_ch(n->weights[3]);
                        in.imm = n->attrs.eps;
                    } else {
                        in.op = NNCB_EW_BN_APPLY;
                        uint32_t st = slot(stats_value(*n));
                        in.b = load(st, 0, true);
                        in.c = load(st, C, true);
                    }
                    break;
                }
                case OpKind::BatchNormGradInput: {
                    // inputs (x, stats, g), weight gamma
                    int64_t C = dims(n->inputs[0]).back();
                    const auto& sums = bn_bundle_sums.at(bundle_key(*n));
                    in.op = NNCB_EW_BN_GRAD;
                    in.a = value(n->inputs[0]);
                    in.b = value(n->inputs[2]);
                    uint32_t st = slot(n->inputs[1]);
                    in.c = load(st, 0, true);
                    in.d = load(st, C, true);
                    in.e = weight_ch(n->weights[0]);
                    in.f = load(sums.first, 0, true);
                    in.h = load(sums.second, 0, true);
                    in.imm = static_cast<double>(element_count(dims(n->inputs[0])) / C);
                    break;
                }
                default:
                    throw Error(Error::Code::UnsupportedInGroup, n->name + ": not elementwise-fusable");
            }
            in.dst = next_reg++;
            L.ew.push_back(in);
            reg_of_value[n->outputs[0]] = in.dst;
            // Store iff visible outside this segment.
            bool visible = keep.count(n->outputs[0]) > 0;
            auto cit = consumers.find(n->outputs[0]);
            if (cit == consumers.end() || cit->second.empty()) visible = true;
            else
                for (const std::string& c : cit->second)
                    if (!in_seg.count(c)) visible = true;
            uint32_t os = slot(n->outputs[0]);
            if (stats_bn) continue;   // statistics pass: nothing leaves registers
            if (visible) {
                nncb_ew_instr st{};
                st.op = NNCB_EW_STORE;
                st.a = in.dst;
                st.slot = arg(os, 0, true);
                L.ew.push_back(st);
                plan.values[os].storage = StorageClass::Buffer;
            } else {
                plan.values[os].storage = StorageClass::FusedRegister;
            }
        }
        if (stats_bn) {
            nncb_ew_instr red{};
            red.op = NNCB_EW_REDUCE_STATS;
            red.dst = red.b = red.c = red.d = red.e = red.f = red.h = -1;
            red.a = reg_of_value.at(stats_bn->inputs[0]);
            red.slot = arg(stats_slot, 0, true);
            red.imm = stats_bn->attrs.eps;
            L.ew.push_back(red);
            label += ".stats(" + stats_bn->name + ")";
        }
        L.ew_regs = next_reg;
        L.label = label;
        L.attrs.out_channels = seg.channels > 0 ? seg.channels : dims(seg.members.front()->outputs[0]).back();
        gk.launches.push_back(std::move(L));
        if (!stats_bn) seg = Segment{};
    }

    /// Recompute (instead of materialize) the input of a training BatchNorm
    /// that the open segment computes: a statistics pass re-evaluates the
    /// chain from the group inputs (SURVEY.md §8(d) C2 mode B: 4 barriers with
    /// recompute = 40 B/element instead of 64 when every barrier stores its
    /// input). Applies when the input is used only inside the group, is not
    /// kept for a backward pass, the chain reads few element-sized inputs, and
    /// the channel-stationary reduction can run.
    bool recompute_stats(const Segment& seg, const Node& bn, const std::unordered_set<std::string>& group_members) const {
        const std::string& x = bn.inputs[0];
        bool produced = false;
        std::unordered_set<std::string> outs, ext;
        for (const Node* m : seg.members) {
            produced = produced || m->outputs[0] == x;
            outs.insert(m->outputs[0]);
        }
        if (!produced || keep.count(x)) return false;
        auto cit = consumers.find(x);
        if (cit != consumers.end())
            for (const std::string& c : cit->second)
                if (!group_members.count(c)) return false;
        for (const Node* m : seg.members)
            for (const std::string& in : m->inputs)
                if (!outs.count(in) && element_count(dims(in)) == seg.elems) ext.insert(in);
        if (ext.size() > 3) return false;
        const int64_t C = dims(x).back(), e = element_count(dims(x));
        if (C < 4 || C > 2048 || (C & (C - 1)) || e % 4 != 0) return false;
        return std::getenv("NNC_NO_STATS_RECOMPUTE") == nullptr;
    }

    // ---- BatchNorm statistics / backward bundles --------------------------
    std::unordered_map<std::string, std::string> stats_of;   // bn node -> stats value
    std::string stats_value(const Node& n) const { return stats_of.at(n.name); }
    static std::string bundle_key(const Node& n) {
        return n.inputs[0] + "|" + n.inputs[1] + "|" + n.inputs[2];
    }
    std::map<std::string, std::pair<uint32_t, uint32_t>> bn_bundle_sums;  // key -> (sum_g, sum_gx)
    std::unordered_set<std::string> absorbed;                              // members lowered by a bundle

    Launch simple(LaunchKind k, const Node& n, std::vector<std::string> ins, std::vector<std::string> outs) {
        Launch L;
        L.kind = k;
        L.label = n.name;
        L.op = n.op;
        L.attrs = n.attrs;
        for (auto& v : ins) { L.args.push_back({slot(v), 0}); L.is_out.push_back(false); }
        for (auto& v : outs) { L.args.push_back({slot(v), 0}); L.is_out.push_back(true); }
        return L;
    }

    void lower_fused(GroupKernel& gk, const FusionGroup& fg) {
        std::vector<const Node*> mem;
        for (const std::string& m : fg.members) mem.push_back(g.find_node(m));
        // BatchNorm backward bundles: members sharing (x, stats, g). The
        // dgamma member and a SumNHW/SumCols(g) dbeta member are produced by
        // the bundle's single reduction launch.
        std::map<std::string, std::vector<const Node*>> bundles;
        for (const Node* n : mem)
            if (n->op == OpKind::BatchNormGradInput || n->op == OpKind::BatchNormGradGamma)
                bundles[bundle_key(*n)].push_back(n);
        std::map<std::string, std::string> bundle_of;   // member -> bundle key
        std::map<std::string, std::pair<std::string, std::string>> sum_values;  // key -> (sum_g, sum_gx)
        for (auto& [key, list] : bundles) {
            const Node* head = list.front();
            int64_t C = dims(head->inputs[0]).back();
            std::string sg, sgx;
            for (const Node* b : list) {
                bundle_of[b->name] = key;
                if (b->op == OpKind::BatchNormGradGamma && sgx.empty()) {
                    sgx = b->outputs[0];
                    absorbed.insert(b->name);
                }
            }
            // each bundle takes its own dbeta sum: BatchNorms fed the same gradient
            // (a residual join) have one SumNHW each, all equal to that bundle's sum_g
            for (const Node* n : mem)
                if ((n->op == OpKind::SumNHW || n->op == OpKind::SumCols) && n->inputs[0] == head->inputs[2] &&
                    sg.empty() && !absorbed.count(n->name)) {
                    sg = n->outputs[0];
                    bundle_of[n->name] = key;
                    absorbed.insert(n->name);
                }
            if (sg.empty()) scratch(sg = head->name + ".sum_g", {C});
            if (sgx.empty()) scratch(sgx = head->name + ".sum_gx", {C});
            sum_values[key] = {sg, sgx};
        }

        // Barriers whose inputs all come from outside the group -- training
        // BatchNorm statistics of a GEMM output, backward reductions of a
        // gradient produced elsewhere -- are hoisted to the head of the group,
        // so they do not split its elementwise segment: e.g. the projection
        // block's two BatchNorms, the add and the ReLU become ONE pass that
        // reads both GEMM outputs and writes the block output (the first BN's
        // result never leaves registers).
        std::unordered_set<std::string> produced_here, hoisted, member_names;
        for (const Node* n : mem) member_names.insert(n->name);
        for (const Node* n : mem)
            for (const std::string& o : n->outputs) produced_here.insert(o);
        for (const Node* n : mem) {
            if (n->op == OpKind::BatchNorm && !n->attrs.inference && !produced_here.count(n->inputs[0])) {
                int64_t C = dims(n->inputs[0]).back();
                std::string st = n->outputs.size() == 2 ? n->outputs[1] : n->name + ".stats";
                if (n->outputs.size() != 2) scratch(st, {2, C});
                stats_of[n->name] = st;
                // the statistics of a GEMM output stay a BnStats launch (the
                // runtime folds them into the GEMM epilogue); any other input
                // is reduced by a one-load statistics pass (channel-stationary,
                // 6.2 TB/s against 4.8 for the generic column reduction)
                const int p = g.producer_of(n->inputs[0]);
                const bool gemm_input = p >= 0 && (g.nodes[p].op == OpKind::Conv2D || g.nodes[p].op == OpKind::Dense);
                const int64_t e = element_count(dims(n->inputs[0]));
                if (!gemm_input && C >= 4 && C <= 2048 && !(C & (C - 1)) && e % 4 == 0 &&
                    !std::getenv("NNC_NO_STATS_RECOMPUTE")) {
                    Launch L;
                    L.kind = LaunchKind::Ew;
                    L.label = n->name + ".stats";
                    L.op = n->op;
                    L.args = {{slot(n->inputs[0]), 0}, {slot(st), 0}};
                    L.is_out = {false, true};
                    L.elem_slot = slot(n->inputs[0]);
                    nncb_ew_instr ld{};
                    ld.op = NNCB_EW_LOAD;
                    ld.a = ld.b = ld.c = ld.d = ld.e = ld.f = ld.h = -1;
                    ld.dst = 0;
                    ld.slot = 0;
                    nncb_ew_instr red{};
                    red.op = NNCB_EW_REDUCE_STATS;
                    red.dst = red.b = red.c = red.d = red.e = red.f = red.h = -1;
                    red.a = 0;
                    red.slot = 1;
                    red.imm = n->attrs.eps;
                    L.ew = {ld, red};
                    L.ew_regs = 1;
                    L.attrs.out_channels = C;
                    gk.launches.push_back(std::move(L));
                } else {
                    gk.launches.push_back(simple(LaunchKind::BnStats, *n, {n->inputs[0]}, {st}));
                }
                hoisted.insert(n->name);
            }
            auto bit = bundle_of.find(n->name);
            if (bit != bundle_of.end() && !bn_bundle_sums.count(bit->second)) {
                const Node* head = bundles[bit->second].front();
                bool outside = true;
                for (int k = 0; k < 3; ++k) outside = outside && !produced_here.count(head->inputs[k]);
                if (outside) {
                    auto [sg, sgx] = sum_values[bit->second];
                    gk.launches.push_back(simple(LaunchKind::BnGradReduce, *head,
                                                 {head->inputs[0], head->inputs[1], head->inputs[2]}, {sg, sgx}));
                    bn_bundle_sums[bit->second] = {slot(sg), slot(sgx)};
                }
            }
        }

        Segment seg;
        for (const Node* n : mem) {
            auto bit = bundle_of.find(n->name);
            if (bit != bundle_of.end() && !bn_bundle_sums.count(bit->second)) {
                flush(seg, gk);
                // (reducing every ready bundle here, so that several BatchNorm
                // grad-input members fed the same gradient share one pass, was
                // measured slower: the merged program carries ~13 per-channel
                // operands and ran at 4.4 TB/s against ~6 TB/s for two passes)
                const Node* head = bundles[bit->second].front();
                auto [sg, sgx] = sum_values[bit->second];
                gk.launches.push_back(simple(LaunchKind::BnGradReduce, *head,
                                             {head->inputs[0], head->inputs[1], head->inputs[2]}, {sg, sgx}));
                bn_bundle_sums[bit->second] = {slot(sg), slot(sgx)};
            }
            if (absorbed.count(n->name)) continue;
            if (n->op == OpKind::BatchNorm && !n->attrs.inference && !hoisted.count(n->name)) {
                int64_t C = dims(n->inputs[0]).back();
                std::string st = n->outputs.size() == 2 ? n->outputs[1] : n->name + ".stats";
                if (n->outputs.size() != 2) scratch(st, {2, C});
                stats_of[n->name] = st;
                if (recompute_stats(seg, *n, member_names)) {
                    flush(seg, gk, n, slot(st));   // statistics pass; the segment stays open
                } else {
                    flush(seg, gk);
                    gk.launches.push_back(simple(LaunchKind::BnStats, *n, {n->inputs[0]}, {st}));
                }
            }
            if (is_elementwise(*n)) {
                int64_t e = element_count(dims(n->outputs[0]));
                bool per_ch = n->op == OpKind::BatchNorm || n->op == OpKind::BatchNormGradInput;
                int64_t c = per_ch ? dims(n->inputs[0]).back() : -1;
                bool clash = !seg.members.empty() && (seg.elems != e || (per_ch && seg.channels > 0 && seg.channels != c));
                if (clash) flush(seg, gk);
                seg.members.push_back(n);
                seg.elems = e;
                if (per_ch) seg.channels = c;
                continue;
            }
            flush(seg, gk);
            switch (n->op) {
                case OpKind::MaxPool2D: {
                    std::vector<std::string> outs(n->outputs.begin(), n->outputs.end());
                    gk.launches.push_back(simple(LaunchKind::MaxPool, *n, {n->inputs[0]}, outs));
                    break;
                }
                case OpKind::MaxPool2DGrad:
                    gk.launches.push_back(simple(LaunchKind::MaxPoolGrad, *n, {n->inputs[0], n->inputs[1]}, {n->outputs[0]}));
                    break;
                case OpKind::AdaptiveAvgPool2D:
                    gk.launches.push_back(simple(LaunchKind::AvgPool, *n, {n->inputs[0]}, {n->outputs[0]}));
                    break;
                case OpKind::AdaptiveAvgPool2DGrad:
                    gk.launches.push_back(simple(LaunchKind::AvgPoolGrad, *n, {n->inputs[0]}, {n->outputs[0]}));
                    break;
                case OpKind::SumCols:
                case OpKind::SumNHW:
                    gk.launches.push_back(simple(LaunchKind::SumRows, *n, {n->inputs[0]}, {n->outputs[0]}));
                    break;
                case OpKind::CumSum:
                    gk.launches.push_back(simple(LaunchKind::CumSum, *n, {n->inputs[0]}, {n->outputs[0]}));
                    break;
                case OpKind::LayerNorm: {
                    Launch L = simple(LaunchKind::LnFwd, *n, {n->inputs[0], n->weights[0], n->weights[1]}, {n->outputs[0]});
                    gk.launches.push_back(std::move(L));
                    break;
                }
                case OpKind::LayerNormGradInput:
                    gk.launches.push_back(simple(LaunchKind::LnBwd, *n, {n->inputs[0], n->weights[0], n->inputs[1]}, {n->outputs[0]}));
                    break;
                case OpKind::LayerNormGradGamma:
                    gk.launches.push_back(simple(LaunchKind::LnDgamma, *n, {n->inputs[0], n->inputs[1]}, {n->outputs[0]}));
                    break;
                default:
                    throw Error(Error::Code::UnsupportedInGroup,
                                n->name + ": op " + hlir::op_name(n->op) + " has no B200 fused lowering");
            }
        }
        flush(seg, gk);
    }

    void lower_gemm(GroupKernel& gk, const FusionGroup& fg) {
        for (const std::string& m : fg.members) {
            const Node& n = *g.find_node(m);
            std::vector<std::string> ins(n.inputs.begin(), n.inputs.end());
            ins.insert(ins.end(), n.weights.begin(), n.weights.end());
            gk.launches.push_back(simple(LaunchKind::Gemm, n, ins, {n.outputs[0]}));
        }
    }
};

}  // namespace

uint64_t next_plan_uid() {
    static std::atomic<uint64_t> next_uid{1};
    return next_uid.fetch_add(1);
}

ExecutionPlan compile_plan(const Graph& input_graph, const std::vector<FusionGroup>& groups, PlanRole role,
                           const autodiff::VersionSet* versions) {
    Graph g = passes::infer_shapes(input_graph).graph;
    if ((role == PlanRole::TrainFwd || role == PlanRole::TrainBwd) && !versions)
        throw Error(Error::Code::BadDocument, "training plans need the version set");
    ExecutionPlan plan;
    plan.uid = next_plan_uid();
    plan.dtype = g.dtype;
    plan.role = role;
    std::unordered_map<std::string, uint32_t> slot_of;
    std::unordered_set<std::string> output_set(g.outputs.begin(), g.outputs.end());
    std::unordered_set<std::string> save_set, grad_outputs;
    if (versions && role != PlanRole::Inference) save_set.insert(versions->save_set.begin(), versions->save_set.end());
    if (versions && role == PlanRole::TrainBwd)
        for (const auto& [w, v] : versions->weight_grads) grad_outputs.insert(v);

    auto add_value = [&](ValueEntry e) {
        auto it = slot_of.find(e.name);
        if (it != slot_of.end()) return it->second;
        uint32_t s = static_cast<uint32_t>(plan.values.size());
        slot_of[e.name] = s;
        plan.values.push_back(std::move(e));
        return s;
    };
    auto dims_of = [&](const std::string& v) {
        const hlir::TensorType* t = g.type_of(v);
        if (!t) throw Error(Error::Code::ShapeMismatch, "plan: untyped value " + v);
        return t->shape.seed_dims();
    };

    // --- value table: parameters, inputs, node outputs in group order ----
    std::set<std::string> referenced;
    for (const Node& n : g.nodes) {
        for (const std::string& w : n.weights)
            if (n.op != OpKind::Const) referenced.insert(w);
        for (const std::string& in : n.inputs)
            if (g.initializers.count(in)) referenced.insert(in);
    }
    for (const std::string& o : g.outputs)
        if (g.initializers.count(o)) referenced.insert(o);
    for (const auto& [name, t] : g.initializers) {
        if (!referenced.count(name)) continue;
        ValueEntry e;
        e.name = name;
        e.category = MemCategory::Parameter;
        e.resident = true;
        e.source_weight = name;
        e.dims = t.dims();
        add_value(std::move(e));
        plan.weight_names.push_back(name);
    }
    for (const Node& n : g.nodes) {
        if (n.op != OpKind::Const) continue;
        ValueEntry e;
        e.name = n.outputs[0];
        e.category = MemCategory::Parameter;
        e.resident = true;
        e.source_weight = n.weights[0];
        e.dims = dims_of(n.outputs[0]);
        add_value(std::move(e));
        if (std::find(plan.weight_names.begin(), plan.weight_names.end(), n.weights[0]) == plan.weight_names.end())
            plan.weight_names.push_back(n.weights[0]);
    }
    for (const auto& gi : g.inputs) {
        ValueEntry e;
        e.name = gi.name;
        bool is_grad_in = versions && std::find(versions->output_grads.begin(), versions->output_grads.end(),
                                                gi.name) != versions->output_grads.end();
        if (role == PlanRole::TrainBwd)
            e.category = is_grad_in ? MemCategory::Input : MemCategory::Saved;
        else
            e.category = save_set.count(gi.name) ? MemCategory::Saved : MemCategory::Input;
        e.resident = output_set.count(gi.name) || (role != PlanRole::TrainBwd && save_set.count(gi.name));
        e.dims = gi.type.shape.seed_dims();
        plan.input_slots.push_back(add_value(std::move(e)));
    }
    auto group_order = order_groups(g, groups);
    for (size_t gi : group_order)
        for (const std::string& m : groups[gi].members)
            for (const std::string& o : g.find_node(m)->outputs) {
                ValueEntry e;
                e.name = o;
                bool grad_out = role == PlanRole::TrainBwd && grad_outputs.count(o);
                if (grad_out) e.category = MemCategory::Intermediate;
                else if (role == PlanRole::TrainFwd && save_set.count(o)) e.category = MemCategory::Saved;
                else if (output_set.count(o)) e.category = MemCategory::Output;
                else e.category = MemCategory::Intermediate;
                e.resident = output_set.count(o) || (role == PlanRole::TrainFwd && save_set.count(o)) || grad_out;
                e.dims = dims_of(o);
                add_value(std::move(e));
            }
    for (const std::string& o : g.outputs) plan.output_slots.push_back(slot_of.at(o));

    // --- lowering --------------------------------------------------------
    Lowering lw{g, plan, slot_of, {}, {}};
    for (const Node& n : g.nodes)
        for (const std::string& in : n.inputs) lw.consumers[in].push_back(n.name);
    lw.keep.insert(output_set.begin(), output_set.end());
    lw.keep.insert(save_set.begin(), save_set.end());
    lw.keep.insert(grad_outputs.begin(), grad_outputs.end());
    for (size_t step = 0; step < group_order.size(); ++step) {
        const FusionGroup& fg = groups[group_order[step]];
        GroupKernel gk;
        gk.id = static_cast<uint32_t>(step);
        gk.backend = fg.backend;
        gk.members = fg.members;
        for (const std::string& m : fg.members) gk.label += (gk.label.empty() ? "" : "+") + m;
        if (fg.backend == BackendId::B200_GEMM)
            lw.lower_gemm(gk, fg);
        else
            lw.lower_fused(gk, fg);
        plan.groups.push_back(std::move(gk));
    }

    // --- exec steps ------------------------------------------------------
    for (size_t gi = 0; gi < plan.groups.size(); ++gi) {
        const GroupKernel& gk = plan.groups[gi];
        if (gk.backend == BackendId::B200_FUSED) {
            ExecStep es{static_cast<uint32_t>(gi), -1, gk.label, {}};
            for (size_t k = 0; k < gk.launches.size(); ++k) es.launches.push_back(static_cast<uint32_t>(k));
            plan.exec_steps.push_back(std::move(es));
        } else {
            for (size_t k = 0; k < gk.launches.size(); ++k)
                plan.exec_steps.push_back({static_cast<uint32_t>(gi), static_cast<int32_t>(k), gk.members[k],
                                           {static_cast<uint32_t>(k)}});
        }
    }

    // --- static schedule -------------------------------------------------
    size_t nv = plan.values.size();
    std::vector<int32_t> prod_step(nv, 0), last_use(nv, 0);
    for (size_t si = 0; si < plan.exec_steps.size(); ++si) {
        const ExecStep& es = plan.exec_steps[si];
        int32_t s = static_cast<int32_t>(si) + 1;
        for (uint32_t li : es.launches) {
            const Launch& L = plan.groups[es.group].launches[li];
            for (size_t a = 0; a < L.args.size(); ++a) {
                uint32_t v = L.args[a].slot;
                if (L.is_out[a]) prod_step[v] = s;
                else last_use[v] = std::max(last_use[v], s);
            }
        }
    }
    for (uint32_t s = 0; s < nv; ++s)
        if (plan.values[s].category == MemCategory::Parameter) plan.events.push_back({0, true, s});
    for (uint32_t s : plan.input_slots) plan.events.push_back({0, true, s});
    for (uint32_t s : plan.input_slots)
        if (!plan.values[s].resident && last_use[s] == 0) plan.events.push_back({0, false, s});
    for (size_t si = 0; si < plan.exec_steps.size(); ++si) {
        const ExecStep& es = plan.exec_steps[si];
        int32_t s = static_cast<int32_t>(si) + 1;
        std::vector<uint32_t> allocs;
        for (uint32_t li : es.launches) {
            const Launch& L = plan.groups[es.group].launches[li];
            for (size_t a = 0; a < L.args.size(); ++a) {
                uint32_t v = L.args[a].slot;
                const ValueEntry& e = plan.values[v];
                if (L.is_out[a] && e.storage == StorageClass::Buffer && e.category != MemCategory::Parameter &&
                    e.category != MemCategory::Input && std::find(allocs.begin(), allocs.end(), v) == allocs.end())
                    allocs.push_back(v);
            }
        }
        for (uint32_t v : allocs) plan.events.push_back({s, true, v});
        for (uint32_t v = 0; v < nv; ++v) {
            const ValueEntry& e = plan.values[v];
            if (e.resident || e.storage != StorageClass::Buffer || e.category == MemCategory::Parameter) continue;
            if (std::max(last_use[v], prod_step[v]) == s) plan.events.push_back({s, false, v});
        }
    }
    return plan;
}

namespace {
// Enabled dims of the plan's graph inputs (Dim::sym after passes::bind_vdims).
void record_vdims(const Graph& g, ExecutionPlan& p) {
    for (const auto& gi : g.inputs) {
        const int s = p.find_value(gi.name);
        if (s < 0) continue;
        for (size_t a = 0; a < gi.type.shape.dims.size(); ++a) {
            const hlir::Dim& d = gi.type.shape.dims[a];
            if (d.is_sym())
                p.vdims.push_back({d.sym_id(), static_cast<uint32_t>(s), static_cast<uint32_t>(a), d.seed_extent()});
        }
    }
}
}  // namespace

VersionPlans compile_version_set(const autodiff::VersionSet& versions,
                                 const std::function<backends::BackendAssignment(const Graph&)>& assign) {
    VersionPlans out;
    auto build = [&](const Graph& g, PlanRole role) {
        ExecutionPlan p = compile_plan(g, backends::group_layers(g, assign(g)), role, &versions);
        record_vdims(g, p);
        return p;
    };
    out.inference = build(versions.inference, PlanRole::Inference);
    out.train_fwd = build(versions.train_fwd, PlanRole::TrainFwd);
    out.train_bwd = build(versions.train_bwd, PlanRole::TrainBwd);
    out.save_set = versions.save_set;
    out.output_grads = versions.output_grads;
    out.weight_grads = versions.weight_grads;
    if (!out.inference.vdims.empty() || !out.train_fwd.vdims.empty()) {
        auto spec = std::make_shared<const Specializer>(versions.source, assign);
        for (ExecutionPlan* p : {&out.inference, &out.train_fwd, &out.train_bwd}) p->spec = spec;
    }
    return out;
}

const VersionPlans& Specializer::plans_for(const std::map<int32_t, int64_t>& binding) const {
    std::lock_guard<std::mutex> lock(mu_);
    auto it = cache_.find(binding);
    if (it != cache_.end()) return *it->second;
    Graph g = source_;
    g.value_types.clear();
    for (auto& gi : g.inputs)
        for (hlir::Dim& d : gi.type.shape.dims)
            if (d.is_sym()) {
                auto b = binding.find(d.sym_id());
                d = hlir::Dim::fixed(b != binding.end() ? b->second : d.seed_extent());
            }
    autodiff::VersionSet vs = autodiff::derive_versions(passes::infer_shapes(g).graph);
    auto plans = std::make_unique<VersionPlans>(compile_version_set(vs, assign_));
    return *cache_.emplace(binding, std::move(plans)).first->second;
}

const ExecutionPlan& Specializer::role_plan(const VersionPlans& v, PlanRole r) {
    return r == PlanRole::Inference ? v.inference : r == PlanRole::TrainFwd ? v.train_fwd : v.train_bwd;
}

namespace {
int64_t value_bytes(const ExecutionPlan& p, uint32_t s, int64_t align) {
    const ValueEntry& e = p.values[s];
    if (e.storage != StorageClass::Buffer) return 0;
    return align_bytes(element_count(e.dims) * static_cast<int64_t>(dtype_size(p.dtype)), align);
}

// Replays events; `live` carries values across plans by name.
int64_t replay(const ExecutionPlan& p, int64_t align, std::map<std::string, int64_t>& live, int64_t& cur) {
    int64_t peak = cur;
    for (const PlanEvent& ev : p.events) {
        const std::string& name = p.values[ev.slot].name;
        if (ev.alloc) {
            if (live.count(name)) continue;
            int64_t b = value_bytes(p, ev.slot, align);
            live[name] = b;
            cur += b;
            peak = std::max(peak, cur);
        } else {
            auto it = live.find(name);
            if (it == live.end()) continue;
            cur -= it->second;
            live.erase(it);
        }
    }
    return peak;
}
}  // namespace

int64_t plan_peak(const ExecutionPlan& p, int64_t align) {
    std::map<std::string, int64_t> live;
    int64_t cur = 0;
    return replay(p, align, live, cur);
}

PeakEstimate estimate_peak(const VersionPlans& plans, int64_t align) {
    PeakEstimate e;
    e.inference_bytes = plan_peak(plans.inference, align);
    std::map<std::string, int64_t> live;
    int64_t cur = 0;
    int64_t p1 = replay(plans.train_fwd, align, live, cur);
    int64_t p2 = replay(plans.train_bwd, align, live, cur);
    e.training_bytes = std::max(p1, p2);
    return e;
}

}  // namespace nnc::plan
