// schedule.cpp -- static memory timelines (reference core/src/schedule.cpp:157-204
// semantics: prefix-sum replay of the plans' alloc/free events; a value already
// live -- carried across the training boundary -- is not allocated twice).
#include "nnc/schedule.hpp"

#include <algorithm>

namespace nnc::schedule {

namespace {

const plan::VersionPlans* specialised(const plan::ExecutionPlan& p, const std::map<int32_t, int64_t>* b) {
    if (!b || b->empty() || !p.spec) return nullptr;
    return &p.spec->plans_for(*b);
}

void replay(const plan::ExecutionPlan& p, int64_t align, std::map<std::string, int64_t>& live, int64_t& cur,
            MemoryTimeline& t, int32_t step_base) {
    for (const plan::PlanEvent& ev : p.events) {
        const plan::ValueEntry& v = p.values[ev.slot];
        MemoryEvent e;
        e.step = step_base + ev.step;
        e.value = v.name;
        e.category = v.category;
        if (ev.alloc) {
            if (live.count(v.name)) continue;
            e.bytes = v.storage == plan::StorageClass::Buffer
                          ? align_bytes(element_count(v.dims) * static_cast<int64_t>(dtype_size(p.dtype)), align)
                          : 0;
            live[v.name] = e.bytes;
            cur += e.bytes;
            if (cur > t.peak_bytes) {
                t.peak_bytes = cur;
                t.peak_step = e.step;
            }
        } else {
            auto it = live.find(v.name);
            if (it == live.end()) continue;
            e.kind = MemoryEvent::Kind::Free;
            e.bytes = it->second;
            cur -= it->second;
            live.erase(it);
        }
        t.events.push_back(std::move(e));
    }
}

}  // namespace

MemoryTimeline plan_timeline(const plan::ExecutionPlan& p, int64_t alignment, const std::map<int32_t, int64_t>* b) {
    if (const plan::VersionPlans* s = specialised(p, b)) return plan_timeline(plan::Specializer::role_plan(*s, p.role), alignment);
    MemoryTimeline t;
    std::map<std::string, int64_t> live;
    int64_t cur = 0;
    replay(p, alignment, live, cur, t, 0);
    t.resident_end_bytes = cur;
    return t;
}

MemoryTimeline training_timeline(const plan::VersionPlans& plans, int64_t alignment, const std::map<int32_t, int64_t>* b) {
    if (const plan::VersionPlans* s = specialised(plans.train_fwd, b)) return training_timeline(*s, alignment);
    MemoryTimeline t;
    std::map<std::string, int64_t> live;
    int64_t cur = 0;
    replay(plans.train_fwd, alignment, live, cur, t, 0);
    replay(plans.train_bwd, alignment, live, cur, t, static_cast<int32_t>(plans.train_fwd.exec_steps.size()) + 1);
    t.resident_end_bytes = cur;
    return t;
}

PeakEstimate estimate_peak(const plan::VersionPlans& plans, int64_t alignment, const std::map<int32_t, int64_t>* b) {
    PeakEstimate e;
    e.inference_bytes = plan_timeline(plans.inference, alignment, b).peak_bytes;
    e.training_bytes = training_timeline(plans, alignment, b).peak_bytes;
    return e;
}

}  // namespace nnc::schedule
