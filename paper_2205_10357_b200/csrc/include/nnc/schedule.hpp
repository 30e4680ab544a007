// nnc/schedule.hpp -- static memory timelines of compiled plans.
// Reference API kept (core/include/nnc/schedule.hpp:25-84): align_bytes,
// MemoryTimeline{peak_bytes, ...}, plan_timeline, training_timeline,
// estimate_peak. The runtime's ExecutionContext high water equals these
// estimates (the reference's invariant, test_runtime.cpp:195-240).
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "nnc/plan.hpp"

namespace nnc::schedule {

using plan::MemCategory;

inline int64_t align_bytes(int64_t bytes, int64_t alignment) { return (bytes + alignment - 1) / alignment * alignment; }

struct MemoryEvent {
    int32_t step = 0;
    enum class Kind : uint8_t { Alloc = 0, Free = 1 } kind = Kind::Alloc;
    std::string value;
    int64_t bytes = 0;   // aligned; 0 for values held in fused-group registers
    MemCategory category = MemCategory::Intermediate;
};

struct MemoryTimeline {
    std::vector<MemoryEvent> events;
    int64_t peak_bytes = 0;
    int32_t peak_step = 0;
    int64_t resident_end_bytes = 0;
};

/// Timeline of one plan at `alignment`; with `bindings` the plan is first
/// specialised for them (its dynamic dims bound).
MemoryTimeline plan_timeline(const plan::ExecutionPlan& p, int64_t alignment,
                             const std::map<int32_t, int64_t>* bindings = nullptr);

/// train_fwd then train_bwd: SaveSet values and parameters stay live across
/// the boundary, gradient buffers survive to the end.
MemoryTimeline training_timeline(const plan::VersionPlans& plans, int64_t alignment,
                                 const std::map<int32_t, int64_t>* bindings = nullptr);

using plan::PeakEstimate;
PeakEstimate estimate_peak(const plan::VersionPlans& plans, int64_t alignment,
                           const std::map<int32_t, int64_t>* bindings = nullptr);

}  // namespace nnc::schedule
