// nnc/backends.hpp -- the B200 backend's support table, assignment and grouping.
//
// The reference has a closed CPU backend enum {REF, FUSED_EW, GEMM_TILED}
// (backends.hpp:20). This backend replaces it with two device backends:
//   B200_FUSED (id 0): every non-contraction op (elementwise, BatchNorm, pooling,
//                      reductions, LayerNorm, ...) -> depth-first fused groups
//   B200_GEMM  (id 2): Conv2D/Dense and all their gradient contractions ->
//                      tcgen05/TMEM tensor-core GEMMs
// The ids equal the reference's REF / GEMM_TILED so that a B200 assignment of a
// forward graph is encodable in the reference for bit-exact partition parity.
// group_layers reproduces the reference algorithm exactly (backends.cpp:232-400):
// greedy join to the latest convex adjacent same-backend group, then pairwise
// merges in index order to a fixpoint.
#pragma once

#include <map>
#include <string>
#include <vector>

#include "nnc/hlir.hpp"

namespace nnc::backends {

enum class BackendId : uint8_t { B200_FUSED = 0, B200_GEMM = 2 };

const char* backend_name(BackendId b);
bool supports(BackendId b, hlir::OpKind op);
bool is_compute(hlir::OpKind op);
bool is_gemm_op(hlir::OpKind op);

using BackendAssignment = std::map<std::string, BackendId>;

/// GEMM ops -> B200_GEMM, everything else -> B200_FUSED (deterministic).
BackendAssignment default_assignment(const hlir::Graph& g);

struct FusionGroup {
    int id = 0;
    BackendId backend = BackendId::B200_FUSED;
    std::vector<std::string> members;   // topological order
};

/* ------------------------------------------------------------------ */
/*  Measured layer-wise tuning (reference backends.hpp:35-73,          */
/*  backends.cpp:73-176), with CUDA-event timings on the B200          */
/* ------------------------------------------------------------------ */

struct CostModel {
    enum class Kind { Measured, Injected };
    Kind kind = Kind::Measured;
    int warmup = 1;
    int trials = 5;
    /// (node, backend) -> cost; must be total over supporting backends.
    std::map<std::pair<std::string, BackendId>, double> injected;
    /// B200: the GEMM precision mode the contractions are timed in (nncb_precision)
    int gemm_precision = 0;

    static CostModel measured() { return {}; }
    static CostModel injected_from(std::map<std::pair<std::string, BackendId>, double> costs);
};

struct TuningRecord {
    std::string node;
    BackendId backend;
    double cost;     // microseconds (median device time); injected costs as given
    bool chosen;
    int32_t tile = 0;   // B200: the tensor-core tile code timed (0: default / not a GEMM)
};

struct TuningReport {
    /// node-major, backend enumeration order; a GEMM node measured on the
    /// device has one record per tensor-core tile candidate, the fastest chosen
    std::vector<TuningRecord> records;
    BackendAssignment assignment;
    /// GEMM nodes -> the chosen tile code (persisted into plans by
    /// plan::attach_tuning, serialized with them in SOLP)
    std::map<std::string, int32_t> tiles;

    std::string render_text() const;
    std::string render_csv() const;
};

/// Layer-by-layer: each compute node is timed in isolation on seed-shaped
/// random inputs on the default device (GEMM nodes: every tile candidate of
/// its contraction through nncb_gemm_time_tile; other nodes: their fused
/// lowering as a one-node plan) and assigned the cheapest supporting backend;
/// ties go to the lowest BackendId. Injected costs skip the device.
TuningReport tune_with_report(const hlir::Graph& g, const CostModel& cost);
BackendAssignment tune(const hlir::Graph& g, const CostModel& cost);

std::vector<FusionGroup> group_layers(const hlir::Graph& g, const BackendAssignment& a);
/// Same algorithm over raw integer backends (for partition-parity tests).
std::vector<std::vector<std::string>> group_layers_ints(const hlir::Graph& g,
                                                        const std::map<std::string, int>& a);
bool is_convex(const hlir::Graph& g, const std::vector<std::string>& members);

}  // namespace nnc::backends
