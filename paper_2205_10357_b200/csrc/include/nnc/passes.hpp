// nnc/passes.hpp -- graph passes that run once before the hot path.
// Mirrors reference core/include/nnc/passes.hpp (infer_shapes :79, eliminate_dead
// :111, canonicalize :119, VdimBinding :81-95, bind_vdims :101, optimize :126).
// Symbolic input dims ("shape": null + "seed_shape" in a DLB document) are
// reported as free vdims #0, #1, ... in order of appearance and bound per the
// VdimBinding (passes.cpp:520-560): Disable (default) collapses to the seed,
// Override substitutes an extent, Enable keeps the dim dynamic -- the plans are
// compiled at the seed and the runtime re-specialises them per call binding
// (runtime::execute, reference runtime.cpp:318-360).
#pragma once

#include <initializer_list>
#include <map>

#include "nnc/hlir.hpp"

namespace nnc::passes {

struct ShapeInfo {
    hlir::Graph graph;
};

/// Annotates every value with a TensorType (fixed extents). Throws
/// Error{RankError, ExtentMismatch, ShapeMismatch} like the reference rules
/// (passes.cpp:168-400), plus rules for the extension ops.
ShapeInfo infer_shapes(const hlir::Graph& g);

/// Keeps exactly the nodes backward-reachable from graph outputs (passes.cpp:574-620).
hlir::Graph eliminate_dead(const hlir::Graph& g);

/// Splices interior Identity nodes and collapses Flatten chains (passes.cpp:704-781).
hlir::Graph canonicalize(const hlir::Graph& g);

struct VdimReport {
    struct FreeSym {
        int32_t id;        // dense report id (#0, #1, ...)
        int64_t seed;      // extent observed at ingest
    };
    std::vector<FreeSym> free_syms;
    std::map<int32_t, int32_t> report_id;   // graph sym id -> report id
    bool is_free(int32_t graph_sym) const { return report_id.count(graph_sym) != 0; }
};

/// Every symbolic dim of the graph inputs is free here (all axes the DLB
/// documents mark dynamic are batch axes; the reference's structural-fixing
/// analysis of infer_vdims is not restated).
VdimReport infer_vdims(const hlir::Graph& g);

struct VdimBinding {
    enum class Action { Enable, Disable, Override };
    struct Item {
        Action action = Action::Disable;
        int64_t extent = 0;   // Override only
    };
    std::map<int32_t, Item> items;   // keyed by report id

    static VdimBinding all_disable() { return {}; }
    static VdimBinding enable(std::initializer_list<int32_t> ids);
};

/// Resolves free symbols per the binding (UnknownSymbol / IllegalOverride as the
/// reference) and re-infers shapes; Enabled dims stay Dim::sym(report id, seed).
hlir::Graph bind_vdims(const hlir::Graph& g, const VdimReport& report, const VdimBinding& binding);

struct OptimizeResult {
    hlir::Graph graph;
    VdimReport report;
};

/// canonicalize -> eliminate_dead -> infer_vdims -> bind_vdims (-> infer_shapes).
OptimizeResult optimize(const hlir::Graph& g, const VdimBinding& binding = {});

}  // namespace nnc::passes
