// nnc/passes.hpp -- graph passes that run once before the hot path.
// Mirrors reference core/include/nnc/passes.hpp (infer_shapes :79, eliminate_dead
// :111, canonicalize :119, optimize :126). This backend binds every symbolic dim
// to its seed at optimize time (the reference's all-Disable binding,
// passes.cpp:520-560); per-call batch rebinding is not supported.
#pragma once

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

struct OptimizeResult {
    hlir::Graph graph;
};

/// canonicalize -> eliminate_dead -> bind symbols to seeds -> infer_shapes.
OptimizeResult optimize(const hlir::Graph& g);

}  // namespace nnc::passes
