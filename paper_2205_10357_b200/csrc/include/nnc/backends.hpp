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

std::vector<FusionGroup> group_layers(const hlir::Graph& g, const BackendAssignment& a);
/// Same algorithm over raw integer backends (for partition-parity tests).
std::vector<std::vector<std::string>> group_layers_ints(const hlir::Graph& g,
                                                        const std::map<std::string, int>& a);
bool is_convex(const hlir::Graph& g, const std::vector<std::string>& members);

}  // namespace nnc::backends
