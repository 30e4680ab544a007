// nnc/autodiff.hpp -- derives inference / train_fwd / train_bwd versions.
// Mirrors reference core/include/nnc/autodiff.hpp:18-44 and follows its
// reverse-topological VJP walk and naming ("d.<value>.relu", "d.<weight>", ...,
// autodiff.cpp:120-212) so SaveSets and gradient names are identical for graphs
// in the reference vocabulary. Extension VJPs (BatchNorm, Gelu, LayerNorm) add
// argmax-style taps: a training BatchNorm grows a "<name>.stats" output [2, C].
#pragma once

#include <map>
#include <string>
#include <vector>

#include "nnc/hlir.hpp"

namespace nnc::autodiff {

struct VersionSet {
    hlir::Graph source;      // the graph the versions were derived from (re-specialisation)
    hlir::Graph inference;
    hlir::Graph train_fwd;
    hlir::Graph train_bwd;
    std::vector<std::string> save_set;
    std::vector<std::string> output_grads;
    std::map<std::string, std::string> weight_grads;
};

/// Conv2D/Dense weights and biases, BatchNorm/LayerNorm gamma+beta.
std::vector<std::string> trainable_weights(const hlir::Graph& g);

VersionSet derive_versions(const hlir::Graph& g);

}  // namespace nnc::autodiff
