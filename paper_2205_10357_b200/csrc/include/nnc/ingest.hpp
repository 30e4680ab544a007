// nnc/ingest.hpp -- model documents (DLB dialect) into the canonical NHWC graph.
// Follows reference core/include/nnc/ingest.hpp:67-107 / ingest.cpp:411-500 for
// the DLB ops the hot path uses, and its deterministic initializer
// (InitStream, ingest.cpp:43-70: U(+-1/sqrt(fan_in)) keyed by seed ^ fnv1a64(name)),
// so a document yields bit-identical weights in the reference and here.
// Extension ops: batch_normalization{epsilon}, gelu, layer_normalization{epsilon}.
#pragma once

#include <map>
#include <string>

#include "nnc/hlir.hpp"

namespace nnc::ingest {

struct Model {
    hlir::Graph graph;
    std::string name;
    uint64_t seed = 0;
};

/// Parses a DLB model document. `weights` (optional) overrides initializers by name.
Model parse_model(const std::string& document, const std::map<std::string, Tensor>* weights = nullptr);

uint64_t fnv1a64(const std::string& text);

class InitStream {
public:
    InitStream(uint64_t document_seed, const std::string& tensor_name);
    double uniform(double lo, double hi);
private:
    uint64_t state_;
};

}  // namespace nnc::ingest
