// backends.cpp -- B200 support table, assignment and convex grouping.
//
// group_layers reproduces the reference partition algorithm bit-exactly
// (backends.cpp:232-400): compute nodes in topo order; pass 1 joins each node
// to the latest (highest-index) adjacent same-backend group that stays convex;
// pass 2 merges touching same-backend group pairs (i<j, index order, restart
// after each merge) while convex. Convexity is the same predicate ("no dataflow
// path between two members leaves the set") evaluated on bitsets: the set's
// descendants outside the set must not reach back into it. This keeps the
// 400-node backward graphs of BatchNorm ResNets at milliseconds.
#include "nnc/backends.hpp"

#include <algorithm>
#include <unordered_map>

namespace nnc::backends {

using hlir::Graph;
using hlir::Node;
using hlir::OpKind;

const char* backend_name(BackendId b) {
    return b == BackendId::B200_GEMM ? "b200_gemm" : "b200_fused";
}

bool is_compute(OpKind op) { return op != OpKind::Input && op != OpKind::Const; }

bool is_gemm_op(OpKind op) {
    switch (op) {
        case OpKind::Conv2D:
        case OpKind::Dense:
        case OpKind::Conv2DGradInput:
        case OpKind::Conv2DGradWeight:
        case OpKind::DenseGradInput:
        case OpKind::DenseGradWeight: return true;
        default: return false;
    }
}

bool supports(BackendId b, OpKind op) {
    if (!is_compute(op)) return false;
    return b == BackendId::B200_GEMM ? is_gemm_op(op) : !is_gemm_op(op);
}

BackendAssignment default_assignment(const Graph& g) {
    BackendAssignment a;
    for (const Node& n : g.nodes)
        if (is_compute(n.op)) a[n.name] = is_gemm_op(n.op) ? BackendId::B200_GEMM : BackendId::B200_FUSED;
    return a;
}

namespace {

struct Bits {
    std::vector<uint64_t> w;
    explicit Bits(size_t n = 0) : w((n + 63) / 64, 0) {}
    void set(size_t i) { w[i >> 6] |= 1ull << (i & 63); }
    bool test(size_t i) const { return (w[i >> 6] >> (i & 63)) & 1; }
    bool intersects(const Bits& o) const {
        for (size_t k = 0; k < w.size(); ++k)
            if (w[k] & o.w[k]) return true;
        return false;
    }
    void operator|=(const Bits& o) {
        for (size_t k = 0; k < w.size(); ++k) w[k] |= o.w[k];
    }
};

struct Ctx {
    std::vector<std::string> order;
    std::vector<Bits> reach;       // reach[u]: nodes with a dataflow path from u
    std::vector<Bits> adj;         // undirected producer/consumer edges
    std::vector<int> backend;
};

Ctx build(const Graph& g, const std::map<std::string, int>& assignment) {
    Ctx c;
    for (const std::string& name : hlir::topo_order(g))
        if (is_compute(g.find_node(name)->op)) c.order.push_back(name);
    size_t n = c.order.size();
    c.reach.assign(n, Bits(n));
    c.adj.assign(n, Bits(n));
    c.backend.resize(n);
    std::unordered_map<std::string, int> producer;
    std::vector<const Node*> nodes(n);
    for (size_t i = 0; i < n; ++i) {
        nodes[i] = g.find_node(c.order[i]);
        auto it = assignment.find(c.order[i]);
        if (it == assignment.end()) throw Error(Error::Code::NoBackend, c.order[i] + ": unassigned node");
        c.backend[i] = it->second;
        for (const std::string& o : nodes[i]->outputs) producer[o] = static_cast<int>(i);
    }
    // ancestors in topo order; reach is the transpose, built at the end.
    std::vector<Bits> anc(n, Bits(n));
    for (size_t v = 0; v < n; ++v)
        for (const std::string& in : nodes[v]->inputs) {
            auto it = producer.find(in);
            if (it == producer.end()) continue;
            size_t u = static_cast<size_t>(it->second);
            c.adj[u].set(v);
            c.adj[v].set(u);
            anc[v].set(u);
            anc[v] |= anc[u];
        }
    for (size_t v = 0; v < n; ++v)
        for (size_t u = 0; u < n; ++u)
            if (anc[v].test(u)) c.reach[u].set(v);
    return c;
}

bool convex(const Ctx& c, const Bits& set) {
    size_t n = c.order.size();
    Bits below(n);
    for (size_t u = 0; u < n; ++u)
        if (set.test(u)) below |= c.reach[u];
    for (size_t w = 0; w < n; ++w)
        if (below.test(w) && !set.test(w) && c.reach[w].intersects(set)) return false;
    return true;
}

bool connected(const Ctx& c, const std::vector<int>& members) {
    if (members.size() <= 1) return true;
    size_t n = c.order.size();
    Bits in(n), seen(n);
    for (int m : members) in.set(m);
    std::vector<int> stack{members[0]};
    seen.set(members[0]);
    size_t visited = 0;
    while (!stack.empty()) {
        int u = stack.back();
        stack.pop_back();
        ++visited;
        for (size_t v = 0; v < n; ++v)
            if (in.test(v) && !seen.test(v) && c.adj[u].test(v)) {
                seen.set(v);
                stack.push_back(static_cast<int>(v));
            }
    }
    return visited == members.size();
}

std::vector<std::vector<int>> partition(const Ctx& c) {
    size_t n = c.order.size();
    std::vector<int> group_of(n, -1);
    std::vector<std::vector<int>> groups;
    auto as_bits = [&](const std::vector<int>& a, const std::vector<int>& b, int extra) {
        Bits s(n);
        for (int m : a) s.set(m);
        for (int m : b) s.set(m);
        if (extra >= 0) s.set(extra);
        return s;
    };
    for (size_t v = 0; v < n; ++v) {
        std::vector<int> cand;
        for (size_t u = 0; u < v; ++u)
            if (c.adj[u].test(v) && c.backend[u] == c.backend[v]) cand.push_back(group_of[u]);
        std::sort(cand.rbegin(), cand.rend());
        cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
        int joined = -1;
        for (int gi : cand)
            if (convex(c, as_bits(groups[gi], {}, static_cast<int>(v)))) {
                joined = gi;
                break;
            }
        if (joined >= 0) {
            groups[joined].push_back(static_cast<int>(v));
            group_of[v] = joined;
        } else {
            group_of[v] = static_cast<int>(groups.size());
            groups.push_back({static_cast<int>(v)});
        }
    }
    for (bool merged = true; merged;) {
        merged = false;
        for (size_t i = 0; i < groups.size() && !merged; ++i) {
            if (groups[i].empty()) continue;
            for (size_t j = i + 1; j < groups.size() && !merged; ++j) {
                if (groups[j].empty() || c.backend[groups[i][0]] != c.backend[groups[j][0]]) continue;
                bool touch = false;
                for (int a : groups[i])
                    for (int b : groups[j]) touch = touch || c.adj[a].test(b);
                if (!touch || !convex(c, as_bits(groups[i], groups[j], -1))) continue;
                groups[i].insert(groups[i].end(), groups[j].begin(), groups[j].end());
                std::sort(groups[i].begin(), groups[i].end());
                groups[j].clear();
                merged = true;
            }
        }
    }
    std::vector<std::vector<int>> out;
    for (auto& m : groups) {
        if (m.empty()) continue;
        if (!connected(c, m)) throw Error(Error::Code::UnsupportedInGroup, "grouping produced a disconnected group");
        out.push_back(m);
    }
    return out;
}

}  // namespace

std::vector<std::vector<std::string>> group_layers_ints(const Graph& g, const std::map<std::string, int>& a) {
    Ctx c = build(g, a);
    std::vector<std::vector<std::string>> out;
    for (const auto& m : partition(c)) {
        std::vector<std::string> names;
        for (int i : m) names.push_back(c.order[i]);
        out.push_back(std::move(names));
    }
    return out;
}

std::vector<FusionGroup> group_layers(const Graph& g, const BackendAssignment& assignment) {
    std::map<std::string, int> a;
    for (const auto& [name, b] : assignment) {
        const Node* n = g.find_node(name);
        if (n && !supports(b, n->op))
            throw Error(Error::Code::NoBackend, name + ": assigned backend does not support op");
        a[name] = static_cast<int>(b);
    }
    Ctx c = build(g, a);
    std::vector<FusionGroup> out;
    for (const auto& m : partition(c)) {
        FusionGroup fg;
        fg.id = static_cast<int>(out.size());
        fg.backend = static_cast<BackendId>(c.backend[m[0]]);
        for (int i : m) fg.members.push_back(c.order[i]);
        out.push_back(std::move(fg));
    }
    return out;
}

bool is_convex(const Graph& g, const std::vector<std::string>& members) {
    std::map<std::string, int> a;
    for (const Node& n : g.nodes)
        if (is_compute(n.op)) a[n.name] = 0;
    Ctx c = build(g, a);
    Bits s(c.order.size());
    for (const std::string& m : members) {
        auto it = std::find(c.order.begin(), c.order.end(), m);
        if (it == c.order.end()) throw Error(Error::Code::UnsupportedInGroup, "unknown member " + m);
        s.set(static_cast<size_t>(it - c.order.begin()));
    }
    return convex(c, s);
}

}  // namespace nnc::backends
