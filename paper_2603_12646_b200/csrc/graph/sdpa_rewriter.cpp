// sdpa_rewriter.cpp -- finds SDPA chains in the graph IR and replaces each with one
// FusedFlashAttention node: the operator-side half of the drop-in boundary.
//
// What must hold (reference proj/core/src/rewrite.cpp): the chain shape
//   Mul(Q, scalar) -> MatMul(., K^T) -> Add(., mask2d) -> Softmax(last axis) -> MatMul(., V)
// anchored on the Softmax (:124-231), intermediates with exactly one consumer that are not graph
// outputs (:118-123), a Transpose that swaps the last two axes folded into K (:189-197), the layer
// kind from a `layer_kind` attr on the Add / mask producer, else from "Where_1" (local) /
// "Where_2" (global) in the mask producer's name, never guessed (:203-207); the rewritten graph
// carries ONE shared chain pad_bias = Cast_f16((1 - attention_mask) * -65504) (:303-318), fused
// nodes [Q, K, V, pad_bias] with attrs scale / window_left / window_right, local w/2-1, w/2 and
// global -1, -1 (:349-362), then dead-code elimination (:233-263).  No [.., S, S] tensor survives.
#include <algorithm>
#include <cmath>
#include <limits>
#include <optional>
#include <unordered_map>
#include <unordered_set>

#include "routefast_b200/graph.hpp"

namespace routefast_b200 {

namespace {

// Producer / consumer lookup tables of one graph.
class GraphIndex {
public:
    explicit GraphIndex(const Graph& g) : g_(g) {
        for (std::size_t i = 0; i < g.nodes.size(); ++i) {
            for (const std::string& t : g.nodes[i].outputs) made_by_[t] = i;
            for (const std::string& t : g.nodes[i].inputs) ++uses_[t];
        }
        for (const Initializer& init : g.initializers) inits_[init.name] = &init;
        for (const std::string& t : g.outputs) outputs_.insert(t);
    }
    // index of the node that writes `tensor`, or npos for graph inputs / initializers
    static constexpr std::size_t npos = static_cast<std::size_t>(-1);
    std::size_t producer(const std::string& tensor) const {
        auto it = made_by_.find(tensor);
        return it == made_by_.end() ? npos : it->second;
    }
    const Node* producer_node(const std::string& tensor) const {
        const std::size_t i = producer(tensor);
        return i == npos ? nullptr : &g_.nodes[i];
    }
    // an intermediate the fusion may swallow: read by exactly one node and not a graph output
    bool private_to_one_reader(const std::string& tensor) const {
        auto it = uses_.find(tensor);
        return outputs_.count(tensor) == 0 && it != uses_.end() && it->second == 1;
    }
    // value of a one-element initializer or of a Constant node (`value` list of one, or `scalar`)
    std::optional<double> scalar(const std::string& tensor) const {
        if (auto it = inits_.find(tensor); it != inits_.end()) {
            if (it->second->data.size() == 1) return it->second->data[0];
            return std::nullopt;
        }
        const Node* n = producer_node(tensor);
        if (n == nullptr || n->op != OpKind::Constant) return std::nullopt;
        if (const std::vector<double>* vs = n->attr_reals("value"); vs != nullptr && vs->size() == 1) return (*vs)[0];
        const double s = n->attr_real("scalar", std::numeric_limits<double>::quiet_NaN());
        if (!std::isnan(s)) return s;
        return std::nullopt;
    }

private:
    const Graph& g_;
    std::unordered_map<std::string, std::size_t> made_by_;
    std::unordered_map<std::string, std::size_t> uses_;
    std::unordered_map<std::string, const Initializer*> inits_;
    std::unordered_set<std::string> outputs_;
};

bool swaps_last_two_axes(const std::vector<int64_t>& perm) {
    const int64_t rank = static_cast<int64_t>(perm.size());
    if (rank < 2) return false;
    for (int64_t i = 0; i + 2 < rank; ++i)
        if (perm[static_cast<std::size_t>(i)] != i) return false;
    return perm[static_cast<std::size_t>(rank - 2)] == rank - 1 && perm[static_cast<std::size_t>(rank - 1)] == rank - 2;
}

std::optional<LayerKind> kind_tag(const Node& node) {
    if (const std::string* s = node.attr_string("layer_kind")) {
        if (*s == "local") return LayerKind::local;
        if (*s == "global") return LayerKind::global;
    }
    return std::nullopt;
}

// the paper's naming convention for the mask construction nodes
std::optional<LayerKind> kind_from_mask_name(const std::string& name) {
    if (name.find("Where_2") != std::string::npos) return LayerKind::global;
    if (name.find("Where_1") != std::string::npos) return LayerKind::local;
    return std::nullopt;
}

// Tries to grow a full SDPA chain around the Softmax node `si`.
std::optional<PatternMatch> match_at_softmax(const Graph& g, const GraphIndex& ix, std::size_t si,
                                             const std::map<std::string, std::vector<int64_t>>& shapes) {
    const Node& sm = g.nodes[si];
    if (sm.op != OpKind::Softmax) return std::nullopt;
    {
        int64_t rank = 0;
        if (auto it = shapes.find(sm.inputs.at(0)); it != shapes.end()) rank = static_cast<int64_t>(it->second.size());
        const int64_t axis = sm.attr_int("axis", -1);
        if (!(axis == -1 || (rank > 0 && axis == rank - 1))) return std::nullopt;
    }
    // Softmax <- Add(scores, mask)
    const std::size_t add_i = ix.producer(sm.inputs.at(0));
    if (add_i == GraphIndex::npos || g.nodes[add_i].op != OpKind::Add) return std::nullopt;
    const Node& add = g.nodes[add_i];
    // Softmax -> first MatMul that takes the probabilities as its left operand
    std::size_t av_i = GraphIndex::npos;
    for (std::size_t i = 0; i < g.nodes.size(); ++i) {
        const Node& n = g.nodes[i];
        if (n.op == OpKind::MatMul && !n.inputs.empty() && n.inputs[0] == sm.outputs[0]) {
            av_i = i;
            break;
        }
    }
    if (av_i == GraphIndex::npos) return std::nullopt;
    if (!ix.private_to_one_reader(sm.outputs[0]) || !ix.private_to_one_reader(add.outputs[0])) return std::nullopt;

    // one Add operand is the QK^T MatMul, the other the 2-D mask
    std::size_t qk_i = GraphIndex::npos;
    std::string mask;
    for (std::size_t side = 0; side < 2; ++side) {
        const std::size_t cand = ix.producer(add.inputs.at(side));
        if (cand != GraphIndex::npos && g.nodes[cand].op == OpKind::MatMul) {
            qk_i = cand;
            mask = add.inputs.at(1 - side);
            break;
        }
    }
    if (qk_i == GraphIndex::npos) return std::nullopt;
    const Node& qk = g.nodes[qk_i];
    if (!ix.private_to_one_reader(qk.outputs[0])) return std::nullopt;

    // QK^T left operand: Mul(Q, scalar constant)
    const std::size_t mul_i = ix.producer(qk.inputs.at(0));
    if (mul_i == GraphIndex::npos || g.nodes[mul_i].op != OpKind::Mul) return std::nullopt;
    const Node& mul = g.nodes[mul_i];
    if (!ix.private_to_one_reader(mul.outputs[0])) return std::nullopt;
    std::optional<double> scale;
    std::string q;
    for (std::size_t side = 0; side < 2 && !scale; ++side) {
        if (auto s = ix.scalar(mul.inputs.at(side))) {
            scale = s;
            q = mul.inputs.at(1 - side);
        }
    }
    if (!scale) return std::nullopt;

    // right operand: K^T, either a graph tensor or Transpose(K) that we fold away
    std::string k = qk.inputs.at(1);
    bool k_is_transposed_tensor = true;
    if (const Node* kt = ix.producer_node(k); kt != nullptr && kt->op == OpKind::Transpose) {
        if (const std::vector<int64_t>* perm = kt->attr_ints("perm"); perm != nullptr && swaps_last_two_axes(*perm)) {
            k = kt->inputs.at(0);
            k_is_transposed_tensor = false;
        }
    }

    // layer kind: Add attr, then mask producer attr, then mask producer name; otherwise leave alone
    std::optional<LayerKind> kind = kind_tag(add);
    const Node* mask_node = ix.producer_node(mask);
    if (!kind && mask_node != nullptr) kind = kind_tag(*mask_node);
    if (!kind && mask_node != nullptr) kind = kind_from_mask_name(mask_node->name);
    if (!kind) return std::nullopt;

    PatternMatch m;
    m.scale_mul = mul_i;
    m.qk_matmul = qk_i;
    m.mask_add = add_i;
    m.softmax = si;
    m.av_matmul = av_i;
    m.q = std::move(q);
    m.k = std::move(k);
    m.v = g.nodes[av_i].inputs.at(1);
    m.mask = std::move(mask);
    m.k_pre_transposed = k_is_transposed_tensor;
    m.scale = *scale;
    m.kind = *kind;
    return m;
}

// a tensor / node name not yet used anywhere in `g`: base, base_1, base_2, ...
std::string fresh_name(const Graph& g, const std::string& base) {
    std::unordered_set<std::string> used;
    for (const Node& n : g.nodes) {
        used.insert(n.name);
        used.insert(n.outputs.begin(), n.outputs.end());
    }
    for (const Initializer& i : g.initializers) used.insert(i.name);
    for (const TensorDecl& i : g.inputs) used.insert(i.name);
    if (used.count(base) == 0) return base;
    for (int suffix = 1;; ++suffix) {
        std::string cand = base + "_" + std::to_string(suffix);
        if (used.count(cand) == 0) return cand;
    }
}

}  // namespace

std::vector<PatternMatch> find_sdpa_patterns(const Graph& graph) {
    const GraphIndex ix(graph);
    std::map<std::string, std::vector<int64_t>> shapes;
    try {
        shapes = infer_shapes(graph);
    } catch (const ValidationError&) {
        // ranks stay unknown; axis == -1 still identifies a last-axis Softmax
    }
    std::vector<PatternMatch> found;
    std::unordered_set<std::size_t> taken;  // nodes already part of a match: matches never overlap
    for (std::size_t si = 0; si < graph.nodes.size(); ++si) {
        if (taken.count(si)) continue;
        std::optional<PatternMatch> m = match_at_softmax(graph, ix, si, shapes);
        if (!m) continue;
        const std::size_t parts[5] = {m->softmax, m->mask_add, m->qk_matmul, m->scale_mul, m->av_matmul};
        if (std::any_of(parts + 1, parts + 5, [&](std::size_t p) { return taken.count(p) != 0; })) continue;
        taken.insert(parts, parts + 5);
        found.push_back(std::move(*m));
    }
    return found;
}

Graph dce(const Graph& graph) {
    std::unordered_map<std::string, std::size_t> made_by;
    for (std::size_t i = 0; i < graph.nodes.size(); ++i)
        for (const std::string& t : graph.nodes[i].outputs) made_by[t] = i;
    // backwards reachability from the graph outputs
    std::unordered_set<std::string> live_tensors;
    std::vector<bool> live_node(graph.nodes.size(), false);
    std::vector<std::string> stack(graph.outputs.begin(), graph.outputs.end());
    while (!stack.empty()) {
        std::string t = std::move(stack.back());
        stack.pop_back();
        if (!live_tensors.insert(t).second) continue;
        auto it = made_by.find(t);
        if (it == made_by.end() || live_node[it->second]) continue;
        live_node[it->second] = true;
        for (const std::string& in : graph.nodes[it->second].inputs) stack.push_back(in);
    }
    Graph out;
    out.inputs = graph.inputs;
    out.outputs = graph.outputs;
    for (std::size_t i = 0; i < graph.nodes.size(); ++i)
        if (live_node[i]) out.nodes.push_back(graph.nodes[i]);
    for (const Initializer& init : graph.initializers)
        if (live_tensors.count(init.name)) out.initializers.push_back(init);
    return out;
}

Graph rewrite(const Graph& graph, const RewriteOptions& options) {
    if (options.head_dim != 32 && options.head_dim != 64 && options.head_dim != 128)
        throw UnsupportedHeadDim("head_dim must be one of {32, 64, 128}, got " + std::to_string(options.head_dim));
    if (options.local_window < 2 || options.local_window % 2 != 0)
        throw std::invalid_argument("local_window must be even and >= 2");

    const std::vector<PatternMatch> matches = find_sdpa_patterns(graph);
    if (matches.empty()) return graph;

    const bool has_mask_input = std::any_of(graph.inputs.begin(), graph.inputs.end(),
                                            [&](const TensorDecl& d) { return d.name == options.mask_input; });
    if (!has_mask_input)
        throw NoAttentionMaskInput("graph has SDPA patterns but no '" + options.mask_input +
                                   "' input for the padding bias");

    const auto shapes = infer_shapes(graph);
    for (const PatternMatch& m : matches) {
        auto it = shapes.find(m.q);
        if (it != shapes.end() && !it->second.empty() && it->second.back() != options.head_dim)
            throw UnsupportedHeadDim("pattern at '" + graph.nodes[m.softmax].name + "' has head_dim " +
                                     std::to_string(it->second.back()) + ", expected " +
                                     std::to_string(options.head_dim));
    }

    Graph out;
    out.inputs = graph.inputs;
    out.outputs = graph.outputs;
    out.initializers = graph.initializers;

    // the shared pad-bias chain: ((1 - attention_mask) * -65504) cast to f16, O(B*S) for the whole graph
    const std::string one = fresh_name(graph, "pad_bias_one");
    const std::string negmax = fresh_name(graph, "pad_bias_negmax");
    const std::string inverted = fresh_name(graph, "pad_bias_inv");
    const std::string bias_f32 = fresh_name(graph, "pad_bias_f32");
    const std::string pad_bias = fresh_name(graph, "pad_bias");
    out.initializers.push_back(Initializer{one, {1}, DType::f32, {1.0}});
    out.initializers.push_back(Initializer{negmax, {1}, DType::f32, {-65504.0}});
    out.nodes.push_back(Node{inverted + "/Sub", OpKind::Sub, {one, options.mask_input}, {inverted}, {}});
    out.nodes.push_back(Node{bias_f32 + "/Mul", OpKind::Mul, {inverted, negmax}, {bias_f32}, {}});
    {
        Node cast{pad_bias + "/Cast", OpKind::Cast, {bias_f32}, {pad_bias}, {}};
        cast.attrs.emplace("to", std::string("f16"));
        out.nodes.push_back(std::move(cast));
    }

    // swallowed nodes disappear, the A*V MatMul position receives the fused node
    std::unordered_set<std::size_t> swallowed;
    std::unordered_map<std::size_t, const PatternMatch*> fuse_here;
    for (const PatternMatch& m : matches) {
        swallowed.insert({m.scale_mul, m.qk_matmul, m.mask_add, m.softmax});
        fuse_here[m.av_matmul] = &m;
    }
    for (std::size_t i = 0; i < graph.nodes.size(); ++i) {
        if (swallowed.count(i)) continue;
        auto hit = fuse_here.find(i);
        if (hit == fuse_here.end()) {
            out.nodes.push_back(graph.nodes[i]);
            continue;
        }
        const PatternMatch& m = *hit->second;
        std::string k_input = m.k;
        if (m.k_pre_transposed) {
            // only K^T exists as a tensor: hand the op a [B,H,S,d] view through one extra Transpose
            std::size_t rank = 4;
            if (auto it = shapes.find(m.k); it != shapes.end()) rank = it->second.size();
            std::vector<int64_t> perm(rank);
            for (std::size_t a = 0; a < rank; ++a) perm[a] = static_cast<int64_t>(a);
            std::swap(perm[rank - 1], perm[rank - 2]);
            k_input = m.k + "_rf_untransposed_" + std::to_string(i);
            Node untranspose{k_input + "/Transpose", OpKind::Transpose, {m.k}, {k_input}, {}};
            untranspose.attrs.emplace("perm", std::move(perm));
            out.nodes.push_back(std::move(untranspose));
        }
        const Node& av = graph.nodes[m.av_matmul];
        Node fused{av.name + "/FlashAttention", OpKind::FusedFlashAttention, {m.q, k_input, m.v, pad_bias}, av.outputs, {}};
        fused.attrs.emplace("scale", m.scale);
        const bool local = m.kind == LayerKind::local;
        fused.attrs.emplace("window_left", local ? options.local_window / 2 - 1 : int64_t{-1});
        fused.attrs.emplace("window_right", local ? options.local_window / 2 : int64_t{-1});
        out.nodes.push_back(std::move(fused));
    }
    return dce(out);
}

}  // namespace routefast_b200
