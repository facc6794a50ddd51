// routefast_b200/graph.hpp -- graph IR, SDPA -> FusedFlashAttention rewriter and GPU graph
// executor: the C++ mirror of the reference's operator boundary
//   proj/core/include/routefast/graph.hpp:17-105      (IR, parse/serialize/validate/topo/shapes)
//   proj/core/include/routefast/rewrite.hpp:14-63     (find_sdpa_patterns, rewrite, dce)
//   proj/core/include/routefast/interpreter.hpp:14-25 (interpret)
// Same names, argument meaning and error types; the implementation is this build's own
// (librf_fa.so).  `interpret` runs every one of the 11 ops on the B200: the un-rewritten graph
// materialises its [B,H,S,S] tensors in HBM with plain CUDA kernels, the rewritten one
// dispatches FusedFlashAttention to the tcgen05 kernel -- so `verify-rewrite`
// (proj/tools/main.cpp:106-149) runs original-vs-rewritten on the GPU.
// There is no CPU fallback: without a CUDA device `interpret` throws std::runtime_error.
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <string_view>
#include <variant>
#include <vector>

#include "attention.hpp"

namespace routefast_b200 {

class SchemaError : public std::runtime_error {  // graph.hpp:17-20
public:
    using std::runtime_error::runtime_error;
};
class ValidationError : public std::runtime_error {  // graph.hpp:23-26
public:
    using std::runtime_error::runtime_error;
};
class NoAttentionMaskInput : public std::runtime_error {  // rewrite.hpp:19-22
public:
    using std::runtime_error::runtime_error;
};
class UnsupportedOp : public std::runtime_error {  // interpreter.hpp:14-17
public:
    using std::runtime_error::runtime_error;
};

std::string_view dtype_name(DType dtype);
DType dtype_from_name(std::string_view name);  // throws SchemaError

enum class OpKind {  // graph.hpp:33-45
    MatMul, Add, Sub, Mul, Softmax, Transpose, Cast, Where, Expand, Constant, FusedFlashAttention,
};
std::string_view op_name(OpKind op);
OpKind op_from_name(std::string_view name);  // throws SchemaError

using AttrValue = std::variant<int64_t, double, std::string, std::vector<int64_t>, std::vector<double>>;

struct TensorDecl {
    std::string name;
    std::vector<int64_t> shape;
    DType dtype = DType::f32;
};

struct Node {
    std::string name;
    OpKind op = OpKind::Constant;
    std::vector<std::string> inputs;
    std::vector<std::string> outputs;
    std::map<std::string, AttrValue> attrs;

    int64_t attr_int(std::string_view key, int64_t fallback) const;
    double attr_real(std::string_view key, double fallback) const;
    const std::vector<int64_t>* attr_ints(std::string_view key) const;
    const std::vector<double>* attr_reals(std::string_view key) const;
    const std::string* attr_string(std::string_view key) const;
};

struct Initializer {
    std::string name;
    std::vector<int64_t> shape;
    DType dtype = DType::f32;
    std::vector<double> data;  // row-major
};

struct Graph {  // single assignment: one producer per tensor name
    std::vector<TensorDecl> inputs;
    std::vector<std::string> outputs;
    std::vector<Node> nodes;
    std::vector<Initializer> initializers;
};

Graph parse_graph(std::string_view json_text);     // parses and validates
std::string serialize_graph(const Graph& graph);   // deterministic, byte-compatible with the reference
void validate_graph(const Graph& graph);           // throws ValidationError
std::vector<std::size_t> topological_order(const Graph& graph);  // stable Kahn, lowest index first
std::map<std::string, std::vector<int64_t>> infer_shapes(const Graph& graph);

// ---- rewriter (rewrite.hpp) ----
enum class LayerKind { local, global };

struct PatternMatch {  // Mul(Q, scale) -> MatMul(., K^T) -> Add(., mask) -> Softmax -> MatMul(., V)
    std::size_t scale_mul = 0, qk_matmul = 0, mask_add = 0, softmax = 0, av_matmul = 0;
    std::string q, k, v, mask;
    bool k_pre_transposed = false;
    double scale = 0.0;
    LayerKind kind = LayerKind::global;
};
std::vector<PatternMatch> find_sdpa_patterns(const Graph& graph);

struct RewriteOptions {  // rewrite.hpp:49-53
    int64_t head_dim = 64;
    int64_t local_window = 128;
    std::string mask_input = "attention_mask";
};
Graph rewrite(const Graph& graph, const RewriteOptions& options);
Graph dce(const Graph& graph);

// ---- executor (interpreter.hpp) ----
using TensorMap = std::map<std::string, Tensor>;

struct InterpretStats {
    std::size_t peak_device_bytes = 0;   // high-water mark of live graph tensors in HBM
    std::size_t launches = 0;            // kernels launched (FusedFlashAttention counts its own)
    std::size_t largest_tensor_bytes = 0;
    double device_ms = 0.0;              // CUDA-event time of the node loop (no host copies)
};

// Host tensors in, host tensors out (the reference's calling convention); every node runs on
// `device`.  Cast(f16) applies binary16 round-trip quantisation (RNE), MatMul accumulates in
// f32.  Shape errors name the failing node.  Tensors are freed after their last use.
TensorMap interpret(const Graph& graph, const TensorMap& inputs, int device = 0, InterpretStats* stats = nullptr);

}  // namespace routefast_b200
