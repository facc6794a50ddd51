// ref_graph_shim.cpp -- C-ABI shim over the UNMODIFIED reference graph sources (TEST
// INFRASTRUCTURE ONLY).  Compiled by oracle/Makefile (target `refgraph`) together with
// /root/reference/proj/core/src/{graph,rewrite,interpreter,attention,tensor}.cpp and the
// reference's own test fixture generator proj/tests/support/graph_fixtures.cpp, where they lie,
// into oracle/_ref/libref_graph.so.  The reference's JSON dependency (nlohmann json.hpp) is not
// vendored in its tree; the copy that ships inside this image's cudnn_frontend package is put on
// the include path for THIS CHECKER ONLY.  Used to pin the graph layer of librf_fa.so: same
// serialised text, same matches, same rewritten graph, same interpreter outputs, same error type.
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>

#include "json.hpp"
#include "routefast/graph.hpp"
#include "routefast/interpreter.hpp"
#include "routefast/rewrite.hpp"
#include "support/graph_fixtures.hpp"

namespace rf = routefast;

namespace {
thread_local std::string g_err;

char* dup_text(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
}

// error text is "<ExceptionType>: <what>"
template <typename F>
char* guarded(F&& f) {
    try {
        return dup_text(f());
    } catch (const rf::SchemaError& e) { g_err = std::string("SchemaError: ") + e.what();
    } catch (const rf::ValidationError& e) { g_err = std::string("ValidationError: ") + e.what();
    } catch (const rf::NoAttentionMaskInput& e) { g_err = std::string("NoAttentionMaskInput: ") + e.what();
    } catch (const rf::UnsupportedHeadDim& e) { g_err = std::string("UnsupportedHeadDim: ") + e.what();
    } catch (const rf::UnsupportedOp& e) { g_err = std::string("UnsupportedOp: ") + e.what();
    } catch (const rf::ShapeMismatch& e) { g_err = std::string("ShapeMismatch: ") + e.what();
    } catch (const std::invalid_argument& e) { g_err = std::string("invalid_argument: ") + e.what();
    } catch (const std::exception& e) { g_err = std::string("exception: ") + e.what(); }
    return nullptr;
}
}  // namespace

extern "C" {

const char* ref_graph_last_error() { return g_err.c_str(); }
void ref_graph_free(char* p) { std::free(p); }

char* ref_graph_normalize(const char* json) {
    return guarded([&] { return rf::serialize_graph(rf::parse_graph(json)); });
}

char* ref_graph_infer_shapes(const char* json) {
    return guarded([&] {
        nlohmann::ordered_json j = nlohmann::ordered_json::object();
        for (const auto& [name, shape] : rf::infer_shapes(rf::parse_graph(json))) j[name] = shape;
        return j.dump(2);
    });
}

char* ref_graph_topological_order(const char* json) {
    return guarded([&] {
        nlohmann::ordered_json j = rf::topological_order(rf::parse_graph(json));
        return j.dump(2);
    });
}

char* ref_graph_find_patterns(const char* json) {
    return guarded([&] {
        nlohmann::ordered_json arr = nlohmann::ordered_json::array();
        for (const auto& m : rf::find_sdpa_patterns(rf::parse_graph(json))) {
            nlohmann::ordered_json o;
            o["scale_mul"] = m.scale_mul;
            o["qk_matmul"] = m.qk_matmul;
            o["mask_add"] = m.mask_add;
            o["softmax"] = m.softmax;
            o["av_matmul"] = m.av_matmul;
            o["q"] = m.q;
            o["k"] = m.k;
            o["v"] = m.v;
            o["mask"] = m.mask;
            o["k_pre_transposed"] = m.k_pre_transposed ? 1 : 0;
            o["scale"] = m.scale;
            o["kind"] = m.kind == rf::LayerKind::local ? "local" : "global";
            arr.push_back(std::move(o));
        }
        return arr.dump(2);
    });
}

char* ref_graph_rewrite(const char* json, int64_t head_dim, int64_t local_window, const char* mask_input) {
    return guarded([&] {
        rf::RewriteOptions opt;
        opt.head_dim = head_dim;
        opt.local_window = local_window;
        if (mask_input) opt.mask_input = mask_input;
        return rf::serialize_graph(rf::rewrite(rf::parse_graph(json), opt));
    });
}

char* ref_graph_dce(const char* json) {
    return guarded([&] { return rf::serialize_graph(rf::dce(rf::parse_graph(json))); });
}

// the reference's own fixture generator (proj/tests/support/graph_fixtures.cpp:16-114);
// `layers` is a string of 'l' (local) / 'g' (global)
char* ref_graph_fixture(int64_t batch, int64_t heads, int64_t seq, int64_t head_dim, int64_t local_window,
                        const char* layers, int pre_transposed_k) {
    return guarded([&] {
        rf::testing::FixtureSpec spec;
        spec.batch = batch;
        spec.heads = heads;
        spec.seq = seq;
        spec.head_dim = head_dim;
        spec.local_window = local_window;
        spec.layers.clear();
        for (const char* c = layers; *c; ++c) spec.layers.push_back(*c == 'l' ? rf::LayerKind::local : rf::LayerKind::global);
        spec.pre_transposed_k = pre_transposed_k != 0;
        return rf::serialize_graph(rf::testing::build_attention_fixture(spec).graph);
    });
}

// interpret(): one named output copied into `out` (capacity in floats); returns its element count,
// or -1 with ref_graph_last_error() set.  out_dims receives up to 8 dims, *out_rank the rank.
int64_t ref_graph_interpret(const char* json, int32_t n_inputs, const char* const* names, const float* const* data,
                            const int64_t* const* dims, const int32_t* ranks, const char* output, float* out,
                            int64_t out_capacity, int64_t* out_dims, int32_t* out_rank) {
    int64_t n = -1;
    char* ok = guarded([&] {
        rf::Graph g = rf::parse_graph(json);
        rf::TensorMap inputs;
        for (int32_t i = 0; i < n_inputs; ++i) {
            rf::Tensor t(std::vector<int64_t>(dims[i], dims[i] + ranks[i]));
            if (!t.data.empty()) std::memcpy(t.data.data(), data[i], t.data.size() * sizeof(float));
            inputs[names[i]] = std::move(t);
        }
        rf::TensorMap outs = rf::interpret(g, inputs);
        const rf::Tensor& t = outs.at(output);
        if (static_cast<int64_t>(t.data.size()) > out_capacity) throw std::invalid_argument("output buffer too small");
        if (!t.data.empty()) std::memcpy(out, t.data.data(), t.data.size() * sizeof(float));
        *out_rank = static_cast<int32_t>(t.shape.size());
        for (std::size_t i = 0; i < t.shape.size() && i < 8; ++i) out_dims[i] = t.shape[i];
        n = static_cast<int64_t>(t.data.size());
        return std::string("ok");
    });
    std::free(ok);
    return n;
}

}  // extern "C"
