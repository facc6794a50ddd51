// graph_capi.cpp -- the C ABI of include/rf_graph.h over the C++ graph layer: JSON text in, JSON
// text (or host tensors) out, the reference's exception types mapped to status codes.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../../include/rf_graph.h"
#include "../fa_internal.h"
#include "json.hpp"
#include "routefast_b200/graph.hpp"

namespace rb = routefast_b200;

struct rf_graph_result {
    std::vector<std::string> names;
    std::vector<rb::Tensor> tensors;
    rb::InterpretStats stats;
};

namespace {

char* dup_text(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    if (p != nullptr) std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
}

// Runs `body`, translating the graph layer's exceptions into status codes.
template <typename Body>
int guarded(Body&& body) {
    try {
        body();
        return RF_OK;
    } catch (const rb::SchemaError& e) {
        return rf::set_last_error(RF_ERR_SCHEMA, e.what());
    } catch (const rb::ValidationError& e) {
        return rf::set_last_error(RF_ERR_VALIDATION, e.what());
    } catch (const rb::NoAttentionMaskInput& e) {
        return rf::set_last_error(RF_ERR_NO_MASK_INPUT, e.what());
    } catch (const rb::UnsupportedOp& e) {
        return rf::set_last_error(RF_ERR_UNSUPPORTED_OP, e.what());
    } catch (const rb::UnsupportedHeadDim& e) {
        return rf::set_last_error(RF_ERR_HEAD_DIM, e.what());
    } catch (const rb::ShapeMismatch& e) {
        return rf::set_last_error(RF_ERR_SHAPE, e.what());
    } catch (const std::invalid_argument& e) {
        return rf::set_last_error(RF_ERR_ARG, e.what());
    } catch (const std::bad_alloc&) {
        return rf::set_last_error(RF_ERR_ARG, "out of host memory");
    } catch (const std::exception& e) {
        return rf::set_last_error(RF_ERR_CUDA, e.what());
    }
}

int text_out(char** out, const std::string& s) {
    *out = dup_text(s);
    return *out != nullptr ? RF_OK : rf::set_last_error(RF_ERR_ARG, "out of host memory");
}

}  // namespace

extern "C" {

void rf_graph_free(char* text) { std::free(text); }

int rf_graph_normalize(const char* json, char** out_json) {
    if (json == nullptr || out_json == nullptr) return rf::set_last_error(RF_ERR_ARG, "null pointer");
    std::string text;
    int rc = guarded([&] { text = rb::serialize_graph(rb::parse_graph(json)); });
    return rc != RF_OK ? rc : text_out(out_json, text);
}

int rf_graph_infer_shapes(const char* json, char** out_json) {
    if (json == nullptr || out_json == nullptr) return rf::set_last_error(RF_ERR_ARG, "null pointer");
    std::string text;
    int rc = guarded([&] {
        rfjson::Value doc = rfjson::Value::object();
        for (const auto& [name, shape] : rb::infer_shapes(rb::parse_graph(json))) {
            rfjson::Value dims = rfjson::Value::array();
            for (int64_t d : shape) dims.push(rfjson::Value::integer(d));
            doc.set(name, std::move(dims));
        }
        rfjson::dump(doc, text, 2);
    });
    return rc != RF_OK ? rc : text_out(out_json, text);
}

int rf_graph_topological_order(const char* json, char** out_json) {
    if (json == nullptr || out_json == nullptr) return rf::set_last_error(RF_ERR_ARG, "null pointer");
    std::string text;
    int rc = guarded([&] {
        rfjson::Value arr = rfjson::Value::array();
        for (std::size_t i : rb::topological_order(rb::parse_graph(json))) arr.push(rfjson::Value::integer(static_cast<int64_t>(i)));
        rfjson::dump(arr, text, 2);
    });
    return rc != RF_OK ? rc : text_out(out_json, text);
}

int rf_graph_find_patterns(const char* json, char** out_json) {
    if (json == nullptr || out_json == nullptr) return rf::set_last_error(RF_ERR_ARG, "null pointer");
    std::string text;
    int rc = guarded([&] {
        rfjson::Value arr = rfjson::Value::array();
        for (const rb::PatternMatch& m : rb::find_sdpa_patterns(rb::parse_graph(json))) {
            rfjson::Value o = rfjson::Value::object();
            o.set("scale_mul", rfjson::Value::integer(static_cast<int64_t>(m.scale_mul)));
            o.set("qk_matmul", rfjson::Value::integer(static_cast<int64_t>(m.qk_matmul)));
            o.set("mask_add", rfjson::Value::integer(static_cast<int64_t>(m.mask_add)));
            o.set("softmax", rfjson::Value::integer(static_cast<int64_t>(m.softmax)));
            o.set("av_matmul", rfjson::Value::integer(static_cast<int64_t>(m.av_matmul)));
            o.set("q", rfjson::Value::string(m.q));
            o.set("k", rfjson::Value::string(m.k));
            o.set("v", rfjson::Value::string(m.v));
            o.set("mask", rfjson::Value::string(m.mask));
            o.set("k_pre_transposed", rfjson::Value::integer(m.k_pre_transposed ? 1 : 0));
            o.set("scale", rfjson::Value::real(m.scale));
            o.set("kind", rfjson::Value::string(m.kind == rb::LayerKind::local ? "local" : "global"));
            arr.push(std::move(o));
        }
        rfjson::dump(arr, text, 2);
    });
    return rc != RF_OK ? rc : text_out(out_json, text);
}

int rf_graph_rewrite(const char* json, int64_t head_dim, int64_t local_window, const char* mask_input, char** out_json,
                     int64_t* n_matches) {
    if (json == nullptr || out_json == nullptr) return rf::set_last_error(RF_ERR_ARG, "null pointer");
    std::string text;
    int rc = guarded([&] {
        rb::RewriteOptions opt;
        opt.head_dim = head_dim;
        opt.local_window = local_window;
        if (mask_input != nullptr) opt.mask_input = mask_input;
        const rb::Graph g = rb::parse_graph(json);
        text = rb::serialize_graph(rb::rewrite(g, opt));
        if (n_matches != nullptr) *n_matches = static_cast<int64_t>(rb::find_sdpa_patterns(g).size());
    });
    return rc != RF_OK ? rc : text_out(out_json, text);
}

int rf_graph_dce(const char* json, char** out_json) {
    if (json == nullptr || out_json == nullptr) return rf::set_last_error(RF_ERR_ARG, "null pointer");
    std::string text;
    int rc = guarded([&] { text = rb::serialize_graph(rb::dce(rb::parse_graph(json))); });
    return rc != RF_OK ? rc : text_out(out_json, text);
}

int rf_graph_interpret(const char* json, int32_t n_inputs, const char* const* names, const float* const* data,
                       const int64_t* const* dims, const int32_t* ranks, int32_t device, rf_graph_result** result) {
    if (json == nullptr || result == nullptr || n_inputs < 0 ||
        (n_inputs > 0 && (names == nullptr || data == nullptr || dims == nullptr || ranks == nullptr)))
        return rf::set_last_error(RF_ERR_ARG, "null pointer");
    *result = nullptr;
    rf_graph_result* res = nullptr;
    int rc = guarded([&] {
        const rb::Graph g = rb::parse_graph(json);
        rb::TensorMap inputs;
        for (int32_t i = 0; i < n_inputs; ++i) {
            if (names[i] == nullptr || dims[i] == nullptr || ranks[i] < 0) throw std::invalid_argument("bad input descriptor");
            rb::Tensor t(std::vector<int64_t>(dims[i], dims[i] + ranks[i]));
            if (!t.data.empty()) {
                if (data[i] == nullptr) throw std::invalid_argument("null input data");
                std::memcpy(t.data.data(), data[i], t.data.size() * sizeof(float));
            }
            inputs[names[i]] = std::move(t);
        }
        res = new rf_graph_result();
        rb::TensorMap outs = rb::interpret(g, inputs, device, &res->stats);
        for (const std::string& name : g.outputs) {  // graph output order
            if (std::find(res->names.begin(), res->names.end(), name) != res->names.end()) continue;
            res->names.push_back(name);
            res->tensors.push_back(std::move(outs.at(name)));
        }
    });
    if (rc != RF_OK) {
        delete res;
        return rc;
    }
    *result = res;
    return RF_OK;
}

int32_t rf_graph_result_count(const rf_graph_result* r) { return r ? static_cast<int32_t>(r->names.size()) : 0; }
// accessors never throw through the C boundary: a null result or an index out of range yields NULL / -1
static bool result_index_ok(const rf_graph_result* r, int32_t i) {
    return r != nullptr && i >= 0 && static_cast<size_t>(i) < r->tensors.size() && static_cast<size_t>(i) < r->names.size();
}
const char* rf_graph_result_name(const rf_graph_result* r, int32_t i) {
    return result_index_ok(r, i) ? r->names[static_cast<size_t>(i)].c_str() : nullptr;
}
int32_t rf_graph_result_rank(const rf_graph_result* r, int32_t i) {
    return result_index_ok(r, i) ? static_cast<int32_t>(r->tensors[static_cast<size_t>(i)].shape.size()) : -1;
}
const int64_t* rf_graph_result_dims(const rf_graph_result* r, int32_t i) {
    return result_index_ok(r, i) ? r->tensors[static_cast<size_t>(i)].shape.data() : nullptr;
}
const float* rf_graph_result_data(const rf_graph_result* r, int32_t i) {
    return result_index_ok(r, i) ? r->tensors[static_cast<size_t>(i)].data.data() : nullptr;
}
int32_t rf_graph_result_is_f16(const rf_graph_result* r, int32_t i) {
    if (!result_index_ok(r, i)) return -1;
    return r->tensors[static_cast<size_t>(i)].dtype == rb::DType::f16 ? 1 : 0;
}
void rf_graph_result_stats(const rf_graph_result* r, rf_graph_stats* stats) {
    if (r == nullptr || stats == nullptr) return;
    stats->peak_device_bytes = r->stats.peak_device_bytes;
    stats->largest_tensor_bytes = r->stats.largest_tensor_bytes;
    stats->launches = r->stats.launches;
    stats->device_ms = r->stats.device_ms;
}
void rf_graph_result_free(rf_graph_result* r) { delete r; }

}  // extern "C"
