/*
 * rf_graph.h -- C ABI of the graph layer around the FusedFlashAttention operator (librf_fa.so):
 * the JSON graph IR, the SDPA -> FusedFlashAttention rewriter and the GPU graph executor.
 *
 *   reference interface                                            replaced by
 *   -------------------------------------------------------------  ---------------------------
 *   parse_graph + serialize_graph   graph.hpp:88-91                rf_graph_normalize
 *   infer_shapes                    graph.hpp:103                  rf_graph_infer_shapes
 *   topological_order               graph.hpp:98                   rf_graph_topological_order
 *   find_sdpa_patterns              rewrite.hpp:47                 rf_graph_find_patterns
 *   rewrite(graph, RewriteOptions)  rewrite.hpp:49-59              rf_graph_rewrite
 *   dce                             rewrite.hpp:63                 rf_graph_dce
 *   interpret(graph, inputs)        interpreter.hpp:25             rf_graph_interpret (on the GPU)
 *   CLI rewrite-graph / verify-rewrite  proj/tools/main.cpp:76-149 the two calls above
 *
 * Graphs cross the boundary as the reference's own JSON text (schema: graph.cpp:143-193), so a
 * binding in any language needs no struct mirroring.  Text results are NUL-terminated strings
 * owned by the library until rf_graph_free.  Status codes are rf_status (rf_fa.h); the
 * reference's exception types map to RF_ERR_SCHEMA (SchemaError), RF_ERR_VALIDATION
 * (ValidationError), RF_ERR_NO_MASK_INPUT (NoAttentionMaskInput), RF_ERR_UNSUPPORTED_OP
 * (UnsupportedOp), RF_ERR_SHAPE (ShapeMismatch), RF_ERR_HEAD_DIM (UnsupportedHeadDim),
 * RF_ERR_ARG (std::invalid_argument); rf_last_error() holds the message.
 */
#ifndef RF_GRAPH_H_
#define RF_GRAPH_H_

#include "rf_fa.h"

#ifdef __cplusplus
extern "C" {
#endif

void rf_graph_free(char* text);

/* serialize_graph(parse_graph(json)): validates, then emits the deterministic form. */
int rf_graph_normalize(const char* json, char** out_json);
/* {"tensor": [dims...], ...} for every tensor, keys sorted. */
int rf_graph_infer_shapes(const char* json, char** out_json);
/* [node indices in execution order] */
int rf_graph_topological_order(const char* json, char** out_json);
/* [{"scale_mul":i,"qk_matmul":i,"mask_add":i,"softmax":i,"av_matmul":i,"q":"..","k":"..","v":"..",
 *   "mask":"..","k_pre_transposed":0|1,"scale":x,"kind":"local"|"global"}, ...] */
int rf_graph_find_patterns(const char* json, char** out_json);
/* RewriteOptions{head_dim, local_window, mask_input}; mask_input NULL = "attention_mask".
 * n_matches (optional) receives the number of fused chains. */
int rf_graph_rewrite(const char* json, int64_t head_dim, int64_t local_window, const char* mask_input,
                     char** out_json, int64_t* n_matches);
int rf_graph_dce(const char* json, char** out_json);

/* interpret(): host f32 tensors in (names/data/dims/ranks arrays of n_inputs entries), every node
 * runs on `device`, graph outputs come back as host tensors held by the result object. */
typedef struct rf_graph_result rf_graph_result;
typedef struct rf_graph_stats {
    uint64_t peak_device_bytes;    /* high-water mark of live graph tensors in HBM */
    uint64_t largest_tensor_bytes; /* the [B,H,S,S] score tensor for an un-rewritten graph */
    uint64_t launches;
    double device_ms;              /* CUDA-event time of the node loop */
} rf_graph_stats;

int rf_graph_interpret(const char* json, int32_t n_inputs, const char* const* names, const float* const* data,
                       const int64_t* const* dims, const int32_t* ranks, int32_t device, rf_graph_result** result);
int32_t rf_graph_result_count(const rf_graph_result* r);
const char* rf_graph_result_name(const rf_graph_result* r, int32_t i);
int32_t rf_graph_result_rank(const rf_graph_result* r, int32_t i);
const int64_t* rf_graph_result_dims(const rf_graph_result* r, int32_t i);
const float* rf_graph_result_data(const rf_graph_result* r, int32_t i);
int32_t rf_graph_result_is_f16(const rf_graph_result* r, int32_t i);
void rf_graph_result_stats(const rf_graph_result* r, rf_graph_stats* stats);
void rf_graph_result_free(rf_graph_result* r);

#ifdef __cplusplus
}
#endif
#endif /* RF_GRAPH_H_ */
