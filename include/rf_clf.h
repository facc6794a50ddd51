/*
 * rf_clf.h -- C ABI of the native classifier session (librf_fa.so): the ModernBERT-style encoder that
 * sits on top of the FusedFlashAttention operator, as one call from token ids to logits.
 *
 *   reference interface                                           replaced by
 *   ------------------------------------------------------------  -------------------------------
 *   JailbreakClassifier / PiiClassifier / DomainClassifier         a model-backed implementation holds
 *     ::classify(std::string_view) -- the pluggable interface       an rf_clf session per classifier and
 *     "real model backends can be dropped in behind"                calls rf_clf_forward on the token ids
 *     proj/core/include/routefast/classifiers.hpp:29-48             (include/routefast_b200/classifiers.hpp)
 *   ClassifierSet (classifiers.hpp:74-80), call site               three sessions (distinct weights)
 *     proj/core/src/stream.cpp:438-443
 *   shared pad-bias chain, one per forward (rewrite.cpp:303-318)   built inside rf_clf_forward from the mask
 *   per-layer window rule: global every `global_every`-th layer,   rf_clf_config.global_every / local_window
 *     else local_window -> (w/2-1, w/2) (rewrite.cpp:355-361)
 *
 * The reference ships keyword stubs and no neural model (classifiers.cpp:63-225): the encoder around the
 * operator (embeddings, pre-norm layers with RoPE and a GeGLU MLP, CLS head) is this build's own
 * construction, sized like ModernBERT-base, the same one paper_2603_12646_b200/classifier.py builds.
 *
 * The session owns its device memory: the weights and one activation arena that grows to the largest
 * (B, S) seen and is reused by every forward (slots are recycled inside a layer, so a 32K-token forward
 * stays under 800 MB including the weights).  The projections are this library's own tcgen05 GEMM (rf_gemm.h)
 * with RoPE and GeGLU fused into its epilogues; selecting RF_CLF_GEMM_CUBLAS routes them to the library GEMM instead
 * (resolved with dlopen at session creation; a missing library is an error, never a fallback).  Everything else
 * is the hand-written kernels of this library.  A (B, S, mask?) shape seen twice in a row is captured into a CUDA
 * graph and replayed from then on (ids / mask / logits go through page-locked staging owned by the session),
 * which removes the launch gaps between the ~200 kernels of a forward (8K tokens: 5.6 -> 5.2 ms).
 * A session is NOT thread-safe; use one per thread or per stream.
 */
#ifndef RF_CLF_H_
#define RF_CLF_H_

#include <stddef.h>
#include <stdint.h>

#include "rf_fa.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rf_clf rf_clf; /* opaque session */

typedef struct rf_clf_config {
    int32_t vocab_size;   /* 50368 */
    int32_t hidden;       /* 768 = heads * head_dim */
    int32_t n_layers;     /* 22 */
    int32_t heads;        /* 12 */
    int32_t head_dim;     /* 64 */
    int32_t mlp;          /* 1152 (GeGLU: Wi produces 2*mlp) */
    int32_t global_every; /* layer i is global iff i % global_every == 0 */
    int32_t local_window; /* 128 -> (63, 64) */
    int32_t n_labels;     /* 3 */
    int32_t mlp_chunk_rows; /* rows of the MLP intermediate computed at once (bounds activation memory) */
    int32_t act_dtype;    /* rf_dtype of weights and activations: RF_DTYPE_F16 (default: 11 significant bits keep the
                             logits within 1e-2 of the fp32 oracle at full depth) or RF_DTYPE_BF16; the residual
                             stream is f32 either way */
    float rope_theta_global; /* 160000 */
    float rope_theta_local;  /* 10000 */
    float eps;               /* 1e-5 */
    int32_t gemm_backend;    /* RF_CLF_GEMM_OWN (default): rf_gemm_nt (rf_gemm.h) with RoPE fused into the QKV projection
                                and GeGLU into the MLP up-projection -- no library on the path, cuBLAS is not even
                                loaded; RF_CLF_GEMM_CUBLAS: library GEMMs + rf_rope_qkv / rf_geglu (the round-1 path,
                                kept as the A/B baseline) */
} rf_clf_config;

enum rf_clf_gemm_backend { RF_CLF_GEMM_OWN = 0, RF_CLF_GEMM_CUBLAS = 1 };

/* ModernBERT-base shape (the defaults of classifier.py's ClassifierConfig). */
void rf_clf_config_default(rf_clf_config* cfg);

/* Number of f32 elements of the weight blob rf_clf_create expects, tensors back to back in this order
 * (row-major, [out, in] for matrices):
 *   tok_emb [vocab, hidden], emb_norm [hidden], final_norm [hidden], head_dense [hidden, hidden],
 *   head_norm [hidden], cls_w [n_labels, hidden], cls_b [n_labels],
 *   then per layer: attn_norm [hidden], wqkv [3*hidden, hidden], wo [hidden, hidden], mlp_norm [hidden],
 *   wi [2*mlp, hidden], wo2 [hidden, mlp].
 * Matrices are stored on the device in act_dtype, norm weights and cls_b in f32. */
size_t rf_clf_weight_elems(const rf_clf_config* cfg);

/* Creates a session on `device` from host f32 weights.  RF_ERR_CUDA without a device / cuBLAS. */
int rf_clf_create(const rf_clf_config* cfg, const float* weights, size_t n_elems, int32_t device, rf_clf** out);

/* One forward: input_ids host int64 [B,S]; attention_mask host f32 [B,S] (1 = token, 0 = padding) or
 * NULL; logits host f32 [B, n_labels].  Synchronous (returns when the logits are in host memory). */
int rf_clf_forward(rf_clf* clf, const int64_t* input_ids, const float* attention_mask, int64_t B, int64_t S,
                   float* logits);

/* Device bytes held by the session: weights, and the activation arena at its high-water mark. */
int rf_clf_session_bytes(const rf_clf* clf, size_t* weight_bytes, size_t* arena_bytes);

/* Device time of the last forward in milliseconds (CUDA events around the whole forward). */
float rf_clf_last_forward_ms(const rf_clf* clf);

void rf_clf_destroy(rf_clf* clf);

/* The classification head rf_clf_forward runs last, as a stand-alone call on device tensors (used by the torch-hosted
 * mirror of the session so that no library GEMM is left on its path): pooled = hf[b * S, :] (CLS token of sequence
 * b); t = gelu(pooled Wd^T) rounded to the 16-bit type; t = LayerNorm(t) * head_norm; logits[b, :] = t Wc^T + cls_b.
 * hf [B*S, hidden], head_dense [hidden, hidden], cls_w [n_labels, hidden] in `dtype` (RF_DTYPE_F16 | RF_DTYPE_BF16);
 * head_norm [hidden], cls_b [n_labels], logits [B, n_labels] f32.  hidden <= 1024, a multiple of 8; head_dense rows
 * 16-byte aligned.  Asynchronous on `stream`. */
int rf_clf_head(const void* hf, int64_t B, int64_t S, int32_t hidden, const void* head_dense, const float* head_norm,
                const void* cls_w, const float* cls_b, int32_t n_labels, float eps, int32_t dtype, float* logits,
                void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RF_CLF_H_ */
