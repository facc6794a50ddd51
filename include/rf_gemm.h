/* rf_gemm.h -- C ABI of the hand-written sm_100a projections either side of the FusedFlashAttention operator
 * ("QKV projection + RoPE + head-split layout glue -> kernel, and O -> out-proj").
 *
 * The reference has no GEMM of its own on this path: its fused node consumes the raw (unscaled) Q and the
 * un-transposed K of whatever produced them (proj/core/src/rewrite.cpp:183,336-353), and its graph fixtures feed
 * Q = K = V = hidden (proj/tests/support/graph_fixtures.cpp:76-103).  In the ModernBERT-style encoder this build
 * wraps around the operator those producers are nn.Linear projections; rf_gemm_nt is that projection with the
 * encoder's element-wise steps fused into its epilogue.  Plain pointers and sizes, asynchronous on `stream`, no
 * allocation, no CPU fallback (RF_ERR_CUDA without a device).  Status codes and rf_last_error() as in rf_fa.h.
 */
#ifndef RF_GEMM_H_
#define RF_GEMM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum rf_gemm_epilogue_kind {
    RF_GEMM_EPI_NONE = 0,  /* y = a w^T                                                                      */
    RF_GEMM_EPI_ROPE = 1,  /* y = packed [tokens, 3, H, 64] QKV projection, rotary embedding ("rotate_half"
                              pairing i, i + 32) applied to the Q and K thirds (what rf_rope_qkv does in place)  */
    RF_GEMM_EPI_GEGLU = 2, /* w = [2*I, K] (input half, then gate half); y[tokens, I] = gelu(in) * gate (erf
                              GELU; what rf_geglu does on a materialised [tokens, 2*I] buffer)                   */
    RF_GEMM_EPI_RESIDUAL = 3 /* y is the f32 residual stream [M, N]: y += a w^T (the f32 accumulators are added
                              in place by TMA reduce-add; the add half of rf_add_layernorm)                      */
};

typedef struct rf_gemm_epilogue {
    int32_t kind;            /* rf_gemm_epilogue_kind */
    int32_t head_dim;        /* ROPE: must be 64 */
    int64_t S;               /* ROPE: token t sits at position t % S */
    const float* cos_table;  /* ROPE: [S, head_dim / 2] f32, device */
    const float* sin_table;
    int32_t out_dtype;       /* ROPE: 0 = same 16-bit type as the operands; 1 + RF_DTYPE_BF16 / 1 + RF_DTYPE_F16 = write
                                Q, K, V in that type (an f16 encoder can hand bf16 Q/K/V to its global attention
                                layers: bf16 P has f32's exponent range, which the dense kernel's row-max skip needs) */
    int32_t head_major;      /* ROPE: 0 = y is the packed projection [tokens, 3, H, 64]; 1 = y is [3, H, tokens, 64]: every
                                head's Q, K and V rows contiguous (ldy ignored), so that the attention kernel's TMA reads
                                whole 16 KiB tiles instead of 128-byte rows 3*H*128 bytes apart */
} rf_gemm_epilogue;

/* y[M, N'] = epilogue(a[M, K] * w[N, K]^T): 16-bit operands and output (dtype = RF_DTYPE_BF16 | RF_DTYPE_F16), f32
 * accumulation.  lda / ldw / ldy are the element strides between rows (0 = dense).  N' = N, or N / 2 for GEGLU.
 * RESIDUAL: y is f32 (ldy in f32 elements) and is accumulated into, not overwritten.
 * Requirements (else RF_ERR_UNSUPPORTED): N % 256 == 0, K % 8 == 0, 16-byte aligned pointers and row strides;
 * ROPE: N = 3 * hidden with hidden % 256 == 0; GEGLU: (N / 2) % 128 == 0.  epi == NULL means RF_GEMM_EPI_NONE. */
int rf_gemm_nt(const void* a, const void* w, void* y, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldw,
               int64_t ldy, int32_t dtype, const rf_gemm_epilogue* epi, void* stream);

/* Every wait inside the kernel is bounded: a protocol failure cannot hang the GPU or kill the context, it leaves a
 * status word behind and lets the grid run to its end with invalid output.  Synchronises `stream`, returns RF_OK or
 * RF_ERR_DEVICE_TIMEOUT (and clears the word): call it where the results of earlier rf_gemm_nt launches on this
 * device are consumed (rf_clf_forward does, once per forward). */
int rf_gemm_launch_status(void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RF_GEMM_H_ */
