/*
 * rf_fa.h -- C ABI of the B200 fused flash-attention operator (librf_fa.so).
 *
 * This is the drop-in boundary for the reference's `FusedFlashAttention` operator:
 *
 *   reference interface                                         replaced by
 *   ----------------------------------------------------------  ---------------------------------
 *   routefast::flash_attention(q,k,v,spec,tile,stats)            rf_fa_fwd_host (host f32 tensors)
 *     proj/core/include/routefast/attention.hpp:46-48            rf_fa_fwd      (device tensors)
 *     proj/core/src/attention.cpp:106-213
 *   FlashStats (attention.hpp:36-40)                             rf_fa_fwd_workspace_bytes / rf_fa_stats
 *   AttentionSpec{scale,window_left,window_right,pad_bias}       fields of rf_fa_params
 *     attention.hpp:18-25
 *   interpret() case OpKind::FusedFlashAttention                 rf_fused_flash_attention_op (attrs + 3|4 inputs)
 *     proj/core/src/interpreter.cpp:308-318
 *   pad-bias chain Cast_f16(-65504*(1-mask))                     rf_pad_bias_from_mask
 *     proj/core/src/rewrite.cpp:303-318
 *   mask_memory_bytes / fa_memory_bytes (attention.cpp:244-252)  rf_mask_memory_bytes / rf_fa_memory_bytes
 *   ShapeMismatch (tensor.hpp:16-19)                             RF_ERR_SHAPE   + rf_last_error()
 *   UnsupportedHeadDim (rewrite.hpp:14-17, rewrite.cpp:266-269)  RF_ERR_HEAD_DIM + rf_last_error()
 *
 * Plain pointers and sizes only; no torch / C++ types.  Every entry point is thread-safe
 * (no mutable global state; rf_last_error() is thread-local).  The launcher never allocates
 * device memory: the caller owns Q/K/V/O and the workspace.  Launches are asynchronous on
 * the given stream.  There is NO CPU fallback: without a CUDA device every compute entry
 * point returns RF_ERR_CUDA.
 */
#ifndef RF_FA_H_
#define RF_FA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RF_FA_ABI_VERSION 1

/* attention.hpp:15-16 */
#define RF_MASK_VALUE (-65504.0f)
#define RF_MASK_THRESHOLD (-30000.0f)

typedef enum rf_status {
    RF_OK = 0,
    RF_ERR_SHAPE = 1,       /* reference: ShapeMismatch */
    RF_ERR_HEAD_DIM = 2,    /* reference: UnsupportedHeadDim (head_dim not in {32,64,128}) */
    RF_ERR_ARG = 3,         /* null pointer, bad enum, bad stride/alignment */
    RF_ERR_CUDA = 4,        /* CUDA runtime/driver failure, or no sm_100 device */
    RF_ERR_WORKSPACE = 5,   /* workspace missing or too small */
    RF_ERR_UNSUPPORTED = 6, /* valid in the reference but not implemented on this path */
    /* graph layer (rf_graph.h) */
    RF_ERR_SCHEMA = 7,         /* reference: SchemaError (graph.hpp:17-20) */
    RF_ERR_VALIDATION = 8,     /* reference: ValidationError (graph.hpp:23-26) */
    RF_ERR_NO_MASK_INPUT = 9,  /* reference: NoAttentionMaskInput (rewrite.hpp:19-22) */
    RF_ERR_UNSUPPORTED_OP = 10, /* reference: UnsupportedOp (interpreter.hpp:14-17) */
    RF_ERR_DEVICE_TIMEOUT = 11  /* a bounded wait inside a kernel ran out (rf_fa_launch_status); the context stays usable */
} rf_status;

typedef enum rf_dtype { RF_DTYPE_BF16 = 0, RF_DTYPE_F16 = 1, RF_DTYPE_F32 = 2 } rf_dtype;

/* Which kernel family runs.  AUTO picks tcgen05 whenever the layout allows (every head_dim of the reference
 * contract, rewrite.cpp:266-269: 64 on the tuned kernels, 32 through the same kernels zero-padded to 64, 128 on
 * its own kernel); SIMT is the generic CUDA-core sm_100a kernel (unaligned layouts, negative scale), also used as
 * an on-device cross-check in tests.  Neither is a CPU path. */
typedef enum rf_kernel { RF_KERNEL_AUTO = 0, RF_KERNEL_TCGEN05 = 1, RF_KERNEL_SIMT = 2 } rf_kernel;

/*
 * One FusedFlashAttention call on device tensors.
 *
 * Q, K, V: [B,H,S,d] logical shape, `dtype` elements (bf16/f16), last dim contiguous,
 * element strides for (batch, head, seq) given explicitly so [B,H,S,d] (the reference
 * layout, attention.cpp:143), [B,S,H,d] and packed [B,S,3,H,d] QKV views are consumed
 * without a transpose.  A stride of 0 in *_stride[2] means "contiguous [B,H,S,d]".
 * O: same logical shape, `out_dtype` (bf16/f16/f32).
 *
 * pad_bias: device f32 [B,S] (the reference's [B,1,1,S] tensor, attention.cpp:111-116) or
 * NULL.  Key j of batch b is masked iff pad_bias[b,j] <= -30000; a live value is ADDED to
 * the scaled score (attention.cpp:160-169).
 *
 * Liveness: (window_left < 0 || i-j <= window_left) && (window_right < 0 || j-i <= window_right)
 * && key unmasked (attention.cpp:132-136,160-161).  Rows with no live key produce 0
 * (attention.cpp:175,204-207).  scale == 0 means 1/sqrt(d) (attention.cpp:34-36).
 *
 * Split-KV (one 32K sequence over several GPUs): when o_partial != NULL the call covers only
 * keys [kv_begin, kv_end) and writes UN-normalised partials instead of `out`:
 *   o_partial f32 [B,H,S,d], m_partial f32 [B,H,S] (running max, log2 domain, -inf if no
 *   live key), l_partial f32 [B,H,S] (running sum relative to m).  rf_fa_merge combines them.
 */
typedef struct rf_fa_params {
    const void* q;
    const void* k;
    const void* v;
    void* out;
    int64_t q_stride[3]; /* elements: batch, head, seq */
    int64_t k_stride[3];
    int64_t v_stride[3];
    int64_t o_stride[3];
    const float* pad_bias;
    int64_t B, H, S, d;
    double scale;
    int64_t window_left;
    int64_t window_right;
    int32_t dtype;     /* rf_dtype of Q/K/V: BF16 or F16 */
    int32_t out_dtype; /* rf_dtype of O */
    int32_t kernel;    /* rf_kernel */
    int32_t flags;     /* reserved, must be 0 */
    int64_t kv_begin; /* split-KV key range.  Full call (o_partial == NULL): both 0 => [0,S).  Partial call: taken
                       * literally; an empty range writes the merge's neutral element (m = -inf, l = 0, O = 0) */
    int64_t kv_end;
    float* o_partial;
    float* m_partial;
    float* l_partial;
    float* debug_scores; /* testing only: raw S tile dump of the first key tile, or NULL */
} rf_fa_params;

/* Scratch sizes of one call, the analogue of FlashStats (attention.hpp:36-40): all O(S). */
typedef struct rf_fa_stats {
    uint64_t workspace_bytes;     /* device workspace the caller must pass (status word, bias + tile flags, schedule state) */
    uint64_t tile_scratch_bytes;  /* on-chip per-CTA scratch (smem + TMEM), independent of S */
    uint64_t row_state_bytes;     /* running max + sum kept in registers: 2*4 bytes per query row */
    uint64_t output_bytes;        /* B*H*S*d*sizeof(out) */
    uint64_t score_matrix_bytes;  /* always 0: no S x S tensor exists */
    int32_t kernel;               /* rf_kernel actually selected */
    int32_t grid_ctas;
} rf_fa_stats;

const char* rf_last_error(void);
int rf_abi_version(void);

/* Fills p with defaults: contiguous strides (0), scale 0, windows -1, bf16 in/out, AUTO. */
void rf_fa_params_init(rf_fa_params* p);

/* Validation only (no CUDA call): same checks, same order, same messages as
 * attention.cpp:14-21,110-116 plus this build's own (head_dim, dtype, alignment). */
int rf_fa_validate(const rf_fa_params* p);

int rf_fa_fwd_workspace_bytes(const rf_fa_params* p, size_t* bytes);
int rf_fa_stats_query(const rf_fa_params* p, rf_fa_stats* stats);

/* Launch on `stream` (cudaStream_t as void*).  workspace may be NULL when
 * rf_fa_fwd_workspace_bytes reports 0. */
int rf_fa_fwd(const rf_fa_params* p, void* workspace, size_t workspace_bytes, void* stream);

/* The launcher's resolved form of one call (the "launcher and workspace allocator" of the operator: the
 * reference has no counterpart because routefast::flash_attention, attention.cpp:106-213, has nothing to
 * prepare).  rf_fa_plan_create does what rf_fa_fwd does before its launches -- validation, kernel and schedule
 * selection, workspace carve-up, the three TMA tensor maps -- once; rf_fa_plan_launch only enqueues the kernels
 * (asynchronous, any stream, any number of times; thread-safe for concurrent launches as long as concurrent
 * launches do not share one workspace).  The plan refers to the tensors and the workspace of `p` by address:
 * they must stay allocated, their contents may change between launches.
 * Plans may share one workspace (a session's layers do) as long as their launches do not overlap in time: the
 * only state that lives across launches -- the split-pair flags of the persistent balanced schedule -- sits at the
 * same offset in every plan's carve-up, is zeroed in-stream by a plan's first launch (the workspace need not be
 * zeroed by the caller) and is left zero by the kernel. */
typedef struct rf_fa_plan rf_fa_plan;
int rf_fa_plan_create(const rf_fa_params* p, void* workspace, size_t workspace_bytes, rf_fa_plan** plan);
int rf_fa_plan_launch(const rf_fa_plan* plan, void* stream);
void rf_fa_plan_destroy(rf_fa_plan* plan);

/* Every wait inside the tcgen05 kernels is bounded.  A wait that runs out (a protocol bug, or a peer CTA that
 * never got scheduled) does not hang or trap: the kernel raises a status word at the head of the workspace, drains
 * and exits normally; its output is then invalid.  This call synchronises `stream`, reads the word, and returns
 * RF_OK or RF_ERR_DEVICE_TIMEOUT (clearing the word).  The CUDA context stays usable either way.  The host entry
 * points (rf_fa_fwd_host, rf_clf_forward) call it themselves. */
int rf_fa_launch_status(void* workspace, void* stream);

/* Split-KV softmax merge (the one exchange step of SURVEY 8(e)):
 *   m* = max_g m_g;  O = sum_g O_g 2^(m_g-m*) / sum_g l_g 2^(m_g-m*), 0 where the sum is 0.
 * o_parts/m_parts/l_parts are arrays of G device pointers (host array of pointers); the
 * reduction order over g is fixed (0..G-1) so the result is run-to-run deterministic.
 * rows = B*H*S. */
int rf_fa_merge(const float* const* o_parts, const float* const* m_parts, const float* const* l_parts,
                int32_t G, int64_t rows, int64_t d, void* out, int32_t out_dtype, void* stream);

/* Rescale step of the NCCL variant: given the all-reduced (max) m_star, turns a partial into
 * summable form in place: O_g *= 2^(m_g-m*), l_g *= 2^(m_g-m*).  After ncclReduceScatter(sum)
 * of [O|l], rf_fa_normalize finishes O/l. */
int rf_fa_rescale_partial(float* o_part, float* l_part, const float* m_part, const float* m_star,
                          int64_t rows, int64_t d, void* stream);
int rf_fa_normalize(const float* o_sum, const float* l_sum, int64_t rows, int64_t d, void* out,
                    int32_t out_dtype, void* stream);

/* pad-bias chain on device (rewrite.cpp:303-318): bias = f16_round(-65504 * (1 - mask)), f32 storage. */
int rf_pad_bias_from_mask(const float* mask, float* pad_bias, int64_t n, void* stream);

/* Layout glue: f32 <-> bf16/f16 casts on device (RNE), used by the host path. */
int rf_cast_f32_to(const float* src, void* dst, int64_t n, int32_t dst_dtype, void* stream);
int rf_cast_to_f32(const void* src, float* dst, int64_t n, int32_t src_dtype, void* stream);

/*
 * Host-buffer entry point with the reference's exact calling convention: f32 host tensors
 * [B,H,S,d] in, f32 host tensor out (routefast::flash_attention on Tensor objects).  The call is
 * PCIe-bound, so it is pipelined: (batch, head-range) chunks -- independent units of the op,
 * attention.cpp:138-142 -- go H2D -> cast to `compute_dtype` -> rf_fa_fwd -> D2H round-robin over
 * four streams, overlapping upload, kernel and download.  Page-locked host buffers get the full
 * overlap; pageable ones work too (O is then fetched with one copy at the end).  Device memory
 * is allocated (stream-ordered pool) and freed inside the call and no result state is retained,
 * like the reference; only the four streams are cached per calling thread and device
 * (rf_fa_host_release destroys the calling thread's).  `tile` is accepted for signature parity
 * and validated (tile < 1 -> RF_ERR_SHAPE, attention.cpp:110); the kernel's tiling is fixed.
 * pad_bias_dims: the 4 dims of the bias tensor as the caller holds it (checked against
 * [B,1,1,S]), or NULL when pad_bias is NULL.
 */
int rf_fa_fwd_host(const float* q, const float* k, const float* v, float* out, int64_t B, int64_t H,
                   int64_t S, int64_t d, double scale, int64_t window_left, int64_t window_right,
                   const float* pad_bias, const int64_t* pad_bias_dims, int64_t tile,
                   int32_t compute_dtype, int32_t device, rf_fa_stats* stats);
void rf_fa_host_release(void);

/* The rounding rf_fa_fwd_host applies to Q, K, V before they cross the link: f32 -> bf16, round to nearest even (NaN
 * stays NaN), on a small pool of host threads (RF_FA_HOST_CAST_THREADS, default min(16, cores - 2); RF_FA_HOST_CAST=0
 * keeps the rounding on the device).  Bit-identical to the device cast.  No CUDA call; exposed for tests and for
 * callers that keep their own 16-bit copies.  The reference has no counterpart (its Tensor is f32 only,
 * proj/core/include/routefast/tensor.hpp). */
int rf_host_round_bf16(const float* src, uint16_t* dst, int64_t n);

/* Bytes the calling thread's rf_fa_fwd_host calls have moved over the link so far (cumulative since the thread's
 * first call) and how many calls completed: what a benchmark reports as host-to-device / device-to-host bytes per
 * call, whichever way the inputs were rounded.  Measurement aid; the reference has no counterpart. */
void rf_fa_host_transfer_counters(uint64_t* h2d_bytes, uint64_t* d2h_bytes, uint64_t* calls);

/* The interpreter's FusedFlashAttention case (interpreter.cpp:308-318) on host tensors:
 * n_inputs is 3 or 4 (4th = pad_bias), each with its rank and dims; attrs default to scale 0.0,
 * windows -1 exactly as node.attr_real/attr_int fall back.  has_* flags say which attrs the
 * node carries. */
int rf_fused_flash_attention_op(const float* const* inputs, const int64_t* const* input_dims,
                                const int32_t* input_ranks, int32_t n_inputs, int32_t has_scale, double scale,
                                int32_t has_window_left, int64_t window_left,
                                int32_t has_window_right, int64_t window_right, float* output,
                                int32_t device);

/* Encoder-layer glue either side of the op, 16-bit activations (`dtype`: bf16 or f16),
 * in place where possible:
 *   rf_rope_qkv      rotary embedding ("rotate_half" pairing i, i+d/2) on the Q and K thirds of a
 *                    packed QKV GEMM output [tokens,3,H,d]; cos/sin f32 [S,d/2]; position = t % S.
 *                    The attention kernel then reads the three thirds as strided views.
 *   rf_add_layernorm x (f32 residual stream [rows,n]) += delta (16-bit, or NULL); y = LN(x)*w (16-bit,
 *                    no bias; y may be NULL to only accumulate).  n % 4 == 0, n <= 4096.
 *   rf_geglu         act[rows,I] = gelu(wi_out[:, :I]) * wi_out[:, I:]   (erf GELU)            */
/* dtype: rf_dtype of the 16-bit activations, RF_DTYPE_BF16 or RF_DTYPE_F16 */
int rf_rope_qkv(void* qkv, const float* cos_table, const float* sin_table, int64_t tokens, int64_t S, int64_t H,
                int64_t d, int32_t dtype, void* stream);
int rf_add_layernorm(float* x, const void* delta, const float* w, void* y, int64_t rows, int64_t n, float eps,
                     int32_t dtype, void* stream);
int rf_geglu(const void* wi_out, void* act, int64_t rows, int64_t I, int32_t dtype, void* stream);

/* Memory model (attention.cpp:244-252). */
uint64_t rf_mask_memory_bytes(uint64_t batch, uint64_t heads, uint64_t seq_len, uint64_t bytes_per_element);
uint64_t rf_fa_memory_bytes(uint64_t batch, uint64_t heads, uint64_t seq_len, uint64_t head_dim,
                            uint64_t tile, uint64_t bytes_per_element);

/* Device info used by bench/tests: 0 if a usable sm_100 device is present. */
int rf_device_check(int32_t device, int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor);

#ifdef __cplusplus
}
#endif
#endif /* RF_FA_H_ */
