// clf_runtime.cu -- native classifier session (include/rf_clf.h): token ids -> logits for the
// ModernBERT-style encoder built on the FusedFlashAttention operator, without Python in the loop.
//
// Same data path as paper_2603_12646_b200/classifier.py (which stays as the torch-hosted mirror):
//   x = LN(emb[ids])                                   embed_gather + rf_add_layernorm
//   per layer: h = LN(x); qkv = rope(h Wqkv^T)         rf_gemm_nt, RoPE in the epilogue -> head-major [3,H,B*S,d]
//              attn = FusedFlashAttention(q, k, v)     rf_fa_fwd on strided views, [B,S,H*d] out
//              x += attn Wo^T; h2 = LN(x)              rf_gemm_nt (residual epilogue: TMA reduce-add into x) + rf_add_layernorm
//              x += (gelu(h2 Wi_a) * h2 Wi_g) Wo2^T    rf_gemm_nt (GeGLU epilogue), rf_gemm_nt (residual epilogue), in row chunks
//   logits = head(LN(x)[CLS])                          clf_head_kernel
// (gemm_backend = RF_CLF_GEMM_CUBLAS keeps the round-1 path for A/B runs: library GEMMs into the packed [B,S,3,H,d]
// layout + rf_rope_qkv / rf_geglu / the add half of rf_add_layernorm.)
// The pad-bias chain is built once per forward and shared by every layer (reference rewrite.cpp:303-318);
// layer i is global iff i % global_every == 0, else local_window -> (w/2-1, w/2) (rewrite.cpp:355-361).
//
// Memory: the session owns the weights and one activation arena with fixed slots that are recycled
// inside a layer: x (f32 stream), `big` (qkv, later the MLP intermediate), two ping-pong slots of one
// bf16 activation each, the attention workspace, RoPE tables, ids, mask/bias.  The arena only grows.
//
// A shape seen twice in a row is captured into a CUDA graph and replayed afterwards; ids, mask and logits
// travel through page-locked staging so that the captured copies have fixed addresses.
//
// cuBLAS is only loaded when RF_CLF_GEMM_CUBLAS is selected: resolved with dlopen/dlsym (five entry points) so that
// librf_fa.so itself has no link-time dependency on it; a missing library is then RF_ERR_CUDA at session creation,
// never a fallback.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/rf_clf.h"
#include "../../include/rf_gemm.h"
#include "fa_internal.h"

namespace {

int fail(int code, const std::string& msg) { return rf::set_last_error(code, msg); }
int cuda_fail(cudaError_t e, const char* what) {
    return fail(RF_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- the five cuBLAS entry points, by hand (cublas_v2.h is not included: no link-time dependency) ----
typedef void* cublasHandle_t;
typedef int (*cublasCreate_fn)(cublasHandle_t*);
typedef int (*cublasDestroy_fn)(cublasHandle_t);
typedef int (*cublasSetStream_fn)(cublasHandle_t, cudaStream_t);
typedef int (*cublasSetWorkspace_fn)(cublasHandle_t, void*, size_t);
typedef int (*cublasGemmEx_fn)(cublasHandle_t, int, int, int, int, int, const void*, const void*, int, int, const void*,
                               int, int, const void*, void*, int, int, int, int);
constexpr int kCublasOpN = 0, kCublasOpT = 1;
constexpr int kCudaR16BF = 14;          // CUDA_R_16BF
constexpr int kCudaR16F = 2;            // CUDA_R_16F
constexpr int kCublasCompute32F = 68;   // CUBLAS_COMPUTE_32F
constexpr int kCublasGemmDefault = -1;  // CUBLAS_GEMM_DEFAULT

struct Cublas {
    void* dl = nullptr;
    cublasCreate_fn create = nullptr;
    cublasDestroy_fn destroy = nullptr;
    cublasSetStream_fn set_stream = nullptr;
    cublasGemmEx_fn gemm_ex = nullptr;
    cublasSetWorkspace_fn set_workspace = nullptr;
    bool load(std::string* why) {
        for (const char* name : {"libcublas.so.12", "libcublas.so", "/usr/local/cuda/lib64/libcublas.so.12"}) {
            dl = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (dl != nullptr) break;
        }
        if (dl == nullptr) {
            *why = "cuBLAS not found (dlopen libcublas.so.12)";
            return false;
        }
        create = reinterpret_cast<cublasCreate_fn>(dlsym(dl, "cublasCreate_v2"));
        destroy = reinterpret_cast<cublasDestroy_fn>(dlsym(dl, "cublasDestroy_v2"));
        set_stream = reinterpret_cast<cublasSetStream_fn>(dlsym(dl, "cublasSetStream_v2"));
        gemm_ex = reinterpret_cast<cublasGemmEx_fn>(dlsym(dl, "cublasGemmEx"));
        set_workspace = reinterpret_cast<cublasSetWorkspace_fn>(dlsym(dl, "cublasSetWorkspace_v2"));
        if (!create || !destroy || !set_stream || !gemm_ex || !set_workspace) {
            *why = "cuBLAS entry points missing";
            return false;
        }
        return true;
    }
};

// ---- kernels of the session that the operator library did not have yet ----

// 16-bit activation / weight element (bf16 or f16) <-> float
template <bool kBf16>
__device__ __forceinline__ float2 pair_to_float2(uint32_t w) {
    if (kBf16) return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w));
    return __half22float2(*reinterpret_cast<const __half2*>(&w));
}
template <bool kBf16>
__device__ __forceinline__ float elem_to_float(uint16_t h) {
    if (kBf16) return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(&h));
    return __half2float(*reinterpret_cast<const __half*>(&h));
}
template <bool kBf16>
__device__ __forceinline__ float round_to_16(float v) {
    if (kBf16) return __bfloat162float(__float2bfloat16_rn(v));
    return __half2float(__float2half_rn(v));
}

// x[row, :] = float(tok_emb[ids[row], :]); one warp per row, 16-byte loads.
template <bool kBf16>
__global__ void __launch_bounds__(128) embed_gather_kernel(const uint16_t* __restrict__ emb, const long long* __restrict__ ids,
                                                           float* __restrict__ x, long long rows, int hidden, int vocab) {
    const long long row = static_cast<long long>(blockIdx.x) * 4 + (threadIdx.x >> 5);
    if (row >= rows) return;
    const int lane = threadIdx.x & 31;
    long long id = ids[row];
    id = id < 0 ? 0 : (id >= vocab ? vocab - 1 : id);
    const uint16_t* src = emb + id * hidden;
    float* dst = x + row * hidden;
    for (int c = lane * 8; c < hidden; c += 256) {
        const uint4 v = *reinterpret_cast<const uint4*>(src + c);
        const float2 t0 = pair_to_float2<kBf16>(v.x), t1 = pair_to_float2<kBf16>(v.y);
        const float2 t2 = pair_to_float2<kBf16>(v.z), t3 = pair_to_float2<kBf16>(v.w);
        *reinterpret_cast<float4*>(dst + c) = make_float4(t0.x, t0.y, t1.x, t1.y);
        *reinterpret_cast<float4*>(dst + c + 4) = make_float4(t2.x, t2.y, t3.x, t3.y);
    }
}

// x (f32) = float(h (16-bit)): the stream restarts from the rounded LN(embeddings), as classifier.py does
template <bool kBf16>
__global__ void __launch_bounds__(256) half_to_f32_kernel(const uint16_t* __restrict__ h, float* __restrict__ x, long long n8) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n8) return;
    const uint4 v = reinterpret_cast<const uint4*>(h)[i];
    const float2 t0 = pair_to_float2<kBf16>(v.x), t1 = pair_to_float2<kBf16>(v.y);
    const float2 t2 = pair_to_float2<kBf16>(v.z), t3 = pair_to_float2<kBf16>(v.w);
    reinterpret_cast<float4*>(x)[2 * i] = make_float4(t0.x, t0.y, t1.x, t1.y);
    reinterpret_cast<float4*>(x)[2 * i + 1] = make_float4(t2.x, t2.y, t3.x, t3.y);
}

// Classification head for one sequence per CTA: pooled = hf[b, 0, :] (CLS); t = gelu(round16(pooled Wd^T));
// t = LN(t) * head_norm; logits = t Wc^T + b.  hidden <= 1024, hidden % 8 == 0.
// 32 warps; the dense layer (hidden x hidden weights, 1.2 MB at 768: all of it read by this one SM) takes four
// output features per warp at a time with 16-byte loads and independent accumulators -- the first version (8 warps,
// one feature per warp, 4-byte loads) was a chain of dependent L2 round trips: 216 us of the 4.4 ms forward.
constexpr int kHeadThreads = 1024;
template <bool kBf16>
__global__ void __launch_bounds__(kHeadThreads) clf_head_kernel(const uint16_t* __restrict__ hf, long long S, int hidden,
                                                                const uint16_t* __restrict__ wd, const float* __restrict__ head_norm,
                                                                const uint16_t* __restrict__ wc, const float* __restrict__ bc,
                                                                int n_labels, float eps, float* __restrict__ logits) {
    __shared__ __align__(16) float pooled[1024];
    __shared__ float t[1024];
    __shared__ float red[2][32];
    const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int kWarps = kHeadThreads / 32;
    const uint16_t* row = hf + static_cast<long long>(b) * S * hidden;
    for (int c = tid; c < hidden; c += kHeadThreads) pooled[c] = elem_to_float<kBf16>(row[c]);
    __syncthreads();
    // dense: four output features per warp per step, lanes stride over the input features in 8-element groups
    for (int j0 = warp * 4; j0 < hidden; j0 += kWarps * 4) {
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (int c = lane * 8; c < hidden; c += 256) {
            const float4 p0 = *reinterpret_cast<const float4*>(pooled + c), p1 = *reinterpret_cast<const float4*>(pooled + c + 4);
#pragma unroll
            for (int f = 0; f < 4; ++f) {
                if (j0 + f < hidden) {
                    const uint4 w8 = __ldg(reinterpret_cast<const uint4*>(wd + static_cast<long long>(j0 + f) * hidden + c));
                    const float2 w0 = pair_to_float2<kBf16>(w8.x), w1 = pair_to_float2<kBf16>(w8.y);
                    const float2 w2 = pair_to_float2<kBf16>(w8.z), w3 = pair_to_float2<kBf16>(w8.w);
                    acc[f] += p0.x * w0.x + p0.y * w0.y + p0.z * w1.x + p0.w * w1.y + p1.x * w2.x + p1.y * w2.y + p1.z * w3.x + p1.w * w3.y;
                }
            }
        }
#pragma unroll
        for (int f = 0; f < 4; ++f) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[f] += __shfl_xor_sync(0xffffffffu, acc[f], o);
            if (lane == 0 && j0 + f < hidden) {
                const float v = round_to_16<kBf16>(acc[f]);  // the GEMM output is 16-bit
                t[j0 + f] = 0.5f * v * (1.0f + erff(v * 0.70710678118654752f));
            }
        }
    }
    __syncthreads();
    float s = 0.f;
    for (int c = tid; c < hidden; c += kHeadThreads) s += t[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[0][warp] = s;
    __syncthreads();
    float mean = 0.f;
    for (int w = 0; w < kWarps; ++w) mean += red[0][w];
    mean /= hidden;
    float v = 0.f;
    for (int c = tid; c < hidden; c += kHeadThreads) v += (t[c] - mean) * (t[c] - mean);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[1][warp] = v;
    __syncthreads();
    float var = 0.f;
    for (int w = 0; w < kWarps; ++w) var += red[1][w];
    const float rstd = rsqrtf(var / hidden + eps);
    for (int c = tid; c < hidden; c += kHeadThreads) pooled[c] = (t[c] - mean) * rstd * head_norm[c];
    __syncthreads();
    for (int k = warp; k < n_labels; k += kWarps) {
        const uint16_t* wr = wc + static_cast<long long>(k) * hidden;
        float acc = 0.f;
        for (int c = lane; c < hidden; c += 32) acc += pooled[c] * elem_to_float<kBf16>(wr[c]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) logits[b * n_labels + k] = acc + bc[k];
    }
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct LayerW {
    const float* attn_norm;
    const uint16_t* wqkv;
    const uint16_t* wo;
    const float* mlp_norm;
    const uint16_t* wi;
    const uint16_t* wo2;
};

}  // namespace

struct rf_clf {
    rf_clf_config cfg{};
    int device = 0;
    Cublas blas;
    cublasHandle_t handle = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // weights: one bf16 block and one f32 block
    void* w16 = nullptr;
    void* w32 = nullptr;
    size_t w16_bytes = 0, w32_bytes = 0;
    const uint16_t *tok_emb = nullptr, *head_dense = nullptr, *cls_w = nullptr;
    const float *emb_norm = nullptr, *final_norm = nullptr, *head_norm = nullptr, *cls_b = nullptr;
    std::vector<LayerW> layers;
    // activation arena
    void* arena = nullptr;
    size_t arena_bytes = 0;
    // RoPE tables (cos, sin) x (global, local), [rope_cap, d/2] f32 each, in their own allocation: they depend on
    // the position only, so the tables of a longer sequence serve every shorter one, whatever B or the mask
    float* rope_buf = nullptr;
    int64_t rope_cap = 0;
    float last_ms = 0.f;
    // library GEMM workspace owned by the session (so that no allocation happens under graph capture)
    void* blas_ws = nullptr;
    // page-locked staging for ids / mask / logits: the captured graph copies from / to fixed addresses
    void* pinned = nullptr;
    size_t pinned_bytes = 0;
    // the forward of the last shape as a CUDA graph: a shape seen twice in a row is captured, then replayed
    cudaGraphExec_t graph_exec = nullptr;
    int64_t graph_key = -1, last_key = -1;
};

namespace {

struct Layout {
    size_t x, big, slot[2], ws, ids, mask, bias, logits, total;
    size_t ws_bytes;
};

Layout make_layout(const rf_clf_config& c, int64_t B, int64_t S, size_t attn_ws) {
    Layout L{};
    const size_t rows = static_cast<size_t>(B) * S, hid = c.hidden;
    const size_t chunk = std::min<size_t>(rows, static_cast<size_t>(c.mlp_chunk_rows));
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t at = off;
        off += align_up(bytes, 256);
        return at;
    };
    L.x = take(rows * hid * 4);
    L.big = take(std::max(rows * 3 * hid * 2, chunk * 3 * static_cast<size_t>(c.mlp) * 2));  // qkv | wi_out + act
    L.slot[0] = take(rows * hid * 2);
    L.slot[1] = take(rows * hid * 2);
    L.ws_bytes = attn_ws;
    L.ws = take(attn_ws);
    L.ids = take(rows * 8);
    L.mask = take(rows * 4);
    L.bias = take(rows * 4);
    L.logits = take(static_cast<size_t>(B) * c.n_labels * 4);
    L.total = off;
    return L;
}

int check_cfg(const rf_clf_config* c) {
    if (c == nullptr) return fail(RF_ERR_ARG, "config is null");
    if (c->hidden != c->heads * c->head_dim) return fail(RF_ERR_SHAPE, "hidden must equal heads * head_dim");
    if (c->head_dim != 64) return fail(RF_ERR_HEAD_DIM, "the classifier session needs head_dim 64");
    if (c->hidden % 8 || c->hidden > 1024 || c->mlp % 8 || c->n_layers < 1 || c->vocab_size < 1 || c->n_labels < 1 ||
        c->global_every < 1 || c->local_window < 2 || c->mlp_chunk_rows < 1 ||
        (c->act_dtype != RF_DTYPE_F16 && c->act_dtype != RF_DTYPE_BF16) ||
        (c->gemm_backend != RF_CLF_GEMM_OWN && c->gemm_backend != RF_CLF_GEMM_CUBLAS))
        return fail(RF_ERR_ARG, "bad classifier config");
    // rf_gemm_nt: accumulator tiles of 256 (or 192) columns, GeGLU slices of 128
    if (c->gemm_backend == RF_CLF_GEMM_OWN && ((c->hidden % 256 && c->hidden % 192) || c->mlp % 128))
        return fail(RF_ERR_UNSUPPORTED, "rf_gemm_nt needs hidden a multiple of 256 (or 192) and mlp a multiple of 128; "
                                        "select RF_CLF_GEMM_CUBLAS for other shapes");
    return RF_OK;
}

}  // namespace

extern "C" {

void rf_clf_config_default(rf_clf_config* c) {
    if (c == nullptr) return;
    c->vocab_size = 50368;
    c->hidden = 768;
    c->n_layers = 22;
    c->heads = 12;
    c->head_dim = 64;
    c->mlp = 1152;
    c->global_every = 3;
    c->local_window = 128;
    c->n_labels = 3;
    c->mlp_chunk_rows = 8192;
    c->act_dtype = RF_DTYPE_F16;
    c->rope_theta_global = 160000.0f;
    c->rope_theta_local = 10000.0f;
    c->eps = 1e-5f;
    c->gemm_backend = RF_CLF_GEMM_OWN;
}

size_t rf_clf_weight_elems(const rf_clf_config* c) {
    if (c == nullptr) return 0;
    const size_t hid = c->hidden, mlp = c->mlp;
    size_t n = static_cast<size_t>(c->vocab_size) * hid + hid + hid + hid * hid + hid + static_cast<size_t>(c->n_labels) * hid +
               c->n_labels;
    n += static_cast<size_t>(c->n_layers) * (hid + 3 * hid * hid + hid * hid + hid + 2 * mlp * hid + hid * mlp);
    return n;
}

int rf_clf_create(const rf_clf_config* cfg, const float* weights, size_t n_elems, int32_t device, rf_clf** out) {
    int rc = check_cfg(cfg);
    if (rc != RF_OK) return rc;
    if (weights == nullptr || out == nullptr) return fail(RF_ERR_ARG, "null pointer");
    if (n_elems != rf_clf_weight_elems(cfg))
        return fail(RF_ERR_SHAPE, "weight blob has " + std::to_string(n_elems) + " elements, expected " +
                                      std::to_string(rf_clf_weight_elems(cfg)));
    int32_t sms = 0, major = 0, minor = 0;
    rc = rf_device_check(device, &sms, &major, &minor);
    if (rc != RF_OK) return rc;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    rf_clf* s = new rf_clf();
    s->cfg = *cfg;
    s->device = device;
    std::string why;
    const bool use_blas = cfg->gemm_backend == RF_CLF_GEMM_CUBLAS;
    if (use_blas && !s->blas.load(&why)) {
        delete s;
        return fail(RF_ERR_CUDA, why);
    }
    auto bail = [&](int code, const std::string& msg) {
        rf_clf_destroy(s);
        return fail(code, msg);
    };
    if ((e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking)) != cudaSuccess) return bail(RF_ERR_CUDA, "cudaStreamCreate");
    cudaEventCreate(&s->ev0);
    cudaEventCreate(&s->ev1);
    if (use_blas) {
        if (s->blas.create(&s->handle) != 0) return bail(RF_ERR_CUDA, "cublasCreate failed");
        s->blas.set_stream(s->handle, s->stream);
        constexpr size_t kBlasWorkspace = 32u << 20;
        if ((e = cudaMalloc(&s->blas_ws, kBlasWorkspace)) != cudaSuccess) return bail(RF_ERR_CUDA, "cudaMalloc(cuBLAS workspace)");
        if (s->blas.set_workspace(s->handle, s->blas_ws, kBlasWorkspace) != 0) return bail(RF_ERR_CUDA, "cublasSetWorkspace failed");
    }

    // split the blob: matrices -> bf16 block, vectors -> f32 block
    const size_t hid = cfg->hidden, mlp = cfg->mlp, V = cfg->vocab_size, NL = cfg->n_labels;
    struct Item { size_t n; bool mat; };
    std::vector<Item> items = {{V * hid, true}, {hid, false}, {hid, false}, {hid * hid, true}, {hid, false}, {NL * hid, true}, {NL, false}};
    for (int i = 0; i < cfg->n_layers; ++i) {
        items.push_back({hid, false});
        items.push_back({3 * hid * hid, true});
        items.push_back({hid * hid, true});
        items.push_back({hid, false});
        items.push_back({2 * mlp * hid, true});
        items.push_back({hid * mlp, true});
    }
    size_t n16 = 0, n32 = 0;
    for (const Item& it : items) (it.mat ? n16 : n32) += align_up(it.n, 128);
    s->w16_bytes = n16 * 2;
    s->w32_bytes = n32 * 4;
    if ((e = cudaMalloc(&s->w16, s->w16_bytes)) != cudaSuccess) return bail(RF_ERR_CUDA, "cudaMalloc(weights)");
    if ((e = cudaMalloc(&s->w32, s->w32_bytes)) != cudaSuccess) return bail(RF_ERR_CUDA, "cudaMalloc(weights)");
    // upload f32 through a staging buffer and cast on the device (same rounding as torch's .to(bfloat16))
    size_t max_mat = 0;
    for (const Item& it : items) if (it.mat) max_mat = std::max(max_mat, it.n);
    float* stage = nullptr;
    if ((e = cudaMalloc(&stage, max_mat * 4)) != cudaSuccess) return bail(RF_ERR_CUDA, "cudaMalloc(staging)");
    std::vector<const void*> ptrs;
    size_t o16 = 0, o32 = 0, src = 0;
    for (const Item& it : items) {
        if (it.mat) {
            uint16_t* dst = static_cast<uint16_t*>(s->w16) + o16;
            cudaMemcpyAsync(stage, weights + src, it.n * 4, cudaMemcpyHostToDevice, s->stream);
            rf::launch_cast_from_f32(stage, dst, static_cast<long long>(it.n), cfg->act_dtype, s->stream);
            ptrs.push_back(dst);
            o16 += align_up(it.n, 128);
        } else {
            float* dst = static_cast<float*>(s->w32) + o32;
            cudaMemcpyAsync(dst, weights + src, it.n * 4, cudaMemcpyHostToDevice, s->stream);
            ptrs.push_back(dst);
            o32 += align_up(it.n, 128);
        }
        src += it.n;
    }
    e = cudaStreamSynchronize(s->stream);
    cudaFree(stage);
    if (e != cudaSuccess) return bail(RF_ERR_CUDA, std::string("weight upload: ") + cudaGetErrorString(e));
    size_t k = 0;
    s->tok_emb = static_cast<const uint16_t*>(ptrs[k++]);
    s->emb_norm = static_cast<const float*>(ptrs[k++]);
    s->final_norm = static_cast<const float*>(ptrs[k++]);
    s->head_dense = static_cast<const uint16_t*>(ptrs[k++]);
    s->head_norm = static_cast<const float*>(ptrs[k++]);
    s->cls_w = static_cast<const uint16_t*>(ptrs[k++]);
    s->cls_b = static_cast<const float*>(ptrs[k++]);
    for (int i = 0; i < cfg->n_layers; ++i) {
        LayerW lw;
        lw.attn_norm = static_cast<const float*>(ptrs[k++]);
        lw.wqkv = static_cast<const uint16_t*>(ptrs[k++]);
        lw.wo = static_cast<const uint16_t*>(ptrs[k++]);
        lw.mlp_norm = static_cast<const float*>(ptrs[k++]);
        lw.wi = static_cast<const uint16_t*>(ptrs[k++]);
        lw.wo2 = static_cast<const uint16_t*>(ptrs[k++]);
        s->layers.push_back(lw);
    }
    *out = s;
    return RF_OK;
}

int rf_clf_forward(rf_clf* s, const int64_t* input_ids, const float* attention_mask, int64_t B, int64_t S, float* logits) {
    if (s == nullptr || input_ids == nullptr || logits == nullptr) return fail(RF_ERR_ARG, "null pointer");
    if (B < 1 || S < 1) return fail(RF_ERR_SHAPE, "B and S must be positive");
    const rf_clf_config& c = s->cfg;
    cudaError_t e = cudaSetDevice(s->device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    const int64_t rows = B * S;
    const int hid = c.hidden, H = c.heads, d = c.head_dim;
    cudaStream_t st = s->stream;

    // attention call template: q/k/v are strided views of the packed [B,S,3,H,d] GEMM output, O is [B,S,H,d]
    rf_fa_params fp;
    rf_fa_params_init(&fp);
    fp.dtype = c.act_dtype;
    fp.out_dtype = c.act_dtype;
    fp.B = B; fp.H = H; fp.S = S; fp.d = d;
    const int64_t tok = 3ll * hid;
    // library GEMM: packed [B,S,3,H,d]; own projection: head-major [3,H,B*S,d] (each head's rows contiguous for the TMA)
    const bool head_major = c.gemm_backend == RF_CLF_GEMM_OWN;
    const int64_t qs_packed[3] = {S * tok, d, tok};
    const int64_t qs_heads[3] = {S * static_cast<int64_t>(d), B * S * static_cast<int64_t>(d), d};
    for (int i = 0; i < 3; ++i) fp.q_stride[i] = fp.k_stride[i] = fp.v_stride[i] = head_major ? qs_heads[i] : qs_packed[i];
    fp.o_stride[0] = S * static_cast<int64_t>(hid); fp.o_stride[1] = d; fp.o_stride[2] = hid;
    // workspace: the larger of the global and the local layer's needs (the pointers only matter for alignment checks)
    size_t ws_need = 0;
    {
        rf_fa_params probe = fp;
        probe.q = probe.k = probe.v = reinterpret_cast<const void*>(uintptr_t{256});
        probe.out = reinterpret_cast<void*>(uintptr_t{256});
        probe.pad_bias = attention_mask != nullptr ? reinterpret_cast<const float*>(uintptr_t{256}) : nullptr;
        size_t need = 0;
        int rc = rf_fa_fwd_workspace_bytes(&probe, &need);
        if (rc != RF_OK) return rc;
        ws_need = need;
        probe.window_left = c.local_window / 2 - 1;
        probe.window_right = c.local_window / 2;
        rc = rf_fa_fwd_workspace_bytes(&probe, &need);
        if (rc != RF_OK) return rc;
        ws_need = std::max(ws_need, need);
    }
    const Layout L = make_layout(c, B, S, ws_need);
    if (L.total > s->arena_bytes) {
        if (s->graph_exec != nullptr) cudaGraphExecDestroy(s->graph_exec);  // it holds arena addresses
        s->graph_exec = nullptr;
        s->graph_key = s->last_key = -1;
        if (s->arena != nullptr) cudaFree(s->arena);
        s->arena = nullptr;
        s->arena_bytes = 0;
        if ((e = cudaMalloc(&s->arena, L.total)) != cudaSuccess) return cuda_fail(e, "cudaMalloc(arena)");
        s->arena_bytes = L.total;
    }
    uint8_t* base = static_cast<uint8_t*>(s->arena);
    float* x = reinterpret_cast<float*>(base + L.x);
    uint16_t* big = reinterpret_cast<uint16_t*>(base + L.big);
    uint16_t* slot[2] = {reinterpret_cast<uint16_t*>(base + L.slot[0]), reinterpret_cast<uint16_t*>(base + L.slot[1])};
    long long* ids = reinterpret_cast<long long*>(base + L.ids);
    float* mask = reinterpret_cast<float*>(base + L.mask);
    float* bias = reinterpret_cast<float*>(base + L.bias);
    float* dlogits = reinterpret_cast<float*>(base + L.logits);
    // RoPE tables, f64 on the host like classifier.py's rope_tables; rebuilt only when S outgrows them
    if (S > s->rope_cap) {
        if (s->graph_exec != nullptr) cudaGraphExecDestroy(s->graph_exec);  // it holds the table addresses
        s->graph_exec = nullptr;
        s->graph_key = s->last_key = -1;
        if (s->rope_buf != nullptr) cudaFree(s->rope_buf);
        s->rope_buf = nullptr;
        s->rope_cap = 0;
        const int half = d / 2;
        const size_t per = static_cast<size_t>(S) * half;
        if ((e = cudaMalloc(reinterpret_cast<void**>(&s->rope_buf), 4 * per * sizeof(float))) != cudaSuccess)
            return cuda_fail(e, "cudaMalloc(rope tables)");
        std::vector<float> tab(4 * per);
        for (int kind = 0; kind < 2; ++kind) {
            const double theta = kind == 0 ? c.rope_theta_global : c.rope_theta_local;
            for (int64_t p = 0; p < S; ++p)
                for (int i = 0; i < half; ++i) {
                    const double ang = static_cast<double>(p) / pow(theta, (2.0 * i) / d);
                    tab[(kind * 2 + 0) * per + static_cast<size_t>(p) * half + i] = static_cast<float>(cos(ang));
                    tab[(kind * 2 + 1) * per + static_cast<size_t>(p) * half + i] = static_cast<float>(sin(ang));
                }
        }
        if ((e = cudaMemcpy(s->rope_buf, tab.data(), tab.size() * sizeof(float), cudaMemcpyHostToDevice)) != cudaSuccess)
            return cuda_fail(e, "rope upload");
        s->rope_cap = S;
    }
    const float* rope[4];
    for (int i = 0; i < 4; ++i) rope[i] = s->rope_buf + static_cast<size_t>(i) * s->rope_cap * (d / 2);

    // page-locked staging: [ids | mask | logits]
    const size_t pin_ids = 0, pin_mask = align_up(rows * 8, 256), pin_logits = pin_mask + align_up(rows * 4, 256);
    const size_t pin_total = pin_logits + align_up(static_cast<size_t>(B) * c.n_labels * 4, 256);
    if (pin_total > s->pinned_bytes) {
        if (s->graph_exec != nullptr) cudaGraphExecDestroy(s->graph_exec);
        s->graph_exec = nullptr;
        s->graph_key = s->last_key = -1;
        if (s->pinned != nullptr) cudaFreeHost(s->pinned);
        s->pinned = nullptr;
        s->pinned_bytes = 0;
        if ((e = cudaMallocHost(&s->pinned, pin_total)) != cudaSuccess) return cuda_fail(e, "cudaMallocHost(staging)");
        s->pinned_bytes = pin_total;
    }
    uint8_t* pin = static_cast<uint8_t*>(s->pinned);
    std::memcpy(pin + pin_ids, input_ids, rows * 8);
    if (attention_mask != nullptr) std::memcpy(pin + pin_mask, attention_mask, rows * 4);
    const float* pad_bias = attention_mask != nullptr ? bias : nullptr;
    fp.pad_bias = pad_bias;

    const int64_t key = (B << 40) | (S << 1) | (attention_mask != nullptr ? 1 : 0);
    auto finish = [&]() -> int {
        cudaEventRecord(s->ev1, st);
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e, "classifier forward");
        if (L.ws_bytes > 0) {  // a bounded wait inside an attention kernel ran out: the logits are invalid
            const int rc_st = rf_fa_launch_status(base + L.ws, st);
            if (rc_st != RF_OK) return rc_st;
        }
        if (c.gemm_backend == RF_CLF_GEMM_OWN) {  // ... or inside a projection
            const int rc_g = rf_gemm_launch_status(st);
            if (rc_g != RF_OK) return rc_g;
        }
        cudaEventElapsedTime(&s->last_ms, s->ev0, s->ev1);
        std::memcpy(logits, pin + pin_logits, static_cast<size_t>(B) * c.n_labels * 4);
        return RF_OK;
    };
    if (s->graph_exec != nullptr && s->graph_key == key) {
        cudaEventRecord(s->ev0, st);
        if ((e = cudaGraphLaunch(s->graph_exec, st)) != cudaSuccess) return cuda_fail(e, "cudaGraphLaunch");
        return finish();
    }
    // A shape seen twice in a row is captured (the first call ran eagerly and loaded every module).
    const bool capture = key == s->last_key;
    s->last_key = key;
    if (capture) {
        if (s->graph_exec != nullptr) cudaGraphExecDestroy(s->graph_exec);
        s->graph_exec = nullptr;
        s->graph_key = -1;
        if ((e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal)) != cudaSuccess) return cuda_fail(e, "cudaStreamBeginCapture");
    } else {
        cudaEventRecord(s->ev0, st);
    }
    auto enqueue = [&]() -> int {
    if ((e = cudaMemcpyAsync(ids, pin + pin_ids, rows * 8, cudaMemcpyHostToDevice, st)) != cudaSuccess) return cuda_fail(e, "ids upload");
    if (attention_mask != nullptr) {
        if ((e = cudaMemcpyAsync(mask, pin + pin_mask, rows * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess) return cuda_fail(e, "mask upload");
        int rc = rf_pad_bias_from_mask(mask, bias, rows, st);  // one shared chain per forward (rewrite.cpp:303-318)
        if (rc != RF_OK) return rc;
    }

    const bool own_gemm = c.gemm_backend == RF_CLF_GEMM_OWN;
    auto gemm = [&](const uint16_t* a, const uint16_t* w, uint16_t* y, int64_t m, int n, int k) {
        if (own_gemm) return rf_gemm_nt(a, w, y, m, n, k, 0, 0, 0, c.act_dtype, nullptr, st);
        // y[m, n] = a[m, k] @ w[n, k]^T, row-major == column-major y^T[n, m] = w^T(k x n)^T * a^T(k x m)
        const float alpha = 1.f, beta = 0.f;
        const int ty = c.act_dtype == RF_DTYPE_BF16 ? kCudaR16BF : kCudaR16F;
        const int r = s->blas.gemm_ex(s->handle, kCublasOpT, kCublasOpN, n, static_cast<int>(m), k, &alpha, w, ty, k, a, ty, k,
                                      &beta, y, ty, n, kCublasCompute32F, kCublasGemmDefault);
        return r == 0 ? RF_OK : fail(RF_ERR_CUDA, "cublasGemmEx failed, status " + std::to_string(r));
    };
#define RF_TRY(expr)               \
    do {                           \
        const int rc_ = (expr);    \
        if (rc_ != RF_OK) return rc_; \
    } while (0)

    // embeddings -> f32 stream; h = LN(x) * emb_norm; the stream restarts from the bf16-rounded h
    const bool bf = c.act_dtype == RF_DTYPE_BF16;
    const int dt = c.act_dtype;
    if (bf) embed_gather_kernel<true><<<static_cast<unsigned>((rows + 3) / 4), 128, 0, st>>>(s->tok_emb, ids, x, rows, hid, c.vocab_size);
    else embed_gather_kernel<false><<<static_cast<unsigned>((rows + 3) / 4), 128, 0, st>>>(s->tok_emb, ids, x, rows, hid, c.vocab_size);
    int cur = 0;  // slot that holds the current bf16 GEMM operand (h)
    RF_TRY(rf_add_layernorm(x, nullptr, s->emb_norm, slot[cur], rows, hid, c.eps, dt, st));
    if (bf) half_to_f32_kernel<true><<<static_cast<unsigned>((rows * hid / 8 + 255) / 256), 256, 0, st>>>(slot[cur], x, rows * hid / 8);
    else half_to_f32_kernel<false><<<static_cast<unsigned>((rows * hid / 8 + 255) / 256), 256, 0, st>>>(slot[cur], x, rows * hid / 8);

    const int64_t chunk = std::min<int64_t>(rows, c.mlp_chunk_rows);
    for (int i = 0; i < c.n_layers; ++i) {
        const LayerW& w = s->layers[i];
        // (for i > 0 the LN that produced h also added the previous layer's MLP output into x: see the loop tail)
        uint16_t* h = slot[cur];
        const bool glob = i % c.global_every == 0;
        if (own_gemm) {  // qkv [rows, 3*hid] == [B,S,3,H,d], rotary embedding applied in the projection's epilogue
            rf_gemm_epilogue ep{};
            ep.kind = RF_GEMM_EPI_ROPE;
            ep.head_dim = d;
            ep.S = S;
            ep.cos_table = rope[glob ? 0 : 2];
            ep.sin_table = rope[glob ? 1 : 3];
            ep.head_major = 1;
            RF_TRY(rf_gemm_nt(h, w.wqkv, big, rows, 3 * hid, hid, 0, 0, 0, dt, &ep, st));
        } else {
            RF_TRY(gemm(h, w.wqkv, big, rows, 3 * hid, hid));
            RF_TRY(rf_rope_qkv(big, rope[glob ? 0 : 2], rope[glob ? 1 : 3], rows, S, H, d, dt, st));
        }
        uint16_t* attn = slot[cur ^ 1];
        fp.q = big;
        fp.k = big + (head_major ? rows * hid : hid);
        fp.v = big + 2 * (head_major ? rows * hid : hid);
        fp.out = attn;
        fp.window_left = glob ? -1 : c.local_window / 2 - 1;                    // rewrite.cpp:355-361
        fp.window_right = glob ? -1 : c.local_window / 2;
        RF_TRY(rf_fa_fwd(&fp, base + L.ws, L.ws_bytes, st));
        uint16_t* o = slot[cur];                                            // h is dead
        uint16_t* h2 = slot[cur ^ 1];                                       // (attn is dead once the projection has run)
        rf_gemm_epilogue res{};
        res.kind = RF_GEMM_EPI_RESIDUAL;
        if (own_gemm) {  // x += attn Wo^T inside the projection (TMA reduce-add of the f32 accumulators); h2 = LN(x)
            RF_TRY(rf_gemm_nt(attn, w.wo, x, rows, hid, hid, 0, 0, 0, dt, &res, st));
            RF_TRY(rf_add_layernorm(x, nullptr, w.mlp_norm, h2, rows, hid, c.eps, dt, st));
        } else {
            RF_TRY(gemm(attn, w.wo, o, rows, hid, hid));
            RF_TRY(rf_add_layernorm(x, o, w.mlp_norm, h2, rows, hid, c.eps, dt, st));    // x += attn out; h2 = LN(x)
        }
        uint16_t* delta = slot[cur];                                        // o is dead
        for (int64_t r0 = 0; r0 < rows; r0 += chunk) {
            const int64_t r1 = std::min(rows, r0 + chunk);
            uint16_t* wi_out = big;                                         // qkv is dead
            uint16_t* act = big + static_cast<size_t>(chunk) * 2 * c.mlp;
            if (own_gemm) {  // act = gelu(h2 Wi_in^T) * (h2 Wi_gate^T) straight out of the up-projection
                rf_gemm_epilogue ep{};
                ep.kind = RF_GEMM_EPI_GEGLU;
                RF_TRY(rf_gemm_nt(h2 + r0 * hid, w.wi, act, r1 - r0, 2 * c.mlp, hid, 0, 0, 0, dt, &ep, st));
                RF_TRY(rf_gemm_nt(act, w.wo2, x + r0 * hid, r1 - r0, hid, c.mlp, 0, 0, 0, dt, &res, st));  // x += mlp out
                continue;
            } else {
                RF_TRY(gemm(h2 + r0 * hid, w.wi, wi_out, r1 - r0, 2 * c.mlp, hid));
                RF_TRY(rf_geglu(wi_out, act, r1 - r0, c.mlp, dt, st));
            }
            RF_TRY(gemm(act, w.wo2, delta + r0 * hid, r1 - r0, hid, c.mlp));
        }
        // x += mlp out; h = LN(x) with the next layer's attn_norm (or the final norm)
        const float* next_norm = i + 1 < c.n_layers ? s->layers[i + 1].attn_norm : s->final_norm;
        RF_TRY(rf_add_layernorm(x, own_gemm ? nullptr : delta, next_norm, slot[cur ^ 1], rows, hid, c.eps, dt, st));  // h2 is dead
        cur ^= 1;
    }
    if (bf)
        clf_head_kernel<true><<<static_cast<unsigned>(B), kHeadThreads, 0, st>>>(slot[cur], S, hid, s->head_dense, s->head_norm, s->cls_w,
                                                                        s->cls_b, c.n_labels, c.eps, dlogits);
    else
        clf_head_kernel<false><<<static_cast<unsigned>(B), kHeadThreads, 0, st>>>(slot[cur], S, hid, s->head_dense, s->head_norm, s->cls_w,
                                                                         s->cls_b, c.n_labels, c.eps, dlogits);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "classifier kernels");
    if ((e = cudaMemcpyAsync(pin + pin_logits, dlogits, static_cast<size_t>(B) * c.n_labels * 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        return cuda_fail(e, "logits download");
    return RF_OK;
    };  // enqueue
    const int rc_enq = enqueue();
    if (capture) {
        cudaGraph_t graph = nullptr;
        e = cudaStreamEndCapture(st, &graph);
        if (rc_enq != RF_OK) {
            if (graph != nullptr) cudaGraphDestroy(graph);
            return rc_enq;
        }
        if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
        e = cudaGraphInstantiate(&s->graph_exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) {
            s->graph_exec = nullptr;
            return cuda_fail(e, "cudaGraphInstantiate");
        }
        s->graph_key = key;
        cudaEventRecord(s->ev0, st);
        if ((e = cudaGraphLaunch(s->graph_exec, st)) != cudaSuccess) return cuda_fail(e, "cudaGraphLaunch");
    } else if (rc_enq != RF_OK) {
        return rc_enq;
    }
    const int rc_fin = finish();
#undef RF_TRY
    return rc_fin;
}

int rf_clf_session_bytes(const rf_clf* s, size_t* weight_bytes, size_t* arena_bytes) {
    if (s == nullptr) return fail(RF_ERR_ARG, "session is null");
    if (weight_bytes != nullptr) *weight_bytes = s->w16_bytes + s->w32_bytes;
    if (arena_bytes != nullptr) *arena_bytes = s->arena_bytes;
    return RF_OK;
}

float rf_clf_last_forward_ms(const rf_clf* s) { return s != nullptr ? s->last_ms : 0.f; }

int rf_clf_head(const void* hf, int64_t B, int64_t S, int32_t hidden, const void* head_dense, const float* head_norm,
                const void* cls_w, const float* cls_b, int32_t n_labels, float eps, int32_t dtype, float* logits,
                void* stream) {
    if (hf == nullptr || head_dense == nullptr || head_norm == nullptr || cls_w == nullptr || cls_b == nullptr || logits == nullptr)
        return fail(RF_ERR_ARG, "rf_clf_head: null pointer");
    if (B < 0 || S < 1 || hidden < 8 || hidden > 1024 || hidden % 8 || n_labels < 1) return fail(RF_ERR_SHAPE, "rf_clf_head: bad shape (hidden must be a multiple of 8, at most 1024)");
    if (dtype != RF_DTYPE_F16 && dtype != RF_DTYPE_BF16) return fail(RF_ERR_ARG, "rf_clf_head: dtype must be bf16 or f16");
    if (B == 0) return RF_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint16_t* h16 = static_cast<const uint16_t*>(hf);
    const uint16_t* wd = static_cast<const uint16_t*>(head_dense);
    const uint16_t* wc = static_cast<const uint16_t*>(cls_w);
    if (dtype == RF_DTYPE_BF16)
        clf_head_kernel<true><<<static_cast<unsigned>(B), kHeadThreads, 0, st>>>(h16, S, hidden, wd, head_norm, wc, cls_b, n_labels, eps, logits);
    else
        clf_head_kernel<false><<<static_cast<unsigned>(B), kHeadThreads, 0, st>>>(h16, S, hidden, wd, head_norm, wc, cls_b, n_labels, eps, logits);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? RF_OK : cuda_fail(e, "rf_clf_head launch");
}

void rf_clf_destroy(rf_clf* s) {
    if (s == nullptr) return;
    cudaSetDevice(s->device);
    if (s->handle != nullptr && s->blas.destroy != nullptr) s->blas.destroy(s->handle);
    if (s->graph_exec != nullptr) cudaGraphExecDestroy(s->graph_exec);
    if (s->arena != nullptr) cudaFree(s->arena);
    if (s->rope_buf != nullptr) cudaFree(s->rope_buf);
    if (s->blas_ws != nullptr) cudaFree(s->blas_ws);
    if (s->pinned != nullptr) cudaFreeHost(s->pinned);
    if (s->w16 != nullptr) cudaFree(s->w16);
    if (s->w32 != nullptr) cudaFree(s->w32);
    if (s->ev0 != nullptr) cudaEventDestroy(s->ev0);
    if (s->ev1 != nullptr) cudaEventDestroy(s->ev1);
    if (s->stream != nullptr) cudaStreamDestroy(s->stream);
    delete s;
}

}  // extern "C"
