// fa_aux.cu -- small HBM-bound kernels around the attention op: padding-bias preparation
// (O(B*S) workspace, never S x S), the split-KV softmax merge, pad-bias chain, dtype casts.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "fa_internal.h"

namespace rf {
namespace {

// One CTA per (128-key tile, batch).  Converts the reference's additive pad bias
// (attention.cpp:160-169: masked iff <= -30000, otherwise added to the score) into the log2
// domain the kernel works in, and classifies the tile so the attention kernel can skip fully
// padded tiles and drop the per-element predicate on fully live, zero-bias tiles.
__global__ void __launch_bounds__(128) bias_prepare_kernel(const float* __restrict__ pad_bias, int S,
                                                           float* __restrict__ bias2,
                                                           uint8_t* __restrict__ tile_flags, int n_kv_tiles) {
    const int n = blockIdx.x, b = blockIdx.y;
    const int j = n * kBlockN + threadIdx.x;
    float v = -CUDART_INF_F;
    bool live = false, plain = false;
    if (j < S) {
        const float raw = pad_bias[static_cast<size_t>(b) * S + j];
        live = raw > kMaskThreshold;
        plain = live && raw == 0.0f;  // -0.0f == 0.0f: the f16-cast chain yields -0 for live keys
        v = live ? raw * kLog2e : -CUDART_INF_F;
    }
    bias2[(static_cast<size_t>(b) * n_kv_tiles + n) * kBlockN + threadIdx.x] = v;
    const int any_live = __syncthreads_or(live ? 1 : 0);
    const int all_plain = __syncthreads_and(plain ? 1 : 0);
    if (threadIdx.x == 0)
        tile_flags[b * n_kv_tiles + n] = !any_live ? kTileSkip : (all_plain ? kTileFull : kTileMixed);
}


// One CTA per (128-key tile, head, batch): the largest key norm of the tile, an upper bound within 1.6 % (the odd
// element of a bf16 pair is squared as it sits in its 32-bit word: the even element's bits below it only lengthen
// the mantissa).  Eight threads share a row (16 bytes each, so a warp reads four whole 128-byte rows per load
// instruction whatever the row stride is), eight passes cover the tile's 128 rows, all loads in flight at once.
// Rows >= S count as 0.
template <bool kBf16>
__device__ __forceinline__ float sumsq8_bound(const uint4& v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    float a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        float lo, hi;
        if (kBf16) {
            lo = __uint_as_float(w[e] << 16);
            hi = __uint_as_float(w[e]);
        } else {
            const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[e]));
            lo = f.x;
            hi = f.y;
        }
        a0 = fmaf(lo, lo, a0);
        a1 = fmaf(hi, hi, a1);
    }
    return a0 + a1;
}

template <bool kBf16>
__global__ void __launch_bounds__(128) k_tile_norms_kernel(const uint16_t* __restrict__ k, long long k_sb, long long k_sh,
                                                           long long k_ss, int H, int S, int d, int n_kv_tiles,
                                                           float* __restrict__ kmax) {
    __shared__ float red[4];
    // let the attention kernel (launched with programmatic stream serialization) start its prologue now; it
    // waits for this grid to complete before it reads anything written here
    asm volatile("griddepcontrol.launch_dependents;");
    const int n = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int sub = threadIdx.x & 7;    // 16-byte chunk of the row
    const int rgrp = threadIdx.x >> 3;  // row inside a pass of 16 rows
    const uint16_t* kb = k + b * k_sb + h * k_sh + sub * 8;
    constexpr int kPasses = kBlockN / 16;
    // head_dim 128: rows are sixteen chunks, a thread takes chunks sub and sub + 8
    uint4 kv[kPasses], kw[kPasses];
#pragma unroll
    for (int pass = 0; pass < kPasses; ++pass) {
        const int row = n * kBlockN + pass * 16 + rgrp;
        kv[pass] = kw[pass] = make_uint4(0u, 0u, 0u, 0u);
        if (row < S && sub * 8 < d)  // head_dim 32: rows are four 16-byte chunks
            kv[pass] = __ldg(reinterpret_cast<const uint4*>(kb + row * k_ss));
        if (row < S && 64 + sub * 8 < d) kw[pass] = __ldg(reinterpret_cast<const uint4*>(kb + row * k_ss + 64));
    }
    float kn_max = 0.f;
#pragma unroll
    for (int pass = 0; pass < kPasses; ++pass) {
        float ks = sumsq8_bound<kBf16>(kv[pass]);
        if (d > 64) ks += sumsq8_bound<kBf16>(kw[pass]);
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) ks += __shfl_xor_sync(0xffffffffu, ks, o);
        kn_max = fmaxf(kn_max, ks);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) kn_max = fmaxf(kn_max, __shfl_xor_sync(0xffffffffu, kn_max, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = kn_max;
    __syncthreads();
    if (threadIdx.x == 0)
        kmax[(static_cast<size_t>(b) * H + h) * n_kv_tiles + n] = sqrtf(fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3])));
}

constexpr int kMaxParts = 16;
struct MergePtrs {
    const float* o[kMaxParts];
    const float* m[kMaxParts];
    const float* l[kMaxParts];
};

template <typename T>
__device__ __forceinline__ void store_out(void* out, size_t idx, float v);
template <>
__device__ __forceinline__ void store_out<float>(void* out, size_t idx, float v) {
    static_cast<float*>(out)[idx] = v;
}
template <>
__device__ __forceinline__ void store_out<__nv_bfloat16>(void* out, size_t idx, float v) {
    static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(v);
}
template <>
__device__ __forceinline__ void store_out<__half>(void* out, size_t idx, float v) {
    static_cast<__half*>(out)[idx] = __float2half_rn(v);
}

__device__ __forceinline__ void store_dyn(void* out, size_t idx, float v, int dtype) {
    if (dtype == 2)
        store_out<float>(out, idx, v);
    else if (dtype == 0)
        store_out<__nv_bfloat16>(out, idx, v);
    else
        store_out<__half>(out, idx, v);
}

// Softmax merge of G split-KV partials; same algebra as the per-tile update of
// attention.cpp:177-196.  One thread per (row, 4 consecutive dims); fixed g order => deterministic.
__global__ void __launch_bounds__(256) merge_kernel(const MergePtrs ptrs, int G, long long rows, int d, void* out,
                                                    int out_dtype) {
    const int d4 = d >> 2;
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= rows * d4) return;
    const long long row = idx / d4;
    const int c4 = static_cast<int>(idx % d4);
    float mstar = -CUDART_INF_F;
    for (int g = 0; g < G; ++g) mstar = fmaxf(mstar, ptrs.m[g][row]);
    float lsum = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int g = 0; g < G; ++g) {
        const float mg = ptrs.m[g][row];
        if (mg == -CUDART_INF_F) continue;  // no live key in this block
        const float w = exp2f(mg - mstar);
        lsum = fmaf(w, ptrs.l[g][row], lsum);
        const float4 og = reinterpret_cast<const float4*>(ptrs.o[g])[row * d4 + c4];
        acc.x = fmaf(w, og.x, acc.x);
        acc.y = fmaf(w, og.y, acc.y);
        acc.z = fmaf(w, og.z, acc.z);
        acc.w = fmaf(w, og.w, acc.w);
    }
    const float inv = lsum > 0.f ? 1.0f / lsum : 0.f;
    const size_t o = static_cast<size_t>(row) * d + c4 * 4;
    store_dyn(out, o + 0, acc.x * inv, out_dtype);
    store_dyn(out, o + 1, acc.y * inv, out_dtype);
    store_dyn(out, o + 2, acc.z * inv, out_dtype);
    store_dyn(out, o + 3, acc.w * inv, out_dtype);
}

__global__ void __launch_bounds__(256) partial_neutral_kernel(float* __restrict__ o_part, float* __restrict__ m_part,
                                                              float* __restrict__ l_part, long long rows, int d) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx < rows * d) o_part[idx] = 0.f;
    if (idx < rows) {
        m_part[idx] = -CUDART_INF_F;
        l_part[idx] = 0.f;
    }
}

__global__ void __launch_bounds__(256) rescale_partial_kernel(float* o_part, float* l_part,
                                                              const float* __restrict__ m_part,
                                                              const float* __restrict__ m_star, long long rows, int d) {
    const int d4 = d >> 2;
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= rows * d4) return;
    const long long row = idx / d4;
    const int c4 = static_cast<int>(idx % d4);
    const float mg = m_part[row];
    const float w = (mg == -CUDART_INF_F) ? 0.f : exp2f(mg - m_star[row]);
    float4* op = reinterpret_cast<float4*>(o_part) + row * d4 + c4;
    float4 v = *op;
    // w == 0 rows may hold garbage-free zeros already; force exact zeros so no NaN can leak
    v = (w == 0.f) ? make_float4(0.f, 0.f, 0.f, 0.f) : make_float4(v.x * w, v.y * w, v.z * w, v.w * w);
    *op = v;
    if (c4 == 0) l_part[row] = (w == 0.f) ? 0.f : l_part[row] * w;
}

__global__ void __launch_bounds__(256) normalize_kernel(const float* __restrict__ o_sum,
                                                        const float* __restrict__ l_sum, long long rows, int d,
                                                        void* out, int out_dtype) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= rows * d) return;
    const long long row = idx / d;
    const float l = l_sum[row];
    store_dyn(out, static_cast<size_t>(idx), l > 0.f ? o_sum[idx] / l : 0.f, out_dtype);
}

// rewrite.cpp:303-318 executed by interpreter.cpp:230-257: Sub, Mul in f32, then Cast(f16)
// = round-trip through binary16 (RNE, tensor.cpp:47-98).
__global__ void __launch_bounds__(256) pad_bias_from_mask_kernel(const float* __restrict__ mask,
                                                                 float* __restrict__ bias, long long n) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float inv = __fsub_rn(1.0f, mask[i]);
    const float scaled = __fmul_rn(inv, -65504.0f);
    bias[i] = __half2float(__float2half_rn(scaled));
}

__global__ void __launch_bounds__(256) cast_from_f32_kernel(const float* __restrict__ src, void* dst, long long n,
                                                            int dst_dtype) {
    const long long i = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    if (i >= n) return;
    if (i + 3 < n) {
        const float4 v = *reinterpret_cast<const float4*>(src + i);
        if (dst_dtype == 0) {
            __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b2 = __floats2bfloat162_rn(v.z, v.w);
            uint2 w = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b2));
            *reinterpret_cast<uint2*>(static_cast<uint16_t*>(dst) + i) = w;
        } else {
            __half2 a = __floats2half2_rn(v.x, v.y), b2 = __floats2half2_rn(v.z, v.w);
            uint2 w = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b2));
            *reinterpret_cast<uint2*>(static_cast<uint16_t*>(dst) + i) = w;
        }
    } else {
        for (long long j = i; j < n; ++j) store_dyn(dst, static_cast<size_t>(j), src[j], dst_dtype);
    }
}

__global__ void __launch_bounds__(256) cast_to_f32_kernel(const void* __restrict__ src, float* __restrict__ dst,
                                                          long long n, int src_dtype) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    dst[i] = src_dtype == 0 ? __bfloat162float(static_cast<const __nv_bfloat16*>(src)[i])
                            : __half2float(static_cast<const __half*>(src)[i]);
}

inline unsigned blocks_for(long long n, int per_block) { return static_cast<unsigned>((n + per_block - 1) / per_block); }

}  // namespace

cudaError_t launch_bias_prepare(const float* pad_bias, int B, int S, float* bias2, uint8_t* tile_flags,
                                int n_kv_tiles, cudaStream_t stream) {
    dim3 grid(n_kv_tiles, B);
    bias_prepare_kernel<<<grid, kBlockN, 0, stream>>>(pad_bias, S, bias2, tile_flags, n_kv_tiles);
    return cudaGetLastError();
}

cudaError_t launch_k_tile_norms(const void* k, const long long ks[3], int dtype, int B, int H, int S, int d, int n_kv_tiles,
                                float* kmax, cudaStream_t stream) {
    dim3 grid(n_kv_tiles, H, B);
    const uint16_t* k16 = static_cast<const uint16_t*>(k);
    if (dtype == 0)
        k_tile_norms_kernel<true><<<grid, kBlockN, 0, stream>>>(k16, ks[0], ks[1], ks[2], H, S, d, n_kv_tiles, kmax);
    else
        k_tile_norms_kernel<false><<<grid, kBlockN, 0, stream>>>(k16, ks[0], ks[1], ks[2], H, S, d, n_kv_tiles, kmax);
    return cudaGetLastError();
}

cudaError_t launch_merge(const float* const* o_parts, const float* const* m_parts, const float* const* l_parts,
                         int G, long long rows, int d, void* out, int out_dtype, cudaStream_t stream) {
    if (G < 1 || G > kMaxParts || (d & 3)) return cudaErrorInvalidValue;
    MergePtrs ptrs{};
    for (int g = 0; g < G; ++g) {
        ptrs.o[g] = o_parts[g];
        ptrs.m[g] = m_parts[g];
        ptrs.l[g] = l_parts[g];
    }
    const long long n = rows * (d >> 2);
    if (n == 0) return cudaSuccess;
    merge_kernel<<<blocks_for(n, 256), 256, 0, stream>>>(ptrs, G, rows, d, out, out_dtype);
    return cudaGetLastError();
}

cudaError_t launch_partial_neutral(float* o_part, float* m_part, float* l_part, long long rows, int d, cudaStream_t stream) {
    const long long n = rows * d;
    if (n == 0) return cudaSuccess;
    partial_neutral_kernel<<<blocks_for(n, 256), 256, 0, stream>>>(o_part, m_part, l_part, rows, d);
    return cudaGetLastError();
}

cudaError_t launch_rescale_partial(float* o_part, float* l_part, const float* m_part, const float* m_star,
                                   long long rows, int d, cudaStream_t stream) {
    if (d & 3) return cudaErrorInvalidValue;
    const long long n = rows * (d >> 2);
    if (n == 0) return cudaSuccess;
    rescale_partial_kernel<<<blocks_for(n, 256), 256, 0, stream>>>(o_part, l_part, m_part, m_star, rows, d);
    return cudaGetLastError();
}

cudaError_t launch_normalize(const float* o_sum, const float* l_sum, long long rows, int d, void* out,
                             int out_dtype, cudaStream_t stream) {
    const long long n = rows * d;
    if (n == 0) return cudaSuccess;
    normalize_kernel<<<blocks_for(n, 256), 256, 0, stream>>>(o_sum, l_sum, rows, d, out, out_dtype);
    return cudaGetLastError();
}

cudaError_t launch_pad_bias_from_mask(const float* mask, float* bias, long long n, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    pad_bias_from_mask_kernel<<<blocks_for(n, 256), 256, 0, stream>>>(mask, bias, n);
    return cudaGetLastError();
}

cudaError_t launch_cast_from_f32(const float* src, void* dst, long long n, int dst_dtype, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    cast_from_f32_kernel<<<blocks_for((n + 3) / 4, 256), 256, 0, stream>>>(src, dst, n, dst_dtype);
    return cudaGetLastError();
}

cudaError_t launch_cast_to_f32(const void* src, float* dst, long long n, int src_dtype, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    cast_to_f32_kernel<<<blocks_for(n, 256), 256, 0, stream>>>(src, dst, n, src_dtype);
    return cudaGetLastError();
}

}  // namespace rf
