// encoder_ops.cu -- the glue either side of the attention op in a ModernBERT-style encoder layer
// (SURVEY.md 8(f) rank 1): all HBM-bound elementwise / row kernels, written so that the QKV GEMM
// output [B,S,3,H,d] feeds the attention kernel in place (no head-split transpose) and the
// attention output [B,S,H*d] feeds the out-projection GEMM in place.
//   rope_qkv      rotary embedding on the Q and K thirds of a packed QKV tensor, in place
//   add_layernorm residual add into the f32 stream + LayerNorm (no bias) -> bf16 GEMM operand
//   geglu         act = gelu(x[:, :I]) * x[:, I:]  on the Wi GEMM output
// The projections themselves are rf_gemm_nt (gemm_sm100.cu), which fuses rope_qkv, geglu and the residual add into its
// epilogues; the stand-alone kernels here serve the library-GEMM A/B path and the tests.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rf_fa.h"

namespace {

// 16-bit activation type of the encoder: bf16 or f16 (rf_dtype), selected per call.  f16 has 11 significant
// bits against bf16's 8 and LayerNorm keeps the activations O(1), so the classifier defaults to f16 (logits
// within 1e-2 of the fp32 oracle at full depth need it); bf16 stays available.
template <bool kBf16>
struct Half2 {
    using type = __nv_bfloat162;
    static __device__ __forceinline__ float2 to_float2(uint32_t w) { return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w)); }
    static __device__ __forceinline__ uint32_t from_floats(float a, float b) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        return *reinterpret_cast<const uint32_t*>(&h);
    }
};
template <>
struct Half2<false> {
    using type = __half2;
    static __device__ __forceinline__ float2 to_float2(uint32_t w) { return __half22float2(*reinterpret_cast<const __half2*>(&w)); }
    static __device__ __forceinline__ uint32_t from_floats(float a, float b) {
        const __half2 h = __floats2half2_rn(a, b);
        return *reinterpret_cast<const uint32_t*>(&h);
    }
};

// qkv: [tokens, 3, H, d] bf16; cos/sin: [S, d/2] f32; token t has position t % S.
// Rotates elements (i, i + d/2) -- the "rotate_half" convention of ModernBERT / HF rotary embeddings.
// One thread per 8 pairs: two 16-byte loads and two 16-byte stores of bf16, cos/sin as float4s, so a
// warp covers whole 128-byte head rows (HBM-bound: Q and K are read and written once).  d % 16 == 0.
template <bool kBf16>
__global__ void __launch_bounds__(256) rope_qkv_kernel(uint16_t* __restrict__ qkv, const float* __restrict__ cosb,
                                                       const float* __restrict__ sinb, long long tokens, int S, int H,
                                                       int d) {
    const int half = d >> 1;
    const int vecs = half >> 3;  // threads per (token, q|k, head) row
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long total = tokens * 2 * H * vecs;
    if (idx >= total) return;
    const int i = static_cast<int>(idx % vecs) * 8;
    long long r = idx / vecs;
    const int h = static_cast<int>(r % H);
    r /= H;
    const int which = static_cast<int>(r % 2);  // 0 = q, 1 = k
    const long long t = r / 2;
    const int pos = static_cast<int>(t % S);
    uint16_t* base = qkv + ((t * 3 + which) * H + h) * d;
    uint4 a = *reinterpret_cast<const uint4*>(base + i);
    uint4 b = *reinterpret_cast<const uint4*>(base + i + half);
    const float4* cp = reinterpret_cast<const float4*>(cosb + static_cast<long long>(pos) * half + i);
    const float4* sp = reinterpret_cast<const float4*>(sinb + static_cast<long long>(pos) * half + i);
    const float4 c0 = __ldg(cp), c1 = __ldg(cp + 1), s0 = __ldg(sp), s1 = __ldg(sp + 1);
    const float cs[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    const float sn[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
    uint32_t* a2 = reinterpret_cast<uint32_t*>(&a);
    uint32_t* b2 = reinterpret_cast<uint32_t*>(&b);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float2 x1 = Half2<kBf16>::to_float2(a2[e]), x2 = Half2<kBf16>::to_float2(b2[e]);
        a2[e] = Half2<kBf16>::from_floats(x1.x * cs[2 * e] - x2.x * sn[2 * e], x1.y * cs[2 * e + 1] - x2.y * sn[2 * e + 1]);
        b2[e] = Half2<kBf16>::from_floats(x2.x * cs[2 * e] + x1.x * sn[2 * e], x2.y * cs[2 * e + 1] + x1.y * sn[2 * e + 1]);
    }
    *reinterpret_cast<uint4*>(base + i) = a;
    *reinterpret_cast<uint4*>(base + i + half) = b;
}

// x (f32 residual stream, [rows, n]) += delta (16-bit, may be null); y = LayerNorm(x) * w -> 16-bit.
// One warp per row, n <= 1024 * 8.  Statistics in f32 (two-pass over registers).
template <int kVecPerLane, bool kBf16>
__global__ void __launch_bounds__(128) add_layernorm_kernel(float* __restrict__ x, const uint16_t* __restrict__ delta,
                                                            const float* __restrict__ w, uint16_t* __restrict__ y,
                                                            long long rows, int n, float eps) {
    // programmatic dependent launch (no-ops under a plain launch): this grid was allowed to start while the previous
    // kernel of the stream -- the projection whose epilogue adds into x -- was still draining; its results are visible
    // after the wait.  The next kernel (a projection: barrier init, TMEM allocation, tensor-map prefetch) may start its
    // prologue right away.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    const long long row = static_cast<long long>(blockIdx.x) * 4 + (threadIdx.x >> 5);
    if (row >= rows) return;
    const int lane = threadIdx.x & 31;
    float* xr = x + row * n;
    float v[kVecPerLane * 4];
    float sum = 0.f;
#pragma unroll
    for (int k = 0; k < kVecPerLane; ++k) {
        const int c = (k * 32 + lane) * 4;
        if (c < n) {
            float4 a = *reinterpret_cast<const float4*>(xr + c);
            if (delta != nullptr) {
                const uint2 dq = *reinterpret_cast<const uint2*>(delta + row * n + c);
                const float2 d0 = Half2<kBf16>::to_float2(dq.x), d1 = Half2<kBf16>::to_float2(dq.y);
                a.x += d0.x;
                a.y += d0.y;
                a.z += d1.x;
                a.w += d1.y;
                *reinterpret_cast<float4*>(xr + c) = a;
            }
            v[4 * k] = a.x; v[4 * k + 1] = a.y; v[4 * k + 2] = a.z; v[4 * k + 3] = a.w;
            sum += a.x + a.y + a.z + a.w;
        } else {
            v[4 * k] = v[4 * k + 1] = v[4 * k + 2] = v[4 * k + 3] = 0.f;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float mean = sum / n;
    float var = 0.f;
#pragma unroll
    for (int k = 0; k < kVecPerLane; ++k) {
        const int c = (k * 32 + lane) * 4;
        if (c < n) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float dlt = v[4 * k + e] - mean;
                var += dlt * dlt;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) var += __shfl_xor_sync(0xffffffffu, var, o);
    const float rstd = rsqrtf(var / n + eps);
    if (y == nullptr) return;
#pragma unroll
    for (int k = 0; k < kVecPerLane; ++k) {
        const int c = (k * 32 + lane) * 4;
        if (c < n) {
            const float4 ww = *reinterpret_cast<const float4*>(w + c);
            const uint2 pk = make_uint2(
                Half2<kBf16>::from_floats((v[4 * k] - mean) * rstd * ww.x, (v[4 * k + 1] - mean) * rstd * ww.y),
                Half2<kBf16>::from_floats((v[4 * k + 2] - mean) * rstd * ww.z, (v[4 * k + 3] - mean) * rstd * ww.w));
            *reinterpret_cast<uint2*>(y + row * n + c) = pk;
        }
    }
}

// wi_out: [rows, 2*I] 16-bit (input half then gate half); act: [rows, I] 16-bit = gelu(input) * gate.
// One thread per 8 outputs (16-byte loads / store); I % 8 == 0.
template <bool kBf16>
__global__ void __launch_bounds__(256) geglu_kernel(const uint16_t* __restrict__ wi_out, uint16_t* __restrict__ act,
                                                    long long rows, int I) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int vecs = I >> 3;
    const long long total = rows * vecs;
    if (idx >= total) return;
    const long long row = idx / vecs;
    const int c = static_cast<int>(idx % vecs) * 8;
    uint4 a = *reinterpret_cast<const uint4*>(wi_out + row * 2 * I + c);
    const uint4 g = *reinterpret_cast<const uint4*>(wi_out + row * 2 * I + I + c);
    auto gelu = [](float v) { return 0.5f * v * (1.0f + erff(v * 0.70710678118654752f)); };
    uint32_t* a2 = reinterpret_cast<uint32_t*>(&a);
    const uint32_t* g2 = reinterpret_cast<const uint32_t*>(&g);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float2 x = Half2<kBf16>::to_float2(a2[e]), y = Half2<kBf16>::to_float2(g2[e]);
        a2[e] = Half2<kBf16>::from_floats(gelu(x.x) * y.x, gelu(x.y) * y.y);
    }
    *reinterpret_cast<uint4*>(act + row * I + c) = a;
}

int fail_cuda(cudaError_t e) { return e == cudaSuccess ? RF_OK : RF_ERR_CUDA; }

}  // namespace

extern "C" {

int rf_rope_qkv(void* qkv, const float* cosb, const float* sinb, int64_t tokens, int64_t S, int64_t H, int64_t d,
                int32_t dtype, void* stream) {
    if (qkv == nullptr || cosb == nullptr || sinb == nullptr || d % 16 || S <= 0) return RF_ERR_ARG;
    if (dtype != RF_DTYPE_BF16 && dtype != RF_DTYPE_F16) return RF_ERR_ARG;
    const long long total = tokens * 2 * H * (d / 16);
    if (total == 0) return RF_OK;
    const unsigned grid = static_cast<unsigned>((total + 255) / 256);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint16_t* p16 = static_cast<uint16_t*>(qkv);
    if (dtype == RF_DTYPE_BF16)
        rope_qkv_kernel<true><<<grid, 256, 0, st>>>(p16, cosb, sinb, tokens, static_cast<int>(S), static_cast<int>(H), static_cast<int>(d));
    else
        rope_qkv_kernel<false><<<grid, 256, 0, st>>>(p16, cosb, sinb, tokens, static_cast<int>(S), static_cast<int>(H), static_cast<int>(d));
    return fail_cuda(cudaGetLastError());
}

int rf_add_layernorm(float* x, const void* delta, const float* w, void* y, int64_t rows, int64_t n, float eps,
                     int32_t dtype, void* stream) {
    if (x == nullptr || (y != nullptr && w == nullptr) || n % 4 || n > 4096) return RF_ERR_ARG;
    if (dtype != RF_DTYPE_BF16 && dtype != RF_DTYPE_F16) return RF_ERR_ARG;
    if (rows == 0) return RF_OK;
    const unsigned grid = static_cast<unsigned>((rows + 3) / 4);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint16_t* dl = static_cast<const uint16_t*>(delta);
    uint16_t* yy = static_cast<uint16_t*>(y);
    const int ni = static_cast<int>(n);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(128);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e;
    if (n <= 1024) {
        if (dtype == RF_DTYPE_BF16) e = cudaLaunchKernelEx(&cfg, add_layernorm_kernel<8, true>, x, dl, w, yy, static_cast<long long>(rows), ni, eps);
        else e = cudaLaunchKernelEx(&cfg, add_layernorm_kernel<8, false>, x, dl, w, yy, static_cast<long long>(rows), ni, eps);
    } else {
        if (dtype == RF_DTYPE_BF16) e = cudaLaunchKernelEx(&cfg, add_layernorm_kernel<32, true>, x, dl, w, yy, static_cast<long long>(rows), ni, eps);
        else e = cudaLaunchKernelEx(&cfg, add_layernorm_kernel<32, false>, x, dl, w, yy, static_cast<long long>(rows), ni, eps);
    }
    return fail_cuda(e);
}

int rf_geglu(const void* wi_out, void* act, int64_t rows, int64_t I, int32_t dtype, void* stream) {
    if (wi_out == nullptr || act == nullptr || I % 8) return RF_ERR_ARG;
    if (dtype != RF_DTYPE_BF16 && dtype != RF_DTYPE_F16) return RF_ERR_ARG;
    const long long total = rows * (I / 8);
    if (total == 0) return RF_OK;
    const unsigned grid = static_cast<unsigned>((total + 255) / 256);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dtype == RF_DTYPE_BF16)
        geglu_kernel<true><<<grid, 256, 0, st>>>(static_cast<const uint16_t*>(wi_out), static_cast<uint16_t*>(act), rows, static_cast<int>(I));
    else
        geglu_kernel<false><<<grid, 256, 0, st>>>(static_cast<const uint16_t*>(wi_out), static_cast<uint16_t*>(act), rows, static_cast<int>(I));
    return fail_cuda(cudaGetLastError());
}

}  // extern "C"
