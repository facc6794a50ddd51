// fa_fwd_simt.cu -- generic FusedFlashAttention forward on CUDA cores (sm_100a), head_dim in
// {32, 64, 128}, any strides, f32 math.  Same semantics as fa_fwd_sm100.cu / reference
// attention.cpp:106-213.  It serves the head dims the tcgen05 kernel does not cover yet and is
// the on-device cross-check for the tensor-core kernel in tests.  It is a GPU kernel, not a
// fallback to the CPU: there is none.
//
// Mapping: 128 threads per CTA = 32 query rows x 4 threads; each thread owns d/4 of the head
// dim for q, the accumulator and the dot product (two shuffles finish the dot).  K/V are
// staged 32 keys at a time in shared memory as f32.  Online softmax per key, log2 domain.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "fa_internal.h"

namespace rf {
namespace {

constexpr int kRows = 32;
constexpr int kKeys = 32;

__device__ __forceinline__ float load_elem(const void* base, long long idx, int dtype) {
    if (dtype == 0) return __bfloat162float(static_cast<const __nv_bfloat16*>(base)[idx]);
    return __half2float(static_cast<const __half*>(base)[idx]);
}

template <int D>
__global__ void __launch_bounds__(128) fa_fwd_simt_kernel(const SimtParams sp, const float* __restrict__ pad_bias) {
    constexpr int DS = D / 4;
    __shared__ float ks[kKeys][D];
    __shared__ float vs[kKeys][D];
    __shared__ float bs[kKeys];

    const FaParams& p = sp.f;
    const int b = blockIdx.z, h = blockIdx.y;
    const int q0 = blockIdx.x * kRows;
    const int rl = threadIdx.x >> 2;
    const int sub = threadIdx.x & 3;
    const int row = q0 + rl;
    const bool row_ok = row < p.S;
    const float c = p.scale_log2;

    float qreg[DS], acc[DS];
    {
        const long long qoff = (long long)b * sp.q_sb + (long long)h * sp.q_sh + (long long)row * sp.q_ss + sub * DS;
#pragma unroll
        for (int i = 0; i < DS; ++i) {
            qreg[i] = row_ok ? load_elem(sp.q, qoff + i, sp.in_dtype) : 0.f;
            acc[i] = 0.f;
        }
    }
    float m = -CUDART_INF_F, l = 0.f;

    const int rows_end = min(q0 + kRows, p.S);
    int j_lo = p.kv_begin, j_hi = min(p.kv_end, p.S);
    if (p.wl >= 0) j_lo = max(j_lo, q0 - p.wl);
    if (p.wr >= 0) j_hi = min(j_hi, rows_end + p.wr);
    // this row's own live range
    int lo = p.kv_begin, hi = min(p.kv_end, p.S) - 1;
    if (p.wl >= 0) lo = max(lo, row - p.wl);
    if (p.wr >= 0) hi = min(hi, row + p.wr);

    for (int kv0 = (j_lo / kKeys) * kKeys; kv0 < j_hi; kv0 += kKeys) {
        // stage K/V rows kv0..kv0+31 (zero beyond S)
        for (int e = threadIdx.x; e < kKeys * D; e += 128) {
            const int jj = e / D, cc = e % D;
            const int j = kv0 + jj;
            float kvv = 0.f, vvv = 0.f;
            if (j < p.S) {
                kvv = load_elem(sp.k, (long long)b * sp.k_sb + (long long)h * sp.k_sh + (long long)j * sp.k_ss + cc,
                                sp.in_dtype);
                vvv = load_elem(sp.v, (long long)b * sp.v_sb + (long long)h * sp.v_sh + (long long)j * sp.v_ss + cc,
                                sp.in_dtype);
            }
            ks[jj][cc] = kvv;
            vs[jj][cc] = vvv;
        }
        if (threadIdx.x < kKeys) {
            const int j = kv0 + threadIdx.x;
            float bv = 0.f;
            if (j >= p.S) {
                bv = -CUDART_INF_F;
            } else if (pad_bias != nullptr) {
                const float raw = pad_bias[(long long)b * p.S + j];
                bv = raw > kMaskThreshold ? raw * kLog2e : -CUDART_INF_F;
            }
            bs[threadIdx.x] = bv;
        }
        __syncthreads();
#pragma unroll 4
        for (int jj = 0; jj < kKeys; ++jj) {
            float part = 0.f;
#pragma unroll
            for (int i = 0; i < DS; ++i) part = fmaf(qreg[i], ks[jj][sub * DS + i], part);
            part += __shfl_xor_sync(0xffffffffu, part, 1);
            part += __shfl_xor_sync(0xffffffffu, part, 2);
            const int j = kv0 + jj;
            const float x = fmaf(part, c, bs[jj]);
            if (j >= lo && j <= hi && x > -CUDART_INF_F) {
                const float m_new = fmaxf(m, x);
                const float alpha = exp2f(m - m_new);  // m = -inf -> 0
                const float pj = exp2f(x - m_new);
                l = fmaf(l, alpha, pj);
#pragma unroll
                for (int i = 0; i < DS; ++i) acc[i] = fmaf(acc[i], alpha, pj * vs[jj][sub * DS + i]);
                m = m_new;
            }
        }
        __syncthreads();
    }

    if (!row_ok) return;
    if (p.o_partial != nullptr) {
        const size_t ridx = (static_cast<size_t>(b) * p.H + h) * p.S + row;
#pragma unroll
        for (int i = 0; i < DS; ++i) p.o_partial[ridx * D + sub * DS + i] = acc[i];
        if (sub == 0) {
            p.m_partial[ridx] = m;
            p.l_partial[ridx] = l;
        }
        return;
    }
    const float inv = l > 0.f ? 1.0f / l : 0.f;
    const size_t off = static_cast<size_t>(b) * p.o_sb + static_cast<size_t>(h) * p.o_sh +
                       static_cast<size_t>(row) * p.o_ss + sub * DS;
#pragma unroll
    for (int i = 0; i < DS; ++i) {
        const float val = acc[i] * inv;
        if (p.out_dtype == 2)
            static_cast<float*>(p.out)[off + i] = val;
        else if (p.out_dtype == 0)
            static_cast<__nv_bfloat16*>(p.out)[off + i] = __float2bfloat16_rn(val);
        else
            static_cast<__half*>(p.out)[off + i] = __float2half_rn(val);
    }
}

}  // namespace

cudaError_t launch_fa_fwd_simt(const SimtParams& sp, cudaStream_t stream, int* grid_ctas) {
    const FaParams& p = sp.f;
    dim3 grid((p.S + kRows - 1) / kRows, p.H, p.B);
    if (grid_ctas) *grid_ctas = static_cast<int>(grid.x * grid.y * grid.z);
    // the raw [B,S] pad_bias travels in f.bias2 for this kernel (no preprocessing needed)
    const float* pad = p.bias2;
    switch (sp.d) {
        case 32: fa_fwd_simt_kernel<32><<<grid, 128, 0, stream>>>(sp, pad); break;
        case 64: fa_fwd_simt_kernel<64><<<grid, 128, 0, stream>>>(sp, pad); break;
        case 128: fa_fwd_simt_kernel<128><<<grid, 128, 0, stream>>>(sp, pad); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace rf
