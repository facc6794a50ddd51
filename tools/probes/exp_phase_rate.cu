// exp_phase_rate.cu -- developer microbenchmark (not part of the product): cost of the softmax
// kernel's exponential phase (64 scores per thread -> 2^(s*c - m), row sum, bf16 pack, tcgen05.st)
// as a function of how many warps per SM sub-partition run it at once.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o exp_phase_rate exp_phase_rate.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <type_traits>

#include "../../paper_2603_12646_b200/csrc/ptx.cuh"
using namespace rfptx;

constexpr int kHalfN = 64;

// variant 0: the kernel's loop (one sum chain, every 8th pair on the FMA pipe)   1: MUFU only, no emulation
// variant 2: four independent sum chains                                         3: MUFU + pack only (no sum)
// variant 4: every 4th pair emulated                                              5: every 2nd pair emulated
template <int kVariant>
__global__ void __launch_bounds__(512, 1) exp_kernel(const float* __restrict__ in, float* __restrict__ out, int iters,
                                                     int active_warps_per_smsp, long long* clk) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        tmem_alloc(smem_u32(&slot), 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const bool active = (warp >> 2) < active_warps_per_smsp;  // warps w, w+4, w+8, w+12 share a sub-partition
    uint32_t su[kHalfN];
    for (int j = 0; j < kHalfN; ++j) su[j] = __float_as_uint(in[(threadIdx.x * kHalfN + j) % 4096]);
    const uint32_t t_p = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp >> 2) * 64;
    float acc = 0.f;
    __syncthreads();
    const long long t0 = clock64();
    if (active) {
        for (int it = 0; it < iters; ++it) {
            const float mul = 0.18f, neg_m = -2.0f - 1e-3f * it;
            uint64_t sum2[4] = {0, 0, 0, 0};
            const uint64_t mul2 = bc2(mul), negm2 = bc2(neg_m);
            constexpr int kEvery = kVariant == 4 ? 4 : (kVariant == 5 ? 2 : 8);
#pragma unroll
            for (int cb = 0; cb < kHalfN / 32; ++cb) {
                uint32_t pk[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    float p0, p1;
                    unpk2(ffma2v(pk2(__uint_as_float(su[cb * 32 + 2 * u]), __uint_as_float(su[cb * 32 + 2 * u + 1])), mul2, negm2), p0, p1);
                    if (kVariant != 1 && kVariant != 3 && (u % kEvery) == kEvery - 1) {
                        exp2_poly2(p0, p1);
                    } else {
                        p0 = ex2(p0);
                        p1 = ex2(p1);
                    }
                    if (kVariant != 3) {
                        const int chain = kVariant == 2 ? (u & 3) : 0;
                        sum2[chain] = fadd2v(sum2[chain], pk2(p0, p1));
                    }
                    pk[u] = pack2<true>(p0, p1);
                }
                tmem_st16(t_p + cb * 16, pk);
            }
            float s0, s1;
            unpk2(fadd2v(fadd2v(sum2[0], sum2[1]), fadd2v(sum2[2], sum2[3])), s0, s1);
            acc += s0 + s1;
            tc_wait_st();
        }
    }
    const long long t1 = clock64();
    if (active && lane == 0 && blockIdx.x == 0) clk[warp] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int kVariant>
void run(const char* name, const float* in, float* out, long long* clk) {
    for (int w : {1, 2, 4}) {
        const int iters = 2000;
        exp_kernel<kVariant><<<148, 512>>>(in, out, iters, w, clk);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("%s: %s\n", name, cudaGetErrorString(e));
            return;
        }
        long long h[16];
        cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
        printf("{\"variant\": \"%s\", \"warps_per_smsp\": %d, \"clk_per_tile_per_warp\": %.0f, \"clk_per_tile_per_smsp_per_warpwork\": %.0f}\n",
               name, w, double(h[0]) / iters, double(h[0]) / iters / w);
    }
}

// Candidate replacement for exp2_poly2 that was measured and NOT adopted: 2^(s*c - m) straight from the
// raw scores for an integer-valued reference m.  With k = 1.5*2^23 - m: t = fma(s,c,k) holds round(x)
// in its low mantissa bits, w = k - t == -m - round(x) exactly, f = fma(s,c,w) in [-0.5,0.5]; three
// packed FMA-pipe instructions for the range reduction instead of four.  Faster in this probe (two
// pairs in eight: 1726 vs 1905 clk per tile), slower inside the attention kernel (756 vs 835 TFLOP/s
// at 8K): the softmax warps are bound by issue slots as much as by MUFU, and every emulated pair
// costs five times the instructions of a MUFU pair.
__device__ __forceinline__ void exp2_emu_pair(float s0, float s1, float smin, uint64_t c2, uint64_t k2, float& p0,
                                              float& p1) {
    const uint64_t s = pk2(fmaxf(s0, smin), fmaxf(s1, smin));
    const uint64_t t = ffma2v(s, c2, k2);
    const uint64_t w = ffma2v(t, bc2(-1.0f), k2);
    const uint64_t f = ffma2v(s, c2, w);
    uint64_t pl = ffma2v(f, bc2(0.055171459913253784f), bc2(0.2426108568906784f));
    pl = ffma2v(pl, f, bc2(0.6932609677314758f));
    pl = ffma2v(pl, f, bc2(0.9999281167984009f));
    float t0, t1, q0, q1;
    unpk2(t, t0, t1);
    unpk2(pl, q0, q1);
    p0 = __int_as_float(__float_as_int(q0) + (__float_as_int(t0) << 23));
    p1 = __int_as_float(__float_as_int(q1) + (__float_as_int(t1) << 23));
}

// mask-driven variants: bit (u % 8) of kMask set -> that element pair takes the FMA-pipe path.
// kNew: exp2_emu_pair (integer reference max, 3-instruction range reduction) instead of exp2_poly2.
// kSum: accumulate the row sum (FADD2) or not (what remains if l came out of the P V MMA).
template <int kMask, bool kNew, bool kSum>
__global__ void __launch_bounds__(512, 1) exp_kernel2(const float* __restrict__ in, float* __restrict__ out, int iters,
                                                      int active_warps_per_smsp, long long* clk) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        tmem_alloc(smem_u32(&slot), 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const bool active = (warp >> 2) < active_warps_per_smsp;
    uint32_t su[kHalfN];
    for (int j = 0; j < kHalfN; ++j) su[j] = __float_as_uint(in[(threadIdx.x * kHalfN + j) % 4096]);
    const uint32_t t_p = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp >> 2) * 64;
    float acc = 0.f;
    __syncthreads();
    const long long t0 = clock64();
    if (active) {
        for (int it = 0; it < iters; ++it) {
            const float mul = 0.18f, neg_m = -2.0f - float(it & 3);
            uint64_t sum2 = 0;
            const uint64_t mul2 = bc2(mul), negm2 = bc2(neg_m), k2 = bc2(12582912.0f + neg_m);
            const float smin = (-neg_m - 125.0f) * (1.0f / 0.18f);
#pragma unroll
            for (int cb = 0; cb < kHalfN / 32; ++cb) {
                uint32_t pk[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    float p0, p1;
                    const float s0 = __uint_as_float(su[cb * 32 + 2 * u]), s1 = __uint_as_float(su[cb * 32 + 2 * u + 1]);
                    if ((kMask >> (u % 8)) & 1) {
                        if (kNew) {
                            exp2_emu_pair(s0, s1, smin, mul2, k2, p0, p1);
                        } else {
                            unpk2(ffma2v(pk2(s0, s1), mul2, negm2), p0, p1);
                            exp2_poly2(p0, p1);
                        }
                    } else {
                        unpk2(ffma2v(pk2(s0, s1), mul2, negm2), p0, p1);
                        p0 = ex2(p0);
                        p1 = ex2(p1);
                    }
                    if (kSum) sum2 = fadd2v(sum2, pk2(p0, p1));
                    pk[u] = pack2<true>(p0, p1);
                }
                tmem_st16(t_p + cb * 16, pk);
            }
            float s0, s1;
            unpk2(sum2, s0, s1);
            acc += s0 + s1;
            tc_wait_st();
        }
    }
    const long long t1 = clock64();
    if (active && lane == 0 && blockIdx.x == 0) clk[warp] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int kMask, bool kNew, bool kSum>
void run2(const char* name, const float* in, float* out, long long* clk) {
    for (int w : {1, 4}) {
        const int iters = 2000;
        exp_kernel2<kMask, kNew, kSum><<<148, 512>>>(in, out, iters, w, clk);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("%s: %s\n", name, cudaGetErrorString(e));
            return;
        }
        long long h[16];
        cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
        printf("{\"variant\": \"%s\", \"warps_per_smsp\": %d, \"clk_per_tile_per_warp\": %.0f, \"clk_per_tile_per_smsp_per_warpwork\": %.0f}\n",
               name, w, double(h[0]) / iters, double(h[0]) / iters / w);
    }
}

int main() {
    float *in, *out;
    long long* clk;
    cudaMalloc(&in, 4096 * 4);
    cudaMalloc(&out, 148 * 512 * 4);
    cudaMalloc(&clk, 16 * 8);
    float h[4096];
    for (int i = 0; i < 4096; ++i) h[i] = float((i * 37) % 101) / 10.f - 5.f;
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    run<0>("kernel loop (1/8 emulated, one sum chain)", in, out, clk);
    run<1>("MUFU only, one sum chain", in, out, clk);
    run<2>("1/8 emulated, four sum chains", in, out, clk);
    run<3>("MUFU + pack only (no sum)", in, out, clk);
    run<4>("1/4 emulated, one sum chain", in, out, clk);
    run<5>("1/2 emulated, one sum chain", in, out, clk);
    run2<0x80, false, true>("old emu 1/8", in, out, clk);
    run2<0x80, true, true>("new emu 1/8", in, out, clk);
    run2<0x88, true, true>("new emu 2/8", in, out, clk);
    run2<0x92, true, true>("new emu 3/8 (bits 1,4,7)", in, out, clk);
    run2<0xAA, true, true>("new emu 4/8", in, out, clk);
    run2<0xAA, false, true>("old emu 4/8", in, out, clk);
    run2<0xB6, true, true>("new emu 5/8", in, out, clk);
    run2<0xFF, true, true>("new emu 8/8", in, out, clk);
    run2<0x92, true, false>("new emu 3/8, no sum", in, out, clk);
    run2<0xAA, true, false>("new emu 4/8, no sum", in, out, clk);
    run2<0x00, true, false>("MUFU only, no sum", in, out, clk);
    return 0;
}
