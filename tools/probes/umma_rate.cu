// umma_rate.cu -- developer microbenchmark (not part of the product): issue/execute rate of
// tcgen05.mma in the operand shapes the attention kernel uses, one CTA per SM, one issuing thread.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o umma_rate umma_rate.cu && ./umma_rate
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../paper_2603_12646_b200/csrc/ptx.cuh"
using namespace rfptx;

constexpr uint32_t kDescHi = (1024u >> 4) | (1u << 14) | (kSwizzle128B << 29);
__device__ __forceinline__ uint64_t dsc(uint32_t lo) { return (static_cast<uint64_t>(kDescHi) << 32) | lo; }

// mode 0: SS M128 N128   1: TS M128 N64 (B MN-major)   2: SS M128 N256   3: SS M128 N64
// mode 4: the kernel's mix per key tile pair: 8 PV, 4 QK, 8 PV, 4 QK     5: TS M128 N128
__global__ void __launch_bounds__(128, 1) rate_kernel(int mode, int rounds, long long* out) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* gen = smem_raw + (base - smem_u32(smem_raw));
    for (int i = threadIdx.x; i < (160 * 1024) / 4; i += 128) reinterpret_cast<uint32_t*>(gen)[i] = 0;
    const uint32_t bar = base + 160 * 1024;
    volatile uint32_t* slot = reinterpret_cast<volatile uint32_t*>(gen + 160 * 1024 + 16);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
    }
    if (threadIdx.x < 32) {
        tmem_alloc(smem_u32(const_cast<uint32_t*>(slot)), 512);
        tmem_relinquish();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (threadIdx.x == 0) {
        const uint32_t sb16 = base >> 4;
        const uint32_t lboK = (16u >> 4) << 16, lboV = (16384u >> 4) << 16;
        const uint32_t i_qk = make_idesc_f16(1, 0, 0, 128, 128), i_pv = make_idesc_f16(1, 0, 1, 128, 64);
        const uint32_t i_256 = make_idesc_f16(1, 0, 0, 128, 256), i_64 = make_idesc_f16(1, 0, 0, 128, 64);
        const uint32_t i_ts128 = make_idesc_f16(1, 0, 1, 128, 128);
        const uint32_t a = lboK | sb16, b = lboK | (sb16 + 32768 / 16), v = lboV | (sb16 + 98304 / 16);
        long long t0 = clock64();
        long long n = 0;
        for (int r = 0; r < rounds; ++r) {
            if (mode == 0) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) mma_ss(tmem + (kk & 4 ? 128 : 0), dsc(a + (kk & 3) * 2), dsc(b + (kk & 3) * 2), i_qk, 1);
                n += 8;
            } else if (mode == 1) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) mma_ts(tmem + 384, tmem + kk * 8, dsc(v + kk * 128), i_pv, 1);
                n += 8;
            } else if (mode == 2) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) mma_ss(tmem, dsc(a + (kk & 3) * 2), dsc(b + (kk & 3) * 2), i_256, 1);
                n += 8;
            } else if (mode == 3) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) mma_ss(tmem, dsc(a + (kk & 3) * 2), dsc(b + (kk & 3) * 2), i_64, 1);
                n += 8;
            } else if (mode == 4) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) mma_ts(tmem + 384, tmem + kk * 8, dsc(v + kk * 128), i_pv, 1);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) mma_ss(tmem + 128, dsc(a + kk * 2), dsc(b + kk * 2), i_qk, kk > 0);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) mma_ts(tmem + 448, tmem + 256 + kk * 8, dsc(v + 1024 + kk * 128), i_pv, 1);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) mma_ss(tmem, dsc(a + 1024 + kk * 2), dsc(b + 1024 + kk * 2), i_qk, kk > 0);
                n += 24;
            } else if (mode == 5) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) mma_ts(tmem + 256, tmem + kk * 8, dsc(v + kk * 128), i_ts128, 1);
                n += 8;
            } else if (mode == 6) {  // TS N64, two accumulators alternating every MMA
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) mma_ts(tmem + 384 + (kk & 1) * 64, tmem + kk * 8, dsc(v + kk * 128), i_pv, 1);
                n += 8;
            } else if (mode == 7) {  // TS N64, four accumulators round robin
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) mma_ts(tmem + 256 + (kk & 3) * 64, tmem + kk * 8, dsc(v + kk * 128), i_pv, 1);
                n += 8;
            } else if (mode == 8) {  // kernel mix with PV and QK interleaved MMA by MMA
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    const uint32_t o = tmem + 384 + half * 64, p_ = tmem + half * 256, s_ = tmem + 128 - half * 128;
                    const uint32_t vv = v + half * 1024, aa = a + half * 1024, bb = b + half * 1024;
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        mma_ts(o, p_ + (2 * g) * 8, dsc(vv + (2 * g) * 128), i_pv, 1);
                        mma_ss(s_, dsc(aa + g * 2), dsc(bb + g * 2), i_qk, g > 0);
                        mma_ts(o, p_ + (2 * g + 1) * 8, dsc(vv + (2 * g + 1) * 128), i_pv, 1);
                    }
                }
                n += 24;
            } else if (mode == 9) {  // SS N128: 4-deep dependent chains vs mode 0 (same)
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) mma_ss(tmem + (kk & 1) * 128, dsc(a + (kk & 3) * 2), dsc(b + (kk & 3) * 2), i_qk, 1);
                n += 8;
            } else if (mode >= 11) {  // 11: SS M64 N128   12: SS M64 N256   13: SS M64 N64   14: SS M64 N128, A MN-major (transposed PV)
                const uint32_t idesc = mode == 11 ? make_idesc_f16(1, 0, 0, 64, 128)
                                     : mode == 12 ? make_idesc_f16(1, 0, 0, 64, 256)
                                     : mode == 13 ? make_idesc_f16(1, 0, 0, 64, 64)
                                                  : make_idesc_f16(1, 1, 0, 64, 128);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_ss(tmem + (kk & 1) * 256, dsc((mode == 14 ? v : a) + (kk & 3) * (mode == 14 ? 128 : 2)), dsc(b + (kk & 3) * 2), idesc, 1);
                n += 8;
            } else {  // mode 10: PV only, A and B interleaved MMA by MMA (two P sources, two accumulators)
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    mma_ts(tmem + 384, tmem + kk * 8, dsc(v + kk * 128), i_pv, 1);
                    mma_ts(tmem + 448, tmem + 256 + kk * 8, dsc(v + kk * 128), i_pv, 1);
                }
                n += 16;
            }
        }
        long long t1 = clock64();
        tc_commit(bar);
        mbar_wait_or_trap(bar, 0);
        long long t2 = clock64();
        if (blockIdx.x == 0) {
            out[0] = t1 - t0;
            out[1] = t2 - t0;
            out[2] = n;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    const int smem = 160 * 1024 + 64 + 1024;
    cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char* names[] = {"SS M128 N128 K16 (QK)", "TS M128 N64 K16 (PV)", "SS M128 N256 K16", "SS M128 N64 K16",
                           "kernel mix 8PV+4QK+8PV+4QK", "TS M128 N128 K16", "TS N64 2 accumulators alternating", "TS N64 4 accumulators", "kernel mix interleaved PV/QK/PV", "SS N128 alternating D", "TS N64 PV_A/PV_B interleaved", "SS M64 N128 K16", "SS M64 N256 K16", "SS M64 N64 K16", "SS M64 N128 K16, A MN-major (transposed PV)"};
    const double macs[] = {128. * 128 * 16, 128. * 64 * 16, 128. * 256 * 16, 128. * 64 * 16, 0, 128. * 128 * 16, 128. * 64 * 16, 128. * 64 * 16, 0, 128. * 128 * 16, 128. * 64 * 16, 64. * 128 * 16, 64. * 256 * 16, 64. * 64 * 16, 64. * 128 * 16};
    for (int grid : {148})
        for (int mode = 0; mode < 15; ++mode) {
            for (int rep = 0; rep < 2; ++rep) {
                rate_kernel<<<grid, 128, smem>>>(mode, 512, d);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) {
                    printf("mode %d: %s\n", mode, cudaGetErrorString(e));
                    return 1;
                }
            }
            long long h[3];
            cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
            const double per = double(h[1]) / double(h[2]);
            printf("{\"grid\": %d, \"mode\": %d, \"shape\": \"%s\", \"mmas\": %lld, \"clk_issue_total\": %lld, \"clk_done_total\": %lld, "
                   "\"clk_per_mma\": %.1f, \"mac_per_clk\": %.0f}\n",
                   grid, mode, names[mode], h[2], h[0], h[1], per, macs[mode] > 0 ? macs[mode] / per : 0.0);
        }
    return 0;
}
