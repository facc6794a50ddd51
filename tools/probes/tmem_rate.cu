// tmem_rate.cu -- developer microbenchmark (not part of the product): tcgen05.ld / tcgen05.st throughput per SM with
// 4, 8 and 16 warps (1, 2, 4 per SM sub-partition; the dense attention kernel runs 4), alone and mixed with MUFU.EX2.
// The dense kernel reads every f32 score once from TMEM: 256 x 128 x 4 B = 128 KiB per (query-tile pair, key tile).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2603_12646_b200/csrc -o tmem_rate.bin tmem_rate.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "ptx.cuh"
using namespace rfptx;

enum Mode { kLd32 = 0, kLd16, kSt32, kSt16, kLd32Mufu, kLd32St16, kTryWait, kNumModes };

template <int kMode>
__global__ void __launch_bounds__(512, 1) probe(int iters, long long* clk_out, uint32_t* sink) {
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t mbar;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&mbar), 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) mbar_arrive(smem_u32(&mbar));  // phase 0 completes: a wait for parity 0 is satisfied from now on
    __syncthreads();
    if (warp == 0) {
        tmem_alloc(smem_u32(&tmem_slot), 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t base = tmem_slot + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    uint32_t r[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) r[i] = threadIdx.x + i;
    float e[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) e[i] = 0.001f * (threadIdx.x + i);
    tmem_st32(base, r);
    tc_wait_st();
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const uint32_t col = ((warp >> 2) * 64 + (it & 1) * 32) & 511;
        if (kMode == kLd32 || kMode == kLd32Mufu || kMode == kLd32St16) {
            uint32_t v[32];
            tmem_ld32(base + col, v);
            if (kMode == kLd32Mufu) {
#pragma unroll
                for (int u = 0; u < 24; ++u) e[u & 7] = ex2(e[u & 7]);  // 24 MUFU per 32 columns = the kernel's 3/4 share
            }
            tc_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] ^= v[i];
            if (kMode == kLd32St16) {
                tmem_st16(base + col, reinterpret_cast<uint32_t(&)[16]>(r[0]));
                tc_wait_st();
            }
        } else if (kMode == kLd16) {
            uint32_t v[16];
            tmem_ld16(base + col, v);
            tc_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) r[i] ^= v[i];
        } else if (kMode == kSt32) {
            tmem_st32(base + col, r);
            tc_wait_st();
        } else if (kMode == kTryWait) {
            // a phase check of a barrier that completed long ago, result consumed (dependent chain: latency)
            r[0] += mbar_try_wait(smem_u32(&mbar), 0);
        } else if (kMode == kSt16) {
            tmem_st16(base + col, reinterpret_cast<uint32_t(&)[16]>(r[0]));
            tc_wait_st();
        }
    }
    const long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) acc ^= r[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc ^= __float_as_uint(e[i]);
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) clk_out[blockIdx.x] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem_slot, 512);
    }
}

template <int kMode>
void run(const char* name, int bytes_per_warp_instr) {
    long long* clk;
    uint32_t* sink;
    cudaMalloc(&clk, 8 * 148);
    cudaMalloc(&sink, 4 * 512 * 148);
    const int iters = 4096;
    for (int warps : {4, 8, 16}) {
        probe<kMode><<<1, warps * 32>>>(iters, clk, sink);
        cudaDeviceSynchronize();
        probe<kMode><<<1, warps * 32>>>(iters, clk, sink);
        cudaError_t e = cudaDeviceSynchronize();
        long long c = 0;
        cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
        const double per_instr = static_cast<double>(c) / iters;  // clk per round of `warps` instructions
        printf("{\"op\": \"%s\", \"warps\": %d, \"clk_per_round\": %.1f, \"bytes_per_clk_per_sm\": %.1f, \"err\": %d}\n", name, warps,
               per_instr, static_cast<double>(bytes_per_warp_instr) * warps / per_instr, static_cast<int>(e));
    }
    cudaFree(clk);
    cudaFree(sink);
}

int main() {
    run<kLd32>("tcgen05.ld 32x32b.x32 (4 KiB per warp)", 4096);
    run<kLd16>("tcgen05.ld 32x32b.x16 (2 KiB per warp)", 2048);
    run<kSt32>("tcgen05.st 32x32b.x32 (4 KiB per warp)", 4096);
    run<kSt16>("tcgen05.st 32x32b.x16 (2 KiB per warp)", 2048);
    run<kLd32Mufu>("tcgen05.ld x32 + 24 MUFU.EX2 (ld bytes counted)", 4096);
    run<kLd32St16>("tcgen05.ld x32 + tcgen05.st x16 (ld bytes counted)", 4096);
    run<kTryWait>("mbarrier.try_wait on a completed phase (clk_per_round = latency per check; bytes n/a)", 0);
    return 0;
}
