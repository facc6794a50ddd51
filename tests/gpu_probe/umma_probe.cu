// umma_probe.cu -- TEST-ONLY bring-up probe (not part of the product library).
// One CTA computes D = A * B with tcgen05.mma in the exact operand configurations the attention
// kernel uses, with shared memory filled by plain stores in the layout the descriptors claim.
// A mismatch here pins a descriptor/layout assumption independently of TMA and of the pipeline.
//   mode 0: SS, A [128x64]  K-major SW128, B [128x64] (N x K) K-major SW128  -> D [128x128]   (S = Q K^T)
//   mode 1: SS, A [128x128] K-major SW128 (two 64-wide sub-tiles), B [128(K) x 64(N)] MN-major SW128 -> D [128x64]
//   mode 2: TS, A [128x128] packed bf16 pairs in TMEM (lo = even k), B as mode 1               -> D [128x64]
//   mode 3: as mode 2 with the pair order swapped (alternate packing hypothesis)
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../paper_2603_12646_b200/csrc/ptx.cuh"

using namespace rfptx;

__global__ void __launch_bounds__(128, 1) umma_probe_kernel(int mode, const uint16_t* __restrict__ A,
                                                            const uint16_t* __restrict__ B, float* __restrict__ D) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* gen = smem_raw + (base - smem_u32(smem_raw));
    // layout: A region 32 KiB @0, B region 16 KiB @32768, barrier @49152, tmem slot @49160
    uint8_t* sA = gen;
    uint8_t* sB = gen + 32768;
    const uint32_t bar = base + 49152;
    volatile uint32_t* slot = reinterpret_cast<volatile uint32_t*>(gen + 49160);
    const int tid = threadIdx.x, warp = tid >> 5;
    const int KA = (mode == 0) ? 64 : 128;   // A columns (reduction dim)
    const int N = (mode == 0) ? 128 : 64;

    if (tid == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
    }
    if (warp == 0) {
        tmem_alloc(smem_u32(const_cast<uint32_t*>(slot)), 256);
        tmem_relinquish();
    }
    // fill shared memory in the swizzled layouts
    if (mode <= 1) {
        for (int e = tid; e < 128 * KA; e += 128) {
            const int r = e / KA, c = e % KA;
            const int sub = c / 64, cc = c % 64;
            const uint32_t off = sub * 16384 + r * 128 + ((((cc >> 3) ^ (r & 7))) << 4) + (cc & 7) * 2;
            *reinterpret_cast<uint16_t*>(sA + off) = A[r * KA + c];
        }
    }
    if (mode == 0) {
        for (int e = tid; e < 128 * 64; e += 128) {
            const int r = e / 64, c = e % 64;
            const uint32_t off = r * 128 + ((((c >> 3) ^ (r & 7))) << 4) + (c & 7) * 2;
            *reinterpret_cast<uint16_t*>(sB + off) = B[r * 64 + c];
        }
    } else {
        for (int e = tid; e < 128 * 64; e += 128) {
            const int k = e / 64, n = e % 64;  // V[k][n], row = key
            const uint32_t off = k * 128 + ((((n >> 3) ^ (k & 7))) << 4) + (n & 7) * 2;
            *reinterpret_cast<uint16_t*>(sB + off) = B[k * 64 + n];
        }
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
    const uint32_t colD = 128, colA = 0;

    if (mode >= 2) {  // stage A in TMEM: lane = row, column c holds (k=2c, k=2c+1)
        for (int cb = 0; cb < 4; ++cb) {
            uint32_t pk[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const uint32_t lo = A[tid * 128 + cb * 32 + 2 * u], hi = A[tid * 128 + cb * 32 + 2 * u + 1];
                pk[u] = (mode == 2) ? (lo | (hi << 16)) : (hi | (lo << 16));
            }
            tmem_st16(tmem + lane_base + colA + cb * 16, pk);
        }
        tc_wait_st();
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    }

    if (tid == 0) {
        if (mode == 0) {
            const uint32_t idesc = make_idesc_f16(1, 0, 0, 128, 128);
            for (int kk = 0; kk < 4; ++kk) {
                const uint64_t ad = make_smem_desc(base + kk * 32, 16, 1024, kSwizzle128B);
                const uint64_t bd = make_smem_desc(base + 32768 + kk * 32, 16, 1024, kSwizzle128B);
                mma_ss(tmem + colD, ad, bd, idesc, kk > 0);
            }
        } else {
            const uint32_t idesc = make_idesc_f16(1, 0, 1, 128, 64);
            for (int kk = 0; kk < 8; ++kk) {
                const uint64_t bd = make_smem_desc(base + 32768 + kk * 2048, 16384, 1024, kSwizzle128B);
                if (mode == 1) {
                    const uint64_t ad = make_smem_desc(base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, kSwizzle128B);
                    mma_ss(tmem + colD, ad, bd, idesc, kk > 0);
                } else {
                    mma_ts(tmem + colD, tmem + colA + kk * 8, bd, idesc, kk > 0);
                }
            }
        }
        tc_commit(bar);
    }
    mbar_wait_or_trap(bar, 0);
    tc_fence_after();
    for (int cb = 0; cb < N / 32; ++cb) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_base + colD + cb * 32, r);
        tc_wait_ld();
#pragma unroll
        for (int u = 0; u < 32; ++u) D[tid * N + cb * 32 + u] = __uint_as_float(r[u]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 256);
}

extern "C" int umma_probe_run(int mode, const void* dA, const void* dB, float* dD) {
    const int smem = 49152 + 64 + 1024;
    cudaFuncSetAttribute(umma_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    umma_probe_kernel<<<1, 128, smem>>>(mode, static_cast<const uint16_t*>(dA), static_cast<const uint16_t*>(dB), dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        fprintf(stderr, "umma_probe mode %d: %s\n", mode, cudaGetErrorString(e));
        return 1;
    }
    return 0;
}
