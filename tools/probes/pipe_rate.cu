// pipe_rate.cu -- developer microbenchmark (not part of the product): issue / pipe throughput of
// the instructions the softmax phase is built from, with 1, 2 and 4 warps per SM sub-partition
// (the attention kernel runs 4 softmax warps per sub-partition).  Prints clk per warp-instruction
// per sub-partition; 1.0 = full issue rate.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o pipe_rate pipe_rate.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

constexpr int kChains = 8;    // independent dependency chains per thread
constexpr int kUnroll = 8;    // body repeats per loop iteration

enum Op {
    kFfma, kFfmaImm, kFfma2, kFadd2, kFmnmx, kFmnmx3, kF2fp, kLea, kShlAdd, kImad, kMufu, kHfma2, kHfma2Bf16,
    kMufuBf16x2, kMufuF16x2, kMufuF16, kPrmt, kHadd2Bf16,
    kMixMufuFfma2,   // 1 MUFU : 1 FFMA2
    kMixFfma2Fmnmx,  // 1 FFMA2 : 1 FMNMX
    kMixFfma2Lea,    // 1 FFMA2 : 1 LEA
    kMixMufuF2fp,    // 1 MUFU : 1 F2FP
    kMixFfmaFfma2,   // 1 FFMA : 1 FFMA2
    kMixAll,         // MUFU + FFMA2 + FMNMX + F2FP (the kernel's MUFU path per element pair: 2 MUFU, 2 FFMA2-class, 1 max3, 1 F2FP)
    kNumOps
};

template <int kOp>
__device__ __forceinline__ void body(uint32_t (&r)[kChains], uint64_t (&w)[kChains], uint32_t a, uint32_t b, uint64_t wa,
                                     uint64_t wb) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        if (kOp == kFfma) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(r[c]) : "r"(a), "r"(b));
        if (kOp == kFfmaImm) asm volatile("fma.rn.f32 %0, %0, %1, 0f3F800000;" : "+r"(r[c]) : "r"(a));
        if (kOp == kFfma2) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(w[c]) : "l"(wa), "l"(wb));
        if (kOp == kFadd2) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(w[c]) : "l"(wa));
        if (kOp == kFmnmx) asm volatile("max.f32 %0, %0, %1;" : "+r"(r[c]) : "r"(a));
        if (kOp == kFmnmx3) asm volatile("max.f32 %0, %0, %1, %2;" : "+r"(r[c]) : "r"(a), "r"(b));
        if (kOp == kF2fp) asm volatile("cvt.rn.bf16x2.f32 %0, %0, %1;" : "+r"(r[c]) : "r"(a));
        if (kOp == kLea) asm volatile("{.reg .u32 t; shl.b32 t, %0, 23; add.u32 %0, t, %1;}" : "+r"(r[c]) : "r"(a));
        if (kOp == kShlAdd) {
            asm volatile("shl.b32 %0, %0, 3;" : "+r"(r[c]));
            asm volatile("add.u32 %0, %0, %1;" : "+r"(r[c]) : "r"(a));
        }
        if (kOp == kImad) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[c]) : "r"(a), "r"(b));
        if (kOp == kMufu) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(r[c]));
        if (kOp == kMufuBf16x2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(r[c]));
        if (kOp == kMufuF16x2) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(r[c]));
        if (kOp == kMufuF16) {
            unsigned short hs = static_cast<unsigned short>(r[c]);
            asm volatile("ex2.approx.f16 %0, %0;" : "+h"(hs));
            r[c] = hs;
        }
        if (kOp == kPrmt) asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(r[c]) : "r"(a));
        if (kOp == kHadd2Bf16) asm volatile("add.rn.bf16x2 %0, %0, %1;" : "+r"(r[c]) : "r"(a));
        if (kOp == kHfma2) asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(r[c]) : "r"(a), "r"(b));
        if (kOp == kHfma2Bf16) asm volatile("fma.rn.bf16x2 %0, %0, %1, %2;" : "+r"(r[c]) : "r"(a), "r"(b));
        if (kOp == kMixMufuFfma2) {
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(r[c]));
            asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(w[c]) : "l"(wa), "l"(wb));
        }
        if (kOp == kMixFfma2Fmnmx) {
            asm volatile("max.f32 %0, %0, %1;" : "+r"(r[c]) : "r"(a));
            asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(w[c]) : "l"(wa), "l"(wb));
        }
        if (kOp == kMixFfma2Lea) {
            asm volatile("{.reg .u32 t; shl.b32 t, %0, 23; add.u32 %0, t, %1;}" : "+r"(r[c]) : "r"(a));
            asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(w[c]) : "l"(wa), "l"(wb));
        }
        if (kOp == kMixMufuF2fp) {
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(r[c]));
            asm volatile("cvt.rn.bf16x2.f32 %0, %0, %1;" : "+r"(r[(c + 1) % kChains]) : "r"(a));
        }
        if (kOp == kMixFfmaFfma2) {
            asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(r[c]) : "r"(a), "r"(b));
            asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(w[c]) : "l"(wa), "l"(wb));
        }
        if (kOp == kMixAll) {
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(r[c]));
            asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(w[c]) : "l"(wa), "l"(wb));
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(r[(c + 3) % kChains]));
            asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(w[(c + 3) % kChains]) : "l"(wa));
            asm volatile("max.f32 %0, %0, %1, %2;" : "+r"(r[(c + 5) % kChains]) : "r"(a), "r"(b));
            asm volatile("cvt.rn.bf16x2.f32 %0, %0, %1;" : "+r"(r[(c + 6) % kChains]) : "r"(a));
        }
    }
}

constexpr int instr_per_body(int op) {
    return op == kShlAdd || op == kMixMufuFfma2 || op == kMixFfma2Fmnmx || op == kMixFfma2Lea || op == kMixMufuF2fp ||
                   op == kMixFfmaFfma2
               ? 2
               : (op == kMixAll ? 6 : 1);
}

template <int kOp>
__global__ void __launch_bounds__(512, 1) rate_kernel(const uint32_t* in, uint32_t* out, int iters, int warps_per_smsp,
                                                      long long* clk) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool active = (warp >> 2) < warps_per_smsp;
    uint32_t r[kChains];
    uint64_t w[kChains];
    for (int c = 0; c < kChains; ++c) {
        r[c] = in[(threadIdx.x + c) & 1023];
        w[c] = (static_cast<uint64_t>(in[(threadIdx.x + c + 7) & 1023]) << 32) | r[c];
    }
    const uint32_t a = in[lane], b = in[lane + 32];
    const uint64_t wa = (static_cast<uint64_t>(a) << 32) | b, wb = (static_cast<uint64_t>(b) << 32) | a;
    __syncthreads();
    const long long t0 = clock64();
    if (active) {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) body<kOp>(r, w, a, b, wa, wb);
        }
    }
    const long long t1 = clock64();
    if (active && lane == 0 && blockIdx.x == 0) clk[warp] = t1 - t0;
    uint32_t acc = 0;
    for (int c = 0; c < kChains; ++c) acc ^= r[c] ^ static_cast<uint32_t>(w[c]) ^ static_cast<uint32_t>(w[c] >> 32);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int kOp>
void run(const char* name, const uint32_t* in, uint32_t* out, long long* clk) {
    for (int wps : {1, 2, 4}) {
        const int iters = 2000;
        rate_kernel<kOp><<<148, 512>>>(in, out, iters, wps, clk);
        if (cudaDeviceSynchronize() != cudaSuccess) {
            printf("%s failed\n", name);
            return;
        }
        long long h[16];
        cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
        const double n = double(iters) * kUnroll * kChains * instr_per_body(kOp) * wps;  // warp-instr per sub-partition
        printf("{\"op\": \"%s\", \"warps_per_smsp\": %d, \"clk_per_warp_instr_per_smsp\": %.3f}\n", name, wps, double(h[0]) / n);
    }
}

int main() {
    uint32_t *in, *out;
    long long* clk;
    cudaMalloc(&in, 1024 * 4);
    cudaMalloc(&out, 148 * 512 * 4);
    cudaMalloc(&clk, 16 * 8);
    uint32_t h[1024];
    for (int i = 0; i < 1024; ++i) {
        float f = 0.25f + float((i * 37) % 101) / 400.f;
        h[i] = *reinterpret_cast<uint32_t*>(&f);
    }
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    run<kFfma>("FFMA r,r,r", in, out, clk);
    run<kFfmaImm>("FFMA r,r,imm", in, out, clk);
    run<kFfma2>("FFMA2", in, out, clk);
    run<kFadd2>("FADD2", in, out, clk);
    run<kFmnmx>("FMNMX", in, out, clk);
    run<kFmnmx3>("FMNMX3", in, out, clk);
    run<kF2fp>("F2FP.BF16 pack", in, out, clk);
    run<kLea>("shl23+add (LEA?)", in, out, clk);
    run<kShlAdd>("SHL ; IADD", in, out, clk);
    run<kImad>("IMAD", in, out, clk);
    run<kMufu>("MUFU.EX2", in, out, clk);
    run<kMufuBf16x2>("ex2.bf16x2 (2 MUFU + PRMT, counted as 1)", in, out, clk);
    run<kMufuF16x2>("ex2.f16x2 (2 MUFU + PRMT, counted as 1)", in, out, clk);
    run<kMufuF16>("ex2.f16 scalar", in, out, clk);
    run<kPrmt>("PRMT", in, out, clk);
    run<kHadd2Bf16>("HADD2.BF16", in, out, clk);
    run<kHfma2>("HFMA2 f16x2", in, out, clk);
    run<kHfma2Bf16>("HFMA2 bf16x2", in, out, clk);
    run<kMixMufuFfma2>("mix MUFU+FFMA2", in, out, clk);
    run<kMixFfma2Fmnmx>("mix FFMA2+FMNMX", in, out, clk);
    run<kMixFfma2Lea>("mix FFMA2+LEA", in, out, clk);
    run<kMixMufuF2fp>("mix MUFU+F2FP", in, out, clk);
    run<kMixFfmaFfma2>("mix FFMA+FFMA2", in, out, clk);
    run<kMixAll>("mix 2MUFU+FFMA2+FADD2+FMNMX3+F2FP", in, out, clk);
    return 0;
}
