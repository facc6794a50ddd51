// fa_fwd_sm100_local.cu -- FusedFlashAttention forward for sm_100a (B200), head_dim 64, specialised
// for NARROW sliding windows: window_left + window_right <= 127 (the reference's local layers use
// (63, 64), rewrite.cpp:355-361).  Same operator contract as fa_fwd_sm100.cu (reference
// attention.cpp:106-213): key j is live for query i iff i-j <= wl, j-i <= wr and pad_bias[b,j] >
// -30000; a live bias value is added to the scaled score; rows with no live key give 0.
//
// Why a second kernel: the general kernel walks 128-key tiles aligned to multiples of 128, so a pair
// of query tiles with a 128-wide band touches four key tiles for each of its two query tiles, every
// one of them on the slow per-element-predicate path, and runs an online softmax over them.  Here a
// 128-row query tile reads exactly the 256 keys [r0 - wl, r0 - wl + 256) it can see -- TMA boxes
// start at any row, rows outside [0, S) are zero-filled -- so that in this strip row r is live on the
// diagonal band of columns [r, r + wl + wr].  The whole row fits one pass: no running max, no
// rescale of O.  This layer is HBM-bound (64 FLOP/B); the point of the design is to keep per-tile
// latency and instruction count down, not to fill the tensor pipe.
//
// One persistent CTA per SM, 10 warps:
//   warps 0-7  softmax/epilogue, two threads per query row: warps 0-3 own strip columns [0,128),
//              warps 4-7 columns [128,256); 32-column chunks that are dead for all 32 rows of a warp
//              are skipped (the band leaves 20 of the 32 chunks of a tile)
//   warp 8     TMA producer: Q (1 box), K and V (2 boxes each, adjacent in smem), two stages
//   warp 9     UMMA issuer: S[128x256] = Q K^T (4 x M128 N256 K16), O[128x64] = P V (16 x M128 N64 K16,
//              P from TMEM)
// TMEM: S [0,256)  P [256,384)  O [384,448).  S is copied to registers in one go and handed back at
// once, so Q K^T of the next tile runs under the softmax of this one; the load/max half of the next
// tile's softmax runs under P V of this one.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "fa_internal.h"
#include "ptx.cuh"

namespace rf {
namespace {

using namespace rfptx;

constexpr int kHeadDim = 64;
constexpr int kStrip = 2 * kBlockN;                 // keys a query tile reads
constexpr int kTileBytes = kBlockN * kHeadDim * 2;  // 16 KiB
constexpr int kStageBytes = 5 * kTileBytes;         // Q | K0 K1 | V0 V1
constexpr int kStages = 2;
constexpr int kSoftmaxWarps = 8;
constexpr int kSoftmaxThreads = kSoftmaxWarps * 32;
constexpr int kProducerWarp = 8;
constexpr int kMmaWarp = 9;
constexpr int kThreads = 320;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColS = 0, kColP = 256, kColO = 384;

struct Smem {
    static constexpr uint32_t stage = 0;
    static constexpr uint32_t bars = stage + kStages * kStageBytes;
    static constexpr uint32_t bar_bytes = 128;
    static constexpr uint32_t xchg = bars + bar_bytes;           // [2 parity][2 halves][128] f32 row max
    static constexpr uint32_t lsum = xchg + 2 * 2 * kBlockM * 4;  // [2 parity][2 halves][128] f32 row sum
    static constexpr uint32_t bias = lsum + 2 * 2 * kBlockM * 4;  // [2 parity][256] f32, log2 domain
    static constexpr uint32_t total = bias + 2 * kStrip * 4;
};
enum : uint32_t {
    kBarFull = 0,   // [2] TMA landed
    kBarEmpty = 2,  // [2] both MMAs of the tile have read the stage
    kBarSFull = 4,
    kBarSFree = 5,  // count 8: S is in the registers of every softmax warp
    kBarPFull = 6,  // count 256
    kBarOFull = 7,
    kNumBars = 8,
};

struct Tile {
    int b, h, r0, kb;  // batch, head, first query row, first key of the strip
};

__device__ __forceinline__ Tile decode_tile(const FaParams& p, int g, int q_tiles) {
    Tile t;
    const int qt = g % q_tiles;
    const int bh = g / q_tiles;
    t.h = bh % p.H;
    t.b = bh / p.H;
    t.r0 = qt * kBlockM;
    t.kb = t.r0 - p.wl;
    return t;
}

template <bool kBf16, bool kHasBias>
__global__ void __launch_bounds__(kThreads, 1)
fa_fwd_sm100_local_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v, const FaParams p,
                          const float* __restrict__ pad_bias) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* smem_gen = smem_raw + (smem_base - smem_u32(smem_raw));
    const uint32_t bars = smem_base + Smem::bars;
    auto bar = [&](uint32_t i) { return bars + 8u * i; };
    volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(smem_gen + Smem::bars + 8 * kNumBars);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int q_tiles = (p.S + kBlockM - 1) / kBlockM;
    const int total = p.B * p.H * q_tiles;
    // tiles blockIdx.x, blockIdx.x + gridDim.x, ...: neighbouring CTAs read overlapping K/V strips
    const int my_tiles = blockIdx.x < total ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

    if (warp == kProducerWarp && lane == 0) {
        prefetch_tensormap(&tm_q);
        prefetch_tensormap(&tm_k);
        prefetch_tensormap(&tm_v);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(bar(kBarFull + s), 1);
            mbar_init(bar(kBarEmpty + s), 1);
        }
        mbar_init(bar(kBarSFull), 1);
        mbar_init(bar(kBarSFree), kSoftmaxWarps);
        mbar_init(bar(kBarPFull), kSoftmaxThreads);
        mbar_init(bar(kBarOFull), 1);
        fence_barrier_init();
    }
    if (warp == kMmaWarp) {
        tmem_alloc(smem_u32(const_cast<uint32_t*>(tmem_slot)), kTmemCols);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == kProducerWarp) {
        // =============================== TMA producer ===============================
        // warp-uniform control flow; only lane 0 issues
        for (int n = 0; n < my_tiles; ++n) {
            const Tile t = decode_tile(p, blockIdx.x + n * gridDim.x, q_tiles);
            const uint32_t s = n & 1;
            const uint32_t dst = smem_base + Smem::stage + s * kStageBytes;
            mbar_wait(bar(kBarEmpty + s), ((n >> 1) & 1) ^ 1);
            if (lane == 0) {
                mbar_arrive_expect_tx(bar(kBarFull + s), kStageBytes);
                tma_load_4d(dst, &tm_q, bar(kBarFull + s), 0, t.r0, t.h, t.b);
                tma_load_4d(dst + 1 * kTileBytes, &tm_k, bar(kBarFull + s), 0, t.kb, t.h, t.b);
                tma_load_4d(dst + 2 * kTileBytes, &tm_k, bar(kBarFull + s), 0, t.kb + kBlockN, t.h, t.b);
                tma_load_4d(dst + 3 * kTileBytes, &tm_v, bar(kBarFull + s), 0, t.kb, t.h, t.b);
                tma_load_4d(dst + 4 * kTileBytes, &tm_v, bar(kBarFull + s), 0, t.kb + kBlockN, t.h, t.b);
            }
            __syncwarp();
        }
    } else if (warp == kMmaWarp) {
        // =============================== UMMA issuer ===============================
        // warp-uniform control flow; only the tcgen05 instructions are predicated on the elected lane
        const bool leader = elect_one() != 0;
        constexpr uint32_t fmt = kBf16 ? 1u : 0u;
        constexpr uint32_t idesc_qk = make_idesc_f16(fmt, 0, 0, kBlockM, kStrip);
        constexpr uint32_t idesc_pv = make_idesc_f16(fmt, 0, 1, kBlockM, kHeadDim);
        const uint32_t t_s = tmem_base + kColS, t_p = tmem_base + kColP, t_o = tmem_base + kColO;
        auto issue_qk = [&](int n) {
            const uint32_t base = smem_base + Smem::stage + (n & 1) * kStageBytes;
            if (leader) {
#pragma unroll
                for (int kk = 0; kk < kHeadDim / 16; ++kk)
                    mma_ss(t_s, make_smem_desc(base + kk * 32, 16, 1024, kSwizzle128B),
                           make_smem_desc(base + kTileBytes + kk * 32, 16, 1024, kSwizzle128B), idesc_qk,
                           kk > 0 ? 1u : 0u);
                tc_commit(bar(kBarSFull));
            }
            __syncwarp();
        };
        if (my_tiles > 0) {
            mbar_wait(bar(kBarFull), 0);
            tc_fence_after();
            issue_qk(0);
        }
        for (int n = 0; n < my_tiles; ++n) {
            if (n + 1 < my_tiles) {
                // S(n) is in registers: Q K^T of the next tile runs under the softmax of this one
                mbar_wait2(bar(kBarFull + ((n + 1) & 1)), ((n + 1) >> 1) & 1, bar(kBarSFree), n & 1);
                tc_fence_after();
                issue_qk(n + 1);
            }
            mbar_wait(bar(kBarPFull), n & 1);
            tc_fence_after();
            if (leader) {
                // V strip [256 keys][64] with d contiguous = MN-major B operand; a K=16 step is 2048 B
                const uint32_t vbase = smem_base + Smem::stage + (n & 1) * kStageBytes + 3 * kTileBytes;
#pragma unroll
                for (int kk = 0; kk < kStrip / 16; ++kk)
                    mma_ts(t_o, t_p + kk * 8, make_smem_desc(vbase + kk * 2048, kTileBytes, 1024, kSwizzle128B),
                           idesc_pv, kk > 0 ? 1u : 0u);
                tc_commit(bar(kBarOFull));
                tc_commit(bar(kBarEmpty + (n & 1)));
            }
            __syncwarp();
        }
    } else {
        // =============================== softmax / epilogue ===============================
        const int hf = warp >> 2;              // 0: strip columns [0,128), 1: [128,256)
        const int quad = warp & 3;
        const int r = quad * 32 + lane;        // row inside the tile == TMEM lane
        const int tid = threadIdx.x;           // 0..255
        const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
        const uint32_t t_s = tmem_base + lane_base + kColS + hf * kBlockN;
        const uint32_t t_p = tmem_base + lane_base + kColP + hf * (kBlockN / 2);
        const uint32_t t_o = tmem_base + lane_base + kColO + hf * (kHeadDim / 2);
        const float c = p.scale_log2;
        const int band = p.wl + p.wr;          // live strip columns of row r: [r, r + band]
        float* xchg = reinterpret_cast<float*>(smem_gen + Smem::xchg);
        float* lsum = reinterpret_cast<float*>(smem_gen + Smem::lsum);
        float* sbias = reinterpret_cast<float*>(smem_gen + Smem::bias);
        const uint32_t pair_bar = 1 + quad;    // named barrier of the two warps that share 32 rows

        auto load_bias = [&](const Tile& t) -> float {  // this thread's strip column, log2 domain
            const int key = t.kb + tid;
            float v = -CUDART_INF_F;
            if (key >= 0 && key < p.S) {
                const float raw = __ldg(pad_bias + static_cast<size_t>(t.b) * p.S + key);
                v = raw > kMaskThreshold ? raw * kLog2e : -CUDART_INF_F;
            }
            return v;
        };

        uint32_t su[kBlockN];  // this thread's 128 scores, then log2-domain x, of the current tile
        uint32_t live_chunks = 0;
        float m_row = -CUDART_INF_F;
        Tile cur = {}, nxt = {};
        float bias_pref = 0.f;
        if (my_tiles > 0) {
            nxt = decode_tile(p, blockIdx.x, q_tiles);
            if (kHasBias) bias_pref = load_bias(nxt);
        }

        // first half of a tile: S -> registers, scale / bias / band predicate, row max
        auto stage_a = [&](int n, const Tile& t) {
            const uint32_t par = n & 1;
            // this thread's live columns, local to its 128-column half
            int lo = max(r, -t.kb);                       // key >= 0
            int hi = min(r + band, p.S - 1 - t.kb);       // key < S
            lo -= hf * kBlockN;
            hi -= hf * kBlockN;
            if (kHasBias) {
                sbias[par * kStrip + tid] = bias_pref;
                named_bar_sync(5, kSoftmaxThreads);
            }
            mbar_wait(bar(kBarSFull), par);
            tc_fence_after();
            uint32_t dead = 0, full = 0;
#pragma unroll
            for (int cb = 0; cb < 4; ++cb) {
                const int c0 = cb * 32;
                if (__all_sync(0xffffffffu, hi < c0 || lo > c0 + 31)) dead |= 1u << cb;
                if (__all_sync(0xffffffffu, lo <= c0 && hi >= c0 + 31)) full |= 1u << cb;
            }
#pragma unroll
            for (int cb = 0; cb < 4; ++cb)
                if (!((dead >> cb) & 1)) tmem_ld32(t_s + cb * 32, reinterpret_cast<uint32_t(&)[32]>(su[cb * 32]));
            tc_wait_ld();
            tc_fence_before();
            if (lane == 0) mbar_arrive(bar(kBarSFree));
            float mx = -CUDART_INF_F;
#pragma unroll
            for (int cb = 0; cb < 4; ++cb) {
                if ((dead >> cb) & 1) continue;
                const bool is_full = (full >> cb) & 1;
                const float* brow = sbias + par * kStrip + hf * kBlockN + cb * 32;
#pragma unroll
                for (int j4 = 0; j4 < 32; j4 += 4) {
                    float4 bb = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (kHasBias) bb = *reinterpret_cast<const float4*>(brow + j4);
                    const float bv[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int j = cb * 32 + j4 + u;
                        float x = fmaf(__uint_as_float(su[j]), c, bv[u]);  // bias -inf => masked key
                        if (!is_full) x = (j >= lo && j <= hi) ? x : -CUDART_INF_F;
                        su[j] = __float_as_uint(x);
                        mx = fmaxf(mx, x);
                    }
                }
            }
            live_chunks = ~dead & 0xfu;
            xchg[(par * 2 + hf) * kBlockM + r] = mx;
            named_bar_sync(pair_bar, 64);
            m_row = fmaxf(mx, xchg[(par * 2 + (hf ^ 1)) * kBlockM + r]);
        };

        for (int n = 0; n < my_tiles; ++n) {
            const uint32_t par = n & 1;
            if (n == 0) stage_a(0, nxt);
            cur = nxt;
            const bool has_next = n + 1 < my_tiles;
            if (has_next) {
                nxt = decode_tile(p, blockIdx.x + (n + 1) * gridDim.x, q_tiles);
                if (kHasBias) bias_pref = load_bias(nxt);
            }
            // ---- second half: P = 2^(x - m), row sum, P -> TMEM ----
            // (P may be overwritten: every thread has seen O-full of the previous tile in its epilogue)
            const float neg_m = (m_row == -CUDART_INF_F) ? 0.f : -m_row;
            const uint64_t negm2 = bc2(neg_m);
            uint64_t sum2 = 0;
#pragma unroll
            for (int cb = 0; cb < 4; ++cb) {
                uint32_t pk[16];
                if ((live_chunks >> cb) & 1) {
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        float p0, p1;
                        unpk2(fadd2v(pk2(__uint_as_float(su[cb * 32 + 2 * u]), __uint_as_float(su[cb * 32 + 2 * u + 1])),
                                     negm2),
                              p0, p1);
                        p0 = ex2(p0);
                        p1 = ex2(p1);
                        sum2 = fadd2v(sum2, pk2(p0, p1));
                        pk[u] = pack2<kBf16>(p0, p1);
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < 16; ++u) pk[u] = 0u;
                }
                tmem_st16(t_p + cb * 16, pk);
            }
            float sum0, sum1;
            unpk2(sum2, sum0, sum1);
            const float l_part = sum0 + sum1;
            lsum[(par * 2 + hf) * kBlockM + r] = l_part;
            tc_wait_st();
            tc_fence_before();
            mbar_arrive(bar(kBarPFull));

            // ---- load / max half of the next tile runs under P V of this one ----
            if (has_next) stage_a(n + 1, nxt);  // (its pair barrier also orders the lsum exchange below)
            else named_bar_sync(pair_bar, 64);

            // ---- epilogue of tile n ----
            const float l_tot = l_part + lsum[(par * 2 + (hf ^ 1)) * kBlockM + r];
            const float inv = l_tot > 0.f ? 1.0f / l_tot : 0.f;
            constexpr int kOutCols = kHeadDim / 2;
            float o[kOutCols];
            mbar_wait(bar(kBarOFull), par);
            tc_fence_after();
            tmem_ld32(t_o, reinterpret_cast<uint32_t(&)[32]>(o));
            tc_wait_ld();
            const int row = cur.r0 + r;
            if (row < p.S) {
                const size_t off = static_cast<size_t>(cur.b) * p.o_sb + static_cast<size_t>(cur.h) * p.o_sh +
                                   static_cast<size_t>(row) * p.o_ss + hf * kOutCols;
                if (p.out_dtype == 2) {
                    float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.out) + off);
#pragma unroll
                    for (int u = 0; u < kOutCols / 4; ++u)
                        dst[u] = make_float4(o[4 * u] * inv, o[4 * u + 1] * inv, o[4 * u + 2] * inv, o[4 * u + 3] * inv);
                } else {
                    uint4* dst = reinterpret_cast<uint4*>(static_cast<uint16_t*>(p.out) + off);
#pragma unroll
                    for (int u = 0; u < kOutCols / 8; ++u) {
                        uint32_t w[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float a0 = o[8 * u + 2 * e] * inv, a1 = o[8 * u + 2 * e + 1] * inv;
                            w[e] = (p.out_dtype == 0) ? pack2<true>(a0, a1) : pack2<false>(a0, a1);
                        }
                        dst[u] = make_uint4(w[0], w[1], w[2], w[3]);
                    }
                }
            }
        }
    }

    // ---------------- teardown ----------------
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc(tmem_base, kTmemCols);
    }
}

}  // namespace

bool fa_fwd_sm100_local_covers(int wl, int wr) { return wl >= 0 && wr >= 0 && wl + wr <= kBlockN - 1; }

size_t fa_fwd_sm100_local_smem_bytes() { return Smem::total + 1024; }

int fa_fwd_sm100_local_grid(const FaParams& p, int sms) {
    const long long tiles = static_cast<long long>(p.B) * p.H * ((p.S + kBlockM - 1) / kBlockM);
    return static_cast<int>(tiles < sms ? tiles : sms);
}

cudaError_t launch_fa_fwd_sm100_local(const CUtensorMap& tmq, const CUtensorMap& tmk, const CUtensorMap& tmv,
                                      const FaParams& p, const float* pad_bias, bool bf16, int grid,
                                      cudaStream_t stream) {
    const bool has_bias = pad_bias != nullptr;
    void (*kern)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const FaParams, const float*) =
        bf16 ? (has_bias ? fa_fwd_sm100_local_kernel<true, true> : fa_fwd_sm100_local_kernel<true, false>)
             : (has_bias ? fa_fwd_sm100_local_kernel<false, true> : fa_fwd_sm100_local_kernel<false, false>);
    const size_t smem = fa_fwd_sm100_local_smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreads, smem, stream>>>(tmq, tmk, tmv, p, pad_bias);
    return cudaGetLastError();
}

}  // namespace rf
