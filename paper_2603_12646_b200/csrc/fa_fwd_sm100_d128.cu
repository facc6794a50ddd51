// fa_fwd_sm100_d128.cu -- FusedFlashAttention forward for sm_100a (B200), head_dim 128.
//
// Same operator contract as fa_fwd_sm100.cu (reference routefast::flash_attention,
// proj/core/src/attention.cpp:106-213; head dims {32, 64, 128}: proj/core/src/rewrite.cpp:266-269).
//
// Why a separate kernel: at head_dim 128 the two O accumulators of a query-tile pair take 256 of the
// 512 TMEM columns, so there is room for exactly two S accumulators -- one per query tile -- instead of
// the three rotating ones of the head_dim-64 kernel, and a K / V tile is 32 KiB, so the rings are two
// deep.  The balance also changes: Q K^T and P V each cost 512 clk of tensor pipe per 128 x 128 tile
// (8 x M128 N128 K16), as much as the 1024 clk the tile's exponentials take on the MUFU pipe, so the
// schedule is the plain ping-pong -- tile A's softmax runs under tile B's MMAs and vice versa:
//
//   warp 17 (UMMA issuer)  S_A = Q_A K^T, S_B = Q_B K^T, then per key tile i:
//                          wait P_A(i): O_A += P_A V(i); S_A = Q_A K(i+1)^T    (in-order pipe: the P V reads
//                          wait P_B(i): O_B += P_B V(i); S_B = Q_B K(i+1)^T     P before Q K^T overwrites S)
//   warp 16 (TMA producer) Q once per pair; K and V as two boxes of 64 head-dim columns per 128-key tile
//   warps 0-7 / 8-15       softmax of tile A / B, two threads per query row (key columns [0,64) / [64,128)),
//                          P (16-bit) written over the thread's own S columns, lazy rescale of O
// TMEM: S_A [0,128)  S_B [128,256)  O_A [256,384)  O_B [384,512).
// Work distribution: whole query-tile pairs -- one per CTA (sched_mode 0: a single wave, split-KV partials) or
// dealt round-robin over a persistent grid (sched_mode 2) -- or, as in fa_fwd_sm100.cu, statically balanced slices of
// the flat (pair x key tile) space (sched_mode 1): a pair cut between CTA c (leading key tiles, its FIRST item) and CTA
// c + 1 (trailing key tiles, its LAST item) is merged in-kernel from the partial c published; a CTA only ever waits
// for a lower-indexed CTA.  (384 pairs on 148 SMs are three rounds of which the last is 60 % full: 13.5 % of the
// SM time idle with whole pairs.)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <type_traits>

#include "fa_internal.h"
#include "ptx.cuh"

namespace rf {
namespace {

using namespace rfptx;

constexpr int kD = 128;
constexpr int kBoxBytes = kBlockN * 64 * 2;   // 16 KiB: one TMA box, 128 rows x 64 head-dim columns
constexpr int kTileBytes = 2 * kBoxBytes;     // 32 KiB: one 128 x 128 16-bit tile = two boxes
constexpr int kStages = 2;                    // K ring and V ring depth
constexpr int kNumSoftmaxWarps = 16;
constexpr int kProducerWarp = 16;
constexpr int kMmaWarp = 17;
constexpr int kThreads = 640;
constexpr int kHalfN = kBlockN / 2;
constexpr int kRegsSoftmax = 112;
constexpr int kRegsOther = 32;
#ifndef RF_FA_D128_EMU_EVERY
#define RF_FA_D128_EMU_EVERY 5  // 326 us at 8K; 8: 328, 16: 329, 4: 334 (same-box sweep)
#endif
constexpr int kEmuEvery = RF_FA_D128_EMU_EVERY;  // every n-th element pair of a full tile: FMA-pipe exp2
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColS = 0;                 // + 128 * X
constexpr uint32_t kColO = 256;               // + 128 * X
constexpr float kRescaleThresholdBf16 = 20.0f;
constexpr float kRescaleThresholdF16 = 14.0f;

struct Smem {
    static constexpr uint32_t q = 0;                             // 2 tiles
    static constexpr uint32_t k = q + 2 * kTileBytes;            // kStages tiles
    static constexpr uint32_t v = k + kStages * kTileBytes;      // kStages tiles
    static constexpr uint32_t bars = v + kStages * kTileBytes;
    static constexpr uint32_t bar_bytes = 256;
    static constexpr uint32_t xchg = bars + bar_bytes;           // [2 parity][2 tile][2 half][128] f32
    static constexpr uint32_t xchg_bytes = 2 * 2 * 2 * kBlockM * 4;
};
enum : uint32_t {
    kBarQFull = 0,
    kBarQEmpty = 1,
    kBarKFull = 2,                     // [kStages]
    kBarKEmpty = kBarKFull + kStages,  // [kStages]
    kBarVFull = kBarKEmpty + kStages,  // [kStages]
    kBarVEmpty = kBarVFull + kStages,  // [kStages]
    kBarSFull = kBarVEmpty + kStages,  // [2] per query tile
    kBarPFull = kBarSFull + 2,         // [2]
    kBarOFull = kBarPFull + 2,         // [2]
    kNumBars = kBarOFull + 2,
};
constexpr uint32_t kTmemSlotOff = kNumBars * 8;
constexpr uint32_t kWaitBlockOff = (kTmemSlotOff + 8 + 15) & ~15u;
static_assert(kWaitBlockOff + 16 <= Smem::bar_bytes, "barrier block too small");

struct Item {
    int b, h, q0;
    int n0, n1;    // key tiles [n0, n1)
    int num_live;  // tiles in the range that are not fully padded
    int kind;      // kItemFull / kItemPublish (leading key tiles of a cut pair) / kItemMerge (its trailing key tiles)
    bool has_b;
};
enum : int { kItemFull = 0, kItemPublish = 1, kItemMerge = 2 };

__device__ __forceinline__ int ld_acquire_gpu(const int* ptr) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int* ptr, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(ptr), "r"(v) : "memory");
}

template <bool kHasBias>
__device__ __forceinline__ bool tile_live(const FaParams& p, int b, int n) {
    return !kHasBias || p.tile_flags[b * p.n_kv_tiles + n] != kTileSkip;
}

// i-th item of this CTA (i = 0, 1, ...): pair blockIdx.x + i * gridDim.x (sched_mode 2), blockIdx.x (mode 0), or the
// i-th pair from the END of the CTA's slice of the flat (pair x key tile) space, cut to the slice (mode 1)
template <bool kHasBias>
__device__ __forceinline__ bool get_item(const FaParams& p, int i, Item& it) {
    int pair_lin, k0 = 0, k1 = 0x7fffffff;
    it.kind = kItemFull;
    if (p.sched_mode == 1) {
        const long long K = p.tiles_per_pair;
        const long long total = static_cast<long long>(p.total_pairs) * K;
        const long long t0 = total * blockIdx.x / gridDim.x, t1 = total * (blockIdx.x + 1) / gridDim.x;
        if (t1 <= t0) return false;
        const long long pl = (t1 - 1) / K - i;
        if (pl < t0 / K) return false;
        const long long pair_start = pl * K;
        pair_lin = static_cast<int>(pl);
        k0 = static_cast<int>(max(t0, pair_start) - pair_start);
        k1 = static_cast<int>(min(t1, pair_start + K) - pair_start);
        it.kind = k0 > 0 ? kItemMerge : (k1 < K ? kItemPublish : kItemFull);
    } else {
        const long long lin = p.sched_mode == 2 ? blockIdx.x + static_cast<long long>(i) * gridDim.x
                                                : (i == 0 ? static_cast<long long>(blockIdx.x) : p.total_pairs);
        if (lin >= p.total_pairs) return false;
        pair_lin = static_cast<int>(lin);
    }
    const int px = pair_lin % p.pairs_per_head;
    const int bh = pair_lin / p.pairs_per_head;
    it.h = bh % p.H;
    it.b = bh / p.H;
    it.q0 = px * kRowsPerCta;
    it.has_b = it.q0 + kBlockM < p.S;
    const int rows_end = min(it.q0 + kRowsPerCta, p.S);
    int j_lo = p.kv_begin, j_hi = p.kv_end;
    if (p.wl >= 0) j_lo = max(j_lo, it.q0 - p.wl);
    if (p.wr >= 0) j_hi = min(j_hi, rows_end + p.wr);
    const int pn0 = j_lo >> 7;
    const int pn1 = (j_hi > j_lo) ? ((j_hi + kBlockN - 1) >> 7) : pn0;
    // the item's slice of the pair's key tiles (mode 1: virtual tile v is real tile pn0 + v; past the last tile: empty)
    it.n0 = min(pn0 + k0, pn1);
    it.n1 = (k1 >= pn1 - pn0) ? pn1 : pn0 + k1;
    it.num_live = 0;
    for (int n = it.n0; n < it.n1; ++n) it.num_live += tile_live<kHasBias>(p, it.b, n) ? 1 : 0;
    return true;
}

// O rows (this thread's 64 columns) *= alpha
__device__ __noinline__ void rescale_o_rows_d128(uint32_t t_o, float alpha) {
#pragma unroll
    for (int cb = 0; cb < 2; ++cb) {
        uint32_t o[32];
        tmem_ld32(t_o + cb * 32, o);
        tc_wait_ld();
#pragma unroll
        for (int u = 0; u < 32; u += 2) {
            float a0 = __uint_as_float(o[u]), a1 = __uint_as_float(o[u + 1]);
            fmul2(a0, a1, alpha);
            o[u] = __float_as_uint(a0);
            o[u + 1] = __float_as_uint(a1);
        }
        tmem_st32(t_o + cb * 32, o);
    }
    tc_wait_st();
}

template <bool kBf16, bool kHasBias>
__global__ void __launch_bounds__(kThreads, 1)
fa_fwd_sm100_d128_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const FaParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* smem_gen = smem_raw + (smem_base - smem_u32(smem_raw));
    const uint32_t bars = smem_base + Smem::bars;
    auto bar = [&](uint32_t i) { return bars + 8u * i; };
    volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(smem_gen + Smem::bars + kTmemSlotOff);
    const WaitCtx wctx{bars + kWaitBlockOff};

    const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);  // warp-uniform by construction: lets roles, buffer indices and TMEM addresses live in uniform registers
    const int lane = threadIdx.x & 31;

    if (warp == kProducerWarp && lane == 0) {
        prefetch_tensormap(&tm_q);
        prefetch_tensormap(&tm_k);
        prefetch_tensormap(&tm_v);
        mbar_init(bar(kBarQFull), 1);
        mbar_init(bar(kBarQEmpty), 1 + kNumSoftmaxWarps);  // the UMMA commit and every softmax warp (row norms from the Q tile)
        for (int s = 0; s < kStages; ++s) {
            mbar_init(bar(kBarKFull + s), 1);
            mbar_init(bar(kBarKEmpty + s), 1);
            mbar_init(bar(kBarVFull + s), 1);
            mbar_init(bar(kBarVEmpty + s), 1);
        }
        for (int x = 0; x < 2; ++x) {
            mbar_init(bar(kBarSFull + x), 1);
            mbar_init(bar(kBarPFull + x), 2 * kBlockM);
            mbar_init(bar(kBarOFull + x), 1);
        }
        wait_block_init(wctx.block_smem, p.status);
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

    static_assert(128 * kRegsOther + 512 * kRegsSoftmax <= kThreads * 96, "setmaxnreg pool must balance");
    if (warp >= kNumSoftmaxWarps) setmaxnreg_dec<kRegsOther>();
    Item item;

    if (warp == kProducerWarp) {
        // =============================== TMA producer ===============================
        const bool leader = elect_one() != 0;
        uint32_t qi = 0, kc = 0, vc = 0;  // items / K tiles / V tiles loaded so far
        auto load_tile = [&](const CUtensorMap* tm, uint32_t dst, uint32_t full_bar, int row0, int h, int b) {
            tma_load_4d(dst, tm, full_bar, 0, row0, h, b);
            tma_load_4d(dst + kBoxBytes, tm, full_bar, 64, row0, h, b);
        };
        for (int ii = 0; get_item<kHasBias>(p, ii, item); ++ii) {
            if (item.num_live == 0) continue;
            const int b = item.b, h = item.h;
            mbar_wait(bar(kBarQEmpty), (qi & 1) ^ 1, wctx);
            if (leader) {
                mbar_arrive_expect_tx(bar(kBarQFull), item.has_b ? 2 * kTileBytes : kTileBytes);
                load_tile(&tm_q, smem_base + Smem::q, bar(kBarQFull), item.q0, h, b);
                if (item.has_b) load_tile(&tm_q, smem_base + Smem::q + kTileBytes, bar(kBarQFull), item.q0 + kBlockM, h, b);
            }
            __syncwarp();
            ++qi;
            auto load_k = [&](int n) {
                const uint32_t st = kc % kStages;
                mbar_wait(bar(kBarKEmpty + st), ((kc / kStages) & 1) ^ 1, wctx);
                if (leader) {
                    mbar_arrive_expect_tx(bar(kBarKFull + st), kTileBytes);
                    load_tile(&tm_k, smem_base + Smem::k + st * kTileBytes, bar(kBarKFull + st), n * kBlockN, h, b);
                }
                __syncwarp();
                ++kc;
            };
            auto load_v = [&](int n) {
                const uint32_t st = vc % kStages;
                mbar_wait(bar(kBarVEmpty + st), ((vc / kStages) & 1) ^ 1, wctx);
                if (leader) {
                    mbar_arrive_expect_tx(bar(kBarVFull + st), kTileBytes);
                    load_tile(&tm_v, smem_base + Smem::v + st * kTileBytes, bar(kBarVFull + st), n * kBlockN, h, b);
                }
                __syncwarp();
                ++vc;
            };
            auto next_live = [&](int n) {
                while (n < item.n1 && !tile_live<kHasBias>(p, b, n)) ++n;
                return n;
            };
            // K runs one tile ahead of V
            int nk = next_live(item.n0);
            if (nk < item.n1) {
                load_k(nk);
                nk = next_live(nk + 1);
            }
            for (int n = next_live(item.n0); n < item.n1; n = next_live(n + 1)) {
                if (nk < item.n1) {
                    load_k(nk);
                    nk = next_live(nk + 1);
                }
                load_v(n);
            }
        }
    } else if (warp == kMmaWarp) {
        // =============================== UMMA issuer ===============================
        // warp-uniform control flow; only the tcgen05 instructions are predicated on the elected lane
        const bool leader = elect_one() != 0;
        constexpr uint32_t fmt = kBf16 ? 1u : 0u;
        constexpr uint32_t idesc_qk = make_idesc_f16(fmt, 0, 0, kBlockM, kBlockN);
        constexpr uint32_t idesc_pv = make_idesc_f16(fmt, 0, 1, kBlockM, kD);
        constexpr uint32_t kDescHi = (1024u >> 4) | (1u << 14) | (kSwizzle128B << 29);  // SBO, version, swizzle
        constexpr uint32_t kLboK = (16u >> 4) << 16;                                    // K-major operands
        constexpr uint32_t kLboV = (static_cast<uint32_t>(kBoxBytes) >> 4) << 16;       // MN-major V: 64-column boxes
        const uint32_t sb16 = smem_base >> 4;
        auto desc = [&](uint32_t lo) { return (static_cast<uint64_t>(kDescHi) << 32) | lo; };
        auto commit = [&](uint32_t b_) {
            if (leader) tc_commit(b_);
            __syncwarp();
        };
        const uint32_t q_lo = kLboK | (sb16 + Smem::q / 16);
        const uint32_t k_lo = kLboK | (sb16 + Smem::k / 16);
        const uint32_t v_lo = kLboV | (sb16 + Smem::v / 16);
        constexpr uint32_t kTile16 = kTileBytes / 16, kBox16 = kBoxBytes / 16;

        // S_X = Q_X K^T: both operands K-major, 128B swizzle; the 128 head-dim columns are two boxes of four
        // K=16 steps each (32 B apart inside the swizzle atom)
        auto issue_qk = [&](uint32_t x, uint32_t kstage) {
            const uint32_t qlo = q_lo + x * kTile16;
            const uint32_t klo = k_lo + kstage * kTile16;
            const uint32_t td = tmem_base + kColS + x * kBlockN;
            if (leader) {
#pragma unroll
                for (int kk = 0; kk < kD / 16; ++kk) {
                    const uint32_t off = (kk >> 2) * kBox16 + (kk & 3) * 2;
                    mma_ss(td, desc(qlo + off), desc(klo + off), idesc_qk, kk > 0 ? 1u : 0u);
                }
                tc_commit(bar(kBarSFull + x));
            }
            __syncwarp();
        };
        // O_X += P V: A = P from TMEM (keys [0,64) in S columns [0,32), keys [64,128) in [64,96)); B = V, MN-major:
        // [key][d] with d contiguous in two 64-column boxes kBoxBytes apart (LBO), 8-key groups 1024 B apart
        // (SBO), a K=16 step advances 16 keys = 2048 B
        auto issue_pv = [&](uint32_t x, uint32_t vstage, uint32_t acc0) {
            const uint32_t vlo = v_lo + vstage * kTile16;
            const uint32_t ta = tmem_base + kColS + x * kBlockN;
            const uint32_t td = tmem_base + kColO + x * kD;
            if (leader) {
#pragma unroll
                for (int kk = 0; kk < kBlockN / 16; ++kk)
                    mma_ts(td, ta + kk * 8 + (kk >= 4 ? 32 : 0), desc(vlo + kk * 128), idesc_pv, kk > 0 ? 1u : acc0);
            }
            __syncwarp();
        };

        uint32_t qi = 0, kc = 0, vc = 0;  // items / K tiles / V tiles consumed so far
        uint32_t sp_a = 0, sp_b = 0;      // phase parity of the next P-full wait of tile A / B (B sits out ragged ends)
        for (int ii = 0; get_item<kHasBias>(p, ii, item); ++ii) {
            const int num_live = item.num_live;
            if (num_live == 0) continue;
            const bool has_b = item.has_b;
            mbar_wait(bar(kBarQFull), qi & 1, wctx);
            mbar_wait(bar(kBarKFull + kc % kStages), (kc / kStages) & 1, wctx);
            tc_fence_after();
            issue_qk(0, kc % kStages);
            if (has_b) issue_qk(1, kc % kStages);
            commit(bar(kBarKEmpty + kc % kStages));
            if (num_live == 1) commit(bar(kBarQEmpty));
            ++kc;
            for (int i = 0; i < num_live; ++i) {
                const bool last = i + 1 == num_live;
                const uint32_t vst = vc % kStages, kst = kc % kStages;
                mbar_wait2(bar(kBarVFull + vst), (vc / kStages) & 1, bar(kBarPFull + 0), sp_a, wctx);
                tc_fence_after();
                issue_pv(0, vst, i > 0 ? 1u : 0u);
                if (last) {
                    commit(bar(kBarOFull + 0));
                } else {
                    mbar_wait(bar(kBarKFull + kst), (kc / kStages) & 1, wctx);
                    tc_fence_after();
                    issue_qk(0, kst);
                }
                if (has_b) {
                    mbar_wait(bar(kBarPFull + 1), sp_b, wctx);
                    tc_fence_after();
                    issue_pv(1, vst, i > 0 ? 1u : 0u);
                    if (last) commit(bar(kBarOFull + 1));
                }
                commit(bar(kBarVEmpty + vst));
                ++vc;
                if (!last) {
                    if (has_b) issue_qk(1, kst);
                    commit(bar(kBarKEmpty + kst));
                    if (i + 2 == num_live) commit(bar(kBarQEmpty));
                    ++kc;
                }
                sp_a ^= 1u;
                if (has_b) sp_b ^= 1u;
            }
            ++qi;
        }
    } else if (warp < kNumSoftmaxWarps) {
        // =============================== softmax / epilogue ===============================
        setmaxnreg_inc<kRegsSoftmax>();
        const int x = warp >> 3;               // 0 = tile A, 1 = tile B
        const int hf = (warp >> 2) & 1;        // which half of the tile's key columns this thread owns
        const int r = (warp & 3) * 32 + lane;  // row inside the tile == TMEM lane
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint32_t t_o = tmem_base + lane_base + kColO + x * kD + hf * (kD / 2);
        const uint32_t t_s = tmem_base + lane_base + kColS + x * kBlockN;
        const int kv_end_eff = min(p.kv_end, p.S);
        const float c = p.scale_log2;
        float* xchg = reinterpret_cast<float*>(smem_gen + Smem::xchg);
        float* xrow_base = xchg + (x * 2) * kBlockM + r;
        const uint32_t bar_id = 1 + x * 4 + (warp & 3);  // named barrier of the two warps that share 32 rows
        constexpr uint32_t kPairThreads = 64;
        constexpr float kThreshold = kBf16 ? kRescaleThresholdBf16 : kRescaleThresholdF16;

        uint32_t oi = 0;    // items with work so far (O-full phase)
        uint32_t qn = 0;    // items with live key tiles so far, whether this tile took part or not (Q-full phase)
        uint32_t sp = 0;    // phase parity of the next S-full wait
        uint32_t xpar = 0;  // exchange double buffer

        for (int ii = 0; get_item<kHasBias>(p, ii, item); ++ii) {
            const int b = item.b, h = item.h;
            const int num_live = item.num_live;
            const bool active = (x == 0) || item.has_b;
            const int tile_r_lo = item.q0 + x * kBlockM;
            const int tile_r_hi = tile_r_lo + kBlockM - 1;
            const int row = tile_r_lo + r;
            float m_ref = -CUDART_INF_F;
            float l_run = 0.f;
            // Row-max skip (fa_fwd_sm100.cu): c |q_row| max_j |k_j| bounds every score of the row in a key tile; |q_row|
            // from the Q tile in shared memory (two 64-column boxes), the key-tile norms from k_tile_norms_kernel.
            float qn_c = CUDART_INF_F;
            const float* kmax_row = nullptr;
            if (num_live > 0) {
                mbar_wait(bar(kBarQFull), qn & 1u, wctx);
                if (active && p.kmax != nullptr) {
                    kmax_row = p.kmax + (static_cast<size_t>(b) * p.H + h) * p.n_kv_tiles;
                    const uint32_t qrow = smem_base + Smem::q + x * kTileBytes + static_cast<uint32_t>(r) * 128u;
                    float sq[2];
                    rows_sumsq<kBf16, 2, static_cast<uint32_t>(kBoxBytes)>(qrow, lane, sq);
                    qn_c = sqrtf(sq[0] + sq[1]) * c * 1.001f;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(bar(kBarQEmpty));
                ++qn;
            }

            if (active && num_live > 0) {
                // key tiles [nf0, nf1) need no window / range predicate for any row of this query tile
                int nf0, nf1;
                {
                    int lo_key = p.kv_begin, hi_key = kv_end_eff - kBlockN;
                    if (p.wl >= 0) lo_key = max(lo_key, tile_r_hi - p.wl);
                    if (p.wr >= 0) hi_key = min(hi_key, tile_r_lo + p.wr - (kBlockN - 1));
                    nf0 = (lo_key + kBlockN - 1) >> 7;
                    nf1 = hi_key >= 0 ? (hi_key >> 7) + 1 : 0;
                }
                const uint8_t* flags_row = kHasBias ? p.tile_flags + b * p.n_kv_tiles : nullptr;
                int it = 0;
                for (int n = item.n0; n < item.n1; ++n) {
                    uint8_t flag = kTileFull;
                    if (kHasBias) {
                        flag = flags_row[n];
                        if (flag == kTileSkip) continue;
                    }
                    const int kv0 = n * kBlockN;
                    const float kmax_n = kmax_row != nullptr ? __ldg(kmax_row + n) : CUDART_INF_F;  // back before S is
                    mbar_wait(bar(kBarSFull + x), sp, wctx);
                    tc_fence_after();
                    uint32_t su[kHalfN];
#pragma unroll
                    for (int cb = 0; cb < kHalfN / 32; ++cb)
                        tmem_ld32(t_s + hf * kHalfN + cb * 32, reinterpret_cast<uint32_t(&)[32]>(su[cb * 32]));
                    tc_wait_ld();

                    const bool full = (n >= nf0) && (n < nf1) && (flag == kTileFull);
                    // no score of this tile can move the reference max (warp-uniform; both halves decide alike)
                    const bool skip_max = full && !__any_sync(0xffffffffu, !(qn_c * kmax_n <= m_ref + kThreshold));
                    float my_max = 0.f, mul;
                    if (skip_max) {
                        mul = c;
                    } else if (full) {
                        float mx[4];
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) mx[q4] = __uint_as_float(su[q4]);
#pragma unroll
                        for (int j = 4; j < kHalfN; j += 8) {
#pragma unroll
                            for (int q4 = 0; q4 < 4; ++q4) {
                                const int j0 = j + 2 * q4;
                                if (j0 + 1 < kHalfN)
                                    mx[q4] = max3(mx[q4], __uint_as_float(su[j0]), __uint_as_float(su[j0 + 1]));
                            }
                        }
                        my_max = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * c;  // scale > 0 (host-checked)
                        mul = c;
                    } else {
                        int lo = p.kv_begin, hi = kv_end_eff - 1;  // live columns of this row inside the tile
                        if (p.wl >= 0) lo = max(lo, row - p.wl);
                        if (p.wr >= 0) hi = min(hi, row + p.wr);
                        lo -= kv0 + hf * kHalfN;
                        hi -= kv0 + hf * kHalfN;
                        const float* brow = (kHasBias && flag == kTileMixed)
                                                ? p.bias2 + static_cast<size_t>(b) * p.bias_stride + kv0 + hf * kHalfN
                                                : nullptr;
                        float mx = -CUDART_INF_F;
#pragma unroll
                        for (int j4 = 0; j4 < kHalfN; j4 += 4) {
                            float4 bb = make_float4(0.f, 0.f, 0.f, 0.f);
                            if (kHasBias && brow != nullptr) bb = __ldg(reinterpret_cast<const float4*>(brow + j4));
                            const float bv[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int j = j4 + u;
                                const float xs = fmaf(__uint_as_float(su[j]), c, bv[u]);  // bias -inf => masked key
                                const float xm = (j >= lo && j <= hi) ? xs : -CUDART_INF_F;
                                su[j] = __float_as_uint(xm);
                                mx = fmaxf(mx, xm);
                            }
                        }
                        my_max = mx;
                        mul = 1.0f;
                    }
                    // row max over both halves (smem, double-buffered); lazy running max
                    float m_new = m_ref, alpha = 1.0f;
                    if (!skip_max) {
                        float* xrow = xrow_base + xpar * (4 * kBlockM);
                        xrow[hf * kBlockM] = my_max;
                        named_bar_sync(bar_id, kPairThreads);
                        const float tile_max = fmaxf(my_max, xrow[(hf ^ 1) * kBlockM]);
                        xpar ^= 1u;
                        m_new = (tile_max > m_ref + kThreshold) ? tile_max : m_ref;
                        alpha = (m_new == m_ref) ? 1.0f : ex2(m_ref - m_new);
                    }
                    const float neg_m = (m_new == -CUDART_INF_F) ? 0.f : -m_new;

                    // P = 2^(s*mul - m); on full tiles every kEmuEvery-th pair takes the FMA-pipe polynomial
                    uint64_t sum2 = 0;
                    const uint64_t mul2 = bc2(mul), negm2 = bc2(neg_m);
                    auto exp_store = [&](auto emu_tag) {
                        constexpr bool kEmu = decltype(emu_tag)::value;
#pragma unroll
                        for (int cb = 0; cb < kHalfN / 32; ++cb) {
                            uint32_t pk[16];
#pragma unroll
                            for (int u = 0; u < 16; ++u) {
                                float p0, p1;
                                unpk2(ffma2v(pk2(__uint_as_float(su[cb * 32 + 2 * u]), __uint_as_float(su[cb * 32 + 2 * u + 1])),
                                             mul2, negm2),
                                      p0, p1);
                                if (kEmu && (u % kEmuEvery) == kEmuEvery - 1) {
                                    exp2_poly2(p0, p1);
                                } else {
                                    p0 = ex2(p0);
                                    p1 = ex2(p1);
                                }
                                sum2 = fadd2v(sum2, pk2(p0, p1));
                                pk[u] = pack2<kBf16>(p0, p1);
                            }
                            tmem_st16(t_s + hf * kHalfN + cb * 16, pk);  // each half keeps P inside its own S columns
                        }
                    };
                    if (full)
                        exp_store(std::true_type{});
                    else
                        exp_store(std::false_type{});
                    float sum0, sum1;
                    unpk2(sum2, sum0, sum1);
                    l_run = l_run * alpha + (sum0 + sum1);
                    m_ref = m_new;
                    // O_X *= alpha where the reference max moved.  S-full of this tile was committed after P V of
                    // the previous one (in-order pipe), so O is stable until this tile's P is published.
                    if (!skip_max && it > 0 && __any_sync(0xffffffffu, alpha != 1.0f)) rescale_o_rows_d128(t_o, alpha);
                    tc_wait_st();
                    tc_fence_before();
                    mbar_arrive(bar(kBarPFull + x));
                    ++it;
                    sp ^= 1u;
                }
            }  // (a tile B that sits the item out -- S ends inside tile A -- moves none of its barriers)

            if (active) {
                // ---------------- epilogue ----------------
                float* lrow = xrow_base;
                named_bar_sync(bar_id, kPairThreads);  // all max-exchange reads of the last tile are done
                lrow[hf * kBlockM] = l_run;
                named_bar_sync(bar_id, kPairThreads);
                const float l_tot = l_run + lrow[(hf ^ 1) * kBlockM];
                named_bar_sync(bar_id, kPairThreads);  // reads done before the next item reuses the slot
                if (num_live > 0) {
                    mbar_wait(bar(kBarOFull + x), oi & 1u, wctx);
                    tc_fence_after();
                }
                const size_t ridx = (static_cast<size_t>(b) * p.H + h) * p.S + row;
                if (item.kind == kItemPublish) {
                    // this CTA owns only the leading key tiles of the pair: un-normalised partial for CTA blockIdx.x + 1
                    const size_t slot = (static_cast<size_t>(blockIdx.x) * 2 + x) * kBlockM + r;
#pragma unroll
                    for (int cb = 0; cb < 2; ++cb) {
                        uint32_t o[32];
                        if (num_live > 0) {
                            tmem_ld32(t_o + cb * 32, o);
                            tc_wait_ld();
                        } else {
#pragma unroll
                            for (int u = 0; u < 32; ++u) o[u] = 0u;
                        }
                        float* dst = p.part_o + slot * kD + hf * (kD / 2) + cb * 32;  // 128-byte aligned
#pragma unroll
                        for (int u = 0; u < 4; ++u) st_global_v8(dst + 8 * u, reinterpret_cast<const uint32_t(&)[8]>(o[8 * u]));
                    }
                    if (hf == 0) {
                        p.part_ml[slot * 2] = m_ref;
                        p.part_ml[slot * 2 + 1] = l_tot;
                    }
                    __threadfence();
                    __syncwarp();
                    if (lane == 0) st_release_gpu(p.part_flag + blockIdx.x * kNumSoftmaxWarps + warp, 1);
                } else {
                    float l_fin = l_tot, w1 = 1.0f, w2 = 0.0f;
                    const float* part_src = nullptr;
                    if (item.kind == kItemMerge) {
                        // the partial CTA blockIdx.x - 1 published for the same rows at the START of its slice (its
                        // half-0 warp of the same quadrant wrote m and l, this warp's twin wrote the columns); own part
                        // first: fixed order, deterministic.  Only ever a wait for a lower-indexed CTA.
                        const int* flag_o = p.part_flag + (blockIdx.x - 1) * kNumSoftmaxWarps + warp;
                        const int* flag_ml = p.part_flag + (blockIdx.x - 1) * kNumSoftmaxWarps + (warp & ~4);
                        uint32_t spins = 0;
                        while (ld_acquire_gpu(flag_o) == 0 || ld_acquire_gpu(flag_ml) == 0) {
                            if (!wait_slow_path(spins, wctx, kStatusPeerTimeout)) break;
                        }
                        const size_t slot = (static_cast<size_t>(blockIdx.x - 1) * 2 + x) * kBlockM + r;
                        const float m2 = __ldcg(p.part_ml + slot * 2);
                        const float l2 = __ldcg(p.part_ml + slot * 2 + 1);
                        const float ms = fmaxf(m_ref, m2);
                        w1 = (m_ref == -CUDART_INF_F) ? 0.f : ex2(m_ref - ms);
                        w2 = (m2 == -CUDART_INF_F) ? 0.f : ex2(m2 - ms);
                        l_fin = l_tot * w1 + l2 * w2;
                        m_ref = ms;
                        part_src = p.part_o + slot * kD + hf * (kD / 2);
                    }
                    const float inv = l_fin > 0.f ? 1.0f / l_fin : 0.f;
                    if (p.o_partial != nullptr && hf == 0 && row < p.S) {
                        p.m_partial[ridx] = m_ref;
                        p.l_partial[ridx] = l_fin;
                    }
#pragma unroll
                    for (int cb = 0; cb < 2; ++cb) {
                        const int col0 = hf * (kD / 2) + cb * 32;
                        float o[32];
                        if (num_live > 0) {
                            tmem_ld32(t_o + cb * 32, reinterpret_cast<uint32_t(&)[32]>(o));
                            tc_wait_ld();
                        } else {
#pragma unroll
                            for (int u = 0; u < 32; ++u) o[u] = 0.f;
                        }
                        if (part_src != nullptr) {
                            const float4* src = reinterpret_cast<const float4*>(part_src + cb * 32);
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                const float4 t = __ldcg(src + u);
                                o[4 * u] = o[4 * u] * w1 + t.x * w2;
                                o[4 * u + 1] = o[4 * u + 1] * w1 + t.y * w2;
                                o[4 * u + 2] = o[4 * u + 2] * w1 + t.z * w2;
                                o[4 * u + 3] = o[4 * u + 3] * w1 + t.w * w2;
                            }
                        }
                        if (row >= p.S) continue;
                        if (p.o_partial != nullptr) {
                            float4* dst = reinterpret_cast<float4*>(p.o_partial + ridx * kD + col0);
#pragma unroll
                            for (int u = 0; u < 8; ++u) dst[u] = make_float4(o[4 * u], o[4 * u + 1], o[4 * u + 2], o[4 * u + 3]);
                        } else {
                            const size_t off = static_cast<size_t>(b) * p.o_sb + static_cast<size_t>(h) * p.o_sh +
                                               static_cast<size_t>(row) * p.o_ss + col0;
                            if (p.out_dtype == 2) {
                                float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.out) + off);
#pragma unroll
                                for (int u = 0; u < 8; ++u)
                                    dst[u] = make_float4(o[4 * u] * inv, o[4 * u + 1] * inv, o[4 * u + 2] * inv, o[4 * u + 3] * inv);
                            } else {
                                uint4* dst = reinterpret_cast<uint4*>(static_cast<uint16_t*>(p.out) + off);
#pragma unroll
                                for (int u = 0; u < 4; ++u) {
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
                    if (item.kind == kItemMerge) {
                        // the flags are left as they were found (zero): this warp and its twin are their only readers
                        named_bar_sync(bar_id, kPairThreads);
                        if (lane == 0) p.part_flag[(blockIdx.x - 1) * kNumSoftmaxWarps + warp] = 0;
                    }
                }
                if (num_live > 0) {
                    // the next item's first P V overwrites O: every thread of the tile has read its columns
                    tc_fence_before();
                    ++oi;
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

bool fa_fwd_sm100_d128_available() { return true; }

size_t fa_fwd_sm100_d128_smem_bytes() { return Smem::xchg + Smem::xchg_bytes + 1024; }

cudaError_t launch_fa_fwd_sm100_d128(const CUtensorMap& tmq, const CUtensorMap& tmk, const CUtensorMap& tmv,
                                     const FaParams& p, bool bf16, int grid, cudaStream_t stream) {
    const bool has_bias = p.tile_flags != nullptr;
    void (*kern)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const FaParams) =
        bf16 ? (has_bias ? fa_fwd_sm100_d128_kernel<true, true> : fa_fwd_sm100_d128_kernel<true, false>)
             : (has_bias ? fa_fwd_sm100_d128_kernel<false, true> : fa_fwd_sm100_d128_kernel<false, false>);
    const size_t smem = fa_fwd_sm100_d128_smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreads, smem, stream>>>(tmq, tmk, tmv, p);
    return cudaGetLastError();
}

}  // namespace rf
