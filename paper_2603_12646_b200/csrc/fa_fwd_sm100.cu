// fa_fwd_sm100.cu -- FusedFlashAttention forward for sm_100a (B200), head_dim 64.
//
// (head_dim 32 runs through the same kernel zero-padded to 64: see FaParams::d.)
// Semantics: reference routefast::flash_attention (proj/core/src/attention.cpp:106-213):
// non-causal, additive padding bias (masked at <= -30000), optional two-sided sliding window,
// online softmax, rows without a live key -> 0.  No S x S tensor is ever materialised.
//
// Hardware mapping (one CTA per SM, 640 threads, two 128-row query tiles "A"/"B" ping-pong):
//   warp 16     TMA producer: Q per work item, K/V 128-key tiles through smem rings
//               (cp.async.bulk.tensor, 128B swizzle, mbarrier complete_tx)
//   warp 17     UMMA issuer: S_X = Q_X K^T  (tcgen05.mma SS, M128 N128 K16 x4)
//                            O_X += P_X V   (tcgen05.mma TS, M128 N64  K16 x8)
//               accumulators in TMEM: three rotating S buffers, cols [0,384) (tile g = 2*t + X of
//               the A,B,A,B,... sequence uses buffer g % 3, so the next S of a warpgroup is computed
//               while it is still busy with the current one), O_A [384,448), O_B [448,512);
//               P (bf16) aliases its S buffer: keys [0,64) in columns [0,32), keys [64,128) in [64,96).
//   warps 0-7   softmax for tile A, warps 8-15 for tile B.  Two threads share one query row
//               (key columns [0,64) and [64,128) of the tile; tcgen05.ld 32x32b), so four softmax
//               warps per SM sub-partition hide each other's MUFU/ALU latencies.  The two halves
//               exchange their row max through shared memory (one 64-thread named barrier per
//               tile); row sums stay per-thread until the epilogue.  exp2 with the scale folded in,
//               packed f32x2 math, lazy rescale of O (only when the running max grows by > 2^20 with
//               bf16 P, 2^14 with f16 P).  Row-max skip: when c |q_row| max_j |k_j| cannot exceed the reference max by more than that slack, the tile's
//               max pass, the exchange and its barrier are skipped (see the softmax loop).
//               setmaxnreg moves registers from the producer/MMA warpgroup to the softmax ones.
//               |q_row| is taken from the Q tile in shared memory by the softmax thread itself; the largest |k_j| of
//               every key tile comes from a pre-pass over K (fa_aux.cu: k_tile_norms_kernel, 4 B per (head, tile)).
//               (Taking the key norms in the kernel too -- two idle warps reading each K tile as it lands -- was
//               measured: 224 us against 212 us at 8K, the extra shared-memory reads and issue slots cost more than
//               the 3 us pre-pass.)
//
// Work distribution.  A work item is (query-tile pair, key-tile range).
//   mode 0: one item per CTA (grid = number of pairs); used when the pairs fit one wave and for split-KV.
//   mode 1: persistent, statically balanced: the flat (pair x key-tile) iteration space is cut
//           into gridDim.x equal contiguous slices, each walked from its LAST pair to its first.
//           A pair cut between CTA c (its leading key tiles: c's first item) and CTA c+1 (its
//           trailing key tiles: c+1's last item) is merged in-kernel: c publishes an un-normalised
//           partial (O, m, l) to the workspace right away, c+1 combines it with its own in a fixed
//           order at the very end.  A CTA therefore only ever waits for a LOWER-indexed CTA (dispatched
//           no later than itself), so the chain cannot starve when other work shares the GPU.  This
//           removes the wave quantisation of the dense global layers (e.g. 384 pairs on 148 SMs) and
//           stays run-to-run deterministic.
//   mode 2: persistent, whole pairs dealt round-robin (pair c, c + gridDim.x, ...): batches whose last
//           partial round wastes little (fa_api.cu).  CTAs that run together work on neighbouring pairs (K/V of a few heads stay in
//           L2), and sequences of different padded lengths spread over all CTAs.
// Narrow sliding windows (wl + wr <= 127) do not come here: fa_fwd_sm100_local.cu.
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

constexpr int kHeadDim = 64;
constexpr int kStagesK = 4;                         // K ring depth (K runs two tiles ahead of V)
constexpr int kStagesV = 3;                         // V ring depth
constexpr int kSBufs = 3;                           // rotating S/P accumulators in TMEM
constexpr int kTileBytes = kBlockN * kHeadDim * 2;  // 16 KiB: one 128 x 64 16-bit tile
constexpr int kNumSoftmaxWarps = 16;
constexpr int kProducerWarp = 16;
constexpr int kMmaWarp = 17;
constexpr int kThreads = 640;        // 5 warpgroups: 4 softmax + 1 (producer, MMA, 2 idle warps)
constexpr int kHalfN = kBlockN / 2;  // key columns per softmax thread
constexpr int kRegsSoftmax = 112;
#ifndef RF_FA_EMU_EVERY
#define RF_FA_EMU_EVERY 5  // 3 of a block's 16 pairs; 4 (a quarter) is 0.8 % slower at 8K, 3 and 6 slower still (same-box A/B)
#endif
constexpr int kEmuEvery = RF_FA_EMU_EVERY;  // every n-th element pair uses the FMA-pipe exp2 (0 = MUFU only)
constexpr int kRegsOther = 32;       // 128*32 + 512*112 == 640*96: the CTA register pool balances exactly
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColS = 0;    // + 128 * buffer
constexpr uint32_t kColO = 384;  // + 64 * X
// Lazy reference max, log2 units: P may reach 2^threshold before a rescale is forced.  bf16 P has the f32
// exponent range (and l, O accumulate in f32), so the slack can be wide -- which also lets the row-max skip
// test pass for looser Cauchy-Schwarz bounds; f16 P must stay below 65504 = 2^16.
constexpr float kRescaleThresholdBf16 = 20.0f;
constexpr float kRescaleThresholdF16 = 14.0f;
// Ping-pong of the exponential phases: on every SM sub-partition the two warps of tile A and the two
// warps of tile B take strict turns on the MUFU pipe (A0, B0, A1, B1, ...), so that one tile's
// max / exchange / TMEM traffic always overlaps the other tile's exponentials instead of all four
// warps convoying through the same phase.
#ifndef RF_FA_PINGPONG
#define RF_FA_PINGPONG 0
#endif
constexpr bool kPingPong = RF_FA_PINGPONG != 0;
// Developer build only (-DRF_FA_TRACE=1): softmax warps of CTA 0 stamp the SM clock at their phase
// boundaries into the debug_scores buffer, [16 warps][64 tiles][8 stamps] u32 (tools/trace_phases.py).
#ifndef RF_FA_TRACE
#define RF_FA_TRACE 0
#endif
// Developer build only (-DRF_FA_MMAONLY=1): the softmax warps skip their work (results are garbage);
// what remains is the TMA + UMMA pipeline, i.e. the tensor-pipe floor of this tiling.
// Developer build only (-DRF_FA_NOEXP=1, results are garbage): the softmax warps keep their TMEM traffic (S loads, P
// stores), barriers and the scale / sum / pack instructions but take no exponential -- what the kernel would cost
// if exponentials were free (171 us at 8K against 124 us for RF_FA_MMAONLY and 207 us shipped).
#ifndef RF_FA_NOEXP
#define RF_FA_NOEXP 0
#endif
#ifndef RF_FA_MMAONLY
#define RF_FA_MMAONLY 0
#endif
// 1: the softmax warps check the V(i) / K(i+2) TMA barriers (while they wait for S) so that the UMMA
// warp's steady-state loop has two barrier waits per key tile; 0: the UMMA warp waits for them itself.
#ifndef RF_FA_VK_IN_SOFTMAX
#define RF_FA_VK_IN_SOFTMAX 0
#endif
#ifndef RF_FA_TRACE_TILES
#define RF_FA_TRACE_TILES 64  // key tiles of CTA 0 the trace buffer holds per warp
#endif
#if RF_FA_TRACE
#define RF_STAMP(slot)                                                                               \
    do {                                                                                             \
        if (blockIdx.x == 0 && lane == 0 && trace_n < RF_FA_TRACE_TILES && p.debug_scores != nullptr)               \
            reinterpret_cast<uint32_t*>(p.debug_scores)[(warp * RF_FA_TRACE_TILES + trace_n) * 8 + (slot)] = clock(); \
    } while (0)
#else
#define RF_STAMP(slot) do { } while (0)
#endif

// dynamic shared memory map (offsets from a 1024B-aligned base)
struct Smem {
    static constexpr uint32_t q = 0;                                   // 2 tiles
    static constexpr uint32_t k = q + 2 * kTileBytes;                  // kStagesK tiles
    static constexpr uint32_t v = k + kStagesK * kTileBytes;           // kStagesV tiles
    static constexpr uint32_t bars = v + kStagesV * kTileBytes;        // barrier block
    static constexpr uint32_t bar_bytes = 512;
    static constexpr uint32_t xchg = bars + bar_bytes;                 // row-max exchange: [2 parity][2 tile][2 half][128] f32
    static constexpr uint32_t xchg_bytes = 2 * 2 * 2 * kBlockM * 4;
};
// barrier indices inside the barrier block (8 bytes each)
enum : uint32_t {
    kBarQFull = 0,
    kBarQEmpty = 1,
    kBarKFull = 2,                       // [kStagesK]
    kBarKEmpty = kBarKFull + kStagesK,   // [kStagesK]
    kBarVFull = kBarKEmpty + kStagesK,   // [kStagesV]
    kBarVEmpty = kBarVFull + kStagesV,   // [kStagesV]
    kBarSFull = kBarVEmpty + kStagesV,   // [kSBufs] one per S buffer: no phase can be skipped
    kBarPFull = kBarSFull + kSBufs,      // [kSBufs]
    kBarOFull = kBarPFull + kSBufs,      // [2]
    kBarTurn = kBarOFull + 2,            // [2 tiles][4 quadrants] exp-phase turn of (tile, SM sub-partition)
    kNumBars = kBarTurn + 8,
};
constexpr uint32_t kTmemSlotOff = kNumBars * 8;                     // u32: TMEM base address
constexpr uint32_t kWaitBlockOff = (kTmemSlotOff + 8 + 15) & ~15u;  // 16 bytes: abort word + status pointer (ptx.cuh)
static_assert(kWaitBlockOff + 16 <= Smem::bar_bytes, "barrier block too small");

// kItemPublish: the CTA owns the LEADING key tiles of a pair cut at the end of its slice: processed first, partial
// published for the next CTA.  kItemMerge: it owns the TRAILING key tiles of the pair its slice starts in:
// processed last, merged with the partial of the previous CTA.
enum : int { kItemFull = 0, kItemPublish = 1, kItemMerge = 2 };

// One unit of work of a CTA: a query-tile pair and a range of key tiles.
struct Item {
    int b, h, q0;
    int n0, n1;    // key tiles [n0, n1)
    int num_live;  // tiles in the range that are not fully padded
    int kind;
    bool has_b;
};

struct Sched {
    long long t, t_end;  // mode 1: the unprocessed part [t, t_end) of the CTA's slice, consumed from the END
    bool done;           // mode 0
};

template <bool kHasBias>
__device__ __forceinline__ bool tile_live(const FaParams& p, int b, int n) {
    return !kHasBias || p.tile_flags[b * p.n_kv_tiles + n] != kTileSkip;
}

__device__ __forceinline__ void sched_init(const FaParams& p, Sched& s) {
    s.done = false;
    if (p.sched_mode == 1) {
        const long long total = static_cast<long long>(p.total_pairs) * p.tiles_per_pair;
        s.t = total * blockIdx.x / gridDim.x;
        s.t_end = total * (blockIdx.x + 1) / gridDim.x;
    } else {
        s.t = s.t_end = 0;
    }
}

template <bool kHasBias>
__device__ __forceinline__ bool next_item(const FaParams& p, Sched& s, Item& it) {
    int pair_lin, k0 = 0, k1 = 0x7fffffff;
    if (p.sched_mode == 1) {
        // The slice is walked from its last pair to its first, so that the piece shared with the NEXT CTA is
        // published before anything else and the piece shared with the PREVIOUS CTA is merged last: a CTA only
        // ever waits for a lower-indexed -- i.e. earlier-dispatched -- CTA, and that one published long ago.
        if (s.t >= s.t_end) return false;
        const int K = p.tiles_per_pair;  // virtual key tiles per pair (upper bound of any pair's range)
        pair_lin = static_cast<int>((s.t_end - 1) / K);
        const long long pair_start = static_cast<long long>(pair_lin) * K;
        k0 = static_cast<int>(max(s.t, pair_start) - pair_start);
        k1 = static_cast<int>(s.t_end - pair_start);
        s.t_end = pair_start + k0;
        it.kind = k0 > 0 ? kItemMerge : (k1 < K ? kItemPublish : kItemFull);
    } else if (p.sched_mode == 2) {
        // whole pairs dealt round-robin: pair blockIdx.x, blockIdx.x + gridDim.x, ...  (s.t counts items)
        const long long lin = blockIdx.x + s.t * gridDim.x;
        if (lin >= p.total_pairs) return false;
        ++s.t;
        pair_lin = static_cast<int>(lin);
        it.kind = kItemFull;
    } else {
        if (s.done) return false;
        s.done = true;
        pair_lin = blockIdx.x;
        it.kind = kItemFull;
    }
    const int px = pair_lin % p.pairs_per_head;
    const int bh = pair_lin / p.pairs_per_head;
    it.h = bh % p.H;
    it.b = bh / p.H;
    it.q0 = px * kRowsPerCta;
    it.has_b = it.q0 + kBlockM < p.S;
    // key-tile range of this pair (union over its rows of window and split range) ...
    const int rows_end = min(it.q0 + kRowsPerCta, p.S);
    int j_lo = p.kv_begin, j_hi = p.kv_end;
    if (p.wl >= 0) j_lo = max(j_lo, it.q0 - p.wl);
    if (p.wr >= 0) j_hi = min(j_hi, rows_end + p.wr);
    const int pn0 = j_lo >> 7;
    const int pn1 = (j_hi > j_lo) ? ((j_hi + kBlockN - 1) >> 7) : pn0;
    // ... cut to this item's slice of it (mode 1: virtual tile v is real tile pn0 + v; slices past
    // the pair's last tile are empty)
    it.n0 = min(pn0 + k0, pn1);
    it.n1 = (k1 >= pn1 - pn0) ? pn1 : pn0 + k1;
    it.num_live = 0;
    for (int n = it.n0; n < it.n1; ++n) it.num_live += tile_live<kHasBias>(p, it.b, n) ? 1 : 0;
    return true;
}

__device__ __forceinline__ int ld_acquire_gpu(const int* ptr) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int* ptr, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(ptr), "r"(v) : "memory");
}

// O rows (32 columns of this thread's lane) *= alpha.  QK^T runs ahead of PV (rotating S buffers),
// so "S ready" does not imply that PV of the previous tile has finished.  The V-empty barrier of
// that tile is committed after both of its PVs: wait for its phase first (it is at most one phase
// away, so the parity wait is exact).
__device__ __noinline__ void rescale_o_rows(uint32_t t_o, float alpha, uint32_t v_empty_bar, uint32_t parity,
                                            WaitCtx wctx) {
    mbar_wait(v_empty_bar, parity, wctx);
    tc_fence_after();
    uint32_t o[32];
    tmem_ld32(t_o, o);
    tc_wait_ld();
#pragma unroll
    for (int u = 0; u < 32; u += 2) {
        float a0 = __uint_as_float(o[u]), a1 = __uint_as_float(o[u + 1]);
        fmul2(a0, a1, alpha);
        o[u] = __float_as_uint(a0);
        o[u + 1] = __float_as_uint(a1);
    }
    tmem_st32(t_o, o);
    tc_wait_st();
}

template <bool kBf16, bool kHasBias>
__global__ void __launch_bounds__(kThreads, 1)
fa_fwd_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const FaParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* smem_gen = smem_raw + (smem_base - smem_u32(smem_raw));
    asm volatile("mov.u32 %0, %0;" : "+r"(smem_base));  // keep in a register: do not rematerialise
    const uint32_t bars = smem_base + Smem::bars;
    auto bar = [&](uint32_t i) { return bars + 8u * i; };
    volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(smem_gen + Smem::bars + kTmemSlotOff);
    const WaitCtx wctx{bars + kWaitBlockOff};

    const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);  // warp-uniform by construction: lets roles, buffer indices and TMEM addresses live in uniform registers
    const int lane = threadIdx.x & 31;
#if RF_FA_TRACE
    // kernel-level stamps of CTA 0 in the row of (idle) warp 18: 0 entry, 1 prologue done, 2 dependencies resolved, 3 teardown
#define RF_KSTAMP(slot)                                                                                          \
    do {                                                                                                         \
        if (blockIdx.x == 0 && threadIdx.x == 18 * 32 && p.debug_scores != nullptr)                              \
            reinterpret_cast<uint32_t*>(p.debug_scores)[(18 * RF_FA_TRACE_TILES) * 8 + (slot)] = clock();        \
    } while (0)
#else
#define RF_KSTAMP(slot) do { } while (0)
#endif
    RF_KSTAMP(0);

    // ---------------- prologue ----------------
    if (warp == kProducerWarp && lane == 0) {
        prefetch_tensormap(&tm_q);
        prefetch_tensormap(&tm_k);
        prefetch_tensormap(&tm_v);
        mbar_init(bar(kBarQFull), 1);
        // Q is also read by every softmax warp (row norms): their arrivals join the UMMA commit on its empty barrier
        mbar_init(bar(kBarQEmpty), 1 + kNumSoftmaxWarps);
        for (int s = 0; s < kStagesK; ++s) {
            mbar_init(bar(kBarKFull + s), 1);
            mbar_init(bar(kBarKEmpty + s), 1);
        }
        for (int s = 0; s < kStagesV; ++s) {
            mbar_init(bar(kBarVFull + s), 1);
            mbar_init(bar(kBarVEmpty + s), 1);
        }
        for (int s = 0; s < kSBufs; ++s) {
            mbar_init(bar(kBarSFull + s), 1);
            mbar_init(bar(kBarPFull + s), 2 * kBlockM);
        }
        for (int x = 0; x < 2; ++x) mbar_init(bar(kBarOFull + x), 1);
        for (int i = 0; i < 8; ++i) mbar_init(bar(kBarTurn + i), 64);  // both warps of the other tile arrive
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
    RF_KSTAMP(1);
    // Programmatic dependent launch: everything above overlapped the tail of the previous kernel in the stream
    // when that one triggers its dependents early; its results are visible after this.  A no-op when the kernel
    // was launched normally.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    RF_KSTAMP(2);

    Sched sched;
    sched_init(p, sched);
    Item item;

    static_assert(128 * kRegsOther + 512 * kRegsSoftmax <= kThreads * 96, "setmaxnreg pool must balance");
    if (warp >= kNumSoftmaxWarps) setmaxnreg_dec<kRegsOther>();

    if (warp == kProducerWarp) {
        // =============================== TMA producer ===============================
        // warp-uniform control flow; only the TMA / expect_tx instructions are predicated
        const bool leader = elect_one() != 0;
        uint32_t qi = 0;  // items with work so far (Q barrier phase)
        uint32_t kc = 0;  // K tiles loaded so far (ring position)
        uint32_t vc = 0;  // V tiles loaded so far
        while (next_item<kHasBias>(p, sched, item)) {
            if (item.num_live == 0) continue;
            const int b = item.b, h = item.h;
            mbar_wait(bar(kBarQEmpty), (qi & 1) ^ 1, wctx);
            if (leader) {
                mbar_arrive_expect_tx(bar(kBarQFull), item.has_b ? 2 * kTileBytes : kTileBytes);
                tma_load_4d(smem_base + Smem::q, &tm_q, bar(kBarQFull), 0, item.q0, h, b);
                if (item.has_b)
                    tma_load_4d(smem_base + Smem::q + kTileBytes, &tm_q, bar(kBarQFull), 0, item.q0 + kBlockM, h, b);
            }
            __syncwarp();
            ++qi;
            // K runs two tiles ahead of V: QK^T of tile t+2 is issued while tile t is in softmax
            auto load_k = [&](int n) {
                const uint32_t st = kc % kStagesK;
                mbar_wait(bar(kBarKEmpty + st), ((kc / kStagesK) & 1) ^ 1, wctx);
                if (leader) {
                    mbar_arrive_expect_tx(bar(kBarKFull + st), kTileBytes);
                    tma_load_4d(smem_base + Smem::k + st * kTileBytes, &tm_k, bar(kBarKFull + st), 0, n * kBlockN, h, b);
                }
                __syncwarp();
                ++kc;
            };
            auto load_v = [&](int n) {
                const uint32_t st = vc % kStagesV;
                mbar_wait(bar(kBarVEmpty + st), ((vc / kStagesV) & 1) ^ 1, wctx);
                if (leader) {
                    mbar_arrive_expect_tx(bar(kBarVFull + st), kTileBytes);
                    tma_load_4d(smem_base + Smem::v + st * kTileBytes, &tm_v, bar(kBarVFull + st), 0, n * kBlockN, h, b);
                }
                __syncwarp();
                ++vc;
            };
            auto next_live = [&](int n) {
                while (n < item.n1 && !tile_live<kHasBias>(p, b, n)) ++n;
                return n;
            };
            int nk = next_live(item.n0);
            for (int pre = 0; pre < 2 && nk < item.n1; ++pre) {
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
        // The whole warp runs this loop with warp-uniform values (so descriptors and addresses
        // live in uniform registers); only the tcgen05 instructions themselves are predicated on
        // one elected lane.  A divergent `if (lane == 0)` around the loop would make ptxas wrap
        // every UTCHMMA in an ELECT / R2UR waterfall loop, which puts ~16 instructions per MMA on
        // the critical path.
        const bool leader = elect_one() != 0;
        constexpr uint32_t fmt = kBf16 ? 1u : 0u;
        constexpr uint32_t idesc_qk = make_idesc_f16(fmt, 0, 0, kBlockM, kBlockN);
        constexpr uint32_t idesc_pv = make_idesc_f16(fmt, 0, 1, kBlockM, kHeadDim);
        // descriptor high words are constants; the low word is (address >> 4) | LBO field
        constexpr uint32_t kDescHi = (1024u >> 4) | (1u << 14) | (kSwizzle128B << 29);  // SBO, version, swizzle
        constexpr uint32_t kLboK = (16u >> 4) << 16;                                    // K-major operands
        constexpr uint32_t kLboV = (static_cast<uint32_t>(kTileBytes) >> 4) << 16;      // MN-major V
        const uint32_t sb16 = smem_base >> 4;
        auto desc = [&](uint32_t lo) { return (static_cast<uint64_t>(kDescHi) << 32) | lo; };
        auto commit = [&](uint32_t b_) {
            if (leader) tc_commit(b_);
            __syncwarp();
        };

        // Loop state is kept incremental (no divisions) and small: this warp runs on 32 registers.
        // K and V tiles live at the same ring positions in every item (kc == vc == tiles so far).
        uint32_t qi = 0;        // items with work so far (Q barrier phase)
        uint32_t kc = 0;        // key tiles consumed in earlier items (K ring position, parity)
        uint32_t ks = 0;        // K ring stage of the item's tile 0
        uint32_t vs = 0;        // V ring stage of the item's tile 0
        uint32_t vp = 0;        // ... and the phase parity of that use
        uint32_t sa = 0;        // S buffer of tile A of the item's key tile 0 (tile B: sa + 1 mod 3)
        uint32_t par_bits = 0;  // bit s = phase parity of the next use of S buffer s (S-full / P-full barriers)
        auto inc_mod = [](uint32_t v, uint32_t add, uint32_t mod) {
            v += add;
            return v >= mod ? v - mod : v;
        };
        // pins a prepared operand word in a register before a barrier wait (keeps the descriptor
        // arithmetic off the wait -> first UMMA critical path)
        auto pin = [](uint32_t& v) { asm volatile("" : "+r"(v)); };
        const uint32_t q_lo = kLboK | (sb16 + Smem::q / 16);
        const uint32_t k_lo = kLboK | (sb16 + Smem::k / 16);
        const uint32_t v_lo = kLboV | (sb16 + Smem::v / 16);
        constexpr uint32_t kTile16 = kTileBytes / 16;

        while (next_item<kHasBias>(p, sched, item)) {
            const int num_live = item.num_live;
            if (num_live == 0) continue;
            const bool has_b = item.has_b;

            // S = Q_X * K^T : both operands K-major (head dim contiguous), 128B swizzle,
            // 8-row core-matrix groups 1024 B apart; a K=16 step advances 32 B inside the atom.
            auto issue_qk = [&](uint32_t x, uint32_t kstage, uint32_t buf) {
                const uint32_t qlo = q_lo + x * kTile16;
                const uint32_t klo = k_lo + kstage * kTile16;
                const uint32_t td = tmem_base + kColS + buf * kBlockN;
                if (leader) {
#pragma unroll
                    for (int kk = 0; kk < kHeadDim / 16; ++kk)
                        mma_ss(td, desc(qlo + kk * 2), desc(klo + kk * 2), idesc_qk, kk > 0 ? 1u : 0u);
                    tc_commit(bar(kBarSFull + buf));
                }
                __syncwarp();
            };
            // O_X += P * V : B operand V is [key][d] with d contiguous = MN-major, 128B swizzle;
            // 8-key groups 1024 B apart (SBO); a K=16 step advances 16 keys = 2048 B.
            // A = P from TMEM: 16 bf16 per row per step = 8 packed 32-bit columns; keys [0,64) sit in S columns
            // [0,32), keys [64,128) in S columns [64,96) (each softmax half writes P over its own scores only).
            auto issue_pv = [&](uint32_t x, uint32_t vlo, uint32_t ta, uint32_t acc0) {
                const uint32_t td = tmem_base + kColO + x * kHeadDim;
                if (leader) {
#pragma unroll
                    for (int kk = 0; kk < kBlockN / 16; ++kk)
                        mma_ts(td, ta + kk * 8 + (kk >= 4 ? 32 : 0), desc(vlo + kk * 128), idesc_pv, kk > 0 ? 1u : acc0);
                }
                __syncwarp();
            };
            // K/V-full barriers are waited for by THIS warp only for the item's first two key tiles;
            // in the steady state the softmax warps check them before they publish P (see there), so
            // that this loop has exactly two waits per key tile.
            auto wait_k = [&](uint32_t i) {
                mbar_wait(bar(kBarKFull + ((kc + i) & (kStagesK - 1))), ((kc + i) / kStagesK) & 1, wctx);
                tc_fence_after();
            };
            static_assert((kStagesK & (kStagesK - 1)) == 0, "K ring depth must be a power of two");
            // every QK^T that reads the K tile in `kstage` has been issued; the item's last one also frees Q
            auto release_k = [&](uint32_t kstage, bool last_of_item) {
                commit(bar(kBarKEmpty + kstage));
                if (last_of_item) commit(bar(kBarQEmpty));
            };

            // prologue: S_A(0), S_B(0), and already S_A(1) into the third buffer
            uint32_t buf_a = sa;                        // S buffer of A(i); B(i) uses the next one
            uint32_t ks1 = inc_mod(ks, 1, kStagesK);    // K stage of tile i+1
            uint32_t vsi = vs, vpi = vp;                // V stage of tile i and its phase parity
            mbar_wait(bar(kBarQFull), qi & 1, wctx);
            wait_k(0);
            issue_qk(0, ks, buf_a);
            if (has_b) issue_qk(1, ks, inc_mod(buf_a, 1, kSBufs));
            release_k(ks, num_live == 1);
            if (num_live > 1) {
                wait_k(1);
                issue_qk(0, ks1, inc_mod(buf_a, 2, kSBufs));
                if (!has_b) release_k(ks1, num_live == 2);
            }

            for (int i = 0; i < num_live; ++i) {
                const bool last = i + 1 == num_live;
                const uint32_t buf_b = inc_mod(buf_a, 1, kSBufs), buf_c = inc_mod(buf_a, 2, kSBufs);
                const uint32_t ks2 = inc_mod(ks1, 1, kStagesK);
#if RF_FA_TRACE
                const int trace_n = i;
#endif
                RF_STAMP(0);
                // ---- P_A(i) ready: O_A += P_A V; its S buffer is then free for S_B(i+1) ----
                uint32_t vlo = v_lo + vsi * kTile16;
                uint32_t ta = tmem_base + kColS + buf_a * kBlockN;
                pin(vlo);
                pin(ta);
                RF_STAMP(1);
                if (!RF_FA_VK_IN_SOFTMAX)  // V(i) was requested tiles ago: check it in the shadow of the P wait
                    mbar_wait2(bar(kBarVFull + vsi), vpi, bar(kBarPFull + buf_a), (par_bits >> buf_a) & 1u, wctx);
                else
                    mbar_wait(bar(kBarPFull + buf_a), (par_bits >> buf_a) & 1u, wctx);  // implies V(i) has landed
                tc_fence_after();
                RF_STAMP(2);
                issue_pv(0, vlo, ta, i > 0 ? 1u : 0u);
                if (last) commit(bar(kBarOFull + 0));
                if (has_b) {
                    if (!last) {
                        issue_qk(1, ks1, buf_a);  // K(i+1) was waited for when S_A(i+1) was issued
                        release_k(ks1, i + 2 == num_live);
                    }
                    RF_STAMP(3);
                    // ---- P_B(i) ready: O_B += P_B V; its S buffer is then free for S_A(i+2) ----
                    ta = tmem_base + kColS + buf_b * kBlockN;
                    pin(ta);
                    if (!RF_FA_VK_IN_SOFTMAX && i + 2 < num_live)  // K(i+2) for the S_A(i+2) issued right after
                        mbar_wait2(bar(kBarKFull + ks2), ((kc + i + 2) / kStagesK) & 1,
                                   bar(kBarPFull + buf_b), (par_bits >> buf_b) & 1u, wctx);
                    else
                        mbar_wait(bar(kBarPFull + buf_b), (par_bits >> buf_b) & 1u, wctx);  // implies K(i+2) has landed
                    tc_fence_after();
                    RF_STAMP(4);
                    issue_pv(1, vlo, ta, i > 0 ? 1u : 0u);
                    if (last) commit(bar(kBarOFull + 1));
                }
                par_bits ^= (1u << buf_a) ^ (has_b ? (1u << buf_b) : 0u);
                commit(bar(kBarVEmpty + vsi));
                RF_STAMP(5);
                if (i + 2 < num_live) {
                    if (!RF_FA_VK_IN_SOFTMAX && !has_b) wait_k(i + 2);
                    RF_STAMP(6);
                    issue_qk(0, ks2, buf_b);
                    if (!has_b) release_k(ks2, i + 3 == num_live);
                }
                RF_STAMP(7);
                buf_a = buf_c;
                ks1 = ks2;
                if (++vsi == kStagesV) {
                    vsi = 0;
                    vpi ^= 1u;
                }
            }
            // ring positions of the next item's tile 0
            kc += num_live;
            ks = (ks + num_live) & (kStagesK - 1);
            vs = vsi;
            vp = vpi;
            sa = buf_a;
            ++qi;
        }
    } else if (warp < kNumSoftmaxWarps) {
        // =============================== softmax / epilogue ===============================
        setmaxnreg_inc<kRegsSoftmax>();
        const int x = warp >> 3;               // 0 = tile A, 1 = tile B
        const int hf = (warp >> 2) & 1;        // which half of the tile's key columns this thread owns
        const int r = (warp & 3) * 32 + lane;  // row inside the tile == TMEM lane
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint32_t t_o = tmem_base + lane_base + kColO + x * kHeadDim + hf * (kHeadDim / 2);
        const uint32_t t_sbase = tmem_base + lane_base + kColS;
        const int kv_end_eff = min(p.kv_end, p.S);
        const float c = p.scale_log2;
        float* xchg = reinterpret_cast<float*>(smem_gen + Smem::xchg);
        float* xrow_base = xchg + (x * 2) * kBlockM + r;
        // named barrier shared by the two warps that own the same 32 rows (ids 1..8)
        const uint32_t bar_id = 1 + x * 4 + (warp & 3);
        // every (batch, head, row, half-row) output segment starts on a 32-byte boundary: 256-bit stores are legal
        const int osz = p.out_dtype == 2 ? 4 : 2;
        const bool wide_ok = (reinterpret_cast<uintptr_t>(p.out) & 31) == 0 && ((p.o_sb * osz) & 31) == 0 &&
                             ((p.o_sh * osz) & 31) == 0 && ((p.o_ss * osz) & 31) == 0;
        constexpr uint32_t kPairThreads = 64;
        uint32_t bars_r = bars;
        asm volatile("mov.u32 %0, %0;" : "+r"(bars_r));
        const WaitCtx wctx{bars_r + kWaitBlockOff};  // (shadows the outer one: derived from the pinned register)

        uint32_t oi = 0;    // items this warpgroup worked on so far (O-full barrier phase)
        uint32_t oa = 0;    // items tile A worked on so far (== oi for tile A's warps): phase of the O_A-full barrier
        uint32_t vc = 0;    // V tiles consumed by the tensor pipe in earlier items (V ring position)
        uint32_t g = x;     // sequence index 2*t + x of this warpgroup's next tile
        uint32_t par_bits = 0;  // bit s = phase parity of the next use of S buffer s (both tiles' uses counted)
        uint32_t xpar = 0;  // exchange double buffer
#if RF_FA_TRACE
        int trace_n = 0;
#endif
        // exp-phase turns: this pair's n-th phase follows the other tile's (n-1)-th (tile A) / n-th (tile B)
        const uint32_t turn_mine = bars_r + 8u * (kBarTurn + x * 4 + (warp & 3));
        const uint32_t turn_other = bars_r + 8u * (kBarTurn + (x ^ 1) * 4 + (warp & 3));
        uint32_t tn = static_cast<uint32_t>(x) + 1u;  // parity of the next turn wait is tn & 1

        bool pub_pending = false;  // this warp wrote a split-pair partial whose flag is not raised yet (warp-uniform)
        auto raise_flag = [&]() {
            __threadfence();
            __syncwarp();
            if (lane == 0) st_release_gpu(p.part_flag + blockIdx.x * kNumSoftmaxWarps + warp, 1);
            pub_pending = false;
        };
        while (next_item<kHasBias>(p, sched, item)) {
            const int b = item.b, h = item.h;
            const int num_live = item.num_live;
            const bool active = (x == 0) || item.has_b;
            const int tile_r_lo = item.q0 + x * kBlockM;
            const int tile_r_hi = tile_r_lo + kBlockM - 1;
            const int row = tile_r_lo + r;

            float m_ref = -CUDART_INF_F;
            float l_run = 0.f;  // this thread's share of the row sum (its 64 columns of every tile)
            // scale * log2e * |q_row| (with a rounding margin): times a key tile's largest |k| it bounds every
            // score of this row in that tile (Cauchy-Schwarz)
            float qn_c = CUDART_INF_F;
            const float* kmax_row = nullptr;
            if (num_live > 0) {
                // |q_row| from the Q tile in shared memory (rows past S arrive as zeros).  Every softmax warp waits
                // for Q and arrives on its empty barrier, tile B's also when it sits the item out: the producer
                // cannot run a Q phase ahead of any of them.
                mbar_wait(bars_r + 8u * kBarQFull, oa & 1u, wctx);
                if (active && p.kmax != nullptr) {
                    kmax_row = p.kmax + (static_cast<size_t>(b) * p.H + h) * p.n_kv_tiles;
                    const uint32_t qrow = bars_r - Smem::bars + Smem::q + x * kTileBytes + static_cast<uint32_t>(r) * 128u;
                    float sq[1];
                    rows_sumsq<kBf16, 1, 0u>(qrow, lane, sq);
                    qn_c = sqrtf(sq[0]) * c * 1.001f;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(bars_r + 8u * kBarQEmpty);
            }

            if (active && num_live > 0) {
                // key tiles [nf0, nf1) need no window / range predicate for any row of this query tile
                int nf0, nf1;
                {
                    int lo_key = p.kv_begin, hi_key = kv_end_eff - kBlockN;  // bounds on the tile's first key
                    if (p.wl >= 0) lo_key = max(lo_key, tile_r_hi - p.wl);
                    if (p.wr >= 0) hi_key = min(hi_key, tile_r_lo + p.wr - (kBlockN - 1));
                    nf0 = (lo_key + kBlockN - 1) >> 7;
                    nf1 = hi_key >= 0 ? (hi_key >> 7) + 1 : 0;
                }
                const uint8_t* flags_row = kHasBias ? p.tile_flags + b * p.n_kv_tiles : nullptr;
                int sb = g % kSBufs;  // S/P buffer of the current tile
                int it = 0;
                // the class byte of a key tile is fetched one tile ahead: with ~10 KB of L1 left beside the
                // shared-memory carve-out the load is an L2 round trip, which would otherwise sit at the top of
                // every tile of a padded call
                uint8_t flag_next = (kHasBias && item.n0 < item.n1) ? flags_row[item.n0] : static_cast<uint8_t>(kTileFull);
                for (int n = item.n0; n < item.n1; ++n) {
                    uint8_t flag = kTileFull;
                    if (kHasBias) {
                        flag = flag_next;
                        if (n + 1 < item.n1) flag_next = flags_row[n + 1];
                        if (flag == kTileSkip) continue;
                    }
                    const int kv0 = n * kBlockN;
                    const uint32_t t_s = t_sbase + sb * kBlockN;
                    const float kmax_n = kmax_row != nullptr ? __ldg(kmax_row + n) : CUDART_INF_F;  // back before S is
                    // The UMMA warp issues PV_A(i) right after P_A(i) and QK_A(i+2) right after P_B(i)
                    // without looking at the TMA barriers itself: this warp checks that V(i) / K(i+2)
                    // have landed (both were requested tiles ago) while it would otherwise idle waiting
                    // for S, long before it publishes P.
                    if (RF_FA_VK_IN_SOFTMAX) {
                        const uint32_t tv = vc + static_cast<uint32_t>(it);
                        if (x == 0) mbar_wait(bars_r + 8u * (kBarVFull + tv % kStagesV), (tv / kStagesV) & 1u, wctx);
                        if ((x == 1 || !item.has_b) && it + 2 < num_live)
                            mbar_wait(bars_r + 8u * (kBarKFull + ((tv + 2u) & (kStagesK - 1))),
                                      ((tv + 2u) / kStagesK) & 1u, wctx);
                    }
                    RF_STAMP(0);
                    mbar_wait(bars_r + 8u * (kBarSFull + sb), (par_bits >> sb) & 1u, wctx);
                    tc_fence_after();
                    RF_STAMP(1);

#if !RF_FA_MMAONLY
                    uint32_t su[kHalfN];
#pragma unroll
                    for (int cb = 0; cb < kHalfN / 32; ++cb)
                        tmem_ld32(t_s + hf * kHalfN + cb * 32, reinterpret_cast<uint32_t(&)[32]>(su[cb * 32]));
                    tc_wait_ld();
                    RF_STAMP(2);
                    if (!RF_FA_TRACE && p.debug_scores != nullptr && it == 0) {
                        float* dst = p.debug_scores +
                                     ((static_cast<size_t>(blockIdx.x) * 2 + x) * kBlockM + r) * kBlockN + hf * kHalfN;
#pragma unroll
                        for (int j = 0; j < kHalfN; ++j) dst[j] = __uint_as_float(su[j]);
                    }

                    // tile class (warp-uniform): "full" tiles need no per-element predicate
                    const bool full = (n >= nf0) && (n < nf1) && (flag == kTileFull);

                    // Row-max skip (warp-uniform): if no score of this tile can exceed the reference max by more
                    // than the lazy-rescale threshold -- bound = c |q_row| max_j |k_j| -- the reference stays,
                    // alpha is 1, and neither the max pass nor the exchange with the other half is needed.
                    // (m_ref == -inf on an item's first tile, and any NaN, fail the test.)  Both halves of a row
                    // hold the same m_ref and bound, so their warps decide alike.
                    const bool skip_max =
                        full && !__any_sync(0xffffffffu, !(qn_c * kmax_n <= m_ref + (kBf16 ? kRescaleThresholdBf16 : kRescaleThresholdF16)));
                    float my_max = 0.f;
                    float mul;
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
                        // live columns of this row inside the tile: [lo, hi]
                        int lo = p.kv_begin, hi = kv_end_eff - 1;
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

                    // row max over both halves: exchange through smem (double-buffered).  (No S/P hazard is
                    // tied to this barrier: each half writes P over its own S columns only.)
                    float m_new = m_ref, alpha = 1.0f;
                    if (!skip_max) {
                        float* xrow = xrow_base + xpar * (4 * kBlockM);
                        xrow[hf * kBlockM] = my_max;
                        RF_STAMP(3);
                        named_bar_sync(bar_id, kPairThreads);
                        const float tile_max = fmaxf(my_max, xrow[(hf ^ 1) * kBlockM]);
                        RF_STAMP(4);
                        xpar ^= 1u;
                        // lazy running max: move the reference only when it would grow by > 2^8
                        m_new = (tile_max > m_ref + (kBf16 ? kRescaleThresholdBf16 : kRescaleThresholdF16)) ? tile_max : m_ref;
                        alpha = (m_new == m_ref) ? 1.0f : ex2(m_ref - m_new);
                    }
                    const float neg_m = (m_new == -CUDART_INF_F) ? 0.f : -m_new;

                    // P = 2^(s*mul - m).  On full tiles every kEmuEvery-th element pair takes the FMA-pipe
                    // polynomial (exp2_poly2) instead of MUFU.EX2 so both pipes share the exponentials;
                    // edge tiles keep MUFU only, because a masked score (-inf) must give exactly 0.
                    uint64_t sum2 = 0;  // packed (0.f, 0.f)
                    const uint64_t mul2 = bc2(mul), negm2 = bc2(neg_m);
                    auto exp_store = [&](auto emu_tag) {
                        constexpr bool kEmu = decltype(emu_tag)::value;
#pragma unroll
                        for (int cb = 0; cb < kHalfN / 32; ++cb) {
                            uint32_t pk[16];
#pragma unroll
                            for (int u = 0; u < 16; ++u) {
                                float p0, p1;
                                unpk2(ffma2v(pk2(__uint_as_float(su[cb * 32 + 2 * u]),
                                                 __uint_as_float(su[cb * 32 + 2 * u + 1])),
                                             mul2, negm2),
                                      p0, p1);
                                if (RF_FA_NOEXP) {
                                    // (developer build: no exponential)
                                } else if (kEmu && (u % (kEmuEvery > 0 ? kEmuEvery : 1)) == (kEmuEvery > 0 ? kEmuEvery - 1 : 0)) {
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
                    if (kPingPong) mbar_wait(turn_mine, tn & 1u, wctx);
                    if (kEmuEvery > 0 && full)
                        exp_store(std::true_type{});
                    else
                        exp_store(std::false_type{});
                    if (kPingPong) {
                        mbar_arrive(turn_other);
                        ++tn;
                    }
                    RF_STAMP(5);
                    float sum0, sum1;
                    unpk2(sum2, sum0, sum1);
                    l_run = l_run * alpha + (sum0 + sum1);
                    m_ref = m_new;

                    // O_X *= alpha for rows whose reference max moved (rare after the first tiles thanks
                    // to the lazy threshold): kept out of line so the hot loop stays compact.
                    if (!skip_max && it > 0 && __any_sync(0xffffffffu, alpha != 1.0f)) {
                        const uint32_t vprev = vc + static_cast<uint32_t>(it) - 1u;
                        rescale_o_rows(t_o, alpha, bars_r + 8u * (kBarVEmpty + vprev % kStagesV),
                                       (vprev / kStagesV) & 1u, wctx);
                    }
                    tc_wait_st();
#endif  // !RF_FA_MMAONLY
                    RF_STAMP(6);
                    tc_fence_before();
                    mbar_arrive(bars_r + 8u * (kBarPFull + sb));
                    if (pub_pending && it >= 3) raise_flag();  // the partial's stores drained long ago: a short fence
                    RF_STAMP(7);
#if RF_FA_TRACE
                    ++trace_n;
#endif
                    ++it;
                    // this tile index used buffer sb for this warpgroup and, if the other tile is
                    // active, its neighbour (A = B - 1, B = A + 1 mod 3) for the other warpgroup
                    {
                        const int other = x == 0 ? (sb + 1 == kSBufs ? 0 : sb + 1) : (sb == 0 ? kSBufs - 1 : sb - 1);
                        par_bits ^= (1u << sb) ^ (item.has_b ? (1u << other) : 0u);
                    }
                    sb += 2;
                    if (sb >= kSBufs) sb -= kSBufs;
                }
            } else if (num_live > 0) {
                // Tile B sits this item out (the last pair of a sequence whose length is 1..128 mod 256).  Its warps
                // must not run ahead into the next item: the S-full barriers carry one phase bit, and a wait issued an
                // odd number of tile-A uses early is satisfied by the phase that is still in flight (a persistent
                // schedule then hung at S = 8193: found by the concurrency driver, tools/cpp/concurrency_table.cpp).
                // O_A-full of this item completes after tile A's last use of every S buffer.
                mbar_wait(bars_r + 8u * (kBarOFull + 0), oa & 1u, wctx);
                // account for tile A's uses of the shared S buffers
                for (int i = 0; i < num_live; ++i) {
                    par_bits ^= 1u << ((g - 1u + 2u * i) % kSBufs);
                    if (kPingPong) {  // keep the turn protocol going: pass every turn straight back
                        mbar_wait(turn_mine, tn & 1u, wctx);
                        mbar_arrive(turn_other);
                        ++tn;
                    }
                }
            }
            // keep the sequence counters of both warpgroups in step even when tile B sat this item out
            g += 2u * static_cast<uint32_t>(num_live);
            vc += static_cast<uint32_t>(num_live);

            if (active) {
                // ---------------- epilogue ----------------
                // combine the two halves' row sums, then each half handles its 32 output columns
                float* lrow = xrow_base;
                named_bar_sync(bar_id, kPairThreads);  // all max-exchange reads of the last tile are done
                lrow[hf * kBlockM] = l_run;
                named_bar_sync(bar_id, kPairThreads);
                float l_tot = l_run + lrow[(hf ^ 1) * kBlockM];
                named_bar_sync(bar_id, kPairThreads);  // reads done before the next item reuses the slot

                constexpr int kOutCols = kHeadDim / 2;
                const int col0 = hf * kOutCols;
                float o[kOutCols];
                if (num_live > 0) {
                    mbar_wait(bars_r + 8u * (kBarOFull + x), oi & 1u, wctx);
                    tc_fence_after();
                    tmem_ld32(t_o, reinterpret_cast<uint32_t(&)[32]>(o));
                    tc_wait_ld();
                } else {
#pragma unroll
                    for (int u = 0; u < kOutCols; ++u) o[u] = 0.f;
                }

                if (item.kind == kItemPublish) {
                    // this CTA owns only the leading key tiles of the pair: publish an un-normalised partial
                    // for CTA blockIdx.x + 1, which holds the trailing key tiles and merges at the end of its slice
                    const size_t slot = (static_cast<size_t>(blockIdx.x) * 2 + x) * kBlockM + r;
                    float* dst = p.part_o + slot * kHeadDim + col0;  // 128-byte aligned
#pragma unroll
                    for (int u = 0; u < kOutCols / 8; ++u)
                        st_global_v8(dst + 8 * u, reinterpret_cast<const uint32_t(&)[8]>(o[8 * u]));
                    if (hf == 0) {
                        p.part_ml[slot * 2] = m_ref;
                        p.part_ml[slot * 2 + 1] = l_tot;
                    }
                    // The flag is raised a few key tiles into the next item (or at the end of the kernel): a fence right
                    // here waits for these 128 KiB of stores to drain (~5 us at every publishing CTA, phase trace), and
                    // the reader only wants the partial at the very end of its own slice.
                    pub_pending = true;
                } else {
                    if (item.kind == kItemMerge) {
                        // merge with the partial CTA blockIdx.x - 1 published for the same rows at the START of
                        // its slice (its half-0 warp of the same quadrant wrote m and l, this warp's twin wrote
                        // the columns); own part first: fixed order, deterministic.  The wait is on a
                        // lower-indexed CTA only, so it cannot starve whatever else is resident on the GPU.
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
                        const float w1 = (m_ref == -CUDART_INF_F) ? 0.f : ex2(m_ref - ms);
                        const float w2 = (m2 == -CUDART_INF_F) ? 0.f : ex2(m2 - ms);
                        const float4* src = reinterpret_cast<const float4*>(p.part_o + slot * kHeadDim + col0);
#pragma unroll
                        for (int u = 0; u < kOutCols / 4; ++u) {
                            const float4 t = __ldcg(src + u);
                            o[4 * u] = o[4 * u] * w1 + t.x * w2;
                            o[4 * u + 1] = o[4 * u + 1] * w1 + t.y * w2;
                            o[4 * u + 2] = o[4 * u + 2] * w1 + t.z * w2;
                            o[4 * u + 3] = o[4 * u + 3] * w1 + t.w * w2;
                        }
                        l_tot = l_tot * w1 + l2 * w2;
                        m_ref = ms;
                        // The flags are left as they were found (zero): this warp and its twin of the other half
                        // are the only readers of the two flags they waited for, and both are done with them.
                        named_bar_sync(bar_id, kPairThreads);
                        if (lane == 0) p.part_flag[(blockIdx.x - 1) * kNumSoftmaxWarps + warp] = 0;
                    }
                    if (row < p.S && col0 < p.d) {  // head_dim 32 runs zero-padded to 64: its columns [32, 64) do not exist
                        if (p.o_partial != nullptr) {
                            const size_t ridx = (static_cast<size_t>(b) * p.H + h) * p.S + row;
                            float4* dst = reinterpret_cast<float4*>(p.o_partial + ridx * p.d + col0);
#pragma unroll
                            for (int u = 0; u < kOutCols / 4; ++u)
                                dst[u] = make_float4(o[4 * u], o[4 * u + 1], o[4 * u + 2], o[4 * u + 3]);
                            if (hf == 0) {
                                p.m_partial[ridx] = m_ref;
                                p.l_partial[ridx] = l_tot;
                            }
                        } else {
                            const float inv = l_tot > 0.f ? 1.0f / l_tot : 0.f;
                            const size_t off = static_cast<size_t>(b) * p.o_sb + static_cast<size_t>(h) * p.o_sh +
                                               static_cast<size_t>(row) * p.o_ss + col0;
                            // A lane owns one row, so a warp-wide store touches 32 rows whatever its width: 32-byte
                            // stores (sm_100's 256-bit st.global) halve the store instructions and their LSU passes.
                            if (p.out_dtype == 2) {
                                float* dst = static_cast<float*>(p.out) + off;
#pragma unroll
                                for (int u = 0; u < kOutCols / 8; ++u) {
                                    uint32_t w[8];
#pragma unroll
                                    for (int e = 0; e < 8; ++e) w[e] = __float_as_uint(o[8 * u + e] * inv);
                                    if (wide_ok) {
                                        st_global_v8(dst + 8 * u, w);
                                    } else {
                                        *reinterpret_cast<uint4*>(dst + 8 * u) = make_uint4(w[0], w[1], w[2], w[3]);
                                        *reinterpret_cast<uint4*>(dst + 8 * u + 4) = make_uint4(w[4], w[5], w[6], w[7]);
                                    }
                                }
                            } else {
                                uint16_t* dst = static_cast<uint16_t*>(p.out) + off;
#pragma unroll
                                for (int u = 0; u < kOutCols / 16; ++u) {
                                    uint32_t w[8];
#pragma unroll
                                    for (int e = 0; e < 8; ++e) {
                                        const float a0 = o[16 * u + 2 * e] * inv, a1 = o[16 * u + 2 * e + 1] * inv;
                                        w[e] = (p.out_dtype == 0) ? pack2<true>(a0, a1) : pack2<false>(a0, a1);
                                    }
                                    if (wide_ok) {
                                        st_global_v8(dst + 16 * u, w);
                                    } else {
                                        *reinterpret_cast<uint4*>(dst + 16 * u) = make_uint4(w[0], w[1], w[2], w[3]);
                                        *reinterpret_cast<uint4*>(dst + 16 * u + 8) = make_uint4(w[4], w[5], w[6], w[7]);
                                    }
                                }
                            }
                        }
                    }
                }
            }
            if (active && num_live > 0) ++oi;
            if (num_live > 0) ++oa;
        }
        if (pub_pending) raise_flag();
    }

    // ---------------- teardown ----------------
    tc_fence_before();
    __syncthreads();
    RF_KSTAMP(3);
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc(tmem_base, kTmemCols);
    }
}

}  // namespace

size_t fa_fwd_sm100_smem_bytes() {
    return Smem::xchg + Smem::xchg_bytes + 1024;  // + alignment slack
}

size_t fa_fwd_sm100_partial_bytes(int grid, int head_dim) {
    // per CTA: O partial [2][128][head_dim] f32 (head_dim 64 here, 128 in fa_fwd_sm100_d128.cu), (m, l) [2][128][2] f32
    return static_cast<size_t>(grid) * (2 * kBlockM * static_cast<size_t>(head_dim) * 4 + 2 * kBlockM * 2 * 4);
}

size_t fa_fwd_sm100_flag_bytes(int grid) {
    return static_cast<size_t>(grid) * kNumSoftmaxWarps * 4;  // one flag per (CTA, softmax warp)
}

// Carves the split-pair workspace.  `flags` (fa_fwd_sm100_flag_bytes) must be zero when the kernel starts; the
// kernel leaves it zero.
void fa_fwd_sm100_partial_carve(void* base, void* flags, int grid, int head_dim, FaParams* p) {
    uint8_t* b = static_cast<uint8_t*>(base);
    p->part_o = reinterpret_cast<float*>(b);
    b += static_cast<size_t>(grid) * 2 * kBlockM * static_cast<size_t>(head_dim) * 4;
    p->part_ml = reinterpret_cast<float*>(b);
    p->part_flag = static_cast<int*>(flags);
}

cudaError_t launch_fa_fwd_sm100(const CUtensorMap& tmq, const CUtensorMap& tmk, const CUtensorMap& tmv,
                                const FaParams& p, bool bf16, int grid, cudaStream_t stream, bool pdl) {
    const bool has_bias = p.tile_flags != nullptr;
    void (*kern)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const FaParams) =
        bf16 ? (has_bias ? fa_fwd_sm100_kernel<true, true> : fa_fwd_sm100_kernel<true, false>)
             : (has_bias ? fa_fwd_sm100_kernel<false, true> : fa_fwd_sm100_kernel<false, false>);
    const size_t smem = fa_fwd_sm100_smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    if (!pdl) {
        kern<<<grid, kThreads, smem, stream>>>(tmq, tmk, tmv, p);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, tmq, tmk, tmv, p);
}

}  // namespace rf
