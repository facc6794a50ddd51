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
// One persistent CTA per SM, 20 warps (five warpgroups, setmaxnreg moves registers to the first four):
//   warps 0-15 softmax/epilogue, four threads per query row (warp w: rows 32*(w%4).., strip columns
//              [64*(w/4), +64)); 32-column chunks that are dead for all 32 rows of a warp are skipped
//              (the band leaves 20 of the 32 chunks of a tile)
//   warp 16    TMA producer: Q double-buffered; K and V as rings of four 128-key boxes.  A CTA owns a
//              contiguous run of query tiles, and the second box of a tile is the first box of the next
//              tile of the same head, so a tile costs one new K box, one new V box and Q (48 KiB, the
//              algorithmic minimum) and loads run two tiles ahead
//   warp 17    UMMA issuer: S[128x256] = Q K^T (2 x 4 M128 N128 K16, one half per box), O[128x64] = P V
//              (16 x M128 N64 K16, P from TMEM)
// TMEM: S [0,256)  P [256,384)  O [384,448) and [448,512) alternating.  S is copied to registers in one go and handed back at
// once, so Q K^T of the next tile runs under the softmax of this one; the load/max half of the next
// tile's softmax runs under P V of this one.
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
constexpr int kStrip = 2 * kBlockN;                 // keys a query tile reads
constexpr int kTileBytes = kBlockN * kHeadDim * 2;  // 16 KiB
constexpr int kQStages = 2;
constexpr int kRing = 4;                            // K / V boxes in flight
constexpr int kParts = 4;                           // softmax threads per query row
constexpr int kPartCols = kStrip / kParts;          // strip columns per softmax thread
constexpr int kOutCols = kHeadDim / kParts;         // output columns per softmax thread
constexpr int kSoftmaxWarps = 4 * kParts;
constexpr int kSoftmaxThreads = kSoftmaxWarps * 32;
constexpr int kProducerWarp = kSoftmaxWarps;
constexpr int kMmaWarp = kSoftmaxWarps + 1;
constexpr int kThreads = kSoftmaxThreads + 128;     // 5 warpgroups: 4 softmax + 1 (producer, MMA, 2 idle warps)
constexpr int kRegsSoftmax = 112;
constexpr int kRegsOther = 32;                      // 128*32 + 512*112 == 640*96
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColS = 0, kColP = 256, kColO = 384;  // O: two buffers of 64 columns, tile n uses n & 1

// Developer build only (-DRF_FA_TRACE=1): CTA 0 stamps the SM clock at phase boundaries into the
// debug_scores buffer, [20 warps][64 tiles][8 stamps] u32 (tools/trace_local.py).
#ifndef RF_FA_TRACE
#define RF_FA_TRACE 0
#endif
#if RF_FA_TRACE
#define RF_STAMP(tile, slot)                                                                          \
    do {                                                                                              \
        if (blockIdx.x == 0 && lane == 0 && (tile) < 64 && p.debug_scores != nullptr)                 \
            reinterpret_cast<uint32_t*>(p.debug_scores)[(warp * 64 + (tile)) * 8 + (slot)] = clock(); \
    } while (0)
#else
#define RF_STAMP(tile, slot) do { } while (0)
#endif

struct Smem {
    static constexpr uint32_t q = 0;
    static constexpr uint32_t k = q + kQStages * kTileBytes;
    static constexpr uint32_t v = k + kRing * kTileBytes;
    static constexpr uint32_t bars = v + kRing * kTileBytes;
    static constexpr uint32_t bar_bytes = 256;
    static constexpr uint32_t xchg = bars + bar_bytes;                // [2 parity][kParts][128] f32 row max
    static constexpr uint32_t lsum = xchg + 2 * kParts * kBlockM * 4;  // [2 parity][kParts][128] f32 row sum
    static constexpr uint32_t bias = lsum + 2 * kParts * kBlockM * 4;  // [2 parity][256] f32, log2 domain
    static constexpr uint32_t total = bias + 2 * kStrip * 4;
};
enum : uint32_t {
    kBarQFull = 0,                     // [2]
    kBarQEmpty = kBarQFull + kQStages, // [2]
    kBarKFull = kBarQEmpty + kQStages, // [kRing]
    kBarKEmpty = kBarKFull + kRing,    // [kRing] the last Q K^T that reads the box has completed
    kBarVFull = kBarKEmpty + kRing,    // [kRing]
    kBarVEmpty = kBarVFull + kRing,    // [kRing]
    kBarSFull = kBarVEmpty + kRing,
    kBarSFree,  // count kSoftmaxWarps: S is in the registers of every softmax warp
    kBarPFull,  // count kSoftmaxThreads
    kBarOFull,
    kNumBars,
};
constexpr uint32_t kTmemSlotOff = kNumBars * 8;                     // u32: TMEM base address
constexpr uint32_t kWaitBlockOff = (kTmemSlotOff + 8 + 15) & ~15u;  // 16 bytes: abort word + status pointer (ptx.cuh)
static_assert(kWaitBlockOff + 16 <= Smem::bar_bytes, "barrier block too small");

struct Tile {
    int b, h, r0, kb;  // batch, head, first query row, first key of the strip
    bool head_start;   // first query tile of its (batch, head): its first K/V box is not shared
};

__device__ __forceinline__ Tile decode_tile(const FaParams& p, int g, int q_tiles) {
    Tile t;
    const int qt = g % q_tiles;
    const int bh = g / q_tiles;
    t.h = bh % p.H;
    t.b = bh / p.H;
    t.r0 = qt * kBlockM;
    t.kb = t.r0 - p.wl;
    t.head_start = qt == 0;
    return t;
}

// next tile of a contiguous run, without the divisions
__device__ __forceinline__ void advance_tile(const FaParams& p, Tile& t, int q_tiles) {
    t.r0 += kBlockM;
    t.head_start = false;
    if (t.r0 >= q_tiles * kBlockM) {
        t.r0 = 0;
        t.head_start = true;
        if (++t.h == p.H) {
            t.h = 0;
            ++t.b;
        }
    }
    t.kb = t.r0 - p.wl;
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
    volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(smem_gen + Smem::bars + kTmemSlotOff);
    const WaitCtx wctx{bars + kWaitBlockOff};

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int q_tiles = (p.S + kBlockM - 1) / kBlockM;
    const int total = p.B * p.H * q_tiles;
    // a contiguous run of query tiles per CTA: consecutive tiles of a head share a K/V box
    const int g0 = static_cast<int>(static_cast<long long>(total) * blockIdx.x / gridDim.x);
    const int my_tiles = static_cast<int>(static_cast<long long>(total) * (blockIdx.x + 1) / gridDim.x) - g0;

    if (warp == kProducerWarp && lane == 0) {
        prefetch_tensormap(&tm_q);
        prefetch_tensormap(&tm_k);
        prefetch_tensormap(&tm_v);
        for (int s = 0; s < kQStages; ++s) {
            mbar_init(bar(kBarQFull + s), 1);
            mbar_init(bar(kBarQEmpty + s), 1);
        }
        for (int s = 0; s < kRing; ++s) {
            mbar_init(bar(kBarKFull + s), 1);
            mbar_init(bar(kBarKEmpty + s), 1);
            mbar_init(bar(kBarVFull + s), 1);
            mbar_init(bar(kBarVEmpty + s), 1);
        }
        mbar_init(bar(kBarSFull), 1);
        mbar_init(bar(kBarSFree), kSoftmaxWarps);
        mbar_init(bar(kBarPFull), kSoftmaxThreads);
        mbar_init(bar(kBarOFull), 1);
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

    static_assert(128 * kRegsOther + kSoftmaxThreads * kRegsSoftmax <= kThreads * 96, "setmaxnreg pool must balance");
    if (warp >= kSoftmaxWarps) setmaxnreg_dec<kRegsOther>();

    if (warp == kProducerWarp) {
        // =============================== TMA producer ===============================
        // warp-uniform control flow; only lane 0 issues
        uint32_t bc = 0;  // K/V boxes requested so far: ring slot bc % kRing, use (bc / kRing)
        auto load_box = [&](const Tile& t, int key0) {
            const uint32_t slot = bc % kRing, par = ((bc / kRing) & 1) ^ 1;
            mbar_wait(bar(kBarKEmpty + slot), par, wctx);
            if (lane == 0) {
                mbar_arrive_expect_tx(bar(kBarKFull + slot), kTileBytes);
                tma_load_4d(smem_base + Smem::k + slot * kTileBytes, &tm_k, bar(kBarKFull + slot), 0, key0, t.h, t.b);
            }
            mbar_wait(bar(kBarVEmpty + slot), par, wctx);
            if (lane == 0) {
                mbar_arrive_expect_tx(bar(kBarVFull + slot), kTileBytes);
                tma_load_4d(smem_base + Smem::v + slot * kTileBytes, &tm_v, bar(kBarVFull + slot), 0, key0, t.h, t.b);
            }
            __syncwarp();
            ++bc;
        };
        for (int n = 0; n < my_tiles; ++n) {
            const Tile t = decode_tile(p, g0 + n, q_tiles);
            const uint32_t s = n & 1;
            mbar_wait(bar(kBarQEmpty + s), ((n >> 1) & 1) ^ 1, wctx);
            if (lane == 0) {
                mbar_arrive_expect_tx(bar(kBarQFull + s), kTileBytes);
                tma_load_4d(smem_base + Smem::q + s * kTileBytes, &tm_q, bar(kBarQFull + s), 0, t.r0, t.h, t.b);
            }
            __syncwarp();
            if (n == 0 || t.head_start) load_box(t, t.kb);
            load_box(t, t.kb + kBlockN);
        }
    } else if (warp == kMmaWarp) {
        // =============================== UMMA issuer ===============================
        // warp-uniform control flow; only the tcgen05 instructions are predicated on the elected lane
        const bool leader = elect_one() != 0;
        constexpr uint32_t fmt = kBf16 ? 1u : 0u;
        constexpr uint32_t idesc_qk = make_idesc_f16(fmt, 0, 0, kBlockM, kBlockN);
        constexpr uint32_t idesc_pv = make_idesc_f16(fmt, 0, 1, kBlockM, kHeadDim);
        const uint32_t t_s = tmem_base + kColS, t_p = tmem_base + kColP, t_o = tmem_base + kColO;
        auto commit = [&](uint32_t b_) {
            if (leader) tc_commit(b_);
            __syncwarp();
        };
        // box stream positions (mirrors the producer): tile n reads boxes first(n), first(n) + 1
        uint32_t nb = 0;        // boxes the producer has requested up to and including the tile being issued
        uint32_t first_qk = 0;  // first box of the tile whose Q K^T is issued next
        auto seg_end = [&](int n) {  // tile n is the last one that reads its second box
            return n + 1 == my_tiles || decode_tile(p, g0 + n + 1, q_tiles).head_start;
        };
        auto issue_qk = [&](int n) {
            const bool fresh = n == 0 || decode_tile(p, g0 + n, q_tiles).head_start;
            first_qk = fresh ? nb : nb - 1;
            nb = first_qk + 2;
            const uint32_t s0 = first_qk % kRing, s1 = (first_qk + 1) % kRing;
            mbar_wait(bar(kBarQFull + (n & 1)), (n >> 1) & 1, wctx);
            mbar_wait2(bar(kBarKFull + s0), (first_qk / kRing) & 1, bar(kBarKFull + s1), ((first_qk + 1) / kRing) & 1, wctx);
            tc_fence_after();
            if (leader) {
                const uint32_t qbase = smem_base + Smem::q + (n & 1) * kTileBytes;
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    const uint32_t kbase = smem_base + Smem::k + (half ? s1 : s0) * kTileBytes;
#pragma unroll
                    for (int kk = 0; kk < kHeadDim / 16; ++kk)
                        mma_ss(t_s + half * kBlockN, make_smem_desc(qbase + kk * 32, 16, 1024, kSwizzle128B),
                               make_smem_desc(kbase + kk * 32, 16, 1024, kSwizzle128B), idesc_qk, kk > 0 ? 1u : 0u);
                }
                tc_commit(bar(kBarSFull));
                tc_commit(bar(kBarQEmpty + (n & 1)));
                tc_commit(bar(kBarKEmpty + s0));
            }
            __syncwarp();
            if (seg_end(n)) commit(bar(kBarKEmpty + s1));
        };
        uint32_t first_pv = 0, nb_pv = 0;
        if (my_tiles > 0) issue_qk(0);
        for (int n = 0; n < my_tiles; ++n) {
            RF_STAMP(n, 0);
            if (n + 1 < my_tiles) {
                // S(n) is in registers: Q K^T of the next tile runs under the softmax of this one
                mbar_wait(bar(kBarSFree), n & 1, wctx);
                RF_STAMP(n, 1);
                issue_qk(n + 1);
            }
            RF_STAMP(n, 2);
            {
                const bool fresh = n == 0 || decode_tile(p, g0 + n, q_tiles).head_start;
                first_pv = fresh ? nb_pv : nb_pv - 1;
                nb_pv = first_pv + 2;
            }
            const uint32_t s0 = first_pv % kRing, s1 = (first_pv + 1) % kRing;
            mbar_wait2(bar(kBarVFull + s0), (first_pv / kRing) & 1, bar(kBarVFull + s1), ((first_pv + 1) / kRing) & 1, wctx);
            RF_STAMP(n, 3);
            mbar_wait(bar(kBarPFull), n & 1, wctx);
            tc_fence_after();
            RF_STAMP(n, 4);
            if (leader) {
                // V box [128 keys][64] with d contiguous = MN-major B operand; a K=16 step is 2048 B
#pragma unroll
                for (int kk = 0; kk < kStrip / 16; ++kk) {
                    const uint32_t vbase = smem_base + Smem::v + (kk < 8 ? s0 : s1) * kTileBytes + (kk & 7) * 2048;
                    mma_ts(t_o + (n & 1) * kHeadDim, t_p + kk * 8, make_smem_desc(vbase, kTileBytes, 1024, kSwizzle128B),
                           idesc_pv, kk > 0 ? 1u : 0u);
                }
                tc_commit(bar(kBarOFull));
                tc_commit(bar(kBarVEmpty + s0));
            }
            __syncwarp();
            if (seg_end(n)) commit(bar(kBarVEmpty + s1));
            RF_STAMP(n, 5);
        }
    } else if (warp < kSoftmaxWarps) {
        // =============================== softmax / epilogue ===============================
        setmaxnreg_inc<kRegsSoftmax>();
        // Four threads per query row (four softmax warps per SM sub-partition hide each other's
        // latencies): warp w owns rows 32*(w%4).. and strip columns [64*(w/4), 64*(w/4) + 64).
        const int part = warp >> 2;            // which 64-column quarter of the strip
        const int quad = warp & 3;
        const int r = quad * 32 + lane;        // row inside the tile == TMEM lane
        const int tid = threadIdx.x;           // 0..511
        const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
        const uint32_t t_s = tmem_base + lane_base + kColS + part * kPartCols;
        const uint32_t t_p = tmem_base + lane_base + kColP + part * (kPartCols / 2);
        const uint32_t t_o = tmem_base + lane_base + kColO + part * kOutCols;
        const float c = p.scale_log2;
        const int band = p.wl + p.wr;          // live strip columns of row r: [r, r + band]
        float* xchg = reinterpret_cast<float*>(smem_gen + Smem::xchg);
        float* lsum = reinterpret_cast<float*>(smem_gen + Smem::lsum);
        float* sbias = reinterpret_cast<float*>(smem_gen + Smem::bias);
        const uint32_t row_bar = 1 + quad;     // named barrier of the four warps that share 32 rows

        auto load_bias = [&](const Tile& t) -> float {  // strip column tid, log2 domain
            const int key = t.kb + tid;
            float v = -CUDART_INF_F;
            if (tid < kStrip && key >= 0 && key < p.S) {
                const float raw = __ldg(pad_bias + static_cast<size_t>(t.b) * p.S + key);
                v = raw > kMaskThreshold ? raw * kLog2e : -CUDART_INF_F;
            }
            return v;
        };

        uint32_t su[kPartCols];  // this thread's 64 scores, then log2-domain x, of the current tile
        uint32_t live_chunks = 0, plain_chunks = 0;
        float m_row = -CUDART_INF_F;
        Tile cur = {}, nxt = {};
        float bias_pref = 0.f;
        if (my_tiles > 0) {
            nxt = decode_tile(p, g0, q_tiles);
            if (kHasBias) bias_pref = load_bias(nxt);
        }

        // first half of a tile: S -> registers, scale / bias / band predicate, row max
        auto stage_a = [&](int n, const Tile& t) {
            const uint32_t par = n & 1;
            // this thread's live columns, local to its 64-column quarter
            int lo = max(r, -t.kb);                       // key >= 0
            int hi = min(r + band, p.S - 1 - t.kb);       // key < S
            lo -= part * kPartCols;
            hi -= part * kPartCols;
            if (kHasBias) {
                if (tid < kStrip) sbias[par * kStrip + tid] = bias_pref;
                named_bar_sync(5, kSoftmaxThreads);
            }
            uint32_t dead = 0, full = 0;
#pragma unroll
            for (int cb = 0; cb < kPartCols / 32; ++cb) {
                const int c0 = cb * 32;
                if (__all_sync(0xffffffffu, hi < c0 || lo > c0 + 31)) dead |= 1u << cb;
                if (__all_sync(0xffffffffu, lo <= c0 && hi >= c0 + 31)) full |= 1u << cb;
            }
            RF_STAMP(n, 2);
            mbar_wait(bar(kBarSFull), par, wctx);
            tc_fence_after();
            RF_STAMP(n, 3);
#pragma unroll
            for (int cb = 0; cb < kPartCols / 32; ++cb)
                if (!((dead >> cb) & 1)) tmem_ld32(t_s + cb * 32, reinterpret_cast<uint32_t(&)[32]>(su[cb * 32]));
            tc_wait_ld();
            tc_fence_before();
            if (lane == 0) mbar_arrive(bar(kBarSFree));
            float mx = -CUDART_INF_F;
            plain_chunks = kHasBias ? 0u : (full & ~dead);  // no predicate, no bias: scaling is left to the exp pass
#pragma unroll
            for (int cb = 0; cb < kPartCols / 32; ++cb) {
                if ((dead >> cb) & 1) continue;
                if ((plain_chunks >> cb) & 1) {
                    float m4[4] = {-CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F};
#pragma unroll
                    for (int j = 0; j < 32; j += 8) {
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4)
                            m4[q4] = max3(m4[q4], __uint_as_float(su[cb * 32 + j + 2 * q4]),
                                          __uint_as_float(su[cb * 32 + j + 2 * q4 + 1]));
                    }
                    mx = fmaxf(mx, fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * c);  // scale > 0 (host-checked)
                    continue;
                }
                const bool is_full = (full >> cb) & 1;
                const float* brow = sbias + par * kStrip + part * kPartCols + cb * 32;
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
            live_chunks = ~dead & ((1u << (kPartCols / 32)) - 1u);
            xchg[(par * kParts + part) * kBlockM + r] = mx;
            named_bar_sync(row_bar, 32 * kParts);
            const float* xr = xchg + par * kParts * kBlockM + r;
            m_row = fmaxf(fmaxf(xr[0], xr[kBlockM]), fmaxf(xr[2 * kBlockM], xr[3 * kBlockM]));
            RF_STAMP(n, 4);
        };

        // epilogue of a tile: this thread owns 16 of the 64 output columns
        auto epilogue = [&](int n, const Tile& t) {
            const uint32_t par = n & 1;
            const float* lr = lsum + par * kParts * kBlockM + r;
            const float l_tot = (lr[0] + lr[kBlockM]) + (lr[2 * kBlockM] + lr[3 * kBlockM]);
            const float inv = l_tot > 0.f ? 1.0f / l_tot : 0.f;
            float o[kOutCols];
            RF_STAMP(n, 6);
            tmem_ld16(t_o + par * kHeadDim, reinterpret_cast<uint32_t(&)[16]>(o));
            tc_wait_ld();
            const int row = t.r0 + r;
            if (row < p.S && part * kOutCols < p.d) {  // head_dim 32 runs zero-padded to 64 (FaParams::d)
                const size_t off = static_cast<size_t>(t.b) * p.o_sb + static_cast<size_t>(t.h) * p.o_sh +
                                   static_cast<size_t>(row) * p.o_ss + part * kOutCols;
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
            RF_STAMP(n, 7);
        };

        // Order per tile n:  [O(n-1) complete -> P is free]  exp(n) -> P-full(n)  |  epilogue(n-1)  |
        // load/max(n+1).  The epilogue of the previous tile and the first half of the next one run under
        // P V of this one; nothing in this loop waits for the MMA it has just triggered.
        Tile prev = {};
        if (my_tiles > 0) stage_a(0, nxt);
        for (int n = 0; n < my_tiles; ++n) {
            const uint32_t par = n & 1;
            prev = cur;
            cur = nxt;
            const bool has_next = n + 1 < my_tiles;
            if (has_next) {
                advance_tile(p, nxt, q_tiles);
                if (kHasBias) bias_pref = load_bias(nxt);
            }
            RF_STAMP(n, 0);
            // P V of tile n-1 must have read P (and written O[(n-1) & 1]) before P is overwritten: test
            // now, the answer is back before the first store needs it
            uint32_t p_free = n > 0 ? mbar_try_wait(bar(kBarOFull), par ^ 1u) : 1u;
            // ---- second half: P = 2^(x - m), row sum, P -> TMEM ----
            const float neg_m = (m_row == -CUDART_INF_F) ? 0.f : -m_row;
            const uint64_t negm2 = bc2(neg_m), c2 = bc2(c);
            uint64_t sum2a = 0, sum2b = 0;
            auto exp_chunk = [&](int cb, auto plain_tag, uint32_t (&pk)[16]) {
                constexpr bool kPlain = decltype(plain_tag)::value;  // raw scores, all live: scale here
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    float p0, p1;
                    const uint64_t sp = pk2(__uint_as_float(su[cb * 32 + 2 * u]), __uint_as_float(su[cb * 32 + 2 * u + 1]));
                    unpk2(kPlain ? ffma2v(sp, c2, negm2) : fadd2v(sp, negm2), p0, p1);
                    // MUFU only: masked scores are -inf and must give exactly 0, and moving a share of
                    // the exponentials to the FMA pipe (as the dense kernel does) measured no gain here --
                    // this pass is latency-bound, not MUFU-bound
                    p0 = ex2(p0);
                    p1 = ex2(p1);
                    if (u & 1) sum2b = fadd2v(sum2b, pk2(p0, p1));
                    else sum2a = fadd2v(sum2a, pk2(p0, p1));
                    pk[u] = pack2<kBf16>(p0, p1);
                }
            };
#pragma unroll
            for (int cb = 0; cb < kPartCols / 32; ++cb) {
                uint32_t pk[16];
                if ((live_chunks >> cb) & 1) {
                    if ((plain_chunks >> cb) & 1) exp_chunk(cb, std::true_type{}, pk);
                    else exp_chunk(cb, std::false_type{}, pk);
                } else {
#pragma unroll
                    for (int u = 0; u < 16; ++u) pk[u] = 0u;
                }
                if (cb == 0) {
                    if (!p_free) mbar_wait(bar(kBarOFull), par ^ 1u, wctx);
                    tc_fence_after();
                }
                tmem_st16(t_p + cb * 16, pk);
            }
            float sum0, sum1;
            unpk2(fadd2v(sum2a, sum2b), sum0, sum1);
            lsum[(par * kParts + part) * kBlockM + r] = sum0 + sum1;
            tc_wait_st();
            tc_fence_before();
            mbar_arrive(bar(kBarPFull));
            RF_STAMP(n, 1);

            if (n > 0) epilogue(n - 1, prev);   // (the row barrier of load/max(n) ordered its lsum exchange)
            if (has_next) stage_a(n + 1, nxt);
        }
        if (my_tiles > 0) {
            const int n = my_tiles - 1;
            named_bar_sync(row_bar, 32 * kParts);  // lsum of the last tile
            mbar_wait(bar(kBarOFull), n & 1, wctx);
            tc_fence_after();
            epilogue(n, cur);
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
