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
// rescale of O.  This layer is HBM-bound (64 FLOP/B): 48 KiB of new data per tile, ~2100 clk of HBM
// time per SM, against a dependent chain Q K^T -> max -> exp -> P V -> store of ~4000 clk per tile.
//
// Round-2 design: TWO small CTAs per SM, each a plain serial chain over its own run of query tiles.  The
// first version ran one CTA per SM with 16 softmax warps in lockstep on one tile and hand-overlapped
// phases; its warps were latency-bound (ncu: issue 39 %, 26 % of SM cycles idle).  Two co-resident CTAs
// interleave their chains through the hardware schedulers instead: while one waits for its MMA the
// other does its exponentials.  It also halves the tile quantisation (296 runs of 2-3 tiles instead of
// 148 runs of 5-6 at B=1, S=8K).
//
// Per CTA, 12 warps (three warpgroups; setmaxnreg moves registers to the first two):
//   warps 0-7  softmax/epilogue, two threads per query row.  Row r of quad q = r / 32 is live on strip
//              columns [32q, 32q + 31 + band] taken over the warp; that range is cut into 16-column
//              pieces and the two warps of a quad take half of them each (<= 5 pieces = 80 columns per
//              thread), so both have the same amount of exponentials whatever the quad
//   warp 8     TMA producer: Q single-buffered, K ring of two 128-key boxes, V ring of three.  A CTA owns
//              a contiguous run of query tiles and the second box of a tile is the first box of the
//              next tile of the same head, so a tile costs one new K box, one new V box and Q (48 KiB,
//              the algorithmic minimum)
//   warp 9     UMMA issuer: S[128x256] = Q K^T (2 x 4 M128 N128 K16, one half per box), O[128x64] = P V
//              (16 x M128 N64 K16, P read from TMEM)
// TMEM (256 columns per CTA): S [0,256); once every softmax thread has its exponentials in registers P
// (bf16/f16 pairs) overwrites [0,128) and O accumulates in [128,192).
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
constexpr int kRingK = 2;                           // K boxes resident: the two of the current tile
constexpr int kRingV = 3;                           // V boxes resident: current tile + the next one's new box
constexpr int kParts = 2;                           // softmax threads per query row
constexpr int kPiece = 16;                          // strip columns per tcgen05.ld piece
constexpr int kMaxPieces = 5;                       // pieces per softmax thread (band <= 127)
constexpr int kOutCols = kHeadDim / kParts;         // output columns per softmax thread
constexpr int kSoftmaxWarps = 4 * kParts;
constexpr int kSoftmaxThreads = kSoftmaxWarps * 32;
constexpr int kProducerWarp = kSoftmaxWarps;
constexpr int kMmaWarp = kSoftmaxWarps + 1;
constexpr int kThreads = kSoftmaxThreads + 128;     // 3 warpgroups: 2 softmax + 1 (producer, MMA, 2 idle warps)
constexpr int kCtasPerSm = 2;
constexpr int kRegsLaunch = 80;                     // 65536 / (2 * 384) rounded down to a multiple of 8
constexpr int kRegsSoftmax = 104;
constexpr int kRegsOther = 32;
static_assert(128 * kRegsOther + kSoftmaxThreads * kRegsSoftmax <= kThreads * kRegsLaunch, "setmaxnreg pool must balance");
constexpr int kBandStride = 392;                    // >= 128 + 256 + 3 entries per copy; 392 % 32 == 8 (bank spread)
static_assert(kBandStride >= kBlockM + kStrip + 3 && kBandStride % 32 == 8, "band table stride");
constexpr uint32_t kTmemCols = 256;
constexpr uint32_t kColS = 0, kColP = 0, kColO = 128;

// Share of the exponentials of predicate-free pieces taken on the FMA pipe (Cody-Waite + cubic, ptx.cuh)
// instead of MUFU: pairs u with (u & 7) < RF_LOCAL_POLY of every 8.  0 = MUFU only.
#ifndef RF_LOCAL_SKEW
#define RF_LOCAL_SKEW 0
#endif
#ifndef RF_LOCAL_SKEW_ODD
#define RF_LOCAL_SKEW_ODD 0
#endif
#ifndef RF_LOCAL_POLY
#define RF_LOCAL_POLY 2
#endif

// Developer build only (-DRF_FA_TRACE=1): CTA 0 stamps the SM clock at phase boundaries into the
// debug_scores buffer, [12 warps][64 tiles][8 stamps] u32 (tools/trace_local.py).
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
    static constexpr uint32_t k = q + kTileBytes;
    static constexpr uint32_t v = k + kRingK * kTileBytes;
    static constexpr uint32_t bars = v + kRingV * kTileBytes;
    static constexpr uint32_t bar_bytes = 256;
    static constexpr uint32_t xchg = bars + bar_bytes;             // [kParts][128] f32 row max
    static constexpr uint32_t lsum = xchg + kParts * kBlockM * 4;  // [kParts][128] f32 row sum
    static constexpr uint32_t xmax = lsum + kParts * kBlockM * 4;  // [kParts][128] f32 max of x - m_ref
    static constexpr uint32_t bias = xmax + kParts * kBlockM * 4;  // [256] f32, log2 domain: per-column additive term
    static constexpr uint32_t band = bias + kStrip * 4;            // [4][kBandStride] f32: band mask table (see softmax)
    static constexpr uint32_t total = band + 4 * kBandStride * 4;
};
// two CTAs must fit one SM: 228 KiB of shared memory, 1 KiB reserved per CTA
static_assert(kCtasPerSm * (Smem::total + 1024 + 1024) <= 228 * 1024, "two CTAs per SM do not fit");
enum : uint32_t {
    kBarQFull = 0,
    kBarQEmpty,
    kBarKFull,                          // [kRingK]
    kBarKEmpty = kBarKFull + kRingK,    // [kRingK] the last Q K^T that reads the box has completed
    kBarVFull = kBarKEmpty + kRingK,    // [kRingV]
    kBarVEmpty = kBarVFull + kRingV,    // [kRingV]
    kBarSFull = kBarVEmpty + kRingV,
    kBarPFull,     // count kSoftmaxWarps: P is in TMEM, every S column has been read
    kBarOFull,
    kBarTmemFree,  // count kSoftmaxWarps: O is in registers, the accumulator columns may be overwritten
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

// tcgen05.wait::ld tied to the registers the loads wrote: nothing that reads them can be scheduled above it
__device__ __forceinline__ void wait_ld16(uint32_t (&r)[16]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
                 :
                 : "memory");
}

template <bool kBf16, bool kHasBias>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
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

    // (shuffled from lane 0 so that the compiler knows it is warp-uniform: roles, piece ranges and TMEM addresses
    // derived from it then live in uniform registers instead of R2UR + spills)
    const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
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
        mbar_init(bar(kBarQFull), 1);
        mbar_init(bar(kBarQEmpty), 1);
        for (int s = 0; s < kRingK; ++s) {
            mbar_init(bar(kBarKFull + s), 1);
            mbar_init(bar(kBarKEmpty + s), 1);
        }
        for (int s = 0; s < kRingV; ++s) {
            mbar_init(bar(kBarVFull + s), 1);
            mbar_init(bar(kBarVEmpty + s), 1);
        }
        mbar_init(bar(kBarSFull), 1);
        mbar_init(bar(kBarPFull), kSoftmaxWarps);
        mbar_init(bar(kBarOFull), 1);
        mbar_init(bar(kBarTmemFree), kSoftmaxWarps);
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
    // Programmatic dependent launch: everything above overlapped the tail of the previous kernel in the stream; its
    // results (Q, K, V come out of the layer's RoPE kernel) are visible, and whatever it still read of the output
    // buffer is done, after the wait.  The next kernel in the stream may then start its own prologue as this
    // grid's CTAs retire.  Both are no-ops under a plain launch.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");

    if (warp >= kSoftmaxWarps) setmaxnreg_dec<kRegsOther>();

    if (warp == kProducerWarp) {
        // =============================== TMA producer ===============================
        // warp-uniform control flow; only lane 0 issues
        uint32_t bc = 0;  // K/V boxes requested so far: K slot bc % kRingK, V slot bc % kRingV
        auto load_k = [&](const Tile& t, uint32_t box, int key0) {
            const uint32_t ks = box % kRingK;
            mbar_wait(bar(kBarKEmpty + ks), ((box / kRingK) & 1) ^ 1, wctx);
            if (lane == 0) {
                mbar_arrive_expect_tx(bar(kBarKFull + ks), kTileBytes);
                tma_load_4d(smem_base + Smem::k + ks * kTileBytes, &tm_k, bar(kBarKFull + ks), 0, key0, t.h, t.b);
            }
            __syncwarp();
        };
        auto load_v = [&](const Tile& t, uint32_t box, int key0) {
            const uint32_t vs = box % kRingV;
            mbar_wait(bar(kBarVEmpty + vs), ((box / kRingV) & 1) ^ 1, wctx);
            if (lane == 0) {
                mbar_arrive_expect_tx(bar(kBarVFull + vs), kTileBytes);
                tma_load_4d(smem_base + Smem::v + vs * kTileBytes, &tm_v, bar(kBarVFull + vs), 0, key0, t.h, t.b);
            }
            __syncwarp();
        };
        for (int n = 0; n < my_tiles; ++n) {
            const Tile t = decode_tile(p, g0 + n, q_tiles);
            mbar_wait(bar(kBarQEmpty), (n & 1) ^ 1, wctx);
            if (lane == 0) {
                mbar_arrive_expect_tx(bar(kBarQFull), kTileBytes);
                tma_load_4d(smem_base + Smem::q, &tm_q, bar(kBarQFull), 0, t.r0, t.h, t.b);
            }
            __syncwarp();
            if (n == 0 || t.head_start) {
                // a fresh strip: both K boxes before the V boxes, so that Q K^T can start on 3/5 of the tile's bytes
                // (every CTA of the grid starts with such a tile: the first 80 KiB per CTA are pure HBM time)
                load_k(t, bc, t.kb);
                load_k(t, bc + 1, t.kb + kBlockN);
                load_v(t, bc, t.kb);
                load_v(t, bc + 1, t.kb + kBlockN);
                bc += 2;
            } else {
                load_k(t, bc, t.kb + kBlockN);
                load_v(t, bc, t.kb + kBlockN);
                bc += 1;
            }
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
        // box stream position (mirrors the producer): tile n reads boxes first, first + 1
        uint32_t nb = 0;
#if RF_LOCAL_SKEW > 0
        // Two co-resident CTAs that start together stay in lockstep (both in their exponentials, then both waiting
        // for the tensor pipe).  The second CTA of an SM starts its chain half a tile period late instead.
        if ((RF_LOCAL_SKEW_ODD ? (blockIdx.x & 1) != 0 : blockIdx.x >= gridDim.x / 2) && gridDim.x > 148) {
            const long long t0 = clock64();
            while (clock64() - t0 < RF_LOCAL_SKEW) { }
        }
#endif
        for (int n = 0; n < my_tiles; ++n) {
            const bool fresh = n == 0 || decode_tile(p, g0 + n, q_tiles).head_start;
            const bool seg_end = n + 1 == my_tiles || decode_tile(p, g0 + n + 1, q_tiles).head_start;
            const uint32_t first = fresh ? nb : nb - 1;
            nb = first + 2;
            const uint32_t k0 = first % kRingK, k1 = (first + 1) % kRingK;
            const uint32_t v0 = first % kRingV, v1 = (first + 1) % kRingV;
            RF_STAMP(n, 0);
            mbar_wait(bar(kBarQFull), n & 1, wctx);
            mbar_wait2(bar(kBarKFull + k0), (first / kRingK) & 1, bar(kBarKFull + k1), ((first + 1) / kRingK) & 1, wctx);
            // the accumulator columns still hold O of the previous tile until its epilogue has read them
            if (n > 0) mbar_wait(bar(kBarTmemFree), (n - 1) & 1, wctx);
            tc_fence_after();
            RF_STAMP(n, 1);
            if (leader) {
                const uint32_t qbase = smem_base + Smem::q;
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    const uint32_t kbase = smem_base + Smem::k + (half ? k1 : k0) * kTileBytes;
#pragma unroll
                    for (int kk = 0; kk < kHeadDim / 16; ++kk)
                        mma_ss(t_s + half * kBlockN, make_smem_desc(qbase + kk * 32, 16, 1024, kSwizzle128B),
                               make_smem_desc(kbase + kk * 32, 16, 1024, kSwizzle128B), idesc_qk, kk > 0 ? 1u : 0u);
                }
                tc_commit(bar(kBarSFull));
                tc_commit(bar(kBarQEmpty));
                tc_commit(bar(kBarKEmpty + k0));
            }
            __syncwarp();
            if (seg_end) commit(bar(kBarKEmpty + k1));
            RF_STAMP(n, 2);
            mbar_wait2(bar(kBarVFull + v0), (first / kRingV) & 1, bar(kBarVFull + v1), ((first + 1) / kRingV) & 1, wctx);
            mbar_wait(bar(kBarPFull), n & 1, wctx);
            tc_fence_after();
            RF_STAMP(n, 3);
            if (leader) {
                // V box [128 keys][64] with d contiguous = MN-major B operand; a K=16 step is 2048 B
#pragma unroll
                for (int kk = 0; kk < kStrip / 16; ++kk) {
                    const uint32_t vbase = smem_base + Smem::v + (kk < 8 ? v0 : v1) * kTileBytes + (kk & 7) * 2048;
                    mma_ts(t_o, t_p + kk * 8, make_smem_desc(vbase, kTileBytes, 1024, kSwizzle128B), idesc_pv,
                           kk > 0 ? 1u : 0u);
                }
                tc_commit(bar(kBarOFull));
                tc_commit(bar(kBarVEmpty + v0));
            }
            __syncwarp();
            if (seg_end) commit(bar(kBarVEmpty + v1));
            RF_STAMP(n, 4);
        }
    } else if (warp < kSoftmaxWarps) {
        // =============================== softmax / epilogue ===============================
        setmaxnreg_inc<kRegsSoftmax>();
        const int part = warp >> 2;            // which half of the quad's live pieces
        const int quad = warp & 3;
        const int r = quad * 32 + lane;        // row inside the tile == TMEM lane
        int tid = threadIdx.x;                 // 0..255
        int seq_len = p.S;
        // pinned in registers: re-reading SR_TID.X / the parameter bank at the top of every tile put ~10 % of the
        // softmax warps' stall samples there (ncu)
        asm volatile("" : "+r"(tid), "+r"(seq_len));
        const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
        const uint32_t t_s = tmem_base + lane_base + kColS;
        const uint32_t t_p = tmem_base + lane_base + kColP;
        const uint32_t t_o = tmem_base + lane_base + kColO + part * kOutCols;
        const float c = p.scale_log2;
        const int band = p.wl + p.wr;          // live strip columns of row r: [r, r + band]
        float* xchg = reinterpret_cast<float*>(smem_gen + Smem::xchg);
        float* lsum = reinterpret_cast<float*>(smem_gen + Smem::lsum);
        float* xmaxs = reinterpret_cast<float*>(smem_gen + Smem::xmax);
        // P = 2^(x - m_ref) must fit the 16-bit type P is stored in (f16: 2^14 < 65504; bf16 has f32's range)
        constexpr float kTau = kBf16 ? 20.0f : 14.0f;
        const float* sbias = reinterpret_cast<const float*>(smem_gen + Smem::bias);
        const uint32_t row_bar = 1 + quad;     // named barrier of the two warps that share 32 rows
        // every (batch, head, row, half-row) output segment starts on a 32-byte boundary
        const int osz = p.out_dtype == 2 ? 4 : 2;
        const bool wide_ok = (reinterpret_cast<uintptr_t>(p.out) & 31) == 0 && ((p.o_sb * osz) & 31) == 0 &&
                             ((p.o_sh * osz) & 31) == 0 && ((p.o_ss * osz) & 31) == 0;

        // Band mask as an additive table instead of two compares and a select per element: f(col - r) = 0 on
        // [0, band], -inf elsewhere.  Four copies, copy k shifted by k entries, so that the lane of row r reads
        // its 16-byte groups f(col - r .. col - r + 3), col % 4 == 0, from copy r % 4 at an aligned address; the
        // copy stride is 8 mod 32 words, which makes the eight lanes of an LDS.128 phase hit distinct banks.
        {
            float* tb = reinterpret_cast<float*>(smem_gen + Smem::band);
            for (int i = tid; i < 4 * kBandStride; i += kSoftmaxThreads) {
                const int d = (i % kBandStride) - kBlockM - (i / kBandStride);
                tb[i] = (d >= 0 && d <= band) ? 0.f : -CUDART_INF_F;
            }
            named_bar_sync(5, kSoftmaxThreads);
        }
        const float* band_row = reinterpret_cast<const float*>(smem_gen + Smem::band) + (r & 3) * kBandStride + kBlockM - (r & ~3);

        // the quad's live pieces [p_lo, p_hi], split evenly between its two warps
        const int p_lo = 2 * quad;
        const int p_hi = min(kStrip / kPiece - 1, (32 * quad + 31 + band) / kPiece);
        const int n_pieces = p_hi - p_lo + 1;
        const int first_piece = p_lo + (part ? (n_pieces + 1) / 2 : 0);
        const int mine = part ? n_pieces / 2 : (n_pieces + 1) / 2;  // <= kMaxPieces
        // strip columns that are inside the band for every row of the warp
        const int lo_all = 32 * quad + 31, hi_all = 32 * quad + band;

        // per-column additive term of strip column tid (log2 domain): the pad bias, -inf for masked keys and for
        // keys outside [0, S)
        auto column_bias = [&](const Tile& t) -> float {
            const int key = t.kb + tid;
            float v = -CUDART_INF_F;
            if (key >= 0 && key < seq_len) {
                v = 0.f;
                if (kHasBias) {
                    const float raw = __ldg(pad_bias + static_cast<size_t>(t.b) * seq_len + key);
                    v = raw > kMaskThreshold ? raw * kLog2e : -CUDART_INF_F;
                }
            }
            return v;
        };
        // without a pad bias only the first and last tiles of a head need the column term (keys outside [0, S))
        auto needs_column_bias = [&](const Tile& t) { return kHasBias || t.kb < 0 || t.kb + kStrip > seq_len; };

        Tile cur = {};
        float bias_pref = 0.f;
        if (my_tiles > 0) {
            cur = decode_tile(p, g0, q_tiles);
            if (needs_column_bias(cur)) bias_pref = column_bias(cur);
        }

        // piece variants: 0 = inside the band for every row, no column term: raw scores, scale folded into the
        // exponent; 1 = band table; 2 = band table + column term
        // x[j] = scale * s[j] + add[j] for four consecutive columns
        auto addend4 = [&](int col, auto var_tag, float (&a)[4]) {
            constexpr int kVar = decltype(var_tag)::value;
            const float4 t4 = *reinterpret_cast<const float4*>(band_row + col);
            a[0] = t4.x; a[1] = t4.y; a[2] = t4.z; a[3] = t4.w;
            if (kVar == 2) {
                const float4 b4 = *reinterpret_cast<const float4*>(sbias + col);
                a[0] += b4.x; a[1] += b4.y; a[2] += b4.z; a[3] += b4.w;
            }
        };
        auto max_piece = [&](const uint32_t (&su)[16], int c0, auto var_tag, float& mx) {
            constexpr int kVar = decltype(var_tag)::value;
            if (kVar == 0) {
                float m4[4] = {-CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F};
#pragma unroll
                for (int j = 0; j < 16; j += 8) {
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4)
                        m4[q4] = max3(m4[q4], __uint_as_float(su[j + 2 * q4]), __uint_as_float(su[j + 2 * q4 + 1]));
                }
                mx = fmaxf(mx, fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * c);  // scale > 0 (host-checked)
            } else {
                float m2[2] = {mx, -CUDART_INF_F};
#pragma unroll
                for (int j = 0; j < 16; j += 4) {
                    float a[4];
                    addend4(c0 + j, var_tag, a);
                    m2[0] = max3(m2[0], fmaf(__uint_as_float(su[j]), c, a[0]), fmaf(__uint_as_float(su[j + 1]), c, a[1]));
                    m2[1] = max3(m2[1], fmaf(__uint_as_float(su[j + 2]), c, a[2]), fmaf(__uint_as_float(su[j + 3]), c, a[3]));
                }
                mx = fmaxf(m2[0], m2[1]);
            }
        };
        auto exp_piece = [&](const uint32_t (&su)[16], int c0, auto var_tag, float neg_m, uint64_t& sum2, float& xmax, uint32_t (&pk)[8]) {
            constexpr int kVar = decltype(var_tag)::value;
            const uint64_t c2 = bc2(c), negm2 = bc2(neg_m);
#pragma unroll
            for (int j = 0; j < 16; j += 4) {
                uint64_t a01 = negm2, a23 = negm2;
                if (kVar != 0) {
                    float a[4];
                    addend4(c0 + j, var_tag, a);
                    a01 = fadd2v(pk2(a[0], a[1]), negm2);  // masked: -inf stays -inf and gives exactly 0
                    a23 = fadd2v(pk2(a[2], a[3]), negm2);
                }
                float p0, p1, p2, p3;
                unpk2(ffma2v(pk2(__uint_as_float(su[j]), __uint_as_float(su[j + 1])), c2, a01), p0, p1);
                unpk2(ffma2v(pk2(__uint_as_float(su[j + 2]), __uint_as_float(su[j + 3])), c2, a23), p2, p3);
                xmax = max3(xmax, p0, p1);
                xmax = max3(xmax, p2, p3);
                if (kVar == 0 && ((j >> 1) & 7) < RF_LOCAL_POLY) {
                    exp2_poly2(p0, p1);
                } else {
                    p0 = ex2(p0);
                    p1 = ex2(p1);
                }
                if (kVar == 0 && (((j >> 1) + 1) & 7) < RF_LOCAL_POLY) {
                    exp2_poly2(p2, p3);
                } else {
                    p2 = ex2(p2);
                    p3 = ex2(p3);
                }
                sum2 = fadd2v(sum2, pk2(p0, p1));
                sum2 = fadd2v(sum2, pk2(p2, p3));
                pk[j >> 1] = pack2<kBf16>(p0, p1);
                pk[(j >> 1) + 1] = pack2<kBf16>(p2, p3);
            }
        };

        for (int n = 0; n < my_tiles; ++n) {
            const uint32_t par = n & 1;
            Tile nxt = cur;
            const bool use_cb = needs_column_bias(cur);  // uniform over the CTA
            if (use_cb) {
                // every read of the previous tile's column terms happened before its P-full, i.e. before this
                // thread's O-full wait returned
                reinterpret_cast<float*>(smem_gen + Smem::bias)[tid] = bias_pref;
                named_bar_sync(5, kSoftmaxThreads);
            }
            if (n + 1 < my_tiles) {
                advance_tile(p, nxt, q_tiles);
                if (needs_column_bias(nxt)) bias_pref = column_bias(nxt);
            }
            auto piece_var = [&](int i) {  // warp-uniform
                const int c0 = (first_piece + i) * kPiece;
                return use_cb ? 2 : (c0 >= lo_all && c0 + kPiece - 1 <= hi_all) ? 0 : 1;
            };

            RF_STAMP(n, 0);
            mbar_wait(bar(kBarSFull), par, wctx);
            tc_fence_after();
            RF_STAMP(n, 1);

            // ---- reference max: the maximum over ONE piece per thread, agreed between the two threads of a row ----
            // A separate max pass would read the 80 KiB of live S twice, five dependent tcgen05.ld round trips of
            // 100-200 clk each per thread and pass (the bandwidth is there -- 436 B/clk/SM with 16 warps,
            // tools/probes/tmem_rate.cu -- the latency is what costs).  So S is read once: exponentials are taken relative to m_ref <= the
            // row max, the true maximum is tracked on the way, and only if it turns out more than kTau above m_ref
            // (P would overflow its 16-bit type) or m_ref was useless (every sampled key masked) the two warps of the
            // quad redo the pass with the exact maximum.  A thread samples the piece of its share that is inside the
            // band for the most rows: the last one of the lower half, the first one of the upper half.
            auto piece_of = [&](int j) { return first_piece + (part ? j : mine - 1 - j); };  // processing order
            auto piece_var_of = [&](int j) { return piece_var(piece_of(j) - first_piece); };
            // Two piece buffers: the load of piece j + 1 is in flight while piece j is worked on (a tcgen05.ld round trip
            // is 100-200 clk under load, five of them in a row were a third of the pass).
            uint32_t su[2][16];
            tmem_ld16(t_s + piece_of(0) * kPiece, su[0]);
            wait_ld16(su[0]);
            if (mine > 1) tmem_ld16(t_s + piece_of(1) * kPiece, su[1]);  // lands during the exchange below
            {
                float mx = -CUDART_INF_F;
                const int c0 = piece_of(0) * kPiece;
                const int var = piece_var_of(0);
                if (var == 0) max_piece(su[0], c0, std::integral_constant<int, 0>{}, mx);
                else if (var == 1) max_piece(su[0], c0, std::integral_constant<int, 1>{}, mx);
                else max_piece(su[0], c0, std::integral_constant<int, 2>{}, mx);
                xchg[part * kBlockM + r] = mx;
            }
            named_bar_sync(row_bar, 32 * kParts);
            const float m_ref = fmaxf(xchg[r], xchg[kBlockM + r]);
            RF_STAMP(n, 2);

            // ---- P = 2^(x - m_ref), row sum, running max of x - m_ref ----
            uint64_t sum2 = 0;
            float xmax = -CUDART_INF_F;
            uint32_t pk[kMaxPieces][8];  // pk[j] = piece piece_of(j)
            auto run_piece = [&](const uint32_t (&sj)[16], int j, float neg_m) {
                const int c0 = piece_of(j) * kPiece;
                const int var = piece_var_of(j);
                if (var == 0) exp_piece(sj, c0, std::integral_constant<int, 0>{}, neg_m, sum2, xmax, pk[j]);
                else if (var == 1) exp_piece(sj, c0, std::integral_constant<int, 1>{}, neg_m, sum2, xmax, pk[j]);
                else exp_piece(sj, c0, std::integral_constant<int, 2>{}, neg_m, sum2, xmax, pk[j]);
            };
            // kPrefetched: piece 0 is in su[0] and the load of piece 1 into su[1] has been issued (first pass);
            // otherwise (redo with the exact maximum, rare) everything is loaded again
            auto run_pass = [&](float neg_m, auto prefetched_tag) {
                constexpr bool kPrefetched = decltype(prefetched_tag)::value;
                sum2 = 0;
                xmax = -CUDART_INF_F;
                if (!kPrefetched) {
                    tmem_ld16(t_s + piece_of(0) * kPiece, su[0]);
                    if (mine > 1) tmem_ld16(t_s + piece_of(1) * kPiece, su[1]);
                    wait_ld16(su[0]);
                }
#pragma unroll
                for (int j = 0; j < kMaxPieces; ++j) {
                    if (j < mine) {
                        if (j >= 1) {
                            wait_ld16(su[j & 1]);  // (waits for every load issued so far)
                            if (j + 1 < mine) tmem_ld16(t_s + piece_of(j + 1) * kPiece, su[(j + 1) & 1]);
                        }
                        run_piece(su[j & 1], j, neg_m);
                    }
                }
                float sum0, sum1;
                unpk2(sum2, sum0, sum1);
                lsum[part * kBlockM + r] = sum0 + sum1;
            };
            const float m_base = (m_ref == -CUDART_INF_F) ? 0.f : m_ref;
            run_pass(-m_base, std::true_type{});
            xmaxs[part * kBlockM + r] = xmax;
            // P overwrites S columns the other warp of the quad may still be reading: both are past their loads
            tc_fence_before();
            named_bar_sync(row_bar, 32 * kParts);
            tc_fence_after();
            {
                // both warps of the quad see the same per-row values, so they take the same branch
                const float xm_row = fmaxf(xmaxs[r], xmaxs[kBlockM + r]);
                const bool redo = xm_row > kTau || (xm_row < -1.0f && xm_row != -CUDART_INF_F);
                if (__any_sync(0xffffffffu, redo)) {
                    // exact row maximum (m_base + xm_row); a row with no live key keeps P = 0, l = 0
                    run_pass(xm_row == -CUDART_INF_F ? 0.f : -(m_base + xm_row), std::false_type{});
                    tc_fence_before();
                    named_bar_sync(row_bar, 32 * kParts);
                    tc_fence_after();
                }
            }
            RF_STAMP(n, 3);
#pragma unroll
            for (int j = 0; j < kMaxPieces; ++j)
                if (j < mine) tmem_st8(t_p + piece_of(j) * (kPiece / 2), pk[j]);
            {
                // the rest of the row is dead: exact zeros (V rows there are finite, 0 * v = 0)
                const uint32_t zero[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
                const int z0 = part ? p_hi + 1 : 0;
                const int z1 = part ? kStrip / kPiece : p_lo;
                for (int z = z0; z < z1; ++z) tmem_st8(t_p + z * (kPiece / 2), zero);
            }
            tc_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(kBarPFull));
            RF_STAMP(n, 4);

            // ---- epilogue: this thread owns 32 of the 64 output columns ----
            const float l_tot = lsum[r] + lsum[kBlockM + r];  // (the second row barrier ordered the exchange)
            const float inv = l_tot > 0.f ? __fdividef(1.0f, l_tot) : 0.f;
            const int row = cur.r0 + r;
            const size_t off = static_cast<size_t>(cur.b) * p.o_sb + static_cast<size_t>(cur.h) * p.o_sh +
                               static_cast<size_t>(row) * p.o_ss + part * kOutCols;
            mbar_wait(bar(kBarOFull), par, wctx);
            tc_fence_after();
            RF_STAMP(n, 5);
            uint32_t ou[kOutCols];
            tmem_ld16(t_o, reinterpret_cast<uint32_t(&)[16]>(ou[0]));
            tmem_ld16(t_o + 16, reinterpret_cast<uint32_t(&)[16]>(ou[16]));
            wait_ld16(reinterpret_cast<uint32_t(&)[16]>(ou[0]));
            wait_ld16(reinterpret_cast<uint32_t(&)[16]>(ou[16]));
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(kBarTmemFree));
            if (row < seq_len && part * kOutCols < p.d) {  // head_dim 32 runs zero-padded to 64 (FaParams::d)
                // A lane owns one row, so a warp-wide store touches 32 rows whatever its width: 32-byte stores (sm_100's
                // 256-bit st.global) halve the number of store instructions -- and of LSU passes, 32 per instruction --
                // against 16-byte ones.  wide_ok: base and strides keep every row segment 32-byte aligned (host-checked).
                if (p.out_dtype == 2) {
                    float* dst = static_cast<float*>(p.out) + off;
#pragma unroll
                    for (int u = 0; u < kOutCols / 8; ++u) {
                        uint32_t w[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) w[e] = __float_as_uint(__uint_as_float(ou[8 * u + e]) * inv);
                        if (wide_ok) {
                            st_global_v8(dst + 8 * u, w);
                        } else {
                            *reinterpret_cast<uint4*>(dst + 8 * u) = make_uint4(w[0], w[1], w[2], w[3]);
                            *reinterpret_cast<uint4*>(dst + 8 * u + 4) = make_uint4(w[4], w[5], w[6], w[7]);
                        }
                    }
                } else {
                    const bool out_bf16 = p.out_dtype == 0;
                    uint16_t* dst = static_cast<uint16_t*>(p.out) + off;
#pragma unroll
                    for (int u = 0; u < kOutCols / 16; ++u) {
                        uint32_t w[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const float a0 = __uint_as_float(ou[16 * u + 2 * e]) * inv;
                            const float a1 = __uint_as_float(ou[16 * u + 2 * e + 1]) * inv;
                            w[e] = out_bf16 ? pack2<true>(a0, a1) : pack2<false>(a0, a1);
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
            RF_STAMP(n, 6);
            cur = nxt;
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

int fa_fwd_sm100_local_grid(long long tiles, int sms) {
    const long long slots = static_cast<long long>(kCtasPerSm) * sms;
    return static_cast<int>(tiles < slots ? tiles : slots);
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
    // the carve-out must leave room for two CTAs' shared memory
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
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
    return cudaLaunchKernelEx(&cfg, kern, tmq, tmk, tmv, p, pad_bias);
}

}  // namespace rf
