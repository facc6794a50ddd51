// gemm_sm100.cu -- the projections either side of the attention operator, hand-written for sm_100a:
//     y[m, n] = sum_k a[m, k] * w[n, k]          (nn.Linear: activations [M, K] times weights [N, K]^T)
// 16-bit operands (bf16 or f16), f32 accumulation in TMEM, 16-bit output, with the encoder's element-wise steps
// fused into the epilogue so that they never make a round trip through HBM (the step either
// side of the op; the fused node consumes the raw Q and the un-transposed K of this projection, rewrite.cpp:183,336-353):
//   RF_GEMM_EPI_NONE    plain store                                         (out-projection, MLP down-projection)
//   RF_GEMM_EPI_ROPE    y is the packed [tokens, 3, H, 64] QKV projection: rotary embedding ("rotate_half" pairing
//                       i, i + 32) on the Q and K thirds before the store   (replaces rf_rope_qkv)
//   RF_GEMM_EPI_GEGLU   w is the MLP up-projection [2*I, K] (input half, then gate half); the kernel computes both
//                       halves of a 128-column slice in one tile and stores act[m, j] = gelu(in) * gate, [M, I]
//                                                                            (replaces rf_geglu and its 2*I-wide buffer)
//   RF_GEMM_EPI_RESIDUAL y is the f32 residual stream: y += a w^T, the f32 accumulators added in place by TMA reduce-add
//                       (out-projection and MLP down-projection inside the encoder: the residual add leaves
//                       rf_add_layernorm, which then only reads the stream)
//
// One persistent CTA per SM, 6 warps:
//   warp 0      TMA producer: per 64-wide K block one 128 x 64 box of A and two 128 x 64 boxes of W (128B swizzle)
//               into a 4-stage ring, mbarrier complete_tx
//   warp 1      UMMA issuer: tcgen05.mma M128 N256 K16, four per K block, accumulators double-buffered in TMEM
//               (2 x 256 columns) so that the epilogue of tile t runs under the MMAs of tile t+1
//   warps 2-5   epilogue: tcgen05.ld (one accumulator row per thread), fused element-wise step, 16-byte stores
// The tensor pipe needs 512 clk per K block of a tile; the 48 KiB it consumes in that time are what bounds the
// kernel (L2 -> shared memory).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "../../include/rf_fa.h"
#include "../../include/rf_gemm.h"
#include "fa_internal.h"
#include "ptx.cuh"

namespace rf {
namespace {

using namespace rfptx;

constexpr int kBM = 128, kBK = 64;
constexpr int kBNMax = 256;                   // accumulator tile width: 256, or 192 where that saves a round of tiles
constexpr int kStages = 4;
constexpr int kABytes = kBM * kBK * 2;        // 16 KiB
constexpr int kStageBytes = kABytes + kBNMax * kBK * 2;  // A + W tile (two boxes of kBN / 2 rows)
constexpr int kThreads = 192;
constexpr int kEpiWarps = 4;
constexpr uint32_t kTmemCols = 512;           // two accumulators of up to 256 columns
constexpr int kCluster = 2;                   // CTA pair: adjacent row tiles of the same column tile share W
constexpr int kOutBoxBytes = 32 * 64 * 2;     // one TMA-store box: 32 rows x 64 columns of 16-bit output

struct GemmParams {
    int64_t M;
    int N, K;             // GEMM N (GEGLU: 2*I)
    int m_pairs, n_tiles; // row-tile pairs (256 rows), 256-column accumulator tiles
    int gate_row0;        // GEGLU: first weight row of the gate half (= I); otherwise unused
    const float* cos_t;   // ROPE: [S, 32]
    const float* sin_t;
    int S;                // ROPE: token t has position t % S
    int rope_cols;        // ROPE: columns [0, rope_cols) are rotated (the Q and K thirds)
    int head_major;       // ROPE: y is [3*H, tokens, 64] (3-D tensor map) instead of [tokens, 3*H*64]
    int out_bf16;         // ROPE: 16-bit type of the output (may differ from the operands': rf_gemm_epilogue.out_dtype)
    int* status;          // bounded-wait status word (ptx.cuh), may be null
};

struct Smem {
    static constexpr uint32_t tiles = 0;
    static constexpr uint32_t out = kStages * kStageBytes;               // [kEpiWarps][2] output boxes (128B swizzle)
    static constexpr uint32_t bars = out + kEpiWarps * 2 * kOutBoxBytes;
    static constexpr uint32_t bar_bytes = 256;
    static constexpr uint32_t total = bars + bar_bytes;
};
static_assert(Smem::total + 1024 <= 227 * 1024, "shared memory budget");
enum : uint32_t {
    kBarFull = 0,                        // [kStages]
    kBarEmpty = kBarFull + kStages,      // [kStages] count kCluster: both CTAs' MMAs are done with the stage
    kBarAccFull = kBarEmpty + kStages,   // [2]
    kBarAccEmpty = kBarAccFull + 2,      // [2] count kEpiWarps
    kNumBars = kBarAccEmpty + 2,
};
constexpr uint32_t kTmemSlotOff = kNumBars * 8;
constexpr uint32_t kWaitBlockOff = (kTmemSlotOff + 8 + 15) & ~15u;
static_assert(kWaitBlockOff + 16 <= Smem::bar_bytes, "barrier block too small");

__device__ __forceinline__ float gelu_erf(float v) { return 0.5f * v * (1.0f + erff(v * 0.70710678118654752f)); }

// Output staging: a 32-row x 64-column box per TMA store, rows of 128 bytes, 128B swizzle (16-byte chunk c of row i
// sits at chunk c ^ (i & 7): conflict-free for the row-per-lane writes, and the layout the tensor map expects).
template <bool kBf16>
__device__ __forceinline__ void stage16(uint32_t box, int lane, int chunk, const float (&v)[8]) {
    const uint32_t addr = box + lane * 128 + ((chunk ^ (lane & 7)) << 4);
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(pack2<kBf16>(v[0], v[1])),
                 "r"(pack2<kBf16>(v[2], v[3])), "r"(pack2<kBf16>(v[4], v[5])), "r"(pack2<kBf16>(v[6], v[7]))
                 : "memory");
}

template <bool kBf16, int kEpi, int kBN>
__global__ void __launch_bounds__(kThreads, 1)
gemm_nt_sm100_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_w,
                     const __grid_constant__ CUtensorMap tm_y, const GemmParams p) {
    static_assert(kBN == 256 || (kBN == 192 && kEpi != RF_GEMM_EPI_GEGLU), "tile widths");
    constexpr int kBBytes = kBN * kBK * 2;     // W tile: two boxes of kBN / 2 rows
    constexpr uint32_t kTxBytes = kABytes + kBBytes;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* smem_gen = smem_raw + (smem_base - smem_u32(smem_raw));
    const uint32_t bars = smem_base + Smem::bars;
    auto bar = [&](uint32_t i) { return bars + 8u * i; };
    volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(smem_gen + Smem::bars + kTmemSlotOff);
    const WaitCtx wctx{bars + kWaitBlockOff};

    const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();          // 0 / 1 inside the CTA pair
    const int k_blocks = (p.K + kBK - 1) / kBK;
    // the pair walks the (row-tile pair, column tile) space together; this CTA owns row tile 2 * pair + rank
    const int total_tiles = p.m_pairs * p.n_tiles;
    const int pair_id = blockIdx.x / kCluster, n_pairs = gridDim.x / kCluster;

    if (warp == 0 && lane == 0) {
        prefetch_tensormap(&tm_a);
        prefetch_tensormap(&tm_w);
        prefetch_tensormap(&tm_y);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(bar(kBarFull + s), 1);
            mbar_init(bar(kBarEmpty + s), kCluster);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(bar(kBarAccFull + s), 1);
            mbar_init(bar(kBarAccEmpty + s), kEpiWarps);
        }
        wait_block_init(wctx.block_smem, p.status);
        fence_barrier_init();
    }
    if (warp == 1) {
        tmem_alloc(smem_u32(const_cast<uint32_t*>(tmem_slot)), kTmemCols);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // the peer's barriers exist before anything of ours can reach them
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // programmatic dependent launch: the prologue above overlapped the previous kernel's tail (no-ops otherwise)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");

    if (warp == 0) {
        // =============================== TMA producer ===============================
        // A: this CTA's 128 rows.  W: each CTA of the pair loads one of the tile's two 128-row boxes and multicasts it
        // to both, so a K block costs 32 KiB of L2 reads per CTA instead of 48.
        uint32_t it = 0;  // K blocks loaded so far (ring position)
        for (int t = pair_id; t < total_tiles; t += n_pairs) {
            const int m0 = ((t / p.n_tiles) * kCluster + static_cast<int>(rank)) * kBM;
            const int nb = t % p.n_tiles;
            // weight rows of the tile's two 128-row boxes; box `rank` is ours to load
            const int w_row = kEpi == RF_GEMM_EPI_GEGLU ? (rank == 0 ? nb * 128 : p.gate_row0 + nb * 128)
                                                        : nb * kBN + static_cast<int>(rank) * (kBN / 2);
            for (int kb = 0; kb < k_blocks; ++kb, ++it) {
                const uint32_t s = it % kStages;
                mbar_wait(bar(kBarEmpty + s), ((it / kStages) & 1) ^ 1, wctx);
                if (lane == 0) {
                    const uint32_t dst = smem_base + Smem::tiles + s * kStageBytes;
                    mbar_arrive_expect_tx(bar(kBarFull + s), kTxBytes);
                    tma_load_2d(dst, &tm_a, bar(kBarFull + s), kb * kBK, m0);
                    tma_load_2d_multicast(dst + kABytes + rank * (kBBytes / 2), &tm_w, bar(kBarFull + s), kb * kBK, w_row,
                                          static_cast<uint16_t>((1u << kCluster) - 1u));
                }
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        // =============================== UMMA issuer ===============================
        const bool leader = elect_one() != 0;
        constexpr uint32_t idesc = make_idesc_f16(kBf16 ? 1u : 0u, 0, 0, kBM, kBN);
        uint32_t it = 0, tile_n = 0;
        for (int t = pair_id; t < total_tiles; t += n_pairs, ++tile_n) {
            const uint32_t acc = tile_n & 1;
            // the epilogue has drained this accumulator (two tiles ago)
            mbar_wait(bar(kBarAccEmpty + acc), ((tile_n >> 1) & 1) ^ 1, wctx);
            tc_fence_after();
            const uint32_t td = tmem_base + acc * kBNMax;
            for (int kb = 0; kb < k_blocks; ++kb, ++it) {
                const uint32_t s = it % kStages;
                mbar_wait(bar(kBarFull + s), (it / kStages) & 1, wctx);
                tc_fence_after();
                if (leader) {
                    const uint32_t a_base = smem_base + Smem::tiles + s * kStageBytes;
                    const uint32_t b_base = a_base + kABytes;
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk)
                        mma_ss(td, make_smem_desc(a_base + kk * 32, 16, 1024, kSwizzle128B),
                               make_smem_desc(b_base + kk * 32, 16, 1024, kSwizzle128B), idesc, (kb | kk) != 0 ? 1u : 0u);
                    // the stage is refilled by both CTAs' loads: tell both producers
                    tc_commit_multicast(bar(kBarEmpty + s), static_cast<uint16_t>((1u << kCluster) - 1u));
                    if (kb + 1 == k_blocks) tc_commit(bar(kBarAccFull + acc));
                }
                __syncwarp();
            }
        }
    } else {
        // =============================== epilogue ===============================
        const int quad = warp & 3;             // TMEM lane quadrant this warp may read
        const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
        const uint32_t out_base = smem_base + Smem::out + (warp - 2) * 2 * kOutBoxBytes;
        uint32_t boxes = 0;                    // output boxes this warp has stored so far (staging buffer = boxes & 1)
        // stage one 32 x 64 box (this warp's 32 rows), then one lane hands it to the TMA; rows and columns outside the
        // output tensor are clipped by the tensor map
        auto begin_box = [&]() -> uint32_t {
            if (lane == 0) bulk_wait_group_read<1>();  // the store that last read this buffer (two boxes ago) is done
            __syncwarp();
            return out_base + (boxes & 1) * kOutBoxBytes;
        };
        auto end_box = [&](int col, int row0) {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                if (kEpi == RF_GEMM_EPI_RESIDUAL) tma_reduce_add_2d(&tm_y, out_base + (boxes & 1) * kOutBoxBytes, col, row0);
                else if (kEpi == RF_GEMM_EPI_ROPE && p.head_major) tma_store_3d(&tm_y, out_base + (boxes & 1) * kOutBoxBytes, 0, row0, col >> 6);
                else tma_store_2d(&tm_y, out_base + (boxes & 1) * kOutBoxBytes, col, row0);
                bulk_commit_group();
            }
            ++boxes;
        };
        uint32_t tile_n = 0;
        for (int t = pair_id; t < total_tiles; t += n_pairs, ++tile_n) {
            const uint32_t acc = tile_n & 1;
            const int row0 = ((t / p.n_tiles) * kCluster + static_cast<int>(rank)) * kBM + quad * 32;  // this warp's rows
            const int nb = t % p.n_tiles;
            mbar_wait(bar(kBarAccFull + acc), (tile_n >> 1) & 1, wctx);
            tc_fence_after();
            const uint32_t ta = tmem_base + lane_base + acc * kBNMax;
            if (kEpi == RF_GEMM_EPI_NONE) {
#pragma unroll 1
                for (int c = 0; c < kBN / 64; ++c) {
                    uint32_t v[64];
                    tmem_ld32(ta + c * 64, reinterpret_cast<uint32_t(&)[32]>(v[0]));
                    tmem_ld32(ta + c * 64 + 32, reinterpret_cast<uint32_t(&)[32]>(v[32]));
                    tc_wait_ld();
                    const uint32_t box = begin_box();
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        float f[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(v[8 * u + e]);
                        stage16<kBf16>(box, lane, u, f);
                    }
                    end_box(nb * kBN + c * 64, row0);
                }
            } else if (kEpi == RF_GEMM_EPI_RESIDUAL) {
                // f32 boxes of 32 x 32 (128-byte rows): 16-byte chunk u of row `lane` holds columns 4u .. 4u + 3
#pragma unroll 1
                for (int c = 0; c < kBN / 32; ++c) {
                    uint32_t v[32];
                    tmem_ld32(ta + c * 32, v);
                    tc_wait_ld();
                    const uint32_t box = begin_box();
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const uint32_t addr = box + lane * 128 + ((u ^ (lane & 7)) << 4);
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v[4 * u]), "r"(v[4 * u + 1]),
                                     "r"(v[4 * u + 2]), "r"(v[4 * u + 3])
                                     : "memory");
                    }
                    end_box(nb * kBN + c * 32, row0);
                }
            } else if (kEpi == RF_GEMM_EPI_ROPE) {
                const int col0 = nb * kBN;
                const bool rotate = col0 < p.rope_cols;  // (a tile never straddles the K | V boundary: host-checked)
                float cs[32], sn[32];
                if (rotate) {
                    const int pos = static_cast<int>(static_cast<int64_t>(row0 + lane) % p.S);
                    const float4* cp = reinterpret_cast<const float4*>(p.cos_t + static_cast<int64_t>(pos) * 32);
                    const float4* sp = reinterpret_cast<const float4*>(p.sin_t + static_cast<int64_t>(pos) * 32);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const float4 c4 = __ldg(cp + u), s4 = __ldg(sp + u);
                        cs[4 * u] = c4.x; cs[4 * u + 1] = c4.y; cs[4 * u + 2] = c4.z; cs[4 * u + 3] = c4.w;
                        sn[4 * u] = s4.x; sn[4 * u + 1] = s4.y; sn[4 * u + 2] = s4.z; sn[4 * u + 3] = s4.w;
                    }
                }
#pragma unroll 1
                for (int hd = 0; hd < kBN / 64; ++hd) {   // one 64-wide head = one output box at a time
                    uint32_t lo[32], hi[32];
                    tmem_ld32(ta + hd * 64, lo);
                    tmem_ld32(ta + hd * 64 + 32, hi);
                    tc_wait_ld();
                    const uint32_t box = begin_box();
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        float f1[8], f2[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const float x1 = __uint_as_float(lo[8 * u + e]), x2 = __uint_as_float(hi[8 * u + e]);
                            f1[e] = rotate ? x1 * cs[8 * u + e] - x2 * sn[8 * u + e] : x1;
                            f2[e] = rotate ? x2 * cs[8 * u + e] + x1 * sn[8 * u + e] : x2;
                        }
                        if (p.out_bf16) {
                            stage16<true>(box, lane, u, f1);
                            stage16<true>(box, lane, 4 + u, f2);
                        } else {
                            stage16<false>(box, lane, u, f1);
                            stage16<false>(box, lane, 4 + u, f2);
                        }
                    }
                    end_box(col0 + hd * 64, row0);
                }
            } else {  // GEGLU: accumulator columns [0,128) = input half, [128,256) = gate half of output columns nb*128..
#pragma unroll 1
                for (int c = 0; c < 2; ++c) {
                    const uint32_t box = begin_box();
#pragma unroll 1
                    for (int h2 = 0; h2 < 2; ++h2) {
                        uint32_t xin[32], xg[32];
                        tmem_ld32(ta + c * 64 + h2 * 32, xin);
                        tmem_ld32(ta + 128 + c * 64 + h2 * 32, xg);
                        tc_wait_ld();
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            float f[8];
#pragma unroll
                            for (int e = 0; e < 8; ++e)
                                f[e] = gelu_erf(__uint_as_float(xin[8 * u + e])) * __uint_as_float(xg[8 * u + e]);
                            stage16<kBf16>(box, lane, h2 * 4 + u, f);
                        }
                    }
                    end_box(nb * 128 + c * 64, row0);
                }
            }
            // every tcgen05.ld of this accumulator has completed (wait::ld above): hand it back
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(kBarAccEmpty + acc));
        }
        if (lane == 0) bulk_wait_group<0>();  // the last stores have left shared memory and are visible
    }

    // ---------------- teardown ----------------
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // no CTA retires while its peer may still multicast into it
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, kTmemCols);
    }
}

// Launch status of the projections (ptx.cuh: written only when a bounded wait inside a CTA runs out, which then lets
// the kernel run through to its teardown with invalid output).  One word per device context; rf_gemm_launch_status
// reads and clears it.
__device__ int g_gemm_status;

int* gemm_status_ptr() {
    void* ptr = nullptr;
    if (cudaGetSymbolAddress(&ptr, g_gemm_status) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return static_cast<int*>(ptr);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                  const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* sym = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &sym, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            sym = nullptr;
        return reinterpret_cast<EncodeTiledFn>(sym);
    }();
    return fn;
}

// [rows, cols] row-major 16-bit matrix with `ld` elements between rows; box = 64 columns x box_rows rows, 128B swizzle
int make_map(CUtensorMap* tm, const void* base, int dtype, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
    const bool f32 = dtype == RF_DTYPE_F32;  // (the residual stream: 32-column boxes, still 128-byte rows)
    EncodeTiledFn enc = encode_fn();
    if (enc == nullptr) return set_last_error(RF_ERR_CUDA, "cuTensorMapEncodeTiled is unavailable (driver too old?)");
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * (f32 ? 4 : 2)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(f32 ? 32 : kBK), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult res = enc(tm, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : dtype == RF_DTYPE_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                             const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS) return set_last_error(RF_ERR_CUDA, "cuTensorMapEncodeTiled failed, CUresult " + std::to_string(res));
    return RF_OK;
}

template <bool kBf16, int kEpi, int kBN>
cudaError_t launch(const CUtensorMap& tma, const CUtensorMap& tmw, const CUtensorMap& tmy, const GemmParams& p, int grid,
                   cudaStream_t stream) {
    auto kern = gemm_nt_sm100_kernel<kBf16, kEpi, kBN>;
    const size_t smem = Smem::total + 1024;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = kCluster;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kern, tma, tmw, tmy, p);
}

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; }

}  // namespace
}  // namespace rf

extern "C" {

int rf_gemm_nt(const void* a, const void* w, void* y, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldw, int64_t ldy,
               int32_t dtype, const rf_gemm_epilogue* epi, void* stream) {
    using namespace rf;
    auto fail = [](int code, const std::string& msg) { return set_last_error(code, msg); };
    if (M < 0 || N < 0 || K <= 0) return fail(RF_ERR_SHAPE, "rf_gemm_nt: negative dimension");
    if (dtype != RF_DTYPE_BF16 && dtype != RF_DTYPE_F16) return fail(RF_ERR_ARG, "rf_gemm_nt: dtype must be bf16 or f16");
    if (M == 0 || N == 0) return RF_OK;
    if (a == nullptr || w == nullptr || y == nullptr) return fail(RF_ERR_ARG, "rf_gemm_nt: a/w/y is null");
    if (lda == 0) lda = K;
    if (ldw == 0) ldw = K;
    const int kind = epi != nullptr ? epi->kind : RF_GEMM_EPI_NONE;
    if (kind < RF_GEMM_EPI_NONE || kind > RF_GEMM_EPI_RESIDUAL) return fail(RF_ERR_ARG, "rf_gemm_nt: bad epilogue kind");
    const int64_t out_cols = kind == RF_GEMM_EPI_GEGLU ? N / 2 : N;
    if (ldy == 0) ldy = out_cols;
    if (!aligned16(a) || !aligned16(w) || !aligned16(y) || lda % 8 || ldw % 8 || ldy % (kind == RF_GEMM_EPI_RESIDUAL ? 4 : 8) || K % 8)
        return fail(RF_ERR_UNSUPPORTED, "rf_gemm_nt: pointers must be 16-byte aligned, K and the leading dimensions multiples of 8");
    if (M > (1ll << 31) - 2 * kBM || N > (1 << 30) || K > (1 << 30)) return fail(RF_ERR_ARG, "rf_gemm_nt: dimension too large");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t m_pairs = (M + kCluster * kBM - 1) / (kCluster * kBM);
    const int64_t slots = std::max(1, sms / kCluster);  // CTA pairs resident at once
    // Accumulator tile width: 256 columns, or 192 where that takes fewer (rounds of tiles) x (tile width) -- e.g. the
    // 768-wide projections at 8K tokens: 96 pair-tiles of 256 run as 2 rounds on 74 pairs, 128 of 192 too, in 3/4 of the time
    auto cost = [&](int bn) { return (N % bn) ? INT64_MAX : ((m_pairs * (N / bn) + slots - 1) / slots) * bn; };
    const bool can192 = kind != RF_GEMM_EPI_GEGLU && (kind != RF_GEMM_EPI_ROPE || (N / 3) % 192 == 0);
    const int bn = (can192 && cost(192) < cost(256)) ? 192 : 256;
    if (N % bn) return fail(RF_ERR_UNSUPPORTED, "rf_gemm_nt: N must be a multiple of 256 (or of 192)");
    GemmParams p{};
    p.M = M;
    p.N = static_cast<int>(N);
    p.K = static_cast<int>(K);
    p.m_pairs = static_cast<int>(m_pairs);
    p.n_tiles = static_cast<int>(N / bn);
    p.status = gemm_status_ptr();
    if (kind == RF_GEMM_EPI_ROPE) {
        if (epi->cos_table == nullptr || epi->sin_table == nullptr || epi->S <= 0 || epi->head_dim != 64)
            return fail(RF_ERR_ARG, "rf_gemm_nt: the RoPE epilogue needs cos/sin tables [S, 32], S > 0 and head_dim 64");
        if (N % 3 || (N / 3) % bn)
            return fail(RF_ERR_UNSUPPORTED, "rf_gemm_nt: the RoPE epilogue needs a packed QKV width 3 * hidden with hidden a multiple of the tile width");
        p.cos_t = epi->cos_table;
        p.sin_t = epi->sin_table;
        p.S = static_cast<int>(epi->S);
        p.rope_cols = static_cast<int>(N / 3 * 2);
        if (epi->out_dtype != 0 && epi->out_dtype != 1 + RF_DTYPE_BF16 && epi->out_dtype != 1 + RF_DTYPE_F16)
            return fail(RF_ERR_ARG, "rf_gemm_nt: bad out_dtype");
        p.out_bf16 = epi->out_dtype == 0 ? (dtype == RF_DTYPE_BF16) : (epi->out_dtype == 1 + RF_DTYPE_BF16);
    } else if (kind == RF_GEMM_EPI_GEGLU) {
        if ((N / 2) % 128) return fail(RF_ERR_UNSUPPORTED, "rf_gemm_nt: the GeGLU epilogue needs an intermediate width that is a multiple of 128");
        p.gate_row0 = static_cast<int>(N / 2);
    }
    CUtensorMap tma, tmw, tmy;
    int rc = make_map(&tma, a, dtype, M, K, lda, 128);
    if (rc != RF_OK) return rc;
    if ((rc = make_map(&tmw, w, dtype, N, K, ldw, bn / 2)) != RF_OK) return rc;
    if (kind == RF_GEMM_EPI_ROPE && epi->head_major) {
        // [3*H, tokens, 64]: one 32-token x 64 box per (head, 32 tokens)
        EncodeTiledFn enc = encode_fn();
        if (enc == nullptr) return fail(RF_ERR_CUDA, "cuTensorMapEncodeTiled is unavailable (driver too old?)");
        const cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(M), static_cast<cuuint64_t>(N / 64)};
        const cuuint64_t strides[2] = {128, static_cast<cuuint64_t>(M) * 128};
        const cuuint32_t box[3] = {64, 32, 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        const CUresult res = enc(&tmy, dtype == RF_DTYPE_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, y,
                                 dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (res != CUDA_SUCCESS) return fail(RF_ERR_CUDA, "cuTensorMapEncodeTiled failed, CUresult " + std::to_string(res));
        p.head_major = 1;
    } else if ((rc = make_map(&tmy, y, kind == RF_GEMM_EPI_RESIDUAL ? RF_DTYPE_F32 : dtype, M, out_cols, ldy, 32)) != RF_OK) {
        return rc;
    }
    // one CTA pair per two SMs, persistent over the (row-tile pair, column tile) space
    const int grid = kCluster * static_cast<int>(std::min<int64_t>(static_cast<int64_t>(p.m_pairs) * p.n_tiles, slots));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const bool bf = dtype == RF_DTYPE_BF16;
    cudaError_t e;
    switch (kind) {
        case RF_GEMM_EPI_ROPE:
            if (bn == 192)
                e = bf ? launch<true, RF_GEMM_EPI_ROPE, 192>(tma, tmw, tmy, p, grid, st) : launch<false, RF_GEMM_EPI_ROPE, 192>(tma, tmw, tmy, p, grid, st);
            else
                e = bf ? launch<true, RF_GEMM_EPI_ROPE, 256>(tma, tmw, tmy, p, grid, st) : launch<false, RF_GEMM_EPI_ROPE, 256>(tma, tmw, tmy, p, grid, st);
            break;
        case RF_GEMM_EPI_GEGLU:
            e = bf ? launch<true, RF_GEMM_EPI_GEGLU, 256>(tma, tmw, tmy, p, grid, st) : launch<false, RF_GEMM_EPI_GEGLU, 256>(tma, tmw, tmy, p, grid, st);
            break;
        case RF_GEMM_EPI_RESIDUAL:
            if (bn == 192)
                e = bf ? launch<true, RF_GEMM_EPI_RESIDUAL, 192>(tma, tmw, tmy, p, grid, st) : launch<false, RF_GEMM_EPI_RESIDUAL, 192>(tma, tmw, tmy, p, grid, st);
            else
                e = bf ? launch<true, RF_GEMM_EPI_RESIDUAL, 256>(tma, tmw, tmy, p, grid, st) : launch<false, RF_GEMM_EPI_RESIDUAL, 256>(tma, tmw, tmy, p, grid, st);
            break;
        default:
            if (bn == 192)
                e = bf ? launch<true, RF_GEMM_EPI_NONE, 192>(tma, tmw, tmy, p, grid, st) : launch<false, RF_GEMM_EPI_NONE, 192>(tma, tmw, tmy, p, grid, st);
            else
                e = bf ? launch<true, RF_GEMM_EPI_NONE, 256>(tma, tmw, tmy, p, grid, st) : launch<false, RF_GEMM_EPI_NONE, 256>(tma, tmw, tmy, p, grid, st);
    }
    if (e != cudaSuccess) return fail(RF_ERR_CUDA, std::string("rf_gemm_nt launch: ") + cudaGetErrorString(e));
    return RF_OK;
}

int rf_gemm_launch_status(void* stream_v) {
    using namespace rf;
    cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
    int* ptr = gemm_status_ptr();
    if (ptr == nullptr) return set_last_error(RF_ERR_CUDA, "rf_gemm_launch_status: no CUDA device");
    uint32_t word = 0;
    cudaError_t e = cudaMemcpyAsync(&word, ptr, sizeof(word), cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return set_last_error(RF_ERR_CUDA, std::string("rf_gemm_launch_status: ") + cudaGetErrorString(e));
    if ((word & 0xffff0000u) != kLaunchStatusMagic) return RF_OK;
    cudaMemsetAsync(ptr, 0, sizeof(word), stream);  // reported once
    return set_last_error(RF_ERR_DEVICE_TIMEOUT, "a barrier wait inside a projection CTA timed out (CTA " + std::to_string(word & 0xfffu) +
                                                     "); the output of that launch is invalid");
}

}  // extern "C"
