// fa_internal.h -- device-side parameter blocks and launcher prototypes shared by the
// kernels (fa_fwd_sm100.cu, fa_fwd_simt.cu, fa_aux.cu) and the C-ABI layer (fa_api.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace rf {

// sets the calling thread's rf_last_error() text and returns `code` (shared by fa_api.cu and the graph C ABI)
int set_last_error(int code, const std::string& message);

constexpr float kLog2e = 1.4426950408889634f;
constexpr uint32_t kLaunchStatusMagic = 0x52460000u;  // == rfptx::kStatusMagic (ptx.cuh)
constexpr float kMaskThreshold = -30000.0f;  // reference attention.hpp:16

// Geometry of the tcgen05 kernel.
constexpr int kBlockM = 128;                  // query rows per UMMA tile
constexpr int kBlockN = 128;                  // keys per tile
constexpr int kQTilesPerCta = 2;              // two query tiles ping-pong on one SM
constexpr int kRowsPerCta = kBlockM * kQTilesPerCta;

// Key-tile classes produced by bias_prepare_kernel (one byte per (batch, 128-key tile)).
enum : uint8_t { kTileSkip = 0, kTileFull = 1, kTileMixed = 2 };

struct FaParams {
    int B, H, S;
    int d;                 // head_dim of the tensors: 64, or 32 (the tcgen05 kernels then run it zero-padded to 64:
                           // TMA boxes are 64 wide and the 32 columns outside the tensor arrive as zeros)
    int* status;           // launch status word (ptx.cuh: written only when a bounded wait times out), may be null
    int kv_begin, kv_end;  // key range [kv_begin, kv_end), 0 <= kv_begin <= kv_end <= S
    int wl, wr;            // window, -1 = unbounded
    float scale_log2;      // effective scale * log2(e)
    // padding bias in the log2 domain: bias2[b*bias_stride + j] = pad_bias*log2e, -inf if masked
    // or j >= S.  nullptr when the op has no pad_bias input.
    const float* bias2;
    const uint8_t* tile_flags;  // [B, n_kv_tiles], nullptr iff bias2 == nullptr
    int bias_stride;            // n_kv_tiles * 128
    int n_kv_tiles;             // ceil(S / 128)
    // output
    void* out;
    long long o_sb, o_sh, o_ss;  // element strides
    int out_dtype;               // rf_dtype
    float* o_partial;            // split-KV partials, contiguous [B,H,S,d] / [B,H,S]
    float* m_partial;
    float* l_partial;
    float* debug_scores;
    // work distribution (see fa_fwd_sm100.cu): 0 = one query-tile pair per CTA, 1 = persistent,
    // statically balanced slices of the flat (pair x key tile) space with in-kernel merge, 2 = persistent,
    // whole pairs dealt round-robin (padded batches: every CTA gets pairs of every sequence)
    int sched_mode;
    int total_pairs;     // B * H * pairs_per_head
    int pairs_per_head;  // ceil(S / 256)
    int tiles_per_pair;  // mode 1: upper bound of the key tiles any pair touches (virtual tiles per pair)
    float* part_o;       // mode 1 workspace: partials of pairs cut between two CTAs
    float* part_ml;
    int* part_flag;
    // Cauchy-Schwarz bound on the scores of a (query row, key tile): |q_i| * max_j |k_j|.  When it cannot
    // exceed the running reference max by more than the lazy-rescale threshold, the softmax warps skip the
    // row-max pass of that tile.  |q_i| is taken from the Q tile in shared memory inside the kernel; kmax
    // [B,H,n_kv_tiles] comes from k_tile_norms_kernel (fa_aux.cu); nullptr = test off.
    const float* kmax;
};

struct SimtParams {
    const void* q;
    const void* k;
    const void* v;
    long long q_sb, q_sh, q_ss, k_sb, k_sh, k_ss, v_sb, v_sh, v_ss;
    int in_dtype;
    int d;
    FaParams f;
};

// launchers (return cudaError_t of the launch)
// pdl: launch with programmatic stream serialization (when the previous kernel in the stream calls
// griddepcontrol.launch_dependents, this one's prologue overlaps its tail)
cudaError_t launch_fa_fwd_sm100(const CUtensorMap& tmq, const CUtensorMap& tmk, const CUtensorMap& tmv,
                                const FaParams& p, bool bf16, int grid, cudaStream_t stream, bool pdl = false);
// narrow-window kernel (fa_fwd_sm100_local.cu): wl + wr <= 127, one 256-key strip per query tile;
// reads the raw pad_bias [B,S] (nullable), needs no workspace
bool fa_fwd_sm100_local_covers(int wl, int wr);
int fa_fwd_sm100_local_grid(long long query_tiles, int sms);  // CTAs: two per SM, at most one per query tile
size_t fa_fwd_sm100_local_smem_bytes();
cudaError_t launch_fa_fwd_sm100_local(const CUtensorMap& tmq, const CUtensorMap& tmk, const CUtensorMap& tmv,
                                      const FaParams& p, const float* pad_bias, bool bf16, int grid,
                                      cudaStream_t stream);
// head_dim 128 kernel (fa_fwd_sm100_d128.cu): sched_mode 0, 1 or 2 as the head_dim-64 kernel
cudaError_t launch_fa_fwd_sm100_d128(const CUtensorMap& tmq, const CUtensorMap& tmk, const CUtensorMap& tmv,
                                     const FaParams& p, bool bf16, int grid, cudaStream_t stream);
size_t fa_fwd_sm100_d128_smem_bytes();
bool fa_fwd_sm100_d128_available();
size_t fa_fwd_sm100_smem_bytes();
size_t fa_fwd_sm100_partial_bytes(int grid, int head_dim);  // head_dim 64 (also for 32, zero-padded) or 128
size_t fa_fwd_sm100_flag_bytes(int grid);
void fa_fwd_sm100_partial_carve(void* base, void* flags, int grid, int head_dim, FaParams* p);
cudaError_t launch_fa_fwd_simt(const SimtParams& p, cudaStream_t stream, int* grid_ctas);

cudaError_t launch_bias_prepare(const float* pad_bias, int B, int S, float* bias2, uint8_t* tile_flags,
                                int n_kv_tiles, cudaStream_t stream);
// max_j |k_j| per (head, 128-key tile): the key side of the row-max skip test.  Triggers programmatic launch of the
// next kernel in the stream right away (the attention kernel's prologue overlaps it).
cudaError_t launch_k_tile_norms(const void* k, const long long k_strides[3], int dtype, int B, int H, int S, int d,
                                int n_kv_tiles, float* kmax, cudaStream_t stream);
cudaError_t launch_merge(const float* const* o_parts, const float* const* m_parts, const float* const* l_parts,
                         int G, long long rows, int d, void* out, int out_dtype, cudaStream_t stream);
// split-KV partial of an empty key block: O = 0, m = -inf, l = 0
cudaError_t launch_partial_neutral(float* o_part, float* m_part, float* l_part, long long rows, int d, cudaStream_t stream);
cudaError_t launch_rescale_partial(float* o_part, float* l_part, const float* m_part, const float* m_star,
                                   long long rows, int d, cudaStream_t stream);
cudaError_t launch_normalize(const float* o_sum, const float* l_sum, long long rows, int d, void* out,
                             int out_dtype, cudaStream_t stream);
cudaError_t launch_pad_bias_from_mask(const float* mask, float* bias, long long n, cudaStream_t stream);
cudaError_t launch_cast_from_f32(const float* src, void* dst, long long n, int dst_dtype, cudaStream_t stream);
cudaError_t launch_cast_to_f32(const void* src, float* dst, long long n, int src_dtype, cudaStream_t stream);

}  // namespace rf
