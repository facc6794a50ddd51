// fa_api.cu -- the C ABI declared in include/rf_fa.h: validation with the reference's error
// behaviour, TMA tensor-map construction, kernel selection, workspace layout, the host-buffer
// entry point and the FusedFlashAttention op dispatch (reference interpreter.cpp:308-318).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <chrono>
#include <cstdlib>
#include <string>

#include "../../include/rf_fa.h"
#include "fa_internal.h"
#include "host_cast.h"

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char* what) {
    return fail(RF_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// Resolved once through the runtime (no link-time dependency on libcuda).
EncodeTiledFn encode_tiled_fn() {
    static EncodeTiledFn fn = [] {
        void* sym = nullptr;
        cudaDriverEntryPointQueryResult qres;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &sym, cudaEnableDefault, &qres) != cudaSuccess ||
            qres != cudaDriverEntryPointSuccess)
            sym = nullptr;
        return reinterpret_cast<EncodeTiledFn>(sym);
    }();
    return fn;
}

struct Resolved {
    int64_t qs[3], ks[3], vs[3], os[3];
    double scale;  // effective
    int64_t kv_begin, kv_end;
    int64_t wl, wr;  // saturated windows: -1 = unbounded (any negative bound, or one that reaches past the sequence)
    bool partial;
};

void resolve_strides(const int64_t in[3], int64_t out[3], int64_t H, int64_t S, int64_t d) {
    if (in[2] == 0) {  // contiguous [B,H,S,d]
        out[0] = H * S * d;
        out[1] = S * d;
        out[2] = d;
    } else {
        out[0] = in[0];
        out[1] = in[1];
        out[2] = in[2];
    }
}

// Checks in the reference's order (attention.cpp:14-21 rank/shape are structural here;
// pad_bias shape is checked by the host-tensor entry points), then this build's own.
int validate(const rf_fa_params* p, Resolved* r) {
    if (p == nullptr) return fail(RF_ERR_ARG, "params is null");
    if (p->B < 0 || p->H < 0 || p->S < 0 || p->d < 0) return fail(RF_ERR_SHAPE, "negative dimension");
    if (p->d != 32 && p->d != 64 && p->d != 128)
        return fail(RF_ERR_HEAD_DIM, "head_dim must be one of {32, 64, 128}, got " + std::to_string(p->d));
    if (p->dtype != RF_DTYPE_BF16 && p->dtype != RF_DTYPE_F16)
        return fail(RF_ERR_ARG, "dtype must be bf16 or f16");
    if (p->out_dtype < RF_DTYPE_BF16 || p->out_dtype > RF_DTYPE_F32) return fail(RF_ERR_ARG, "bad out_dtype");
    if (p->kernel < RF_KERNEL_AUTO || p->kernel > RF_KERNEL_SIMT) return fail(RF_ERR_ARG, "bad kernel selector");
    if (p->flags != 0) return fail(RF_ERR_ARG, "flags is reserved and must be 0");
    // any negative window bound means "unbounded", as in attention.cpp:132-136
    // B and H index grid.y / grid.z of the auxiliary kernels (65535 each)
    if (p->S > (1ll << 30) || p->B > 65535 || p->H > 65535) return fail(RF_ERR_ARG, "dimension too large");
    r->partial = p->o_partial != nullptr;
    if (r->partial && (p->m_partial == nullptr || p->l_partial == nullptr))
        return fail(RF_ERR_ARG, "split-KV needs o_partial, m_partial and l_partial");
    const bool empty = p->B == 0 || p->H == 0 || p->S == 0;
    if (!empty) {
        if (p->q == nullptr || p->k == nullptr || p->v == nullptr) return fail(RF_ERR_ARG, "q/k/v is null");
        if (!r->partial && p->out == nullptr) return fail(RF_ERR_ARG, "out is null");
    }
    resolve_strides(p->q_stride, r->qs, p->H, p->S, p->d);
    resolve_strides(p->k_stride, r->ks, p->H, p->S, p->d);
    resolve_strides(p->v_stride, r->vs, p->H, p->S, p->d);
    resolve_strides(p->o_stride, r->os, p->H, p->S, p->d);
    r->scale = p->scale != 0.0 ? p->scale : 1.0 / std::sqrt(static_cast<double>(p->d));  // attention.cpp:34-36
    if (!std::isfinite(r->scale)) return fail(RF_ERR_ARG, "scale is not finite");
    // any negative bound means unbounded (attention.cpp:132-136); so does one of S or more, which keeps every
    // later sum of the two inside int64 whatever the caller passes for "no limit"
    r->wl = (p->window_left < 0 || p->window_left >= p->S) ? -1 : p->window_left;
    r->wr = (p->window_right < 0 || p->window_right >= p->S) ? -1 : p->window_right;
    r->kv_begin = p->kv_begin;
    r->kv_end = p->kv_end;
    // "both 0" means the whole sequence only for a full call; a split-KV partial takes its range literally, so
    // an honestly empty key block [0, 0) yields the neutral element of the merge (m = -inf, l = 0, O = 0)
    if (!r->partial && r->kv_begin == 0 && r->kv_end == 0) r->kv_end = p->S;
    if (r->kv_begin < 0 || r->kv_end > p->S || r->kv_begin > r->kv_end)
        return fail(RF_ERR_ARG, "kv range must satisfy 0 <= kv_begin <= kv_end <= S");
    return RF_OK;
}

// Streams (and the one event) of the host entry point, cached per calling thread and device:
// creating and destroying four streams costs ~0.3 ms per call otherwise.  They carry no data
// between calls; rf_fa_host_release() destroys the calling thread's.
constexpr int kHostStreams = 4;
constexpr int kMaxDevices = 64;
struct HostCtx {
    cudaStream_t streams[kHostStreams] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t ready = nullptr;
    int n = 0;
    // host-side cast (host_cast.h): page-locked 16-bit staging, one slot per stream, and the event that says a
    // slot's upload has been read
    uint16_t* stage[kHostStreams] = {nullptr, nullptr, nullptr, nullptr};
    size_t stage_bytes = 0;  // per slot
    cudaEvent_t uploaded[kHostStreams] = {nullptr, nullptr, nullptr, nullptr};
};
thread_local HostCtx g_host_ctx[kMaxDevices];

// Which way large rf_fa_fwd_host calls round their inputs: seconds per byte of the best call seen each way.  The
// first three eligible calls go through the host cores (the first pays for the pool and the page-locked staging),
// the next three through the device, after that the faster way wins (ties to the host: fewer bytes on the link)
// and every 16th call tries the other way again, so a choice made on a noisy start does not stick.
// RF_FA_HOST_CAST=1 pins the host way, =0 the device way.
struct HostCastChoice {
    std::mutex m;
    double best[2] = {1e30, 1e30};  // [0] device cast, [1] host cast
    int calls[2] = {0, 0};
    bool want_host() {
        static const int pinned = [] {
            const char* env = std::getenv("RF_FA_HOST_CAST");
            return env == nullptr ? -1 : (env[0] == '0' ? 0 : 1);
        }();
        if (pinned >= 0) return pinned == 1;
        std::lock_guard<std::mutex> lk(m);
        if (calls[1] < 3) return true;
        if (calls[0] < 3) return false;
        const bool host = best[1] <= best[0];
        return ((calls[0] + calls[1]) % 16 == 15) ? !host : host;
    }
    void record(bool host, double s_per_byte) {
        std::lock_guard<std::mutex> lk(m);
        const int i = host ? 1 : 0;
        ++calls[i];
        best[i] = std::min(best[i], s_per_byte);
    }
};
HostCastChoice g_cast_choice;
// bytes rf_fa_fwd_host moved over the link on the calling thread, cumulative (rf_fa_host_transfer_counters)
thread_local uint64_t g_h2d_total = 0, g_d2h_total = 0, g_host_calls = 0;

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; }
bool strides_ok_tma(const int64_t s[3]) { return s[0] > 0 && s[1] > 0 && s[2] > 0 && s[0] % 8 == 0 && s[1] % 8 == 0 && s[2] % 8 == 0; }

// Can a tcgen05 kernel take this call?  (scale > 0, TMA-compatible layout.)  head_dim 64 has the tuned kernels,
// 32 runs through the same kernels zero-padded to 64 (the TMA box is 64 wide, the 32 columns outside the tensor
// arrive as zeros: the call is exponential-bound either way), 128 has its own kernel (fa_fwd_sm100_d128.cu).
bool tcgen05_eligible(const rf_fa_params* p, const Resolved& r, std::string* why) {
    if (p->d == 128 && !rf::fa_fwd_sm100_d128_available()) {
        *why = "head_dim 128 tcgen05 kernel is not built in";
        return false;
    }
    if (!(r.scale > 0.0)) {
        *why = "tcgen05 kernel needs scale > 0";
        return false;
    }
    if (!aligned16(p->q) || !aligned16(p->k) || !aligned16(p->v) || !strides_ok_tma(r.qs) ||
        !strides_ok_tma(r.ks) || !strides_ok_tma(r.vs)) {
        *why = "q/k/v must be 16-byte aligned with strides that are multiples of 8 elements";
        return false;
    }
    if (!r.partial) {
        const int64_t al = p->out_dtype == RF_DTYPE_F32 ? 4 : 8;
        if (!aligned16(p->out) || r.os[0] % al || r.os[1] % al || r.os[2] % al) {
            *why = "out rows must be 16-byte aligned";
            return false;
        }
    } else if (!aligned16(p->o_partial)) {
        *why = "o_partial must be 16-byte aligned";
        return false;
    }
    return true;
}

int select_kernel(const rf_fa_params* p, const Resolved& r, int* kernel) {
    std::string why;
    const bool ok = tcgen05_eligible(p, r, &why);
    if (p->kernel == RF_KERNEL_TCGEN05 && !ok) return fail(RF_ERR_UNSUPPORTED, why);
    *kernel = (p->kernel == RF_KERNEL_SIMT || !ok) ? RF_KERNEL_SIMT : RF_KERNEL_TCGEN05;
    return RF_OK;
}

int64_t n_kv_tiles(int64_t S) { return (S + rf::kBlockN - 1) / rf::kBlockN; }
size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// SM count of the current device (148 on B200; also the answer when no device is visible, so
// that workspace queries work on a CPU-only build box).
int sm_count_or_default() {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0)
        return sms;
    cudaGetLastError();  // clear the sticky "no device" status
    return 148;
}

constexpr size_t kStatusBlockBytes = 256;  // head of every tcgen05 workspace: the launch status word (ptx.cuh)

struct Plan {
    int kernel;
    bool local;       // tcgen05 only: the narrow-window kernel takes the call
    bool d128;        // tcgen05 only: head_dim 128 kernel
    int sched_mode;   // tcgen05 only
    int grid;         // CTAs
    int64_t total_pairs, pairs_per_head, tiles_per_pair;
    size_t status_bytes;
    // Split-pair flags of the persistent balanced schedule: ALWAYS the first block after the status block in a
    // workspace that has anything after the status block at all, whatever the plan, so that plans of different
    // shapes sharing one workspace never put data where another plan keeps flags.  The flags are zero between
    // launches: a plan zeroes them with its first launch, the kernel leaves them as it found them.
    size_t sched_flag_bytes;
    size_t bias_bytes, flag_bytes_bias, part_bytes;
    size_t kmax_bytes;  // row-max skip test, key side: largest key norm per (head, key tile) (dense kernel, S >= 1024)
    size_t tail_bytes() const { return bias_bytes + flag_bytes_bias + part_bytes + kmax_bytes; }
    size_t workspace_bytes() const { return status_bytes + (tail_bytes() > 0 ? sched_flag_bytes + tail_bytes() : 0); }
};

Plan make_plan(const rf_fa_params* p, const Resolved& r, int kernel) {
    Plan pl{};
    pl.kernel = kernel;
    if (p->B == 0 || p->H == 0 || p->S == 0) return pl;
    if (kernel != RF_KERNEL_TCGEN05) {
        pl.grid = static_cast<int>(((p->S + 31) / 32) * p->H * p->B);
        return pl;
    }
    pl.status_bytes = kStatusBlockBytes;
    const int sms = sm_count_or_default();
    pl.sched_flag_bytes = align_up(rf::fa_fwd_sm100_flag_bytes(sms), 256);
    pl.pairs_per_head = (p->S + rf::kRowsPerCta - 1) / rf::kRowsPerCta;
    pl.total_pairs = pl.pairs_per_head * p->H * p->B;
    if (r.partial && r.kv_begin == r.kv_end) {  // empty key block: one fill kernel, no workspace
        pl.status_bytes = 0;
        return pl;
    }
    // narrow sliding window (the reference's local layers): one 256-key strip per query tile, no
    // workspace.  RF_FA_LOCAL=0 routes these calls to the general kernel (A/B measurements).
    static const bool local_enabled = [] {
        const char* env = std::getenv("RF_FA_LOCAL");
        return env == nullptr || env[0] != '0';
    }();
    if (p->d != 128 && local_enabled && !r.partial && r.kv_begin == 0 && r.kv_end == p->S && r.wl >= 0 && r.wr >= 0 &&
        r.wl < rf::kBlockN && r.wr < rf::kBlockN && r.wl + r.wr < rf::kBlockN &&
        rf::fa_fwd_sm100_local_covers(static_cast<int>(r.wl), static_cast<int>(r.wr))) {
        pl.local = true;
        const int64_t tiles = static_cast<int64_t>(p->B) * p->H * ((p->S + rf::kBlockM - 1) / rf::kBlockM);
        pl.grid = rf::fa_fwd_sm100_local_grid(tiles, sm_count_or_default());  // two CTAs per SM
        return pl;
    }
    pl.grid = static_cast<int>(pl.total_pairs);
    if (p->pad_bias != nullptr) {
        const size_t nt = static_cast<size_t>(n_kv_tiles(p->S));
        pl.bias_bytes = align_up(static_cast<size_t>(p->B) * nt * rf::kBlockN * sizeof(float), 256);
        pl.flag_bytes_bias = align_up(static_cast<size_t>(p->B) * nt, 256);
    }
    // more query-tile pairs than SMs: persistent, statically balanced schedule over the flat
    // (pair x key tile) space.  tiles_per_pair bounds the key tiles any pair touches.
    {
        const int64_t t_begin = r.kv_begin / rf::kBlockN;
        const int64_t t_end = (r.kv_end + rf::kBlockN - 1) / rf::kBlockN;
        int64_t tiles = t_end - t_begin;
        if (r.wl >= 0 && r.wr >= 0) {
            const int64_t span = rf::kRowsPerCta + r.wl + r.wr;  // keys a pair can see
            tiles = std::min<int64_t>(tiles, (span + rf::kBlockN - 1) / rf::kBlockN + 1);
        }
        pl.tiles_per_pair = std::max<int64_t>(tiles, 1);
    }
    // Row-max skip test (fa_fwd_sm100.cu): max |k_j| per key tile from a pre-pass over K (4 B per (head, tile));
    // |q_i| is taken inside the kernel.  RF_FA_SKIP_MAX=0 turns it off (A/B measurements).
    static const bool skip_max_enabled = [] {
        const char* env = std::getenv("RF_FA_SKIP_MAX");
        return env == nullptr || env[0] != '0';
    }();
    if (p->d == 128) pl.d128 = true;  // own kernel (fa_fwd_sm100_d128.cu): same schedules, same row-max skip
    if (skip_max_enabled && p->S >= 1024)
        pl.kmax_bytes = align_up(static_cast<size_t>(p->B) * p->H * n_kv_tiles(p->S) * sizeof(float), 256);
    if (!r.partial && pl.total_pairs > sms) {
        pl.sched_mode = 1;
        pl.grid = sms;
        pl.part_bytes = align_up(rf::fa_fwd_sm100_partial_bytes(pl.grid, pl.d128 ? 128 : 64), 256);
        // Batches with many pairs per SM are dealt round-robin as whole pairs instead (mode 2), for two reasons.
        // (i) CTAs that run at the same time work on neighbouring pairs, i.e. on a handful of heads whose K/V
        // stay in L2; contiguous slices put the 148 CTAs on as many different heads at once, and with B*H*S*256 B
        // of K/V beyond the L2 that costs 5-15 % (B=4, S=16K: 785 -> 899 TFLOP/s).  (ii) With padding, sequence
        // lengths live on the device and usually differ: equal slices of the virtual (pair x tile) space leave
        // the CTAs that drew short sequences idle (efficiency ~ mean/max length), round-robin gives every CTA
        // pairs of every sequence.  No pair is split; the price is a last partial round ...
        // A single sequence keeps mode 1 (B=1, S=16K: 921 vs 799 TFLOP/s).
        // RF_FA_SCHED_MODE=1|2 forces a schedule (developer aid for A/B measurements)
        static const int forced = [] {
            const char* env = std::getenv("RF_FA_SCHED_MODE");
            return env != nullptr ? std::atoi(env) : 0;
        }();
        // ... chosen when that last round wastes little: its idle share is rounds*sms/pairs - 1 (at most 5 % for
        // dense batches, where the gain is L2 locality, at most 10 % for padded ones, where lengths differ)
        const int64_t rounds = (pl.total_pairs + sms - 1) / sms;
        const double waste = static_cast<double>(rounds * sms) / static_cast<double>(pl.total_pairs) - 1.0;
        // A single long sequence also goes round-robin once its K/V no longer sit in the L2 next to each other: with
        // contiguous slices all H heads are in flight at once (S = 32K: 100 MB of K/V on a 126 MB L2), round-robin
        // keeps the 148 CTAs on one or two heads (S = 32K: 3.24 vs 3.32-3.39 ms although its last round idles 6 %;
        // at 16K, 50 MB, contiguous slices stay ahead: 0.79 vs 0.90 ms).
        const double kv_bytes = 4.0 * static_cast<double>(p->B) * p->H * p->S * p->d;  // K and V, 16-bit
        const bool kv_beyond_l2 = kv_bytes > 64.0e6;
        const bool want2 = (p->B > 1 || kv_beyond_l2) && pl.total_pairs >= 4ll * sms &&
                           waste <= ((p->pad_bias != nullptr || (p->B == 1 && kv_beyond_l2)) ? 0.10 : 0.05);
        if (forced == 2 || (forced == 0 && want2)) {
            pl.sched_mode = 2;
            pl.part_bytes = 0;
        }
    }
    return pl;
}

int make_tmap(CUtensorMap* tm, const void* base, int dtype, int64_t d, int64_t S, int64_t H, int64_t B,
              const int64_t st[3]) {
    EncodeTiledFn enc = encode_tiled_fn();
    if (enc == nullptr) return fail(RF_ERR_CUDA, "cuTensorMapEncodeTiled is unavailable (driver too old?)");
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(S), static_cast<cuuint64_t>(H),
                                static_cast<cuuint64_t>(B)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(st[2]) * 2, static_cast<cuuint64_t>(st[1]) * 2,
                                   static_cast<cuuint64_t>(st[0]) * 2};
    // box: 64 head-dim columns x 128 rows.  d = 32: the upper 32 columns are out of bounds and arrive as zeros;
    // d = 128: a tile is two boxes (columns [0,64) and [64,128))
    const cuuint32_t box[4] = {64, static_cast<cuuint32_t>(rf::kBlockN), 1, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult res =
        enc(tm, dtype == RF_DTYPE_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4,
            const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS) return fail(RF_ERR_CUDA, "cuTensorMapEncodeTiled failed, CUresult " + std::to_string(res));
    return RF_OK;
}

void fill_fa_params(const rf_fa_params* p, const Resolved& r, rf::FaParams* f) {
    std::memset(f, 0, sizeof(*f));
    f->B = static_cast<int>(p->B);
    f->H = static_cast<int>(p->H);
    f->S = static_cast<int>(p->S);
    f->d = static_cast<int>(p->d);
    f->kv_begin = static_cast<int>(r.kv_begin);
    f->kv_end = static_cast<int>(r.kv_end);
    f->wl = static_cast<int>(r.wl);
    f->wr = static_cast<int>(r.wr);
    f->scale_log2 = static_cast<float>(r.scale * 1.4426950408889634);
    f->n_kv_tiles = static_cast<int>(n_kv_tiles(p->S));
    f->bias_stride = f->n_kv_tiles * rf::kBlockN;
    f->out = p->out;
    f->o_sb = r.os[0];
    f->o_sh = r.os[1];
    f->o_ss = r.os[2];
    f->out_dtype = p->out_dtype;
    f->o_partial = p->o_partial;
    f->m_partial = p->m_partial;
    f->l_partial = p->l_partial;
    f->debug_scores = p->debug_scores;
}

// Everything one call needs, resolved once: kernel choice, schedule, workspace carve-up, tensor maps and the
// pre-pass arguments.  rf_fa_fwd builds one on the stack per call; an rf_fa_plan keeps it, so that steady-state
// launches do no validation, no planning and no cuTensorMapEncodeTiled (three driver calls) at all.
struct Launch {
    int kernel = RF_KERNEL_SIMT;
    bool empty = false;    // B, H or S is 0: nothing to launch
    bool neutral = false;  // split-KV partial over an empty key block
    bool bf16 = true;
    Plan pl{};
    rf::FaParams f{};
    rf::SimtParams sp{};
    CUtensorMap tmq{}, tmk{}, tmv{};
    const float* pad_bias = nullptr;  // raw [B,S]
    // pre-pass
    float* bias2 = nullptr;
    uint8_t* tile_flags = nullptr;
    // split-pair flag block of the persistent balanced schedule: zeroed in-stream by the first launch (and by
    // the first one after any launch reported a timeout), left zero by the kernel itself
    void* memset_ptr = nullptr;
    size_t memset_bytes = 0;
    mutable std::atomic<int> zeroed_epoch{-1};
    // key-norm pre-pass of the row-max skip test
    float* kmax = nullptr;
    const void* k = nullptr;
    long long ks[3] = {0, 0, 0};
    int dtype = 0;
    // neutral partial
    float* o_partial = nullptr;
    float* m_partial = nullptr;
    float* l_partial = nullptr;
    long long rows = 0;
    int d = 0;
};

int build_launch(const rf_fa_params* p, void* workspace, size_t workspace_bytes, Launch* L) {
    Resolved r;
    int rc = validate(p, &r);
    if (rc != RF_OK) return rc;
    int kernel;
    rc = select_kernel(p, r, &kernel);
    if (rc != RF_OK) return rc;
    L->kernel = kernel;
    if (p->B == 0 || p->H == 0 || p->S == 0) {
        L->empty = true;
        return RF_OK;
    }
    L->bf16 = p->dtype == RF_DTYPE_BF16;
    L->d = static_cast<int>(p->d);
    if (r.partial && r.kv_begin == r.kv_end) {  // empty key block: the neutral element of the merge
        L->neutral = true;
        L->o_partial = p->o_partial;
        L->m_partial = p->m_partial;
        L->l_partial = p->l_partial;
        L->rows = static_cast<long long>(p->B) * p->H * p->S;
        return RF_OK;
    }
    rf::FaParams& f = L->f;
    fill_fa_params(p, r, &f);
    L->pad_bias = p->pad_bias;

    if (kernel == RF_KERNEL_SIMT) {
        rf::SimtParams& sp = L->sp;
        std::memset(&sp, 0, sizeof(sp));
        sp.q = p->q;
        sp.k = p->k;
        sp.v = p->v;
        sp.q_sb = r.qs[0]; sp.q_sh = r.qs[1]; sp.q_ss = r.qs[2];
        sp.k_sb = r.ks[0]; sp.k_sh = r.ks[1]; sp.k_ss = r.ks[2];
        sp.v_sb = r.vs[0]; sp.v_sh = r.vs[1]; sp.v_ss = r.vs[2];
        sp.in_dtype = p->dtype;
        sp.d = static_cast<int>(p->d);
        sp.f = f;
        sp.f.bias2 = p->pad_bias;  // raw [B,S] bias; see launch_fa_fwd_simt
        return RF_OK;
    }

    // ---- tcgen05 path ----
    const Plan pl = make_plan(p, r, kernel);
    L->pl = pl;
    const size_t need = pl.workspace_bytes();
    if (need > 0) {
        if (workspace == nullptr || workspace_bytes < need)
            return fail(RF_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need) + " bytes");
        if (!aligned16(workspace)) return fail(RF_ERR_WORKSPACE, "workspace must be 16-byte aligned");
    }
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    f.status = reinterpret_cast<int*>(ws);
    ws += pl.status_bytes;
    if ((rc = make_tmap(&L->tmq, p->q, p->dtype, p->d, p->S, p->H, p->B, r.qs)) != RF_OK) return rc;
    if ((rc = make_tmap(&L->tmk, p->k, p->dtype, p->d, p->S, p->H, p->B, r.ks)) != RF_OK) return rc;
    if ((rc = make_tmap(&L->tmv, p->v, p->dtype, p->d, p->S, p->H, p->B, r.vs)) != RF_OK) return rc;
    if (pl.local) return RF_OK;
    void* sched_flags = nullptr;
    if (pl.tail_bytes() > 0) {
        sched_flags = ws;
        ws += pl.sched_flag_bytes;
    }
    if (pl.bias_bytes > 0) {
        L->bias2 = reinterpret_cast<float*>(ws);
        L->tile_flags = ws + pl.bias_bytes;
        f.bias2 = L->bias2;
        f.tile_flags = L->tile_flags;
    }
    f.sched_mode = pl.sched_mode;
    f.total_pairs = static_cast<int>(pl.total_pairs);
    f.pairs_per_head = static_cast<int>(pl.pairs_per_head);
    f.tiles_per_pair = static_cast<int>(pl.tiles_per_pair);
    if (pl.sched_mode == 1) {
        rf::fa_fwd_sm100_partial_carve(ws + pl.bias_bytes + pl.flag_bytes_bias, sched_flags, pl.grid, pl.d128 ? 128 : 64, &f);
        L->memset_ptr = sched_flags;
        L->memset_bytes = rf::fa_fwd_sm100_flag_bytes(pl.grid);
    }
    if (pl.kmax_bytes > 0) {
        L->kmax = reinterpret_cast<float*>(ws + pl.bias_bytes + pl.flag_bytes_bias + pl.part_bytes);
        L->k = p->k;
        for (int i = 0; i < 3; ++i) L->ks[i] = r.ks[i];
        L->dtype = p->dtype;
        f.kmax = L->kmax;
    }
    return RF_OK;
}

// Bumped whenever a launch reported a timed-out wait (rf_fa_launch_status): the kernel that gave up may have left
// split-pair flags set, so every plan zeroes its flag block again with its next launch.
std::atomic<int> g_flag_epoch{0};

int run_launch(const Launch& L, cudaStream_t stream) {
    if (L.empty) return RF_OK;
    cudaError_t e;
    if (L.neutral) {
        e = rf::launch_partial_neutral(L.o_partial, L.m_partial, L.l_partial, L.rows, L.d, stream);
        return e == cudaSuccess ? RF_OK : cuda_fail(e, "partial_neutral launch");
    }
    if (L.kernel == RF_KERNEL_SIMT) {
        int grid = 0;
        e = rf::launch_fa_fwd_simt(L.sp, stream, &grid);
        return e == cudaSuccess ? RF_OK : cuda_fail(e, "fa_fwd_simt launch");
    }
    const rf::FaParams& f = L.f;
    if (L.pl.local) {
        e = rf::launch_fa_fwd_sm100_local(L.tmq, L.tmk, L.tmv, f, L.pad_bias, L.bf16, L.pl.grid, stream);
        return e == cudaSuccess ? RF_OK : cuda_fail(e, "fa_fwd_sm100_local launch");
    }
    if (L.bias2 != nullptr) {
        e = rf::launch_bias_prepare(L.pad_bias, f.B, f.S, L.bias2, L.tile_flags, f.n_kv_tiles, stream);
        if (e != cudaSuccess) return cuda_fail(e, "bias_prepare launch");
    }
    if (L.memset_bytes > 0) {
        const int epoch = g_flag_epoch.load(std::memory_order_acquire);
        if (L.zeroed_epoch.exchange(epoch, std::memory_order_acq_rel) != epoch) {
            e = cudaMemsetAsync(L.memset_ptr, 0, L.memset_bytes, stream);
            if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(split-pair flags)");
        }
    }
    if (L.kmax != nullptr) {
        e = rf::launch_k_tile_norms(L.k, L.ks, L.dtype, f.B, f.H, f.S, f.d, f.n_kv_tiles, L.kmax, stream);
        if (e != cudaSuccess) return cuda_fail(e, "k_tile_norms launch");
    }
    if (L.pl.d128)
        e = rf::launch_fa_fwd_sm100_d128(L.tmq, L.tmk, L.tmv, f, L.bf16, L.pl.grid, stream);
    else
        e = rf::launch_fa_fwd_sm100(L.tmq, L.tmk, L.tmv, f, L.bf16, L.pl.grid, stream, /*pdl=*/true);
    return e == cudaSuccess ? RF_OK : cuda_fail(e, "fa_fwd_sm100 launch");
}

}  // namespace

struct rf_fa_plan {
    Launch launch;
};

namespace rf {
int set_last_error(int code, const std::string& message) { return fail(code, message); }
}  // namespace rf

extern "C" {

const char* rf_last_error(void) { return g_last_error.c_str(); }
int rf_abi_version(void) { return RF_FA_ABI_VERSION; }

void rf_fa_params_init(rf_fa_params* p) {
    if (p == nullptr) return;
    std::memset(p, 0, sizeof(*p));
    p->window_left = -1;
    p->window_right = -1;
    p->dtype = RF_DTYPE_BF16;
    p->out_dtype = RF_DTYPE_BF16;
    p->kernel = RF_KERNEL_AUTO;
}

int rf_fa_validate(const rf_fa_params* p) {
    Resolved r;
    int rc = validate(p, &r);
    if (rc != RF_OK) return rc;
    int kernel;
    return select_kernel(p, r, &kernel);
}

int rf_fa_fwd_workspace_bytes(const rf_fa_params* p, size_t* bytes) {
    if (bytes == nullptr) return fail(RF_ERR_ARG, "bytes is null");
    Resolved r;
    int rc = validate(p, &r);
    if (rc != RF_OK) return rc;
    int kernel;
    rc = select_kernel(p, r, &kernel);
    if (rc != RF_OK) return rc;
    *bytes = make_plan(p, r, kernel).workspace_bytes();
    return RF_OK;
}

int rf_fa_stats_query(const rf_fa_params* p, rf_fa_stats* st) {
    if (st == nullptr) return fail(RF_ERR_ARG, "stats is null");
    Resolved r;
    int rc = validate(p, &r);
    if (rc != RF_OK) return rc;
    int kernel;
    rc = select_kernel(p, r, &kernel);
    if (rc != RF_OK) return rc;
    std::memset(st, 0, sizeof(*st));
    const Plan pl = make_plan(p, r, kernel);
    st->kernel = kernel;
    st->workspace_bytes = pl.workspace_bytes();
    st->tile_scratch_bytes = kernel == RF_KERNEL_TCGEN05
                                 ? rf::fa_fwd_sm100_smem_bytes() + 512ull * 128 * 4  // smem + TMEM
                                 : (2ull * 32 * p->d + 32) * sizeof(float);
    st->row_state_bytes = 2ull * sizeof(float) * static_cast<uint64_t>(p->S);
    const uint64_t esz = p->out_dtype == RF_DTYPE_F32 ? 4 : 2;
    st->output_bytes = static_cast<uint64_t>(p->B) * p->H * p->S * p->d * (r.partial ? 4 : esz);
    st->score_matrix_bytes = 0;
    st->grid_ctas = pl.grid;
    return RF_OK;
}

int rf_fa_fwd(const rf_fa_params* p, void* workspace, size_t workspace_bytes, void* stream_v) {
    Launch L;
    const int rc = build_launch(p, workspace, workspace_bytes, &L);
    if (rc != RF_OK) return rc;
    return run_launch(L, static_cast<cudaStream_t>(stream_v));
}

int rf_fa_plan_create(const rf_fa_params* p, void* workspace, size_t workspace_bytes, rf_fa_plan** plan) {
    if (plan == nullptr) return fail(RF_ERR_ARG, "plan is null");
    *plan = nullptr;
    rf_fa_plan* pl = new (std::nothrow) rf_fa_plan();
    if (pl == nullptr) return fail(RF_ERR_ARG, "out of host memory");
    const int rc = build_launch(p, workspace, workspace_bytes, &pl->launch);
    if (rc != RF_OK) {
        delete pl;
        return rc;
    }
    *plan = pl;
    return RF_OK;
}

int rf_fa_plan_launch(const rf_fa_plan* plan, void* stream) {
    if (plan == nullptr) return fail(RF_ERR_ARG, "plan is null");
    return run_launch(plan->launch, static_cast<cudaStream_t>(stream));
}

void rf_fa_plan_destroy(rf_fa_plan* plan) { delete plan; }

int rf_fa_launch_status(void* workspace, void* stream_v) {
    if (workspace == nullptr) return RF_OK;  // kernels without a workspace have no cross-warp waits to time out
    cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
    uint32_t word = 0;
    cudaError_t e = cudaMemcpyAsync(&word, workspace, sizeof(word), cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return cuda_fail(e, "launch status read");
    if ((word & 0xffff0000u) != rf::kLaunchStatusMagic) return RF_OK;
    cudaMemsetAsync(workspace, 0, sizeof(word), stream);  // reported once
    g_flag_epoch.fetch_add(1, std::memory_order_acq_rel);  // plans zero their split-pair flags again
    const unsigned code = (word >> 12) & 0xfu, cta = word & 0xfffu;
    return fail(RF_ERR_DEVICE_TIMEOUT,
                std::string(code == 2 ? "a CTA timed out waiting for the partial of its predecessor"
                                      : "a barrier wait inside a CTA timed out") +
                    " (CTA " + std::to_string(cta) + "); the output of that launch is invalid");
}

int rf_fa_merge(const float* const* o_parts, const float* const* m_parts, const float* const* l_parts, int32_t G,
                int64_t rows, int64_t d, void* out, int32_t out_dtype, void* stream) {
    if (o_parts == nullptr || m_parts == nullptr || l_parts == nullptr || out == nullptr)
        return fail(RF_ERR_ARG, "null pointer");
    if (G < 1 || G > 16) return fail(RF_ERR_ARG, "G must be in [1,16]");
    if (d <= 0 || d % 4) return fail(RF_ERR_ARG, "d must be a positive multiple of 4");
    cudaError_t e = rf::launch_merge(o_parts, m_parts, l_parts, G, rows, static_cast<int>(d), out, out_dtype,
                                     static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "merge launch");
    return RF_OK;
}

int rf_fa_rescale_partial(float* o_part, float* l_part, const float* m_part, const float* m_star, int64_t rows,
                          int64_t d, void* stream) {
    if (o_part == nullptr || l_part == nullptr || m_part == nullptr || m_star == nullptr)
        return fail(RF_ERR_ARG, "null pointer");
    cudaError_t e = rf::launch_rescale_partial(o_part, l_part, m_part, m_star, rows, static_cast<int>(d),
                                               static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "rescale_partial launch");
    return RF_OK;
}

int rf_fa_normalize(const float* o_sum, const float* l_sum, int64_t rows, int64_t d, void* out, int32_t out_dtype,
                    void* stream) {
    if (o_sum == nullptr || l_sum == nullptr || out == nullptr) return fail(RF_ERR_ARG, "null pointer");
    cudaError_t e = rf::launch_normalize(o_sum, l_sum, rows, static_cast<int>(d), out, out_dtype,
                                         static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "normalize launch");
    return RF_OK;
}

int rf_pad_bias_from_mask(const float* mask, float* pad_bias, int64_t n, void* stream) {
    if (n < 0 || (n > 0 && (mask == nullptr || pad_bias == nullptr))) return fail(RF_ERR_ARG, "null pointer");
    cudaError_t e = rf::launch_pad_bias_from_mask(mask, pad_bias, n, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "pad_bias_from_mask launch");
    return RF_OK;
}

int rf_cast_f32_to(const float* src, void* dst, int64_t n, int32_t dst_dtype, void* stream) {
    if (dst_dtype != RF_DTYPE_BF16 && dst_dtype != RF_DTYPE_F16) return fail(RF_ERR_ARG, "bad dtype");
    cudaError_t e = rf::launch_cast_from_f32(src, dst, n, dst_dtype, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "cast launch");
    return RF_OK;
}

int rf_cast_to_f32(const void* src, float* dst, int64_t n, int32_t src_dtype, void* stream) {
    if (src_dtype != RF_DTYPE_BF16 && src_dtype != RF_DTYPE_F16) return fail(RF_ERR_ARG, "bad dtype");
    cudaError_t e = rf::launch_cast_to_f32(src, dst, n, src_dtype, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "cast launch");
    return RF_OK;
}

int rf_device_check(int32_t device, int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    if (device < 0 || device >= n) return fail(RF_ERR_CUDA, "no CUDA device " + std::to_string(device));
    cudaDeviceProp prop;
    e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
    if (sm_count) *sm_count = prop.multiProcessorCount;
    if (cc_major) *cc_major = prop.major;
    if (cc_minor) *cc_minor = prop.minor;
    if (prop.major != 10) return fail(RF_ERR_CUDA, "device is not sm_100 (Blackwell B200)");
    return RF_OK;
}

uint64_t rf_mask_memory_bytes(uint64_t batch, uint64_t heads, uint64_t seq_len, uint64_t bpe) {
    return batch * heads * seq_len * seq_len * bpe;  // attention.cpp:244-247
}
uint64_t rf_fa_memory_bytes(uint64_t batch, uint64_t heads, uint64_t seq_len, uint64_t head_dim, uint64_t tile,
                            uint64_t bpe) {
    return batch * heads * (2 * tile * head_dim + seq_len * head_dim) * bpe;  // attention.cpp:249-252
}

// ---------------------------------------------------------------------------------------------
// Host-tensor entry points (the reference's calling convention)
// ---------------------------------------------------------------------------------------------
int rf_fa_fwd_host(const float* q, const float* k, const float* v, float* out, int64_t B, int64_t H, int64_t S,
                   int64_t d, double scale, int64_t window_left, int64_t window_right, const float* pad_bias,
                   const int64_t* pad_bias_dims, int64_t tile, int32_t compute_dtype, int32_t device,
                   rf_fa_stats* stats) {
    // reference check order: check_qkv (structural here), tile, pad_bias shape (attention.cpp:107-116)
    if (B < 0 || H < 0 || S < 0 || d < 0) return fail(RF_ERR_SHAPE, "negative dimension");
    if (tile < 1) return fail(RF_ERR_SHAPE, "tile must be >= 1");
    if (pad_bias != nullptr) {
        if (pad_bias_dims == nullptr || pad_bias_dims[0] != B || pad_bias_dims[1] != 1 || pad_bias_dims[2] != 1 ||
            pad_bias_dims[3] != S)
            return fail(RF_ERR_SHAPE, "pad_bias must be [B,1,1,S]");
    }
    rf_fa_params p;
    rf_fa_params_init(&p);
    p.B = B; p.H = H; p.S = S; p.d = d;
    p.scale = scale;
    p.window_left = window_left;
    p.window_right = window_right;
    p.dtype = compute_dtype;
    p.out_dtype = RF_DTYPE_F32;
    const int64_t n = B * H * S * d;
    if (n == 0) {
        Resolved r;
        int rc0 = validate(&p, &r);
        if (rc0 != RF_OK) return rc0;
        if (stats) std::memset(stats, 0, sizeof(*stats));
        return RF_OK;
    }
    if (q == nullptr || k == nullptr || v == nullptr || out == nullptr) return fail(RF_ERR_ARG, "null host pointer");
    if (device < 0 || device >= kMaxDevices) return fail(RF_ERR_ARG, "device index out of range");

    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    {
        // keep freed staging buffers in the device's default pool so that steady-state calls do
        // not go back to the driver for memory (idempotent; the pool belongs to the runtime)
        cudaMemPool_t pool = nullptr;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess && pool != nullptr) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }

    // The call is PCIe-bound (3 f32 tensors in, 1 out), so it is pipelined over (batch, head-range)
    // chunks -- every (b, h) slice is an independent unit of the op (attention.cpp:138-142):
    // chunk c runs H2D -> cast -> attention -> D2H on stream c % kStreams, so the upload of the
    // next chunk, the kernel of this one and the download of the previous one overlap.  Small
    // problems run as one chunk.
    // RF_FA_HOST_TIMING=1 prints the host-side timeline of the call to stderr (developer aid)
    static const bool host_timing = std::getenv("RF_FA_HOST_TIMING") != nullptr;
    const auto t_begin = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (host_timing)
            std::fprintf(stderr, "[rf_fa_fwd_host] %-10s %8.3f ms\n", what,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_begin).count());
    };
    constexpr int kStreams = kHostStreams;
    const size_t nb32 = static_cast<size_t>(n) * sizeof(float);
    // Q, K, V rounded to bf16 on the host cores, chunk c + 1 under the transfers of chunk c: half the bytes cross the
    // link (the call is PCIe-bound) and no f32 upload or cast kernel is needed on the device.  Not for f16, small
    // calls, hosts without spare threads, or while another thread holds the pool; and since how fast the host cores
    // round depends on the host, large calls try both ways twice and then stay with the faster one (HostCastChoice).
    const bool cast_candidate = compute_dtype == RF_DTYPE_BF16 && 3 * nb32 >= (16u << 20) && rf::hostcast::threads() > 0;
    bool cast_pool = cast_candidate && g_cast_choice.want_host() && rf::hostcast::try_acquire();  // this call holds the pool
    bool cast_in_flight = false;
    const size_t slice_elems = static_cast<size_t>(S) * d;          // one (b, h) slice
    const size_t slice_in_bytes = 3 * slice_elems * sizeof(float);
    int64_t hpc = H;                                                // heads per chunk
    bool per_batch = false;                                         // chunks never cross a batch
    if (static_cast<size_t>(B) * H * slice_in_bytes >= (16u << 20)) {
        per_batch = true;
        // ~8 MiB of f32 input per chunk (RF_FA_HOST_CHUNK_MB overrides: developer knob)
        // ~8 MiB of f32 input per chunk, ~4 MiB when the host rounds (shorter pipeline fill and drain; measured)
        static const long chunk_env = [] {
            const char* env = std::getenv("RF_FA_HOST_CHUNK_MB");  // developer knob
            return env != nullptr ? std::atol(env) : 0L;
        }();
        const size_t chunk_target = static_cast<size_t>(chunk_env > 0 ? chunk_env : (cast_pool ? 4 : 8)) << 20;
        hpc = std::max<int64_t>(1, static_cast<int64_t>((chunk_target + slice_in_bytes - 1) / slice_in_bytes));
        hpc = std::max<int64_t>(hpc, (B * H + 63) / 64);            // at most ~64 chunks
        hpc = std::min<int64_t>(hpc, H);
    }
    const int64_t chunks_per_batch = per_batch ? (H + hpc - 1) / hpc : 1;
    const int64_t n_chunks = per_batch ? B * chunks_per_batch : 1;
    const int64_t cb = per_batch ? 1 : B;                           // batches per chunk
    const int n_streams = static_cast<int>(std::min<int64_t>(kStreams, n_chunks));
    const size_t chunk_elems = static_cast<size_t>(cb) * hpc * slice_elems;  // largest chunk, per tensor

    // A download into pageable host memory blocks the calling thread until it has finished, which
    // would serialise the pipeline chunk by chunk: in that case O is kept on the device and fetched
    // with one copy at the end.  Page-locked (or registered) host memory gets per-chunk downloads.
    bool out_pinned = false;
    {
        cudaPointerAttributes attr;
        if (cudaPointerGetAttributes(&attr, out) == cudaSuccess)
            out_pinned = attr.type == cudaMemoryTypeHost || attr.type == cudaMemoryTypeManaged;
        else
            cudaGetLastError();
    }
    float* d_out_full = nullptr;

    HostCtx& ctx = g_host_ctx[device];
    cudaStream_t* streams = ctx.streams;
    float* d_f32[kStreams] = {nullptr, nullptr, nullptr, nullptr};    // f32 staging: 3 inputs, then reused for O
    uint16_t* d_qkv[kStreams] = {nullptr, nullptr, nullptr, nullptr}; // 16-bit Q, K, V of the chunk
    void* d_ws[kStreams] = {nullptr, nullptr, nullptr, nullptr};
    float* d_bias = nullptr;
    cudaEvent_t& bias_ready = ctx.ready;
    int rc = RF_OK;
    auto cleanup = [&]() {
        if (cast_in_flight) rf::hostcast::wait();  // the workers read the caller's tensors
        cast_in_flight = false;
        if (cast_pool) rf::hostcast::release();
        cast_pool = false;
        // work queued on any stream may still read the shared buffers: drain all of them before freeing
        for (int i = 0; i < kStreams; ++i)
            if (streams[i] != nullptr) cudaStreamSynchronize(streams[i]);
        for (int i = 0; i < kStreams; ++i) {
            if (streams[i] == nullptr) continue;
            if (d_f32[i]) cudaFreeAsync(d_f32[i], streams[i]);
            if (d_qkv[i]) cudaFreeAsync(d_qkv[i], streams[i]);
            if (d_ws[i]) cudaFreeAsync(d_ws[i], streams[i]);
            if (i == 0 && d_bias) cudaFreeAsync(d_bias, streams[0]);
            if (i == 0 && d_out_full) cudaFreeAsync(d_out_full, streams[0]);
        }
        for (int i = 0; i < kStreams; ++i)
            if (streams[i] != nullptr) cudaStreamSynchronize(streams[i]);
    };
#define RF_TRY_CUDA(call, what)            \
    do {                                   \
        cudaError_t _e = (call);           \
        if (_e != cudaSuccess) {           \
            rc = cuda_fail(_e, what);      \
            cleanup();                     \
            return rc;                     \
        }                                  \
    } while (0)
#define RF_TRY_RC(call)       \
    do {                      \
        rc = (call);          \
        if (rc != RF_OK) {    \
            cleanup();        \
            return rc;        \
        }                     \
    } while (0)

    for (int i = 0; i < n_streams; ++i)
        if (streams[i] == nullptr)
            RF_TRY_CUDA(cudaStreamCreateWithFlags(&streams[i], cudaStreamNonBlocking), "cudaStreamCreate");

    if (cast_pool) {
        const size_t need = 3 * chunk_elems * sizeof(uint16_t);
        if (ctx.stage_bytes < need) {
            for (int i = 0; i < kStreams; ++i) {
                if (ctx.stage[i] != nullptr) cudaFreeHost(ctx.stage[i]);
                ctx.stage[i] = nullptr;
            }
            ctx.stage_bytes = 0;
            for (int i = 0; i < kStreams; ++i)
                RF_TRY_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctx.stage[i]), need, cudaHostAllocDefault), "cudaHostAlloc");
            ctx.stage_bytes = need;
        }
        for (int i = 0; i < n_streams; ++i)
            if (ctx.uploaded[i] == nullptr)
                RF_TRY_CUDA(cudaEventCreateWithFlags(&ctx.uploaded[i], cudaEventDisableTiming), "cudaEventCreate");
    }

    // the params of the largest chunk size the workspace of every stream
    p.B = cb;
    p.H = hpc;
    p.q = p.k = p.v = reinterpret_cast<const void*>(uintptr_t{256});  // placeholders for the size query only
    p.out = reinterpret_cast<void*>(uintptr_t{256});
    p.pad_bias = pad_bias != nullptr ? reinterpret_cast<const float*>(uintptr_t{256}) : nullptr;
    size_t ws = 0;
    RF_TRY_RC(rf_fa_fwd_workspace_bytes(&p, &ws));
    for (int i = 0; i < n_streams; ++i) {
        RF_TRY_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_f32[i]), 3 * chunk_elems * sizeof(float), streams[i]),
                    "cudaMallocAsync");
        RF_TRY_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_qkv[i]), 3 * chunk_elems * 2, streams[i]),
                    "cudaMallocAsync");
        if (ws > 0) RF_TRY_CUDA(cudaMallocAsync(&d_ws[i], ws, streams[i]), "cudaMallocAsync");
    }
    if (!out_pinned && n_chunks > 1)
        RF_TRY_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_out_full), nb32, streams[0]), "cudaMallocAsync");
    if ((pad_bias != nullptr || d_out_full != nullptr) && bias_ready == nullptr)
        RF_TRY_CUDA(cudaEventCreateWithFlags(&bias_ready, cudaEventDisableTiming), "cudaEventCreate");
    if (pad_bias != nullptr) {
        const size_t nb = static_cast<size_t>(B) * S * sizeof(float);
        RF_TRY_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_bias), nb, streams[0]), "cudaMallocAsync");
        RF_TRY_CUDA(cudaMemcpyAsync(d_bias, pad_bias, nb, cudaMemcpyHostToDevice, streams[0]), "H2D copy");
        g_h2d_total += nb;
    }
    if (pad_bias != nullptr || d_out_full != nullptr) {  // stream 0 allocated the shared buffers (and uploads the bias)
        RF_TRY_CUDA(cudaEventRecord(bias_ready, streams[0]), "cudaEventRecord");
        for (int i = 1; i < n_streams; ++i) RF_TRY_CUDA(cudaStreamWaitEvent(streams[i], bias_ready, 0), "cudaStreamWaitEvent");
    }
    if (stats) {
        rf_fa_params full = p;
        full.B = B;
        full.H = H;
        rf_fa_stats_query(&full, stats);
        stats->workspace_bytes = static_cast<uint64_t>(ws) * n_streams;
    }

    lap("setup");
    const float* host_in[3] = {q, k, v};
    struct ChunkGeom {
        int si;
        int64_t b0, nh;
        size_t off, ne;
    };
    auto geom = [&](int64_t c) {
        ChunkGeom g;
        g.si = static_cast<int>(c % n_streams);
        g.b0 = per_batch ? c / chunks_per_batch : 0;
        const int64_t h0 = per_batch ? (c % chunks_per_batch) * hpc : 0;
        g.nh = per_batch ? std::min<int64_t>(hpc, H - h0) : H;
        g.off = (static_cast<size_t>(g.b0) * H + h0) * slice_elems;      // first element of the chunk
        g.ne = static_cast<size_t>(cb) * g.nh * slice_elems;            // elements per tensor
        return g;
    };
    auto start_cast = [&](int64_t c) {
        const ChunkGeom g = geom(c);
        const float* src[3] = {host_in[0] + g.off, host_in[1] + g.off, host_in[2] + g.off};
        rf::hostcast::start(src, ctx.stage[g.si], g.ne);
        cast_in_flight = true;
    };
    if (cast_pool) start_cast(0);
    for (int64_t c = 0; c < n_chunks; ++c) {
        const ChunkGeom g = geom(c);
        const int si = g.si;
        cudaStream_t st = streams[si];
        const size_t off = g.off, ne = g.ne;
        if (cast_pool) {
            rf::hostcast::wait();
            cast_in_flight = false;
            if (c + 1 < n_chunks) {
                // the next chunk's slot was last uploaded n_streams chunks ago: that copy must have read it
                if (c + 1 >= n_streams) RF_TRY_CUDA(cudaEventSynchronize(ctx.uploaded[(c + 1) % n_streams]), "cudaEventSynchronize");
                start_cast(c + 1);
            }
            RF_TRY_CUDA(cudaMemcpyAsync(d_qkv[si], ctx.stage[si], 3 * ne * sizeof(uint16_t), cudaMemcpyHostToDevice, st), "H2D copy");
            g_h2d_total += 3 * ne * sizeof(uint16_t);
            RF_TRY_CUDA(cudaEventRecord(ctx.uploaded[si], st), "cudaEventRecord");
        } else {
            for (int t = 0; t < 3; ++t)
                RF_TRY_CUDA(cudaMemcpyAsync(d_f32[si] + static_cast<size_t>(t) * ne, host_in[t] + off, ne * sizeof(float),
                                            cudaMemcpyHostToDevice, st),
                            "H2D copy");
            g_h2d_total += 3 * ne * sizeof(float);
            RF_TRY_CUDA(rf::launch_cast_from_f32(d_f32[si], d_qkv[si], static_cast<long long>(3 * ne), compute_dtype, st),
                        "cast launch");
        }
        p.B = cb;
        p.H = g.nh;
        p.q = d_qkv[si];
        p.k = d_qkv[si] + ne;
        p.v = d_qkv[si] + 2 * ne;
        // the f32 staging slab holds O (device cast: its inputs are already cast when the kernel runs)
        p.out = d_out_full != nullptr ? d_out_full + off : d_f32[si];
        p.pad_bias = d_bias != nullptr ? d_bias + static_cast<size_t>(g.b0) * S : nullptr;
        RF_TRY_RC(rf_fa_fwd(&p, d_ws[si], ws, st));
        if (d_out_full == nullptr)
            RF_TRY_CUDA(cudaMemcpyAsync(out + off, d_f32[si], ne * sizeof(float), cudaMemcpyDeviceToHost, st), "D2H copy");
    }
    lap("enqueued");
    for (int i = 0; i < n_streams; ++i) RF_TRY_CUDA(cudaStreamSynchronize(streams[i]), "stream sync");
    for (int i = 0; i < n_streams; ++i)
        if (d_ws[i] != nullptr) RF_TRY_RC(rf_fa_launch_status(d_ws[i], streams[i]));
    lap("synced");
    if (d_out_full != nullptr) RF_TRY_CUDA(cudaMemcpy(out, d_out_full, nb32, cudaMemcpyDeviceToHost), "D2H copy");
#undef RF_TRY_CUDA
#undef RF_TRY_RC
    const bool used_host_cast = cast_pool;
    g_d2h_total += nb32;
    ++g_host_calls;
    cleanup();
    lap("cleanup");
    if (cast_candidate)
        g_cast_choice.record(used_host_cast,
                             std::chrono::duration<double>(std::chrono::steady_clock::now() - t_begin).count() / static_cast<double>(nb32));
    return RF_OK;
}

void rf_fa_host_transfer_counters(uint64_t* h2d_bytes, uint64_t* d2h_bytes, uint64_t* calls) {
    if (h2d_bytes != nullptr) *h2d_bytes = g_h2d_total;
    if (d2h_bytes != nullptr) *d2h_bytes = g_d2h_total;
    if (calls != nullptr) *calls = g_host_calls;
}

int rf_host_round_bf16(const float* src, uint16_t* dst, int64_t n) {
    if (n < 0 || (n > 0 && (src == nullptr || dst == nullptr))) return fail(RF_ERR_ARG, "null pointer or negative count");
    if (n == 0) return RF_OK;
    if (n >= (1 << 16) && rf::hostcast::try_acquire()) {
        const float* srcs[3] = {src, nullptr, nullptr};
        rf::hostcast::start(srcs, dst, static_cast<size_t>(n), 1);
        rf::hostcast::wait();
        rf::hostcast::release();
    } else {
        rf::hostcast::round_bf16_serial(src, dst, static_cast<size_t>(n));
    }
    return RF_OK;
}

void rf_fa_host_release(void) {
    for (int dev = 0; dev < kMaxDevices; ++dev) {
        HostCtx& ctx = g_host_ctx[dev];
        bool any = ctx.ready != nullptr;
        for (int i = 0; i < kHostStreams; ++i) any = any || ctx.streams[i] != nullptr || ctx.stage[i] != nullptr;
        if (!any) continue;
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(dev);
        for (int i = 0; i < kHostStreams; ++i)
            if (ctx.streams[i] != nullptr) {
                cudaStreamSynchronize(ctx.streams[i]);
                cudaStreamDestroy(ctx.streams[i]);
                ctx.streams[i] = nullptr;
            }
        if (ctx.ready != nullptr) {
            cudaEventDestroy(ctx.ready);
            ctx.ready = nullptr;
        }
        for (int i = 0; i < kHostStreams; ++i) {
            if (ctx.stage[i] != nullptr) cudaFreeHost(ctx.stage[i]);
            ctx.stage[i] = nullptr;
            if (ctx.uploaded[i] != nullptr) cudaEventDestroy(ctx.uploaded[i]);
            ctx.uploaded[i] = nullptr;
        }
        ctx.stage_bytes = 0;
        cudaSetDevice(cur);
    }
    rf::hostcast::shutdown();
}

int rf_fused_flash_attention_op(const float* const* inputs, const int64_t* const* input_dims,
                                const int32_t* input_ranks, int32_t n_inputs, int32_t has_scale, double scale,
                                int32_t has_window_left, int64_t window_left, int32_t has_window_right,
                                int64_t window_right, float* output, int32_t device) {
    if (inputs == nullptr || input_dims == nullptr || input_ranks == nullptr) return fail(RF_ERR_ARG, "null pointer");
    if (n_inputs < 3) return fail(RF_ERR_SHAPE, "FusedFlashAttention: missing input tensor");  // interpreter.cpp:209-214
    // check_qkv (attention.cpp:14-21)
    for (int t = 0; t < 3; ++t)
        if (input_ranks[t] != 4) return fail(RF_ERR_SHAPE, "attention inputs must be [B,H,S,d]");
    for (int t = 1; t < 3; ++t)
        for (int a = 0; a < 4; ++a)
            if (input_dims[t][a] != input_dims[0][a]) return fail(RF_ERR_SHAPE, "Q, K, V must have identical shapes");
    const int64_t* qd = input_dims[0];
    const float* bias = nullptr;
    int64_t bias_dims[4] = {0, 0, 0, 0};
    if (n_inputs > 3) {  // interpreter.cpp:313-315
        bias = inputs[3];
        if (input_ranks[3] != 4) return fail(RF_ERR_SHAPE, "pad_bias must be [B,1,1,S]");
        for (int a = 0; a < 4; ++a) bias_dims[a] = input_dims[3][a];
        if (bias == nullptr) return fail(RF_ERR_ARG, "pad_bias input is null");
    }
    // attrs default exactly like node.attr_real("scale", 0.0) / attr_int("window_*", -1)
    return rf_fa_fwd_host(inputs[0], inputs[1], inputs[2], output, qd[0], qd[1], qd[2], qd[3],
                          has_scale ? scale : 0.0, has_window_left ? window_left : -1,
                          has_window_right ? window_right : -1, bias, bias ? bias_dims : nullptr, 64,
                          RF_DTYPE_BF16, device, nullptr);
}

}  // extern "C"
