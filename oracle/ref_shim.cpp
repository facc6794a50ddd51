// ref_shim.cpp -- C-ABI shim over the UNMODIFIED reference sources (TEST INFRASTRUCTURE ONLY).
//
// Compiled by oracle/Makefile together with /root/reference/proj/core/src/{attention,tensor}.cpp
// (where they lie; no reference source is copied into this repo) into
// oracle/_ref/libref_attn.so.  It exists to (1) pin oracle/rf_oracle.c bit-for-bit,
// (2) generate the golden vectors under tests/golden/, and (3) serve as the
// `cpu_baseline.kind == "reference"` timing arm of bench.py.
//
// The reference operator is single-threaded (attention.cpp has no threads).  Because every
// (batch, head) slice is independent (attention.cpp:138-142) and the function is pure,
// calling it on [1,1,S,d] slices from several threads gives bit-identical output; that is
// what `threads > 1` does here.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "routefast/attention.hpp"
#include "routefast/tensor.hpp"

namespace rf = routefast;

namespace {
thread_local std::string g_err;

rf::Tensor wrap(const float* p, std::vector<int64_t> shape) {
    rf::Tensor t(std::move(shape));
    if (!t.data.empty()) std::memcpy(t.data.data(), p, t.data.size() * sizeof(float));
    return t;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// routefast::flash_attention (attention.hpp:46-48).  Returns 0, or 1 with ref_last_error()
// holding the ShapeMismatch text.  pad_bias_dims (4 ints) lets tests pass a wrong-shaped bias
// to exercise the reference's own error path.
int ref_flash_attention(const float* q, const float* k, const float* v, float* out, int64_t B,
                        int64_t H, int64_t S, int64_t d, double scale, int64_t wl, int64_t wr,
                        const float* pad_bias, const int64_t* pad_bias_dims, int64_t tile,
                        int threads, uint64_t* stats3) {
    try {
        std::vector<int64_t> pdims = {B, 1, 1, S};
        if (pad_bias && pad_bias_dims) pdims.assign(pad_bias_dims, pad_bias_dims + 4);
        const bool whole = threads <= 1 || B * H <= 1 || pdims != std::vector<int64_t>{B, 1, 1, S};
        if (whole) {
            rf::AttentionSpec spec;
            spec.scale = scale;
            spec.window_left = wl;
            spec.window_right = wr;
            if (pad_bias) spec.pad_bias = wrap(pad_bias, pdims);
            rf::FlashStats st;
            rf::Tensor o = rf::flash_attention(wrap(q, {B, H, S, d}), wrap(k, {B, H, S, d}),
                                               wrap(v, {B, H, S, d}), spec, tile, &st);
            std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
            if (stats3) {
                stats3[0] = st.tile_scratch_floats;
                stats3[1] = st.row_state_floats;
                stats3[2] = st.output_floats;
            }
            return 0;
        }
        // sliced, threaded: each slice is a [1,1,S,d] call into the same reference function
        const int64_t slices = B * H;
        std::atomic<int64_t> next{0};
        std::atomic<bool> bad{false};
        std::string first_err;
        std::vector<std::thread> pool;
        const int n = static_cast<int>(std::min<int64_t>(threads, slices));
        for (int t = 0; t < n; ++t) {
            pool.emplace_back([&] {
                for (;;) {
                    const int64_t s = next.fetch_add(1);
                    if (s >= slices || bad.load()) return;
                    try {
                        const int64_t b = s / H;
                        const std::size_t base = static_cast<std::size_t>(s * S * d);
                        rf::AttentionSpec spec;
                        spec.scale = scale;  // slice keeps head_dim, so scale==0 resolves identically
                        spec.window_left = wl;
                        spec.window_right = wr;
                        if (pad_bias) spec.pad_bias = wrap(pad_bias + b * S, {1, 1, 1, S});
                        rf::Tensor o =
                            rf::flash_attention(wrap(q + base, {1, 1, S, d}), wrap(k + base, {1, 1, S, d}),
                                                wrap(v + base, {1, 1, S, d}), spec, tile, nullptr);
                        std::memcpy(out + base, o.data.data(), o.data.size() * sizeof(float));
                    } catch (const std::exception& e) {
                        if (!bad.exchange(true)) first_err = e.what();
                    }
                }
            });
        }
        for (auto& th : pool) th.join();
        if (bad.load()) {
            g_err = first_err;
            return 1;
        }
        if (stats3) {
            stats3[0] = static_cast<uint64_t>(tile);
            stats3[1] = static_cast<uint64_t>(2 * S);
            stats3[2] = static_cast<uint64_t>(B * H * S * d);
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// routefast::sdpa (attention.hpp:31-32); mask dims are [mB, mH, S, S] when mask2d != NULL.
int ref_sdpa(const float* q, const float* k, const float* v, float* out, int64_t B, int64_t H,
             int64_t S, int64_t d, const float* mask2d, int64_t mB, int64_t mH, double scale) {
    try {
        rf::Tensor m;
        if (mask2d) m = wrap(mask2d, {mB, mH, S, S});
        rf::Tensor o = rf::sdpa(wrap(q, {B, H, S, d}), wrap(k, {B, H, S, d}), wrap(v, {B, H, S, d}),
                                mask2d ? &m : nullptr, scale);
        std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// routefast::window_to_mask2d (attention.hpp:53-54); pad_bias is [B,1,1,S] or NULL (then B=1).
int ref_window_to_mask2d(int64_t S, int64_t wl, int64_t wr, const float* pad_bias, int64_t B,
                         float* mask) {
    try {
        rf::Tensor p;
        if (pad_bias) p = wrap(pad_bias, {B, 1, 1, S});
        rf::Tensor m = rf::window_to_mask2d(S, wl, wr, pad_bias ? &p : nullptr);
        std::memcpy(mask, m.data.data(), m.data.size() * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

float ref_quantize_f16(float v) { return rf::quantize_f16(v); }
uint16_t ref_float_to_half(float v) { return rf::float_to_half(v); }
float ref_half_to_float(uint16_t b) { return rf::half_to_float(b); }

double ref_effective_scale(double scale, int64_t head_dim) {
    rf::AttentionSpec s;
    s.scale = scale;
    return s.effective_scale(head_dim);
}

uint64_t ref_mask_memory_bytes(uint64_t b, uint64_t h, uint64_t s, uint64_t bpe) {
    return rf::mask_memory_bytes(b, h, s, bpe);
}
uint64_t ref_fa_memory_bytes(uint64_t b, uint64_t h, uint64_t s, uint64_t d, uint64_t tile, uint64_t bpe) {
    return rf::fa_memory_bytes(b, h, s, d, tile, bpe);
}

// Tensor::random stream (tensor.cpp:35-45): fills n_tensors consecutive tensors of `each`
// elements from one std::mt19937_64(seed), as bench_attention.cpp:16-23 does for q, k, v.
void ref_random_fill(uint64_t seed, float* out, int64_t each, int64_t n_tensors, int as_f16) {
    std::mt19937_64 rng(seed);
    for (int64_t t = 0; t < n_tensors; ++t) {
        rf::Tensor x = rf::Tensor::random({each}, rng, as_f16 ? rf::DType::f16 : rf::DType::f32);
        std::memcpy(out + t * each, x.data.data(), static_cast<std::size_t>(each) * sizeof(float));
    }
}

}  // extern "C"
