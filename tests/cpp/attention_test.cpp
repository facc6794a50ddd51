// attention_test.cpp -- C++ test of the routefast_b200 mirror, written the way the reference's own
// (missing-from-snapshot) proj/tests/attention_test.cpp is specified in SPEC.md:504-507,540-549:
// flash_attention against an independently coded double-precision reference
// (the role of proj/tests/support/oracles.cpp:83-129) over S x window x padding, plus the
// known answers and the error behaviour.  Built with g++ against librf_fa.so; needs a B200.
// Tolerance: bf16 kernel vs f64 math, inputs rounded to bf16 first: max-abs <= 2e-2.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

#include "routefast_b200/attention.hpp"

namespace rf = routefast_b200;

static float round_bf16(float v) {
    uint32_t b;
    std::memcpy(&b, &v, 4);
    b += 0x7FFFu + ((b >> 16) & 1u);
    b &= 0xFFFF0000u;
    std::memcpy(&v, &b, 4);
    return v;
}

static rf::Tensor random_tensor(std::vector<int64_t> shape, std::mt19937_64& rng) {
    rf::Tensor t(std::move(shape));
    for (auto& v : t.data) {  // tensor.cpp:37-43, then the parity convention (bf16 on both sides)
        double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
        v = round_bf16(static_cast<float>(2.0 * u - 1.0));
    }
    return t;
}

// independent double-precision masked attention (brute force, O(S^2))
static std::vector<double> reference(const rf::Tensor& q, const rf::Tensor& k, const rf::Tensor& v,
                                     const rf::AttentionSpec& spec) {
    const int64_t B = q.shape[0], H = q.shape[1], S = q.shape[2], d = q.shape[3];
    const double scale = spec.effective_scale(d);
    std::vector<double> out(q.data.size(), 0.0), w(static_cast<size_t>(S));
    for (int64_t b = 0; b < B; ++b)
        for (int64_t h = 0; h < H; ++h) {
            const size_t base = static_cast<size_t>((b * H + h) * S * d);
            for (int64_t i = 0; i < S; ++i) {
                double mx = -INFINITY;
                for (int64_t j = 0; j < S; ++j) {
                    bool live = (spec.window_left < 0 || i - j <= spec.window_left) &&
                                (spec.window_right < 0 || j - i <= spec.window_right);
                    double bias = 0.0;
                    if (spec.pad_bias) {
                        bias = spec.pad_bias->data[static_cast<size_t>(b * S + j)];
                        live = live && bias > rf::kMaskThreshold;
                    }
                    if (!live) { w[j] = -INFINITY; continue; }
                    double dot = 0.0;
                    for (int64_t c = 0; c < d; ++c) dot += double(q.data[base + i * d + c]) * double(k.data[base + j * d + c]);
                    w[j] = dot * scale + bias;
                    mx = std::max(mx, w[j]);
                }
                if (std::isinf(mx)) continue;  // no live key -> zeros
                double den = 0.0;
                for (int64_t j = 0; j < S; ++j) { w[j] = std::isinf(w[j]) ? 0.0 : std::exp(w[j] - mx); den += w[j]; }
                for (int64_t c = 0; c < d; ++c) {
                    double acc = 0.0;
                    for (int64_t j = 0; j < S; ++j) acc += w[j] * double(v.data[base + j * d + c]);
                    out[base + i * d + c] = acc / den;
                }
            }
        }
    return out;
}

static int failures = 0;
#define CHECK(cond, ...) do { if (!(cond)) { ++failures; std::printf("FAIL %s:%d: ", __FILE__, __LINE__); std::printf(__VA_ARGS__); std::printf("\n"); } } while (0)

int main() {
    std::mt19937_64 rng(11);
    // grid: S x windows x random padding, head_dim 64 (tcgen05) and 32 (generic kernel)
    const int64_t sizes[] = {1, 2, 5, 8, 37, 100, 257, 512};
    const int64_t windows[][2] = {{-1, -1}, {0, 0}, {1, 2}, {63, 64}};
    double worst = 0.0;
    for (int64_t d : {64, 32, 128})
        for (int64_t S : sizes)
            for (auto& w : windows) {
                rf::Tensor q = random_tensor({2, 2, S, d}, rng), k = random_tensor({2, 2, S, d}, rng),
                           v = random_tensor({2, 2, S, d}, rng);
                rf::AttentionSpec spec;
                spec.window_left = w[0];
                spec.window_right = w[1];
                spec.pad_bias = rf::Tensor({2, 1, 1, S});
                for (auto& x : spec.pad_bias->data) x = (rng() % 4 == 0) ? rf::kMaskValue : 0.0f;
                rf::FlashStats st;
                rf::Tensor o = rf::flash_attention(q, k, v, spec, 64, &st);
                auto ref = reference(q, k, v, spec);
                double err = 0.0;
                for (size_t i = 0; i < ref.size(); ++i) err = std::max(err, std::abs(double(o.data[i]) - ref[i]));
                worst = std::max(worst, err);
                CHECK(err <= 2e-2, "S=%ld d=%ld window=(%ld,%ld) max-abs %.3e", (long)S, (long)d, (long)w[0], (long)w[1], err);
                CHECK(st.score_matrix_bytes == 0 && st.row_state_floats == size_t(2 * S), "stats");
                CHECK(st.kernel == RF_KERNEL_TCGEN05, "kernel selection d=%ld", (long)d);  // every head dim of the contract
            }
    std::printf("grid worst max-abs error %.3e\n", worst);

    // known answers: window (0,0) -> O = V; S = 1 -> O = V
    {
        rf::Tensor q = random_tensor({1, 2, 70, 64}, rng), k = random_tensor({1, 2, 70, 64}, rng),
                   v = random_tensor({1, 2, 70, 64}, rng);
        rf::AttentionSpec self;
        self.window_left = self.window_right = 0;
        rf::Tensor o = rf::flash_attention(q, k, v, self);
        double err = 0.0;
        for (size_t i = 0; i < o.data.size(); ++i) err = std::max(err, std::abs(double(o.data[i]) - double(v.data[i])));
        CHECK(err <= 1e-6, "window (0,0) must return V exactly (bf16-representable), err %.3e", err);
    }
    // fully masked batch row -> zeros, not NaN (attention.cpp:175,204-207)
    {
        rf::Tensor q = random_tensor({1, 1, 40, 64}, rng);
        rf::AttentionSpec spec;
        spec.pad_bias = rf::Tensor::full({1, 1, 1, 40}, rf::kMaskValue);
        rf::Tensor o = rf::flash_attention(q, q, q, spec);
        bool all_zero = std::all_of(o.data.begin(), o.data.end(), [](float x) { return x == 0.0f; });
        CHECK(all_zero, "fully masked rows must be exactly zero");
    }
    // error behaviour (attention.cpp:14-21,110-116; rewrite.cpp:266-269)
    {
        rf::Tensor a({1, 1, 4, 64}), b({1, 1, 5, 64}), r3({1, 4, 64});
        auto throws_shape = [&](auto&& fn, const char* what) {
            try { fn(); CHECK(false, "expected ShapeMismatch: %s", what); }
            catch (const rf::ShapeMismatch& e) { CHECK(std::strstr(e.what(), what) != nullptr, "message '%s' lacks '%s'", e.what(), what); }
        };
        throws_shape([&] { rf::flash_attention(a, a, b, {}); }, "identical shapes");
        throws_shape([&] { rf::flash_attention(r3, r3, r3, {}); }, "[B,H,S,d]");
        throws_shape([&] { rf::flash_attention(a, a, a, {}, 0); }, "tile must be >= 1");
        rf::AttentionSpec bad;
        bad.pad_bias = rf::Tensor({1, 1, 1, 5});
        throws_shape([&] { rf::flash_attention(a, a, a, bad); }, "pad_bias must be [B,1,1,S]");
        rf::Tensor h48({1, 1, 4, 48});
        try { rf::flash_attention(h48, h48, h48, {}); CHECK(false, "expected UnsupportedHeadDim"); }
        catch (const rf::UnsupportedHeadDim&) {}
    }
    // memory model
    CHECK(rf::mask_memory_bytes(1, 12, 8192, 2) == 1610612736ull, "mask_memory_bytes");
    CHECK(rf::fa_memory_bytes(1, 12, 8192, 64, 64, 2) == 12779520ull, "fa_memory_bytes");

    std::printf(failures ? "attention_test: %d FAILURE(S)\n" : "attention_test: all checks passed\n", failures);
    return failures ? 1 : 0;
}
