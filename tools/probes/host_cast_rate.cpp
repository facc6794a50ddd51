// host_cast_rate.cpp -- developer probe: how fast can the host round f32 -> bf16 (RNE) with OpenMP threads?
// (decides whether casting on the host, which halves the H2D bytes of rf_fa_fwd_host, can pay)
//   g++ -O3 -fopenmp -o host_cast_rate host_cast_rate.cpp
#include <omp.h>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

static inline uint16_t bf16_rne(uint32_t x) {
    if ((x & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((x >> 16) | 0x40u);  // NaN stays NaN
    return static_cast<uint16_t>((x + 0x7fffu + ((x >> 16) & 1u)) >> 16);
}

int main() {
    const size_t n = 3ull * 12 * 8192 * 64;
    std::vector<float> src(n);
    std::vector<uint16_t> dst(n);
    for (size_t i = 0; i < n; ++i) src[i] = float(i % 1000) * 0.001f - 0.5f;
    std::printf("{\"hw_threads\": %d}\n", omp_get_max_threads());
    for (int threads : {1, 4, 8, 12, 16, 24, 32}) {
        if (threads > omp_get_max_threads()) break;
        double best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            const auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel for num_threads(threads) schedule(static)
            for (long long i = 0; i < static_cast<long long>(n); ++i) {
                uint32_t x;
                std::memcpy(&x, &src[i], 4);
                dst[i] = bf16_rne(x);
            }
            const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            if (ms < best) best = ms;
        }
        std::printf("{\"threads\": %d, \"ms_for_75MB_in\": %.3f, \"GBps_read\": %.1f}\n", threads, best, n * 4 / best / 1e6);
    }
    return dst[123] == 7 ? 1 : 0;
}
