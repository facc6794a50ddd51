// host_cast.h -- f32 -> bf16 rounding on the host cores, for the host-tensor entry point (fa_api.cu: rf_fa_fwd_host).
// The call is PCIe-bound; rounding Q, K, V on the host halves the bytes that cross the link, and a small pool of
// worker threads does it chunk by chunk under the previous chunk's transfers.
#pragma once
#include <cstddef>
#include <cstdint>

namespace rf {
namespace hostcast {

// Worker threads the pool would use (0 = host-side casting is off: RF_FA_HOST_CAST=0, or a single hardware thread).
int threads();
// One job at a time, process-wide.  try_acquire() returns false when another host thread holds the pool (the caller
// then casts on the device as before); release() gives it back.
bool try_acquire();
void release();
// Starts rounding three f32 arrays of `ne` elements each (round-to-nearest-even, NaN stays NaN: bit-identical to the
// device cast) into dst[0, ne), dst[ne, 2 ne), dst[2 ne, 3 ne); returns at once.  wait() blocks until it is done.
// arrays: how many of the three sources are used (1..3).
void start(const float* const src[3], uint16_t* dst, size_t ne, int arrays = 3);
void wait();
// The same rounding on the calling thread (no pool).
void round_bf16_serial(const float* src, uint16_t* dst, size_t n);
// Joins the workers (rf_fa_host_release); the pool restarts on the next start().
void shutdown();

}  // namespace hostcast
}  // namespace rf
