// host_cast.cpp -- see host_cast.h.  Plain C++ (no CUDA): a fork-join pool with one job in flight.
#include "host_cast.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace rf {
namespace hostcast {
namespace {

// f32 -> bf16, round to nearest even; NaN keeps its sign and becomes quiet (what __float2bfloat16_rn gives)
inline uint16_t bf16_rne(uint32_t x) {
    const uint32_t rounded = x + 0x7fffu + ((x >> 16) & 1u);
    const uint32_t nan = x | 0x00400000u;
    return static_cast<uint16_t>((((x & 0x7fffffffu) > 0x7f800000u) ? nan : rounded) >> 16);
}

void cast_range_generic(const float* src, uint16_t* dst, size_t n) {
    for (size_t i = 0; i < n; ++i) {
        uint32_t x;
        std::memcpy(&x, src + i, 4);
        dst[i] = bf16_rne(x);
    }
}
#if defined(__x86_64__) && defined(__GNUC__)
// same loop, auto-vectorised for AVX2 (chosen at run time; the library itself is built for baseline x86-64)
__attribute__((target("avx2"))) void cast_range_avx2(const float* src, uint16_t* dst, size_t n) {
    for (size_t i = 0; i < n; ++i) {
        uint32_t x;
        std::memcpy(&x, src + i, 4);
        dst[i] = bf16_rne(x);
    }
}
#endif

#if defined(__x86_64__) && defined(__GNUC__)
// ... and for AVX-512 (16 lanes, vpmovdw packs).  The integer formulation is kept on purpose: AVX512-BF16's
// vcvtneps2bf16 flushes subnormals, the device cast does not.
__attribute__((target("avx512f,avx512bw,avx512vl,prefer-vector-width=512"))) void cast_range_avx512(const float* src, uint16_t* dst,
                                                                                                    size_t n) {
    for (size_t i = 0; i < n; ++i) {
        uint32_t x;
        std::memcpy(&x, src + i, 4);
        dst[i] = bf16_rne(x);
    }
}
#endif

using CastFn = void (*)(const float*, uint16_t*, size_t);
CastFn pick_cast() {
#if defined(__x86_64__) && defined(__GNUC__)
    const char* isa = std::getenv("RF_FA_HOST_CAST_ISA");  // developer knob: "avx2" keeps the 256-bit path
    const bool allow512 = isa == nullptr || std::strcmp(isa, "avx2") != 0;
    if (allow512 && __builtin_cpu_supports("avx512bw") && __builtin_cpu_supports("avx512vl")) return cast_range_avx512;
    if (__builtin_cpu_supports("avx2")) return cast_range_avx2;
#endif
    return cast_range_generic;
}

inline void cpu_relax() {
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
}

// Jobs of one call arrive every ~0.2 ms; a futex wake-up of fifteen sleeping workers costs about as much as the job
// itself.  So a worker that ran out of work polls the job counter for a while (kSpinUs) before it goes to sleep on the
// condition variable, and the thread that waits for a job polls the completion counter.
//
// Work is handed out in blocks through an atomic counter, and the posting thread takes blocks too while it waits:
// a worker that the hypervisor parks for a millisecond then costs one block, not 1/T of the job (the bench boxes are
// VMs; with fixed shares the same call took 1.5 or 2.1 ms depending on the minute).  A job is complete when all its
// blocks are, not when every worker has looked at it; the two job slots alternate, and a slot is only rewritten once
// no worker is inside it (active == 0) -- a latecomer finds the slot's generation changed and leaves.
constexpr int kSpinUs = 400;
constexpr size_t kBlockElems = 8192;  // per tensor: 32 KiB read, 16 KiB written

struct Job {
    const float* src[3] = {nullptr, nullptr, nullptr};
    uint16_t* dst = nullptr;
    size_t ne = 0, n_blocks = 0;
    int arrays = 3;
    std::atomic<uint64_t> gen{0};      // sequence number of the job in this slot, 0 while it is being rewritten
    std::atomic<size_t> next{0};       // next block to hand out
    std::atomic<size_t> done{0};       // blocks finished
    std::atomic<int> active{0};        // threads inside the slot
};

struct Pool {
    std::mutex m;
    std::condition_variable cv_work;
    std::vector<std::thread> workers;
    Job jobs[2];
    std::atomic<uint64_t> posted{0};  // sequence number of the newest job
    std::atomic<bool> stop{false};
    int sleepers = 0;                 // workers blocked on cv_work (under m)
    CastFn fn = nullptr;

    // takes blocks of job `seq` until none is left; returns at once if the slot holds another job by now
    void help(uint64_t seq) {
        Job& j = jobs[seq & 1];
        j.active.fetch_add(1, std::memory_order_acq_rel);
        if (j.gen.load(std::memory_order_acquire) == seq) {
            for (;;) {
                const size_t b = j.next.fetch_add(1, std::memory_order_relaxed);
                if (b >= j.n_blocks) break;
                const size_t e0 = b * kBlockElems, e1 = std::min(j.ne, e0 + kBlockElems);
                for (int t = 0; t < j.arrays; ++t) fn(j.src[t] + e0, j.dst + static_cast<size_t>(t) * j.ne + e0, e1 - e0);
                j.done.fetch_add(1, std::memory_order_release);
            }
        }
        j.active.fetch_sub(1, std::memory_order_release);
    }

    void worker() {
        uint64_t seen = 0;
        for (;;) {
            // poll, then sleep
            const auto t0 = std::chrono::steady_clock::now();
            while (posted.load(std::memory_order_acquire) == seen && !stop.load(std::memory_order_relaxed)) {
                for (int i = 0; i < 64; ++i) cpu_relax();
                if (std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(kSpinUs)) {
                    std::unique_lock<std::mutex> lk(m);
                    ++sleepers;
                    cv_work.wait(lk, [&] { return stop.load(std::memory_order_relaxed) || posted.load(std::memory_order_acquire) != seen; });
                    --sleepers;
                    break;
                }
            }
            if (stop.load(std::memory_order_relaxed)) return;
            seen = posted.load(std::memory_order_acquire);
            help(seen);
        }
    }
    void ensure_started(int count) {
        if (!workers.empty()) return;
        fn = pick_cast();
        stop.store(false);
        for (int i = 0; i < count; ++i) workers.emplace_back([this] { worker(); });
    }
    void join_all() {
        {
            std::lock_guard<std::mutex> lk(m);
            stop.store(true);
        }
        cv_work.notify_all();
        for (auto& t : workers) t.join();
        workers.clear();
        // (sequence numbers keep counting: a restarted pool's workers start from seen = 0 and simply find the newest job)
    }
};

Pool& pool() {
    static Pool* p = new Pool();  // never destroyed: worker threads may outlive static destruction order otherwise
    return *p;
}
std::atomic<bool> g_busy{false};

int configured_threads() {
    static const int n = [] {
        const char* off = std::getenv("RF_FA_HOST_CAST");
        if (off != nullptr && off[0] == '0') return 0;
        int hw = static_cast<int>(std::thread::hardware_concurrency());
        if (const char* lw = std::getenv("LOCAL_WORLD_SIZE")) {  // one process per GPU: share the cores
            const int ranks = std::atoi(lw);
            if (ranks > 1) hw /= ranks;
        }
        int t = std::min(16, hw - 2);  // leave cores to the thread that drives the copies and to the driver's own threads
        if (const char* env = std::getenv("RF_FA_HOST_CAST_THREADS")) t = std::atoi(env);
        return t < 2 ? 0 : std::min(t, 64);
    }();
    return n;
}

}  // namespace

int threads() { return configured_threads(); }

bool try_acquire() {
    if (configured_threads() == 0) return false;
    bool expected = false;
    return g_busy.compare_exchange_strong(expected, true, std::memory_order_acq_rel);
}

void release() { g_busy.store(false, std::memory_order_release); }

void start(const float* const src[3], uint16_t* dst, size_t ne, int arrays) {
    Pool& p = pool();
    p.ensure_started(configured_threads());  // (one caller at a time: try_acquire)
    const uint64_t seq = p.posted.load(std::memory_order_relaxed) + 1;
    Job& j = p.jobs[seq & 1];
    j.gen.store(0, std::memory_order_release);                          // nobody may enter the slot any more ...
    while (j.active.load(std::memory_order_acquire) != 0) cpu_relax();  // ... and whoever is inside leaves (its job is long done)
    j.src[0] = src[0]; j.src[1] = arrays > 1 ? src[1] : nullptr; j.src[2] = arrays > 2 ? src[2] : nullptr;
    j.dst = dst;
    j.ne = ne;
    j.arrays = arrays;
    j.n_blocks = (ne + kBlockElems - 1) / kBlockElems;
    j.next.store(0, std::memory_order_relaxed);
    j.done.store(0, std::memory_order_relaxed);
    j.gen.store(seq, std::memory_order_release);
    p.posted.store(seq, std::memory_order_release);
    bool wake;
    {
        std::lock_guard<std::mutex> lk(p.m);
        wake = p.sleepers > 0;
    }
    if (wake) p.cv_work.notify_all();
}

void wait() {
    Pool& p = pool();
    const uint64_t seq = p.posted.load(std::memory_order_acquire);
    if (seq == 0) return;
    p.help(seq);  // the waiting thread takes blocks too
    Job& j = p.jobs[seq & 1];
    int spins = 0;
    while (j.done.load(std::memory_order_acquire) != j.n_blocks) {
        cpu_relax();
        if (++spins > (1 << 14)) {
            std::this_thread::yield();
            spins = 0;
        }
    }
}

void round_bf16_serial(const float* src, uint16_t* dst, size_t n) { pick_cast()(src, dst, n); }

void shutdown() {
    if (!try_acquire()) {
        if (configured_threads() == 0) return;
        return;  // another thread is mid-call: leave its pool alone
    }
    Pool& p = pool();
    if (!p.workers.empty()) p.join_all();
    release();
}

}  // namespace hostcast
}  // namespace rf
