// ptx.cuh -- thin inline-PTX wrappers for sm_100a: mbarrier, TMA, tcgen05 (MMA / TMEM).
// No CUTLASS/CuTe: the descriptor bit layouts below are the hardware formats (PTX ISA 8.7,
// "tcgen05 matrix descriptors" / "instruction descriptor").
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace rfptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ------------------------------------------------------------------------------------------
// mbarrier
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// generic-proxy writes (st.shared) -> visible to the async proxy (TMA / UMMA smem reads)
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ uint32_t mbar_try_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.b32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok;
}

// Bounded waits.  A wait that exhausts its poll budget (a protocol bug, or a dependency that is never
// scheduled) must neither hang the GPU nor kill the context: it records a code in a status word in global
// memory (the host reads it: rf_fa_launch_status) and raises the CTA's abort word in shared memory.  Every
// wait of the CTA polls that word from its slow path and returns as soon as it is set, so the kernel runs
// through to its normal teardown (results are garbage, the status word says so).  The fast path -- the
// barrier is ready on the first polls -- is unchanged.
#ifndef RF_MBAR_SPIN_LIMIT
#define RF_MBAR_SPIN_LIMIT (1u << 24)
#endif
// The CTA's 16-byte wait block in shared memory: [0,4) abort word (0 = running), [8,16) the launch's global
// status word pointer (may be null).  Keeping the pointer there instead of in a WaitCtx member costs the
// 32-register producer / MMA warps nothing.
struct WaitCtx {
    uint32_t block_smem;  // shared-memory address of the wait block
};
// Status word values: kStatusMagic | code << 12 | (CTA index & 0xfff).  The workspace is caller-owned and never
// cleared on the launch path (a memset node would cost the 20 us local-window layer 5-10 %), so the word is only
// meaningful when it carries the magic tag; the host clears it after reporting.
enum : int { kStatusBarrierTimeout = 1, kStatusPeerTimeout = 2 };
constexpr uint32_t kStatusMagic = 0x52460000u;

__device__ __forceinline__ void wait_block_init(uint32_t block_smem, int* status) {
    asm volatile("st.shared::cta.u32 [%0], %1;" ::"r"(block_smem), "r"(0u) : "memory");
    asm volatile("st.shared::cta.u64 [%0], %1;" ::"r"(block_smem + 8u), "l"(reinterpret_cast<uint64_t>(status)) : "memory");
}
__device__ __forceinline__ uint32_t ld_shared_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.volatile.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
static __device__ __noinline__ void wait_timed_out(uint32_t block_smem, int code) {
    asm volatile("st.volatile.shared::cta.u32 [%0], %1;" ::"r"(block_smem), "r"(1u) : "memory");
    uint64_t ptr;
    asm volatile("ld.shared::cta.u64 %0, [%1];" : "=l"(ptr) : "r"(block_smem + 8u) : "memory");
    int* status = reinterpret_cast<int*>(ptr);
    if (status != nullptr)
        *reinterpret_cast<volatile uint32_t*>(status) = kStatusMagic | (static_cast<uint32_t>(code) << 12) | (blockIdx.x & 0xfffu);
}
// true = keep polling
__device__ __forceinline__ bool wait_slow_path(uint32_t& spins, const WaitCtx& w, int code) {
    if ((++spins & 0xffu) != 0) return true;
    if (ld_shared_u32(w.block_smem) != 0) return false;
    if (spins > RF_MBAR_SPIN_LIMIT) {
        wait_timed_out(w.block_smem, code);
        return false;
    }
    return true;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity, const WaitCtx& w) {
    uint32_t spins = 0;
    while (!mbar_try_wait(bar, parity)) {
        if (!wait_slow_path(spins, w, kStatusBarrierTimeout)) break;
    }
}

// Test probes only (tests/gpu_probe, tools/probes): a single-CTA micro-kernel with no status word traps instead.
__device__ __forceinline__ void mbar_wait_or_trap(uint32_t bar, uint32_t parity) {
    uint32_t spins = 0;
    while (!mbar_try_wait(bar, parity)) {
        if (++spins > RF_MBAR_SPIN_LIMIT) __trap();
    }
}

// Two barriers at once: both try_waits are in flight together, so the (long) latency of a
// phase check is paid once, not twice.
__device__ __forceinline__ void mbar_wait2(uint32_t bar_a, uint32_t parity_a, uint32_t bar_b, uint32_t parity_b,
                                           const WaitCtx& w) {
    uint32_t spins = 0;
    for (;;) {
        const uint32_t oa = mbar_try_wait(bar_a, parity_a);
        const uint32_t ob = mbar_try_wait(bar_b, parity_b);
        if (oa & ob) break;
        if (!wait_slow_path(spins, w, kStatusBarrierTimeout)) break;
    }
}

// ------------------------------------------------------------------------------------------
// TMA (cp.async.bulk.tensor), 4-D tiled tensor maps
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void prefetch_tensormap(const void* tmap) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t smem_dst, const void* tmap, uint32_t bar, int c0, int c1,
                                            int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
        "%6}], [%2];"
        ::"r"(smem_dst),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t smem_dst, const void* tmap, uint32_t bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(smem_dst),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}

// multicast to the CTAs of the cluster named in cta_mask: the box lands at the same shared-memory offset, and
// completes bytes on the mbarrier at the same offset, in every destination CTA
__device__ __forceinline__ void tma_load_2d_multicast(uint32_t smem_dst, const void* tmap, uint32_t bar, int c0, int c1,
                                                      uint16_t cta_mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, "
        "%4}], [%2], %5;"
        ::"r"(smem_dst),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar), "r"(c0), "r"(c1), "h"(cta_mask)
        : "memory");
}
// TMA store of one box from (swizzled) shared memory; rows / columns outside the tensor are not written
__device__ __forceinline__ void tma_store_2d(const void* tmap, uint32_t smem_src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(tmap)),
                 "r"(smem_src), "r"(c0), "r"(c1)
                 : "memory");
}
// global[box] += shared[box], element-wise in the tensor map's type (f32 here), performed by the TMA unit / L2
__device__ __forceinline__ void tma_reduce_add_2d(const void* tmap, uint32_t smem_src, int c0, int c1) {
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(tmap)),
                 "r"(smem_src), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void tma_store_3d(const void* tmap, uint32_t smem_src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(tmap)),
                 "r"(smem_src), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit_group() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// at most kPending of this thread's bulk groups may still be READING their shared-memory source
template <int kPending>
__device__ __forceinline__ void bulk_wait_group_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kPending) : "memory");
}
template <int kPending>
__device__ __forceinline__ void bulk_wait_group() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(kPending) : "memory");
}

// ------------------------------------------------------------------------------------------
// thread-block clusters
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ------------------------------------------------------------------------------------------
// tcgen05: TMEM allocation, fences, commit
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t smem_result_addr, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_result_addr),
                 "r"(ncols)
                 : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// mbarrier arrives once all tcgen05 async ops previously issued by this thread have completed
// (implies tcgen05.fence::before_thread_sync).
__device__ __forceinline__ void tc_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}

// the same arrival on the barrier at this offset in every CTA of cta_mask (a shared-memory stage that a peer CTA's
// multicast load also fills is free only when both consumers are done with it)
__device__ __forceinline__ void tc_commit_multicast(uint32_t bar, uint16_t cta_mask) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
                 "h"(cta_mask)
                 : "memory");
}

// ------------------------------------------------------------------------------------------
// tcgen05.mma, kind::f16 (bf16/f16 inputs, f32 accumulate in TMEM)
// ------------------------------------------------------------------------------------------
// D[tmem] (+)= A[smem desc] * B[smem desc]
__device__ __forceinline__ void mma_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem desc]
__device__ __forceinline__ void mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Shared-memory matrix descriptor (64-bit):
//   [0,14)  start address >> 4        [16,30) leading-dim byte offset >> 4
//   [32,46) stride-dim byte offset>>4 [46,48) version = 1 (sm_100)
//   [49,52) base offset (0: tiles are 1024B aligned)   [52] LBO mode = 0
//   [61,64) swizzle: 0 none, 2 = 128B, 4 = 64B, 6 = 32B
enum : uint32_t { kSwizzleNone = 0, kSwizzle128B = 2, kSwizzle64B = 4, kSwizzle32B = 6 };

__device__ __forceinline__ uint64_t make_smem_desc(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                                   uint32_t swizzle) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(swizzle & 7u) << 61;
    return d;
}

// Instruction descriptor (32-bit) for kind::f16:
//   [4,6) D format (1 = f32)   [7,10) A format (0 f16, 1 bf16)   [10,13) B format
//   [15] A major (0 = K)       [16] B major (0 = K, 1 = MN)
//   [17,23) N >> 3             [24,29) M >> 4
__host__ __device__ constexpr uint32_t make_idesc_f16(uint32_t ab_format, uint32_t a_mn_major, uint32_t b_mn_major,
                                                      uint32_t m, uint32_t n) {
    return (1u << 4) | (ab_format << 7) | (ab_format << 10) | (a_mn_major << 15) | (b_mn_major << 16) |
           ((n >> 3) << 17) | ((m >> 4) << 24);
}

// ------------------------------------------------------------------------------------------
// tcgen05.ld / tcgen05.st, shape 32x32b: thread t of the warp <-> TMEM lane (lane_base + t),
// .xN = N consecutive 32-bit columns.  lane_base (bits 31:16 of the address) must be the
// warp's own quadrant: 32 * (warp_id % 4).
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
          "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
          "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%8], {%0, %1, %2, %3, %4, %5, %6, %7};" ::"r"(r[0]),
        "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%32], "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31};" ::"r"(r[0]),
        "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
        "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]),
        "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]), "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%16], "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15};" ::"r"(r[0]),
        "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(taddr)
        : "memory");
}

// ------------------------------------------------------------------------------------------
// math helpers
// ------------------------------------------------------------------------------------------
// 256-bit global store (sm_100): eight 32-bit words, 32-byte aligned
__device__ __forceinline__ void st_global_v8(void* dst, const uint32_t (&w)[8]) {
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst), "r"(w[0]), "r"(w[1]), "r"(w[2]),
                 "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                 : "memory");
}

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float max3(float a, float b, float c) {
    float y;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(y) : "f"(a), "f"(b), "f"(c));
    return y;
}
// pack (lo, hi) -> two 16-bit floats in one 32-bit word, lo in bits [0,16)
template <bool kBf16>
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
    uint32_t y;
    if (kBf16)
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(y) : "f"(hi), "f"(lo));
    else
        asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(y) : "f"(hi), "f"(lo));
    return y;
}

// packed f32x2 math (sm_100): one instruction for two lanes of a register pair
__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b, float c) {
    uint64_t a, bb, cc, d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(b));
    asm("mov.b64 %0, {%1, %1};" : "=l"(cc) : "f"(c));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(bb), "l"(cc));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(d));
}
__device__ __forceinline__ void fadd2(float& acc0, float& acc1, float a0, float a1) {
    uint64_t a, d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(acc0), "f"(acc1));
    asm("add.rn.f32x2 %0, %0, %1;" : "+l"(d) : "l"(a));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(acc0), "=f"(acc1) : "l"(d));
}
__device__ __forceinline__ void fmul2(float& d0, float& d1, float b) {
    uint64_t a, bb;
    asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(d0), "f"(d1));
    asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(b));
    asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(a) : "l"(bb));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(a));
}

// 64-bit register-pair forms (avoid pack/unpack moves when chaining packed ops)
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ uint64_t bc2(float v) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(v));
    return r;
}
__device__ __forceinline__ void unpk2(uint64_t v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2v(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t fadd2v(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

// 2^x for two lanes on the FMA/ALU pipes only (no MUFU): Cody-Waite split x = n + f with the
// 1.5*2^23 rounding trick, degree-3 minimax polynomial for 2^f on [-0.5, 0.5] (max relative
// error 7.5e-5, far below the bf16 rounding applied to P afterwards), exponent insertion by an
// integer add.  x <= ~100; -inf (masked) is clamped to -126 and yields ~1e-38 (a denormal that
// flushes to 0 in the bf16 pack).
__device__ __forceinline__ void exp2_poly2(float& x0, float& x1) {
    constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
    x0 = fmaxf(x0, -126.0f);
    x1 = fmaxf(x1, -126.0f);
    const uint64_t x = pk2(x0, x1);
    const uint64_t t = fadd2v(x, bc2(kMagic));            // low mantissa bits = round(x)
    const uint64_t r = fadd2v(t, bc2(-kMagic));           // round(x) as float
    const uint64_t f = ffma2v(r, bc2(-1.0f), x);          // x - round(x) in [-0.5, 0.5]
    uint64_t pl = ffma2v(f, bc2(0.055171459913253784f), bc2(0.2426108568906784f));
    pl = ffma2v(pl, f, bc2(0.6932609677314758f));
    pl = ffma2v(pl, f, bc2(0.9999281167984009f));
    float t0, t1, p0, p1;
    unpk2(t, t0, t1);
    unpk2(pl, p0, p1);
    x0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
    x1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
}

// named barrier among a subset of the CTA's warps (id 1..15; id 0 is __syncthreads)
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// warpgroup register reallocation (all 128 threads of an aligned warpgroup must execute it)
template <int kRegs>
__device__ __forceinline__ void setmaxnreg_inc() {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegs));
}
template <int kRegs>
__device__ __forceinline__ void setmaxnreg_dec() {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegs));
}

__device__ __forceinline__ uint32_t elect_one() {
    uint32_t pred;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "elect.sync _|p, 0xffffffff;\n"
        "selp.b32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(pred));
    return pred;
}

// ---- norms for the row-max skip test (fa_fwd_sm100.cu, fa_fwd_sm100_d128.cu) ----
// An UPPER bound (within 1.6 %) of the sum of squares of the eight 16-bit values of a 16-byte chunk, added to two
// independent accumulators.  bf16: the odd element of a word is used as it sits in the word -- the even element's
// bits below it only lengthen the mantissa, |w| >= |hi| and at most 2^-7 larger -- which saves the mask; the skip test
// needs a bound, not the norm.
template <bool kBf16>
__device__ __forceinline__ void sumsq_chunk(const uint4& v, float& a0, float& a1) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        float lo, hi;
        if (kBf16) {
            lo = __uint_as_float(w[e] << 16);
            hi = __uint_as_float(w[e]);
        } else {
            const float2 f2 = __half22float2(*reinterpret_cast<const __half2*>(&w[e]));
            lo = f2.x;
            hi = f2.y;
        }
        a0 = fmaf(lo, lo, a0);
        a1 = fmaf(hi, hi, a1);
    }
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
// Bound of |row|^2 for kRows 128-byte rows (kStride bytes apart) of a 128B-swizzled tile at once.  The swizzle
// permutes a row's eight chunks, which a sum does not care about; lane l starts at chunk l mod 8 so that the warp's
// 32 rows hit all banks (4 wavefronts per LDS.128).  Loads go out in batches, and every row has two accumulators.
template <bool kBf16, int kRows, uint32_t kStride>
__device__ __forceinline__ void rows_sumsq(uint32_t row_addr, int lane, float (&out)[kRows]) {
    float a0[kRows], a1[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) a0[r] = a1[r] = 0.f;
#pragma unroll
    for (int c = 0; c < 8; c += 2) {
        uint4 v[kRows][2];
#pragma unroll
        for (int r = 0; r < kRows; ++r)
#pragma unroll
            for (int u = 0; u < 2; ++u) v[r][u] = lds128(row_addr + r * kStride + (((c + u + lane) & 7) << 4));
#pragma unroll
        for (int r = 0; r < kRows; ++r)
#pragma unroll
            for (int u = 0; u < 2; ++u) sumsq_chunk<kBf16>(v[r][u], a0[r], a1[r]);
    }
#pragma unroll
    for (int r = 0; r < kRows; ++r) out[r] = a0[r] + a1[r];
}

}  // namespace rfptx
