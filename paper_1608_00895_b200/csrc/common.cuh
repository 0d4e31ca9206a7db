// common.cuh -- sm_100a building blocks shared by the kernels of libblstm.so:
// mbarriers, TMA (cp.async.bulk.tensor), tcgen05 (TMEM alloc / MMA / commit /
// ld) and the UMMA shared-memory + instruction descriptors.
//
// Descriptor bit layouts follow the PTX ISA "tcgen05 matrix descriptor" and
// "instruction descriptor" tables (kind::f16): see DESIGN.md §5.1.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#define DEVI __device__ __forceinline__

namespace blstm {

// ---------------------------------------------------------------------------
// generic
// ---------------------------------------------------------------------------
DEVI uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

DEVI uint32_t lane_id() { return threadIdx.x & 31u; }
DEVI uint32_t warp_id() { return threadIdx.x >> 5; }

DEVI bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(pred));
    return pred != 0;
}

// ---------------------------------------------------------------------------
// mbarrier
// ---------------------------------------------------------------------------
DEVI void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
DEVI void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
DEVI void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
DEVI void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
DEVI bool mbar_try_wait(uint32_t addr, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    return ok != 0;
}
DEVI uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// try_wait with a suspend-time hint: a thread whose phase is not complete is parked by the
// hardware until the phase completes (or the hint expires) instead of re-polling; a polling warp
// takes issue slots from the warps of its sub-partition that do the step's work (measured: the
// MMA-completion wait alone was ~70 instructions per warp per step of the forward recurrence)
#ifndef BLSTM_WAIT_HINT_NS
#define BLSTM_WAIT_HINT_NS 10000000u
#endif
DEVI bool mbar_try_wait_sleep(uint32_t addr, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity), "r"(BLSTM_WAIT_HINT_NS)
        : "memory");
    return ok != 0;
}
// Watchdog for every spin: a synchronisation bug traps (kernel error) instead of hanging the GPU.
constexpr uint64_t SPIN_TIMEOUT_NS = 20ull * 1000 * 1000 * 1000;
DEVI void mbar_wait(uint64_t *bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    if (mbar_try_wait(a, parity)) return;
#if BLSTM_WAIT_HINT_NS
    const uint64_t t0 = globaltimer_ns();
    while (!mbar_try_wait_sleep(a, parity))
        if (globaltimer_ns() - t0 > SPIN_TIMEOUT_NS) __trap();
#else
    // (the timer is read every 256 polls only: each read is an issue slot on the critical path)
    uint64_t t0 = 0;
    for (uint32_t n = 1; !mbar_try_wait(a, parity); ++n) {
        if ((n & 255) == 0) {
            const uint64_t t = globaltimer_ns();
            if (!t0) t0 = t;
            else if (t - t0 > SPIN_TIMEOUT_NS) __trap();
        }
    }
#endif
}

// ---------------------------------------------------------------------------
// thread-block clusters / distributed shared memory
// ---------------------------------------------------------------------------
DEVI uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
DEVI void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address -> shared::cluster address of the same offset in CTA `rank`
DEVI uint32_t mapa_shared(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
// bulk copy local smem -> (possibly remote) smem, completing tx bytes on the destination's mbarrier
DEVI void bulk_s2c(uint32_t dst_cluster, uint32_t src_cta, uint32_t bytes, uint32_t mbar_cluster) {
    asm volatile(
        "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            dst_cluster),
        "r"(src_cta), "r"(bytes), "r"(mbar_cluster)
        : "memory");
}
// bulk copy global -> this CTA's smem (16-byte aligned, size % 16 == 0), completing tx bytes on bar
DEVI void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// per-thread asynchronous copies global -> own smem through the LSU (not the bulk-copy engine);
// completion is per thread (cp.async.commit_group / wait_group), no register scoreboard involved
DEVI void cp_async16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
DEVI void cp_async8(uint32_t dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
DEVI void cp_async4(uint32_t dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
// 4-byte copy reading src_bytes (0 or 4) bytes; the rest of the destination is zero-filled
DEVI void cp_async4_zfill(uint32_t dst, const void *src, uint32_t src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
template <int BYTES>
DEVI void cp_async(uint32_t dst, const void *src) {
    static_assert(BYTES == 4 || BYTES == 8 || BYTES == 16, "cp.async size");
    if constexpr (BYTES == 16) cp_async16(dst, src);
    else if constexpr (BYTES == 8) cp_async8(dst, src);
    else cp_async4(dst, src);
}
DEVI void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
DEVI void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// order this thread's (acquired) view of global memory before its later async-proxy reads of it
DEVI void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
DEVI void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
DEVI void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
// 16-byte store into a (possibly remote) CTA's shared memory, completing tx bytes on its mbarrier
DEVI void st_async_v4u(uint32_t dst_cluster, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t mbar_cluster) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
            dst_cluster),
        "r"(a), "r"(b), "r"(c), "r"(d), "r"(mbar_cluster)
        : "memory");
}
DEVI void st_async_v2u(uint32_t dst_cluster, uint32_t a, uint32_t b, uint32_t mbar_cluster) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];" ::"r"(
                     dst_cluster),
                 "r"(a), "r"(b), "r"(mbar_cluster)
                 : "memory");
}
DEVI void st_async_v4(uint32_t dst_cluster, float a, float b, float c, float d, uint32_t mbar_cluster) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
            dst_cluster),
        "f"(a), "f"(b), "f"(c), "f"(d), "r"(mbar_cluster)
        : "memory");
}

// ---------------------------------------------------------------------------
// proxy fences
// ---------------------------------------------------------------------------
// generic-proxy writes to shared memory -> visible to the async proxy (tcgen05.mma, TMA store)
DEVI void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// generic-proxy global writes (possibly by other SMs, acquired) -> async-proxy (TMA) reads
DEVI void fence_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// ---------------------------------------------------------------------------
// TMA
// ---------------------------------------------------------------------------
DEVI void tma_prefetch_desc(const CUtensorMap *m) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
DEVI void tma_load_2d(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// ---------------------------------------------------------------------------
// tcgen05
// ---------------------------------------------------------------------------
DEVI void tmem_alloc(uint32_t *dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
}
DEVI void tmem_relinquish() { asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory"); }
DEVI void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
DEVI void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
DEVI void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T   (kind::f16: fp16 operands, fp32 accumulate)
DEVI void mma_f16_ss(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]^T
DEVI void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Warp-collective issue: the whole (converged) warp executes these and one elected lane issues.
// With warp-uniform operands ptxas keeps them in uniform registers (UIADD3 + UTCHMMA, no
// per-MMA ELECT / R2UR waterfall as when a single divergent thread issues).
DEVI void mma_f16_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
        " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
DEVI void mma_f16_ss_w(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
        " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
DEVI void mma_commit_w(uint64_t *bar) {
    asm volatile(
        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
        " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
            smem_u32(bar))
        : "memory");
}
// ---- CTA pairs (cta_group::2): cluster ranks 2p and 2p+1, on the two SMs of a TPC ----------------
// Verified on B200 by scripts/pair_test.cu: alloc/relinquish/dealloc are executed by one warp in
// EACH CTA of the pair; an MMA issued by the even CTA computes M = 256 rows, A (TMEM, TS mode)
// supplying rows 128r.. from CTA r's TMEM, B split by N (CTA r holds columns [rN/2, (r+1)N/2)
// at the same smem offset), and CTA r's TMEM receives its 128 rows x all N columns of D.
DEVI void tmem_alloc2(uint32_t *dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
}
DEVI void tmem_relinquish2() { asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory"); }
DEVI void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
DEVI void mma_f16_ts2_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
        " @e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// arrive (once) on the mbarrier at this smem offset in every CTA of cta_mask when the pair MMAs
// issued so far by this thread complete
DEVI void mma_commit2_w(uint64_t *bar, uint16_t cta_mask) {
    asm volatile(
        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
        " @e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(
            smem_u32(bar)),
        "h"(cta_mask)
        : "memory");
}
// arrive on an mbarrier of another CTA of the cluster.  Relaxed: a release would first wait for
// this thread's earlier global stores to become visible (measured ~0.9 us on the recurrence's
// critical path); the data announced here was written by bulk copies whose completion this thread
// has just observed on its own mbarrier.
DEVI void mbar_remote_arrive(uint32_t bar_cluster) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
DEVI bool mbar_try_wait_cluster(uint32_t addr, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    return ok != 0;
}
DEVI bool mbar_try_wait_cluster_sleep(uint32_t addr, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity), "r"(BLSTM_WAIT_HINT_NS)
        : "memory");
    return ok != 0;
}
// wait for a phase completed by a remote (cluster-scope) arrive
DEVI void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    if (mbar_try_wait_cluster(a, parity)) return;
#if BLSTM_WAIT_HINT_NS
    const uint64_t t0 = globaltimer_ns();
    while (!mbar_try_wait_cluster_sleep(a, parity))
        if (globaltimer_ns() - t0 > SPIN_TIMEOUT_NS) __trap();
#else
    uint64_t t0 = 0;
    for (uint32_t n = 1; !mbar_try_wait_cluster(a, parity); ++n) {
        if ((n & 255) == 0) {
            const uint64_t t = globaltimer_ns();
            if (!t0) t0 = t;
            else if (t - t0 > SPIN_TIMEOUT_NS) __trap();
        }
    }
#endif
}

// a warp-uniform copy of v (lane 0's), so the compiler may keep it in a uniform register
DEVI int warp_uniform(int v) { return __shfl_sync(0xffffffffu, v, 0); }

// Four TS-mode MMAs in one asm block (operands made warp-uniform once per block, not per
// MMA): D += A[a + 8i] . B[bdesc + i*binc]^T for i = 0..3; the first one accumulates iff acc0.
// a + 8 columns = the next 16 fp16 of K in TMEM; binc = descriptor start-address step (16-B units).
DEVI void mma_f16_ts_x4(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t binc, uint32_t idesc,
                        uint32_t acc0) {
    asm volatile(
        "{\n .reg .pred p, t;\n .reg .b32 a1, a2, a3;\n .reg .b64 inc, b1, b2, b3;\n"
        " setp.ne.b32 p, %5, 0;\n setp.eq.b32 t, %5, %5;\n"
        " cvt.u64.u32 inc, %4;\n"
        " add.u32 a1, %1, 8;\n add.u32 a2, %1, 16;\n add.u32 a3, %1, 24;\n"
        " add.u64 b1, %2, inc;\n add.u64 b2, b1, inc;\n add.u64 b3, b2, inc;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, t;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], b2, %3, t;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], b3, %3, t;\n}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(binc), "r"(acc0)
        : "memory");
}
// arrive on an mbarrier when all previously issued tcgen05 ops of this thread complete
DEVI void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
DEVI void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
DEVI void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 32 lanes x 16 columns of 32-bit: thread i gets lane (base_lane + i), columns col..col+15
DEVI void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
// 32 lanes x 16 columns store (thread i writes lane base_lane + i)
DEVI void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

// 32 lanes x 8 columns store
DEVI void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

// ---------------------------------------------------------------------------
// UMMA descriptors
// ---------------------------------------------------------------------------
// Shared-memory matrix descriptor, SWIZZLE_128B, sm_100 version field = 1.
//   K-major : rows of 128 B (64 fp16 of K), 8-row atoms of 1024 B; SBO = 1024 (next 8 rows).
//             Advance along K by +32 B per 16 elements.
//   MN-major: rows of 128 B (64 fp16 of M/N) per k; 8 k-rows per 1024 B atom; SBO = 1024
//             (next 8 k), LBO = byte distance between 64-element M/N blocks.
//             Advance along K by +2048 B per 16 elements.
DEVI uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // version
    d |= (uint64_t)2 << 61;  // SWIZZLE_128B
    return d;
}

// Shared-memory matrix descriptor without swizzle (K-major "interleave" layout): core matrices
// of 8 rows x 16 B stored contiguously (128 B); SBO = byte distance between 8-row groups,
// LBO = byte distance between the two 8-element K halves of one 16-element MMA step.
DEVI uint64_t sdesc_noswz(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // version; layout type 0 = SWIZZLE_NONE
    return d;
}

// Instruction descriptor, kind::f16 with fp16 A/B and fp32 D.
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, int a_mn_major, int b_mn_major) {
    return (1u << 4)                          // D format = F32
           | (0u << 7) | (0u << 10)           // A, B = F16
           | ((uint32_t)a_mn_major << 15)     // A major
           | ((uint32_t)b_mn_major << 16)     // B major
           | ((uint32_t)(N >> 3) << 17)       // N / 8
           | ((uint32_t)(M >> 4) << 24);      // M / 16
}

// byte offset of element (row, col) inside a K-major SW128 tile made of
// 64-column blocks of `rows` rows each ([col/64][row][128 B], 16-B chunks XOR row%8)
DEVI uint32_t sw128_offset(uint32_t row, uint32_t col, uint32_t rows) {
    const uint32_t kb = col >> 6, c = col & 63u;
    const uint32_t chunk = (c >> 3) ^ (row & 7u);
    return kb * rows * 128u + row * 128u + (chunk << 4) + ((c & 7u) << 1);
}

// ---------------------------------------------------------------------------
// numerics (fp32; no approximate transcendentals on c or h: DESIGN.md R9)
// ---------------------------------------------------------------------------
DEVI float sigmoidf_acc(float z) {
    if (z >= 0.f) return 1.f / (1.f + expf(-z));
    const float e = expf(z);
    return e / (1.f + e);
}

// ---------------------------------------------------------------------------
// gpu-scope flag helpers for the persistent kernels' step barriers
// ---------------------------------------------------------------------------
DEVI uint32_t ld_acquire_gpu(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
DEVI void spin_until_geq(const uint32_t *p, uint32_t target) {
    if (ld_acquire_gpu(p) >= target) return;
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_gpu(p) < target) {
        if (globaltimer_ns() - t0 > SPIN_TIMEOUT_NS) __trap();
    }
}
DEVI void red_release_gpu_add(uint32_t *p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---------------------------------------------------------------------------
// Start arbitration between a persistent consumer and the concurrent producer it spins on (the
// forward recurrence and its Z GEMM, launched as a programmatic dependent: PDL lets the GEMM start
// early but does not guarantee it -- a profiler that serializes kernels, CUDA_LAUNCH_BLOCKING, an
// MPS SM cap or a co-tenant can keep it off the GPU until the consumer exits).  Two words per
// launch pair, zeroed before it: arb[0] counts resident producer CTAs (each adds 1 at entry),
// arb[1] is the decision, set once by compare-and-swap: ARB_GO by a consumer CTA that saw every
// producer CTA resident (count == target), ARB_ABORT by one that waited ARB_TIMEOUT_NS without
// seeing it.  Every consumer CTA follows the one decision: an aborted consumer exits at once and
// a conditional re-launch after the producer does the work (api.cu stack_forward).
// (A compare-and-swap loop on a single word by the 52 producer CTAs cost ~20 us per launch.)
// ---------------------------------------------------------------------------
constexpr uint32_t ARB_GO = 1u, ARB_ABORT = 2u;
constexpr uint64_t ARB_TIMEOUT_NS = 20ull * 1000 * 1000;
DEVI void arb_checkin(uint32_t *arb) { red_release_gpu_add(arb, 1u); }  // producer CTA, one thread
DEVI bool arb_decide(uint32_t *arb, uint32_t target) {  // consumer CTA, one thread: true = go
    const uint64_t t0 = globaltimer_ns();
    for (;;) {
        uint32_t d = ld_acquire_gpu(arb + 1);
        if (d == 0) {
            if (ld_acquire_gpu(arb) >= target) d = atomicCAS(arb + 1, 0u, ARB_GO);
            else if (globaltimer_ns() - t0 > ARB_TIMEOUT_NS) d = atomicCAS(arb + 1, 0u, ARB_ABORT);
            else { __nanosleep(128); continue; }
            if (d == 0) d = ld_acquire_gpu(arb + 1);  // our CAS won: re-read the word we wrote
        }
        return d == ARB_GO;
    }
}

}  // namespace blstm
