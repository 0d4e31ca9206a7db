// dsmem_bench.cu -- microbenchmark of the recurrence kernels' per-step exchange: a cluster of
// 16 CTAs (1 per SM) repeatedly all-gathers a slice of `bytes` per CTA through distributed
// shared memory (cp.async.bulk shared::cta -> shared::cluster, complete_tx on the receiver's
// mbarrier, double-buffered), exactly the forward kernel's h exchange.  Reports ns per round.
//   modes: 0 = one thread issues all 16 copies, 1 = lane 0 of 16 warps issues one each,
//          2 = st.async.v4 from registers by all threads (no staging)
//          3 = half the peers by bulk copy (mode 1), the other half by st.async (mode 2): tests
//              whether the bulk-copy engine and the LSU st.async path add bandwidth
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o dsmem_bench dsmem_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define DEVI __device__ __forceinline__
DEVI uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
DEVI uint32_t rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
DEVI void csync() { asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
DEVI uint32_t mapa(uint32_t a, uint32_t r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
DEVI void minit(uint64_t *b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c)); }
DEVI void mexpect(uint64_t *b, uint32_t tx) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory"); }
DEVI bool mtry(uint32_t a, uint32_t ph) {
    uint32_t ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(a), "r"(ph) : "memory");
    return ok;
}
DEVI void mwait(uint64_t *b, uint32_t ph) { while (!mtry(smem_u32(b), ph)) {} }
DEVI void bulk(uint32_t dst, uint32_t src, uint32_t n, uint32_t mb) {
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "r"(src), "r"(n), "r"(mb) : "memory");
}
DEVI void stas(uint32_t dst, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t mb) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];" ::"r"(dst), "r"(a), "r"(b), "r"(c), "r"(d), "r"(mb) : "memory");
}

__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(512, 1) kern(int rounds, int bytes, int mode, long long *out) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int NC = 16;
    uint8_t *buf = sm;                              // [2][NC][bytes]
    uint8_t *stg = sm + 2 * NC * bytes;             // [bytes]
    uint64_t *full = (uint64_t *)(stg + bytes);     // [2]
    const uint32_t c = rank(), w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (threadIdx.x == 0) { minit(&full[0], 1); minit(&full[1], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    if (threadIdx.x == 0) { mexpect(&full[0], NC * bytes); mexpect(&full[1], NC * bytes); }
    csync();
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int s = 0; s < rounds; ++s) {
        const int b = s & 1;
        // "compute": write the staging slice
        for (int i = threadIdx.x * 16; i < bytes; i += 512 * 16) *(uint4 *)(stg + i) = make_uint4(s, c, i, 0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        const uint32_t dst = smem_u32(buf + (b * NC + c) * bytes), mb = smem_u32(&full[b]);
        if (mode == 0) {
            if (threadIdx.x == 0) {
                for (int r = 0; r < NC; ++r) bulk(mapa(dst, r), smem_u32(stg), bytes, mapa(mb, r));
                asm volatile("cp.async.bulk.commit_group;");
            }
        } else if (mode == 1) {
            if (l == 0 && w < NC) { bulk(mapa(dst, w), smem_u32(stg), bytes, mapa(mb, w)); asm volatile("cp.async.bulk.commit_group;"); }
        } else if (mode == 2) {
            // each thread stores 16 B pieces of the slice to every peer
            for (int i = threadIdx.x * 16; i < bytes; i += 512 * 16)
                for (int r = 0; r < NC; ++r) stas(mapa(dst + i, r), s, c, i, 0, mapa(mb, r));
        } else {
            if (l == 0 && w < NC / 2) { bulk(mapa(dst, w), smem_u32(stg), bytes, mapa(mb, w)); asm volatile("cp.async.bulk.commit_group;"); }
            for (int i = threadIdx.x * 16; i < bytes; i += 512 * 16)
                for (int r = NC / 2; r < NC; ++r) stas(mapa(dst + i, r), s, c, i, 0, mapa(mb, r));
        }
        mwait(&full[b], (ph >> b) & 1);
        ph ^= 1u << b;
        if (threadIdx.x == 0 && s + 2 < rounds) mexpect(&full[b], NC * bytes);
        if (mode != 2 && threadIdx.x < 32 * NC && l == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
    }
    long long t1 = clock64();
    csync();
    if (threadIdx.x == 0 && c == 0) out[blockIdx.x / 16] = t1 - t0;
}

int main() {
    long long *d;
    cudaMalloc(&d, 64 * sizeof(long long));
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const int rounds = 2000;
    for (int mode = 0; mode < 4; ++mode)
        for (int bytes : {1024, 2048, 4096}) {
            const size_t smem = 2 * 16 * bytes + bytes + 64;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            for (int clusters : {1, 6}) {
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0); cudaEventCreate(&e1);
                kern<<<16 * clusters, 512, smem>>>(100, bytes, mode, d);
                cudaEventRecord(e0);
                kern<<<16 * clusters, 512, smem>>>(rounds, bytes, mode, d);
                cudaEventRecord(e1);
                cudaError_t err = cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                long long cyc = 0;
                cudaMemcpy(&cyc, d, sizeof(cyc), cudaMemcpyDeviceToHost);
                printf("mode %d  bytes/CTA %5d  clusters %d : %7.1f ns/round (events), %6.0f cycles/round (clock64) %s\n",
                       mode, bytes, clusters, ms * 1e6 / rounds, (double)cyc / rounds, err == cudaSuccess ? "" : cudaGetErrorString(err));
            }
        }
    return 0;
}
