// mma_rate.cu -- tcgen05 MMA issue rate for the C5 persistent BPTT's per-step shape:
// 33.5 MFLOP per CTA and step = 64 MMAs of M = 128, N = 128 (batch), K = 16, A (R) from TMEM.
// Each mode issues the same work per CTA `reps` times (commit + wait per rep, like one step) on
// 32 two-CTA clusters (64 SMs, the shipped grid), operands are constant garbage:
//   mode 0: cta_group::1, M = 128, N = 128, A from TMEM (ts)         -- as shipped
//   mode 1: cta_group::2, M = 256, N = 128, A from TMEM, B split by N -- a CTA pair per 2 unit tiles
//   mode 2: cta_group::1, M = 128, N = 128, A from shared memory (ss)
//   mode 3: cta_group::1, M = 128, N = 256, ts (32 MMAs: same flops)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1608_00895_b200/csrc -o mma_rate mma_rate.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_fp16.h>
#include "common.cuh"

using namespace blstm;

constexpr int THREADS = 128;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1) rate_kernel(int mode, int reps, int *sink) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t *sm = (uint8_t *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *bs = sm;              // B: 256 rows x 64 K fp16 SW128 (32 KB)
    uint8_t *as = sm + 32768;      // A (ss mode): 128 rows x 64 K (16 KB)
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int r = (int)cluster_ctarank(), t = threadIdx.x, w = t >> 5;
    for (int i = t; i < 49152 / 16; i += THREADS)
        reinterpret_cast<uint4 *>(sm)[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u);
    if (t == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (w == 0) {
        if (mode == 1) {
            tmem_alloc2(&tslot, 512);
            tmem_relinquish2();
        } else {
            tmem_alloc(&tslot, 512);
            tmem_relinquish();
        }
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tslot;
    uint32_t ph = 0;
    const uint32_t sb = smem_u32(bs), sa = smem_u32(as);
    for (int rep = 0; rep < reps; ++rep) {
        if (w == 0) {
            if (mode == 0 || mode == 2) {
                const uint32_t idesc = idesc_f16(128, 128, 0, 0);
                for (int i = 0; i < 64; ++i) {
                    const int kk = i & 3;
                    if (mode == 0)
                        mma_f16_ts_w(tmem + 384, tmem + (uint32_t)((i * 8) % 384), sdesc_sw128(sb + kk * 32, 16, 1024),
                                     idesc, i != 0);
                    else
                        mma_f16_ss_w(tmem + 384, sdesc_sw128(sa + kk * 32, 16, 1024), sdesc_sw128(sb + kk * 32, 16, 1024),
                                     idesc, i != 0);
                }
                mma_commit_w(&bar);
            } else if (mode == 3) {
                const uint32_t idesc = idesc_f16(128, 256, 0, 0);
                for (int i = 0; i < 32; ++i) {
                    const int kk = i & 3;
                    mma_f16_ts_w(tmem + 256, tmem + (uint32_t)((i * 8) % 256), sdesc_sw128(sb + kk * 32, 16, 1024), idesc,
                                 i != 0);
                }
                mma_commit_w(&bar);
            } else if (r == 0) {  // mode 1: the even CTA issues for the pair
                const uint32_t idesc = idesc_f16(256, 128, 0, 0);
                for (int i = 0; i < 64; ++i) {
                    const int kk = i & 3;
                    mma_f16_ts2_w(tmem + 384, tmem + (uint32_t)((i * 8) % 384), sdesc_sw128(sb + kk * 32, 16, 1024),
                                  idesc, i != 0);
                }
                mma_commit2_w(&bar, (uint16_t)3);
            }
        }
        mbar_wait(&bar, ph);
        ph ^= 1;
        tc_fence_after();
        __syncthreads();
        if (mode == 1) cluster_sync();  // the pair's next rep starts together
    }
    if (t == 0) sink[blockIdx.x] = reps;
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (w == 0) {
        tc_fence_after();
        if (mode == 1) tmem_dealloc2(tmem, 512);
        else tmem_dealloc(tmem, 512);
    }
}

int main(int argc, char **argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 1000;
    int *sink;
    cudaMalloc(&sink, 4096);
    const int smem = 49152 + 1024;
    cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char *names[4] = {"cg1 ts M128 N128 (shipped)", "cg2 ts M256 N128 (pair)", "cg1 ss M128 N128", "cg1 ts M128 N256"};
    for (int mode = 0; mode < 4; ++mode) {
        for (int ctas : {2, 64}) {
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            rate_kernel<<<ctas, THREADS, smem>>>(mode, 10, sink);
            cudaEventRecord(a);
            rate_kernel<<<ctas, THREADS, smem>>>(mode, reps, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            const double ns = ms * 1e6 / reps;
            const double tf = 33.554432e6 / (ns * 1e-9) / 1e12;  // per CTA (SM)
            printf("mode %d %-28s CTAs %3d: %7.1f ns per step (33.5 MFLOP per SM) = %5.2f TF/s per SM  %s\n", mode,
                   names[mode], ctas, ns, tf, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
