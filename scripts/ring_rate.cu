// ring_rate.cu -- the C5 persistent BPTT's per-step operand pipeline in isolation:
// 16 chunks of dA (128 batch rows x 64 gate columns fp16 = 16 KB, SW128) per CTA and step through a
// 7-slot ring (TMA warp -> full barrier -> MMA warp -> commit -> empty barrier), 64 CTAs in 32
// two-CTA clusters, one 2 MB "dA step" [128 rows][8192 columns] in L2 that every CTA reads a
// 1024-column K-split of (8 CTAs per split, as in the kernel).
//   mode 4: MMAs through the ring handshake, no loads (the producer arrives on full itself)
//   mode 5: TMA loads through the ring, no MMAs (the consumer commits at once)
//   mode 6: as 5 with a contiguous source (row pitch 128 B instead of 16 KB)
//   mode 7: TMA + MMAs (M = N = 128, A from TMEM)                          -- as shipped
//   mode 9: MMAs, no ring (every chunk's full barrier pre-armed), a commit after every chunk
//   mode 10: as 9 with one commit per step (the cost of the per-chunk commits)
//   mode 11: as 7 with 6 slots in 3 pairs: one commit (and one empty barrier) per pair of chunks
//   mode 8: CTA pair (cta_group::2): each CTA loads 64 batch rows (8 KB) into its own ring slot,
//           completing on the even CTA's full barrier (TMA .cta_group::2); the even CTA issues
//           M = 256 MMAs (its rows + the odd CTA's), commits multicast to both CTAs' empty barriers
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1608_00895_b200/csrc -o ring_rate ring_rate.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_fp16.h>
#include "common.cuh"

using namespace blstm;

constexpr int THREADS = 128, S = 7, KC = 16;
constexpr uint32_t CHUNK = 16384;

DEVI void tma_load_2d_pair(uint32_t dst, const CUtensorMap *m, uint32_t bar_cluster, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(c0), "r"(c1)
        : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    ring_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tmh, int mode, int reps,
                int *sink) {
    extern __shared__ uint8_t sm_raw[];
    uint8_t *ring = (uint8_t *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[S], empty[S], done, f16[KC], dummy;
    __shared__ uint32_t tslot;
    const int r = (int)cluster_ctarank(), t = threadIdx.x, w = t >> 5;
    const bool pair = mode == 8;
    if (t == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(&done, 1);
        for (int i = 0; i < KC; ++i) mbar_init(&f16[i], 1);
        mbar_init(&dummy, 1);
        fence_mbar_init();
    }
    if (w == 1) {
        if (pair) {
            tmem_alloc2(&tslot, 512);
            tmem_relinquish2();
        } else {
            tmem_alloc(&tslot, 512);
            tmem_relinquish();
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tslot;
    const int col0 = (blockIdx.x / 2 % 8) * 1024;
    int stage = 0;
    uint32_t phase = 0, dph = 0;
    const uint32_t idesc = idesc_f16(pair ? 256 : 128, 128, 0, 0);
    for (int rep = 0; rep < reps && mode >= 9; ++rep) {
        if (t == 0)
            for (int i = 0; i < KC; ++i) mbar_arrive(&f16[i]);
        __syncthreads();
        if (w == 1) {
            for (int kc = 0; kc < KC; ++kc) {
                mbar_wait(&f16[kc], (uint32_t)(rep & 1));
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    mma_f16_ts_w(tmem + 384, tmem + (uint32_t)((kc * 32 + kk * 8) % 384), sdesc_sw128(smem_u32(ring) + kk * 32, 16, 1024),
                                 idesc, (kc | kk) != 0);
                if (mode == 9) mma_commit_w(&dummy);
                __syncwarp();
            }
            mma_commit_w(&done);
            __syncwarp();
        }
        mbar_wait(&done, dph);
        dph ^= 1;
        tc_fence_after();
        __syncthreads();
    }
    for (int rep = 0; rep < reps && mode == 11; ++rep) {
        // 3 groups of 2 slots; group g's empty barrier = empty[g]; chunk kc -> slot kc % 6
        if (w == 0) {
            for (int kc = 0; kc < KC; ++kc) {
                const int c = rep * KC + kc, sl = c % 6, g = sl >> 1;
                const uint32_t use = (uint32_t)(c / 6);  // how many times this slot was used before
                if ((sl & 1) == 0) mbar_wait(&empty[g], (use & 1) ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(&full[sl], CHUNK);
                    tma_load_2d(ring + sl * CHUNK, &tm, &full[sl], col0 + kc * 64, 0);
                }
                __syncwarp();
            }
        } else if (w == 1) {
            for (int kc = 0; kc < KC; ++kc) {
                const int c = rep * KC + kc, sl = c % 6, g = sl >> 1;
                mbar_wait(&full[sl], (uint32_t)(c / 6) & 1);
                tc_fence_after();
                const uint32_t sb = smem_u32(ring + sl * CHUNK);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    mma_f16_ts_w(tmem + 384, tmem + (uint32_t)((kc * 32 + kk * 8) % 384), sdesc_sw128(sb + kk * 32, 16, 1024),
                                 idesc, (kc | kk) != 0);
                if ((sl & 1) == 1) mma_commit_w(&empty[g]);
                __syncwarp();
            }
            mma_commit_w(&done);
            __syncwarp();
        }
        mbar_wait(&done, dph);
        dph ^= 1;
        tc_fence_after();
        __syncthreads();
    }
    for (int rep = 0; rep < reps && mode < 9; ++rep) {
        if (w == 0) {  // producer
            int st2 = stage;
            uint32_t ph2 = phase;
            for (int kc = 0; kc < KC; ++kc) {
                mbar_wait(&empty[st2], ph2 ^ 1);
                if (mode == 4) {
                    if (elect_one()) mbar_arrive(&full[st2]);
                } else if (pair) {
                    if (elect_one()) {
                        // both CTAs' halves complete on the even CTA's full barrier (16 KB in all)
                        if (r == 0) mbar_arrive_expect_tx(&full[st2], CHUNK);
                        tma_load_2d_pair(smem_u32(ring + st2 * CHUNK), &tmh, mapa_shared(smem_u32(&full[st2]), 0),
                                         col0 + kc * 64, 64 * r);
                    }
                } else if (elect_one()) {
                    mbar_arrive_expect_tx(&full[st2], CHUNK);
                    tma_load_2d(ring + st2 * CHUNK, mode == 6 ? &tmh : &tm, &full[st2], mode == 6 ? 0 : col0 + kc * 64,
                                mode == 6 ? (blockIdx.x % 64) * 128 + kc * 0 : 0);
                }
                __syncwarp();
                if (++st2 == S) { st2 = 0; ph2 ^= 1; }
            }
        } else if (w == 1 && (!pair || r == 0)) {  // MMA issuer
            int st2 = stage;
            uint32_t ph2 = phase;
            for (int kc = 0; kc < KC; ++kc) {
                mbar_wait(&full[st2], ph2);
                tc_fence_after();
                const uint32_t sb = smem_u32(ring + st2 * CHUNK);
                if (mode == 4 || mode == 7) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        mma_f16_ts_w(tmem + 384, tmem + (uint32_t)((kc * 32 + kk * 8) % 384), sdesc_sw128(sb + kk * 32, 16, 1024),
                                     idesc, (kc | kk) != 0);
                    mma_commit_w(&empty[st2]);
                } else if (pair) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        mma_f16_ts2_w(tmem + 384, tmem + (uint32_t)((kc * 32 + kk * 8) % 384),
                                      sdesc_sw128(sb + kk * 32, 16, 1024), idesc, (kc | kk) != 0);
                    mma_commit2_w(&empty[st2], (uint16_t)3);
                } else {
                    mma_commit_w(&empty[st2]);
                }
                __syncwarp();
                if (++st2 == S) { st2 = 0; ph2 ^= 1; }
            }
            if (pair) mma_commit2_w(&done, (uint16_t)3);
            else mma_commit_w(&done);
            __syncwarp();
        }
        {
            const int adv = stage + KC;
            phase ^= (uint32_t)((adv / S) & 1);
            stage = adv % S;
        }
        mbar_wait(&done, dph);
        dph ^= 1;
        tc_fence_after();
        __syncthreads();
        if (pair) cluster_sync();
    }
    if (t == 0) sink[blockIdx.x] = reps;
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (w == 1) {
        tc_fence_after();
        if (pair) tmem_dealloc2(tmem, 512);
        else tmem_dealloc(tmem, 512);
    }
}

static int tmap(CUtensorMap *m, void *p, uint64_t inner, uint64_t outer, uint32_t box_outer) {
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {inner * 2};
    cuuint32_t box[2] = {64, box_outer};
    cuuint32_t estr[2] = {1, 1};
    return (int)cuTensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, p, dims, strides, box, estr,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

int main(int argc, char **argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 1000;
    void *dA, *cont;
    int *sink;
    cudaMalloc(&dA, 128 * 8192 * 2);
    cudaMalloc(&cont, 64 * 128 * 64 * 2);
    cudaMemset(dA, 0, 128 * 8192 * 2);
    cudaMemset(cont, 0, 64 * 128 * 64 * 2);
    cudaMalloc(&sink, 4096);
    CUtensorMap tm, tmc, tmh;
    int e1 = tmap(&tm, dA, 8192, 128, 128), e2 = tmap(&tmc, cont, 64, 64 * 128, 128), e3 = tmap(&tmh, dA, 8192, 128, 64);
    if (e1 || e2 || e3) {
        printf("tensor map error %d %d %d\n", e1, e2, e3);
        return 1;
    }
    const int smem = S * CHUNK + 1024;
    cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char *names[12] = {"", "", "", "", "MMA + ring, no loads", "loads, no MMA (16 KB row pitch)",
                             "loads, no MMA (contiguous)", "loads + MMA (shipped)", "pair: half loads + M256 MMA",
                             "MMA, no ring, commit per chunk", "MMA, no ring, one commit",
                             "loads + MMA, commit per slot pair"};
    for (int mode = 4; mode <= 11; ++mode) {
        const CUtensorMap &second = mode == 6 ? tmc : tmh;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        ring_kernel<<<64, THREADS, smem>>>(tm, second, mode, 10, sink);
        cudaEventRecord(a);
        ring_kernel<<<64, THREADS, smem>>>(tm, second, mode, reps, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("mode %d %-34s: %7.1f ns per step (256 KB dA + 33.5 MFLOP per CTA)  %s\n", mode, names[mode],
               ms * 1e6 / reps, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
