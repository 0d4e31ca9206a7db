// step_floor.cu -- microbenchmarks of the per-timestep floor of the C3 recurrence kernels
// (t_floor = max(t_mma + t_epi + t_xchg + t_bar, bytes_step / BW_hbm)), on the
// shipped launch shape: 6 clusters x 16 CTAs = 96 SMs, CTA pairs (cta_group::2), N = 32 batch
// columns per group, Hq = 512 (lstm_rec.cu).  Each mode runs one phase alone for `reps` steps;
// the kernel time / reps is the phase's per-step floor.  t_xchg + t_bar is scripts/dsmem_bench.cu
// (the same 16-CTA all-gather the kernels do).
//   mode 0 (t_mma): the pair MMA of one step: D[256 x 32] over K = 512 (32 MMAs of 256x32x16, A from
//          TMEM, B from shared memory) issued by 4 warps into 4 K-split accumulators, then one
//          commit multicast to both CTAs and the wait -- exactly the forward step's MMA phase; the
//          BPTT step's MMA (2 pair tiles of M = 256, K = 256) is the same 32 MMAs.
//   mode 1 (t_epi, forward): tcgen05.ld of the 4 accumulators, their sum, sigmoid / tanh of 4 gates,
//          the 4x4 lane transpose, the cell update, fp16 h into shared memory, CTA barrier.
//   mode 2 (t_epi, BPTT): per (unit, column): the 16-slot partial-sum gather of dh from shared memory,
//          tanh(c), the four gate gradients, dc, scaled fp16 dA into shared memory, CTA barrier.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1608_00895_b200/csrc -o step_floor step_floor.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_fp16.h>
#include "common.cuh"

using namespace blstm;

constexpr int N = 32, NH = N / 2, KF = 512, THREADS = 512;

DEVI void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
DEVI float sg(float z) { return __fdividef(1.f, 1.f + __expf(-z)); }
DEVI float th(float z) { return 2.f * sg(2.f * z) - 1.f; }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1) floor_kernel(int mode, int reps, float *sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *bs = sm;                                   // B operand: NH x K fp16, no-swizzle core matrices (16 KB)
    __half *stage = reinterpret_cast<__half *>(sm + NH * KF * 2);  // epilogue output staging (8 KB)
    __half *slots = stage + 4096;                       // BPTT: 16 partial slots [16][32 units][32 cols] fp16 (32 KB)
    float *inp = reinterpret_cast<float *>(slots + 16 * 1024);     // BPTT: per-cell inputs [8][1024] fp32 (32 KB)
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int r = (int)cluster_ctarank(), t = threadIdx.x, w = t >> 5, l = t & 31;
    for (int i = t; i < (NH * KF * 2 + 8192 + 32768 + 32768) / 16; i += THREADS)
        reinterpret_cast<uint4 *>(sm)[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u);
    if (t == 0) {
        mbar_init(&bar, 4);
        fence_mbar_init();
    }
    if (w == 0) {
        tmem_alloc2(&tslot, 512);
        tmem_relinquish2();
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tslot;
    const uint32_t ACC = 256;  // A: columns [0, 256) = K 512 fp16; accumulators: 4 x 32 columns from 256
    const uint32_t idesc = idesc_f16(256, N, 0, 0);
    float keep = 0.f;
    uint32_t ph = 0;
    float c_state[2] = {0.1f, 0.2f};
    for (int it = 0; it < reps; ++it) {
        if (mode == 0) {
            if (r == 0 && w < 4) {
                const int ks0 = w * 8;
                for (int ks = ks0; ks < ks0 + 8; ++ks)
                    mma_f16_ts2_w(tmem + ACC + 32 * w, tmem + ks * 8,
                                  sdesc_noswz(smem_u32(bs) + ks * 2 * NH * 16, NH * 16, 128), idesc, ks != ks0);
                mma_commit2_w(&bar, 0x3);
            }
            mbar_wait(&bar, ph);
            ph ^= 1;
            tc_fence_after();
        } else if (mode == 1) {
            // warp w: lane quarter q = w & 3, 8 columns cb = w >> 2; 4 K-split accumulators
            const int q = w & 3, cb = w >> 2;
            uint32_t v[4][8];
            const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + ACC + 8 * cb;
#pragma unroll
            for (int a = 0; a < 4; ++a) tmem_ld8(ta + 32 * a, v[a]);
            tmem_ld_wait();
            float pre[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
                pre[i] = ((__uint_as_float(v[0][i]) + __uint_as_float(v[1][i])) + __uint_as_float(v[2][i])) +
                         __uint_as_float(v[3][i]) + 0.01f * it;
            const int gam = l & 3;  // this lane's gate row: 4j + gam
            float act[8];  // one exp + one divide per gate (lstm_rec.cu gate_act: tanh z = 2 sigmoid(2z) - 1)
            const bool is_g = gam == 2;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float sgv = sg(is_g ? 2.f * pre[i] : pre[i]);
                act[i] = is_g ? 2.f * sgv - 1.f : sgv;
            }
            // 4x4 lane transpose (two butterfly stages) over columns i = 4c' + e
            float g4[2][4];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float a0 = act[4 * h], a1 = act[4 * h + 1], a2 = act[4 * h + 2], a3 = act[4 * h + 3];
                const bool o1 = l & 1, o2 = l & 2;
                float s0 = __shfl_xor_sync(0xffffffffu, o1 ? a0 : a1, 1), s1 = __shfl_xor_sync(0xffffffffu, o1 ? a2 : a3, 1);
                a0 = o1 ? s0 : a0; a1 = o1 ? a1 : s0; a2 = o1 ? s1 : a2; a3 = o1 ? a3 : s1;
                s0 = __shfl_xor_sync(0xffffffffu, o2 ? a0 : a2, 2); s1 = __shfl_xor_sync(0xffffffffu, o2 ? a1 : a3, 2);
                a0 = o2 ? s0 : a0; a2 = o2 ? a2 : s0; a1 = o2 ? s1 : a1; a3 = o2 ? a3 : s1;
                g4[h][0] = a0; g4[h][1] = a1; g4[h][2] = a2; g4[h][3] = a3;
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                c_state[h] = g4[h][1] * c_state[h] + g4[h][0] * g4[h][2];
                const float hv = g4[h][3] * th(c_state[h]);
                stage[(q * 32 + l) * 16 + cb * 2 + h] = __float2half_rn(hv);
            }
            __syncthreads();
        } else {
            // BPTT: 1024 cells (32 units x 32 columns) per CTA, 2 per thread
            const float scale = 1024.f;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int cell = 2 * t + h;  // unit = cell >> 5, column = cell & 31
                float dh = 0.f;
#pragma unroll
                for (int sl = 0; sl < 16; ++sl) dh += __half2float(slots[sl * 1024 + cell]);
                const float gi = inp[cell], gf = inp[1024 + cell], gg = inp[2048 + cell], go = inp[3072 + cell];
                const float c = inp[4096 + cell], cp = inp[5120 + cell], dy = inp[6144 + cell];
                const float dH = dh * (1.f / 16.f) + dy;
                const float tc = th(c);
                const float dct = c_state[h] + dH * go * (1.f - tc * tc);
                const float da_i = dct * gg * gi * (1.f - gi), da_f = dct * cp * gf * (1.f - gf);
                const float da_g = dct * gi * (1.f - gg * gg), da_o = dH * tc * go * (1.f - go);
                c_state[h] = dct * gf;
                __half2 *o = reinterpret_cast<__half2 *>(stage) + 2 * ((cell ^ (it & 7)) & 1023);
                o[0] = __floats2half2_rn(da_i * scale, da_f * scale);
                o[1] = __floats2half2_rn(da_g * scale, da_o * scale);
            }
            __syncthreads();
        }
    }
    keep += c_state[0] + c_state[1];
    if (sink && keep == 12345.f) sink[0] = keep;
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (w == 0) {
        tc_fence_after();
        tmem_dealloc2(tmem, 512);
    }
}

int main(int argc, char **argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 20000;
    const size_t smem = NH * KF * 2 + 8192 + 32768 + 32768 + 1024;
    cudaFuncSetAttribute(floor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float *sink;
    cudaMalloc(&sink, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char *names[3] = {"t_mma (pair MMA 256x32, K=512, 4 issuing warps, commit + wait)",
                            "t_epi forward (tmem ld x4, gates, transpose, cell, fp16 h -> smem, barrier)",
                            "t_epi BPTT (16-slot dh gather, tanh c, dA x4, dc, fp16 dA -> smem, barrier)"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int ctas : {2, 96}) {
            floor_kernel<<<ctas, THREADS, smem>>>(mode, 100, sink);  // warm-up
            cudaEventRecord(e0);
            floor_kernel<<<ctas, THREADS, smem>>>(mode, reps, sink);
            cudaEventRecord(e1);
            cudaError_t e = cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("mode %d  CTAs %3d : %8.1f ns/step  (%s)  %s\n", mode, ctas, ms * 1e6 / reps, names[mode],
                   cudaGetErrorString(e));
        }
    }
    return 0;
}
