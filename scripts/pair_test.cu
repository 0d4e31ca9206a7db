// pair_test.cu -- checks the tcgen05 cta_group::2 semantics the recurrence kernels rely on, on a
// 2-CTA cluster:
//   * tcgen05.alloc / relinquish / dealloc .cta_group::2 executed by one warp in EACH CTA;
//   * tcgen05.mma.cta_group::2.kind::f16, A from TMEM (TS), issued by rank 0 only:
//     D (M=256) = A (rank r holds rows 128r..128r+127 in its TMEM) x B^T, where rank r holds
//     B columns [r*N/2, (r+1)*N/2) in its smem at the SAME offset;
//   * tcgen05.commit.cta_group::2 ... multicast::cluster to both CTAs' mbarriers;
//   * each CTA then reads D rows of its half, all N columns, from its own TMEM.
// Also times a chain of dependent pair MMAs vs single-CTA MMAs.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1608_00895_b200/csrc -o pair_test pair_test.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_fp16.h>
#include "common.cuh"

using namespace blstm;

constexpr int K = 64, N = 32, NH = N / 2;

DEVI void alloc2(uint32_t *dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols)
                 : "memory");
}
DEVI void relinquish2() { asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory"); }
DEVI void dealloc2(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
DEVI void mma2_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
        "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
DEVI void commit2(uint64_t *bar, uint16_t mask) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     smem_u32(bar)),
                 "h"(mask)
                 : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    pair_kernel(const __half *A, const __half *B, float *D, int reps, long long *cycles) {
    __shared__ __align__(1024) uint8_t bs[K * NH * 2];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int r = (int)cluster_ctarank(), t = threadIdx.x, w = t >> 5, l = t & 31;
    if (t == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (w == 0) {
        alloc2(&tslot, 128);
        relinquish2();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    // A rows of this CTA -> TMEM columns [0, K/2) (two fp16 per 32-bit column), lane = row
    {
        const int row = 128 * r + t;
        uint32_t v[16];
        for (int c0 = 0; c0 < K / 2; c0 += 16) {
            for (int u = 0; u < 16; ++u) {
                __half2 h2 = __halves2half2(A[row * K + 2 * (c0 + u)], A[row * K + 2 * (c0 + u) + 1]);
                v[u] = *reinterpret_cast<uint32_t *>(&h2);
            }
            tmem_st16(tmem + ((uint32_t)(32 * w) << 16) + c0, v);
        }
        tmem_st_wait();
    }
    // this CTA's B columns (n' = n - r*NH) in no-swizzle K-major core matrices: (n', k) at
    // ((k/8)*NH + n')*16 + (k%8)*2
    for (int e = t; e < NH * K; e += 128) {
        const int nl = e / K, k = e % K;
        *reinterpret_cast<__half *>(bs + ((k / 8) * NH + nl) * 16 + (k % 8) * 2) = B[(r * NH + nl) * K + k];
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // both halves of A and B in place
    tc_fence_after();
    const uint32_t idesc = idesc_f16(256, N, 0, 0);
    long long c0 = clock64();
    uint32_t ph = 0;
    for (int it = 0; it < reps; ++it) {
        if (r == 0 && t == 0) {
            for (int ks = 0; ks < K / 16; ++ks)
                mma2_ts(tmem + 64, tmem + ks * 8, sdesc_noswz(smem_u32(bs) + ks * 2 * NH * 16, NH * 16, 128), idesc, ks != 0);
            commit2(&bar, 0x3);
        }
        mbar_wait(&bar, ph);
        ph ^= 1;
        tc_fence_after();
    }
    long long c1 = clock64();
    if (t == 0 && cycles) cycles[r] = (c1 - c0) / (reps > 0 ? reps : 1);
    // D rows of this CTA, all N columns
    {
        float v[16];
        for (int c = 0; c < N; c += 16) {
            tmem_ld16(tmem + ((uint32_t)(32 * w) << 16) + 64 + c, v);
            tmem_ld_wait();
            for (int j = 0; j < 16; ++j) D[(128 * r + t) * N + c + j] = v[j];
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (w == 0) {
        tc_fence_after();
        dealloc2(tmem, 128);
    }
}

int main() {
    std::vector<__half> hA(256 * K), hB(N * K);
    std::vector<float> fA(256 * K), fB(N * K);
    srand(1);
    for (int i = 0; i < 256 * K; ++i) { fA[i] = (rand() % 17 - 8) / 8.f; hA[i] = __float2half(fA[i]); }
    for (int i = 0; i < N * K; ++i) { fB[i] = (rand() % 13 - 6) / 4.f; hB[i] = __float2half(fB[i]); }
    __half *dA, *dB;
    float *dD;
    long long *dc;
    cudaMalloc(&dA, 256 * K * 2);
    cudaMalloc(&dB, N * K * 2);
    cudaMalloc(&dD, 256 * N * 4);
    cudaMalloc(&dc, 16);
    cudaMemcpy(dA, hA.data(), 256 * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB.data(), N * K * 2, cudaMemcpyHostToDevice);
    for (int reps : {1, 1000}) {
        cudaMemset(dD, 0, 256 * N * 4);
        pair_kernel<<<2, 128>>>(dA, dB, dD, reps, dc);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> hD(256 * N);
        cudaMemcpy(hD.data(), dD, 256 * N * 4, cudaMemcpyDeviceToHost);
        long long cyc[2];
        cudaMemcpy(cyc, dc, 16, cudaMemcpyDeviceToHost);
        double maxerr = 0;
        int bad = 0, first_bad = -1;
        for (int m = 0; m < 256; ++m)
            for (int n = 0; n < N; ++n) {
                double ref = 0;
                for (int k = 0; k < K; ++k) ref += (double)fA[m * K + k] * fB[n * K + k];
                const double err = fabs(ref - hD[m * N + n]);
                if (err > maxerr) maxerr = err;
                if (err > 1e-3 && bad++ == 0) first_bad = m * N + n;
            }
        printf("reps %4d: %s; max |err| %.3g, %d bad of %d (first bad m=%d n=%d); %lld cycles per pair step "
               "(%d MMAs of 256x%dx16)\n",
               reps, cudaGetErrorString(e), maxerr, bad, 256 * N, first_bad < 0 ? -1 : first_bad / N,
               first_bad < 0 ? -1 : first_bad % N, cyc[0], K / 16, N);
    }
    return 0;
}
