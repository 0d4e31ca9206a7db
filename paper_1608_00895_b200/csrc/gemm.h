// gemm.h -- internal interface of the tcgen05 GEMM (gemm.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

namespace blstm {

struct GemmOperand {
    const void *ptr;  // fp16, 16-byte aligned
    long ld;          // row stride in elements (multiple of 8)
    int mn_major;     // 0: element (r, k) at ptr[r*ld + k]; 1: at ptr[k*ld + r]
};

struct GemmParams {
    int M, N, K;
    float *C;           // fp32 [M, ldc]
    long ldc;
    float alpha;
    int beta;           // 1: C += result
    const float *bias;  // [N] or nullptr
    int a_mn, b_mn;     // filled by gemm_f16
    // > 0: C is written in the recurrence kernels' CTA-native layout (lstm_rec.h, rec_native_index)
    int natB = 0, natBg = 0, natG = 0, natNQ = 0, natNC = 0, natHq4 = 0, natNdir = 0;
};

int gemm_f16(const GemmOperand &A, const GemmOperand &B, const GemmParams &p, int max_ctas, cudaStream_t st);
int make_tmap_f16(CUtensorMap *map, const void *ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                  uint32_t box_outer);
int num_sms();

}  // namespace blstm
