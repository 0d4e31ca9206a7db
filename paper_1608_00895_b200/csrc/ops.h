// ops.h -- internal interface of the helper kernels (ops.cu).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

namespace blstm {

// Input dropout (R20): element (row r, logical feature j) of site s is kept iff the
// counter-based draw h(seed, s, r * width + j) >= thr; kept elements are scaled by `scale`.
struct Dropout {
    int on;
    uint32_t thr, seed;
    float scale;
};
int cast_x_f16(const float *x, long ldx, int D, __half *x16, int Dp, long rows, cudaStream_t st,
               const Dropout &dr = Dropout{0, 0, 0, 1.f});
// in place on a [rows, 2Hq] layer output (fp16) or input gradient (fp32): logical feature
// d*H + u of column d*Hq + u (u < H), site `site`, width 2H
int dropout_f16(__half *y, long rows, int H, int Hq, int site, const Dropout &dr, cudaStream_t st);
int dropout_f32(float *y, long rows, int H, int Hq, int site, const Dropout &dr, cudaStream_t st);
// rowmode 0: input rows are W rows (rows >= Drows are padding); 1: input rows are the padded
// [fwd (Hq) | bwd (Hq)] halves of the layer below (row half*Hq + jj <-> W row half*H + jj).
// lo_rows > 0 (BLSTM_PREC_FP16X2W): also write lo = fp16(W - hi) at row r + lo_rows (W16 then has
// 2 * lo_rows rows: [W_hi; W_lo] stacked along K)
int pack_w(const float *W0, const float *W1, int Drows, int H, int Hq, int ndir, int Dn, int rowmode, __half *W16,
           cudaStream_t st, int lo_rows = 0);
int pack_rt(const float *R0, const float *R1, int H, int Hq, int ndir, __half *RT16, cudaStream_t st);
int pack_bias(const float *b0, const float *b1, int H, int Hq, int ndir, float *bq, cudaStream_t st);
// every layer of a bidirectional stack at once (pack_w, pack_rt, pack_bias of each layer, both
// directions): three launches
constexpr int PACK_MAXL = 16;
struct HistLayers {
    __half *hist[PACK_MAXL];
};

struct PackLayers {
    int L, H, Hq;
    const float *W[PACK_MAXL][2], *R[PACK_MAXL][2], *b[PACK_MAXL][2];
    int Drows[PACK_MAXL], Dn[PACK_MAXL], rowmode[PACK_MAXL];
    int lo_rows[PACK_MAXL];  // > 0: W_lo rows at that offset (pack_w)
    __half *W16[PACK_MAXL], *RT16[PACK_MAXL];
    float *bq[PACK_MAXL];
};
int pack_layers(const PackLayers &a, cudaStream_t st);
// The stack step's preamble in ONE launch (it was bound by the host's launch rate: ~7 small
// launches / memsets of a few us each): x -> x16 (cast_x_f16), the operand packs of layers
// [0, pk.L) (pack_layers), the mask (mask_mode 1: pack_mask, 2: check_mask), zero words (the Z
// flags), every layer's zero h0 history slots (init_hist) and the head's operands (pack_wout).
// Jobs are independent and
// take disjoint block ranges.
struct StackPrep {
    const float *x; long ldx; int D; __half *x16; int Dp; long rows; Dropout dr;
    PackLayers pk;  // pk.L = 0: no packs
    int mask_mode; const uint8_t *mask; int T, B, G, Bg, N; uint8_t *maskN; long mask_n;
    uint32_t *zero; long zero_n;
    HistLayers hl; int hist_L, hT, hB, hHq;
    const float *Wo, *bo; int K, Kp; __half *Wo16; float *boq;  // the head's operands (pack_wout); Wo16 = nullptr: none
    int maxDn;
    unsigned *err;
    int nb[8];  // blocks per job: cast, pack_w, pack_rt, pack_bias, mask, zero, hist, head (set by stack_prep)
};
int stack_prep(StackPrep &p, cudaStream_t st);
int pack_wout(const float *Wo, const float *bo, int H, int Hq, int K, int Kp, __half *Wo16, float *boq,
              cudaStream_t st);
int init_hist(__half *hist, const float *h0, int T, int B, int H, int Hq, int ndir, int dir0, cudaStream_t st);
int ce_head(const float *logits, long ldl, int K, int Kp, const uint8_t *mask, const int32_t *labels, float scale,
            __half *dlog16, double *rowloss, int32_t *rowerr, long rows, cudaStream_t st);
int reduce_loss(const double *rowloss, const int32_t *rowerr, long rows, double *loss, int32_t *ferr,
                cudaStream_t st);
size_t colsum_scratch_bytes(long rows, int cols);
int colsum_f16_add(const __half *src, long rows, int cols, long ld, float alpha, float *out, float *scratch,
                   cudaStream_t st);
int scatter_w(float *gW, int Drows, int H, int Hq, const float *dWT, long ldw, int d, int rowmode, cudaStream_t st);
int scatter_r(float *gR, int H, int Hq, const float *dRT, cudaStream_t st);
int scatter_b(float *gb, int H, int Hq, const float *dbpart, int G, int d, cudaStream_t st);
int scatter_wout(float *gWo, int H, int Hq, int K, const float *dWoT, long ldw, cudaStream_t st);
// recurrence kernels' mask rows: maskN[(t*G + g)*N + n] = mask[t*B + g*Bg + n] for n < Bg,
// g*Bg + n < B, else 0 (one N-byte row per step and batch group, bulk-copyable)
int pack_mask(const uint8_t *mask, int T, int B, int G, int Bg, int N, uint8_t *maskN, cudaStream_t st);
// mask entries outside {0,1}: pack_mask and check_mask set a process-wide flag (mapped host memory);
// mask_flag_take() returns 1 (and clears it) if a kernel that has completed saw one
int check_mask(const uint8_t *mask, long n, cudaStream_t st);
int mask_flag_take();
// dst[r*ldd + j] = src[r*lds + j] for j < cols (a row-strided copy into an aligned buffer)
int copy_rows(const float *src, long lds, long rows, int cols, float *dst, long ldd, cudaStream_t st);
int pad_halves(const float *src, int H, int Hq, long rows, float *dst, cudaStream_t st);
int store_dx(float *dx, long ldx, const float *dX, long ldX, int D, long rows, int accum, cudaStream_t st);
// one-thread kernel: returns once *flag >= target (acquire) or after 2 ms (placement guard of
// side-stream work behind a recurrence launch)
int wait_count(const uint32_t *flag, uint32_t target, cudaStream_t st);
int gather_chunks(const float *frames, const int32_t *flab, int D, const int64_t *cstart, const int32_t *clen, int B,
                  int T, float *x, uint8_t *mask, int32_t *labels, cudaStream_t st);
int sgd(float *theta, float *grad, long n, float lr, int zero, cudaStream_t st);

}  // namespace blstm
