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

// Scatter output (gemm.h GemmParams::scat): element (m, n) of alpha * A B^T is ADDED to
// dst[row_off(m) + col_off(n)] instead of being stored to C -- the weight gradients land in the flat
// parameter vector's layout (blstm.h) directly, with no staging matrix and no scatter pass.
//   rowmode 0: m -> m (m < nrows);  1: gate-interleaved m = d 4Hq + 4u + gamma -> d dstride + gamma H + u
//              (skipped for u >= H)
//   colmode 0: n -> n ld (n < ncols);  1: padded halves n = h Hq + u -> (h H + u) ld (skipped for u >= H)
struct GemmScatter {
    float *dst = nullptr;
    int rowmode = 0, colmode = 0, H = 0, Hq = 0, nrows = 0, ncols = 0;
    long dstride = 0, ld = 0;
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
    // != nullptr (CTA-native mode only): the Z GEMM feeds a recurrence running concurrently on other
    // SMs.  Tiles are then visited M-tile by M-tile in each direction's time order (bit d of
    // flag_desc: direction d consumes time steps in descending order) and, after a tile's stores,
    // the epilogue adds 1 (release, gpu scope) to flags[d * ceil(M/128) + m_tile]; a (direction,
    // M-tile) is complete when its counter reaches natHq4 / gemm_bn(N).
    uint32_t *flags = nullptr;
    int flag_desc = 0;
    // launch as a programmatic dependent of the previous kernel in the stream (which triggers it
    // once all its CTAs are resident: lstm_rec_fwd), so the GEMM runs beside it on the free SMs
    int pdl = 0;
    // != nullptr (with pdl): the start-arbitration word shared with the recurrence (common.cuh
    // arb_checkin); every CTA checks in at entry
    uint32_t *arb = nullptr;
    // != nullptr: split-K scratch (fp32, splitk_elems floats).  GEMMs with few output tiles and a long
    // K (the weight gradients, K = T*B) split K over idle SMs; partial tiles land in the scratch and
    // a fixed-order reduction writes C (deterministic).
    float *splitk_ws = nullptr;
    long splitk_elems = 0;
    int ksplit = 1;          // set by gemm_f16
    long split_stride = 0;   // set by gemm_f16: C offset of split s (elements)
    int bn = 0;              // N tile: 0 = gemm_bn(N); 128 forces the narrow tile (more CTAs for small M)
    // > 0: split K exactly this many ways and leave the fp32 partials in splitk_ws (split s at
    // s * M * N, row-major [M][N]) for the consumer to sum -- no reduction launch (alpha applies
    // to each partial; beta / bias unsupported)
    int partials = 0;
    // != nullptr: a second, independent product in the same launch (the two directions of a
    // step-launched recurrence step): batch 1 takes its A operand from a2 (same shape and ld as A),
    // its B rows / columns at b_boff further along B's outer dimension (B's tensor map spans both),
    // and writes C at c_bstride elements further
    const void *a2 = nullptr;
    long b_boff = 0, c_bstride = 0;
    int nbatch = 1;          // set by gemm_f16
    // 1: programmatic dependent launch in a chain of dependent kernels (rec_step.cu): the prologue
    // overlaps the previous kernel's tail; every thread waits (griddepcontrol.wait) for the
    // previous grid's completion before any load of its outputs or any store, then lets the next
    // kernel of the chain launch
    int pdl_chain = 0;
    // > 0 (K-major A, single product): A is read with its K index wrapped modulo a_kwrap k-blocks
    // (a_kwrap * 64 elements), so one launch computes A.[B_0; B_1; ...] over K = nseg * a_kwrap * 64
    // with B's segments stacked along K -- BLSTM_PREC_FP16X2W's Z = X W_hi + X W_lo (R9)
    int a_kwrap = 0;
    GemmScatter scat;  // scat.dst != nullptr: scatter-add output (C, ldc, beta and bias unused; no flags / partials)
    // != nullptr: a plain GEMM (no split-K, flags, batch, scatter or PDL) whose tiles leave a partial
    // last wave splits that wave's tiles over K, tail_split ways, into fp32 partial tiles here
    // (tail_elems floats); a fixed-order reduction then writes them (deterministic).  The idle SMs
    // of the last wave share its work (e.g. C3's dX: 636 tiles = 4.3 waves on 148 SMs)
    float *tail_ws = nullptr;
    long tail_elems = 0;
    int full_items = 0, tail_split = 0;  // set by gemm_f16
};
// floats of a tail_ws that lets every shape use the tail split (one partial tile per SM)
long gemm_tail_elems();

constexpr int GEMM_BM_ROWS = 128;           // M tile
constexpr int GEMM_BK_ELEMS = 64;           // K block (a_kwrap unit)
inline int gemm_bn(int N) { return N > 128 ? 256 : 128; }  // N tile chosen by gemm_f16

// CTAs of a launch of gemm_f16 without split-K (e.g. the flagged Z GEMM): the arbitration target
int gemm_grid(int M, int N, int bn, int max_ctas);
int gemm_f16(const GemmOperand &A, const GemmOperand &B, const GemmParams &p, int max_ctas, cudaStream_t st);
// load + configure the GEMM kernels now: with lazy module loading the first launch of a kernel
// synchronizes the context, which must not happen while a recurrence waits on that GEMM (pdl)
int gemm_prepare();
int make_tmap_f16(CUtensorMap *map, const void *ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                  uint32_t box_outer);
int make_tmap_f32_rows(CUtensorMap *map, const void *ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                       uint32_t box_outer);
int num_sms();

}  // namespace blstm
