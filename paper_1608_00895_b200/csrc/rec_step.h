// rec_step.h -- step-launched recurrence for layers beyond the persistent kernels' on-chip
// capacity (rec_supported false, e.g. BASELINE C5: H = 1024).  DESIGN.md §5.7.
//
// Same operation as lstm_rec_fwd / lstm_rec_bwd (§4.2, readings R1-R4), same
// HBM layouts for everything the rest of the step reads (h history, cell states, dA), but each
// time step is launched: per step and direction one tcgen05 GEMM (h_{t-1} R^T, or dA_t R) with R
// streamed from L2, plus one fused gate / cell-update kernel for both directions.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace blstm {

struct RecStepFwd {
    int T, B, H, Hq;
    int ndir, dir0;          // directions (1 or 2); scan direction of index 0 (index 1 is always -1)
    const float *Z;          // [T*B][ndir*4Hq] row-major, column d*4Hq + 4u + gamma, bias included
    const uint8_t *mask;     // [T*B]
    const __half *RT16;      // [2][4Hq][Hq] (R^T per direction, gate-interleaved rows)
    float *P;                // [2][SF][B][4Hq] scratch: this step's h_{t-1} R^T as split-K partials,
                             // followed by [2][B][Hq]: the fp32 h carried across masked frames
    float *C;                // cell state after frame t: C[d*c_doff + r*ldc + u]
    long ldc, c_doff;
    float *y;                // [T*B][ldy] (+ d*y_doff), u < H; nullable
    long ldy, y_doff;
    __half *y16;             // [T*B][2Hq] (+ d*Hq); nullable
    __half *gates;           // [T*B][ndir*4Hq] fp16 activations (i, f, g, o at 4u + gamma)
    __half *hist;            // [ndir][T+1][B][Hq]: h before frame t at slot t + (dir < 0); slot 0 / T = h0
    const float *h0, *c0;    // [ndir][B][H] or nullptr (0)
    float *hT, *cT;          // [ndir][B][H] state after the scan, or nullptr
};

struct RecStepBwd {
    int T, B, H, Hq;
    int ndir, dir0;
    const uint8_t *mask;
    const __half *RT16;      // [2][4Hq][Hq]
    const float *C;          // as written by the forward (ldc = Hq, c_doff = T*B*Hq)
    long ldc, c_doff;
    const __half *gates;     // [T*B][8Hq]
    const float *dy;         // [T*B][lddy] (+ d*dy_doff), u < H
    long lddy, dy_doff;
    __half *dA;              // [T*B][ndir*4Hq], scaled by 2^DA_SHIFT
    const float *c0;         // [ndir][B][H] or nullptr
    const float *dhT, *dcT;  // [ndir][B][H] gradients at the end of the scan, or nullptr
    float *dh0, *dc0;        // [ndir][B][H] gradients w.r.t. h0 / c0 (overwritten), or nullptr
    float *dhR;              // [2][SB][B][Hq] scratch: dA_t R of the previous step (split-K partials)
                             // (layout of the scratch: rec_step_bwd_partial_floats)
    float *dhc, *dcc;        // [2][B][Hq] carried dh (masked frames) and dc
    float *splitk_ws;        // split-K scratch of the per-step GEMM
    long splitk_elems;
    // the persistent BPTT (rec_step.cu step_bwd_persist_kernel) also needs: R in the K-major layout
    // of pack_w ([Hq][2 * 4Hq]: R16[k][d 4Hq + 4u + gamma] = R_d[k][gamma H + u]; nullptr: chain only),
    // the db partials output ([ndir][rec_step_bwd_db_groups()][4Hq]; nullptr: not written) and an
    // optional "CTAs placed" counter (side-stream guard)
    const __half *R16;
    float *dbpart;
    uint32_t *started;
    int exp;  // trace builds only (BLSTM_PB_EXP): 1 = MMAs without the dA loads, 2 = loads without MMAs
};

size_t rec_step_fwd_scratch_bytes(int B, int Hq);
size_t rec_step_bwd_scratch_bytes(int B, int Hq);
// floats of the dA R partials at the start of the BPTT scratch ([2][SB][B][Hq]); dhc and dcc
// ([2][B][Hq] each) follow
size_t rec_step_bwd_partial_floats(int B, int Hq);
int rec_step_fwd(const RecStepFwd &p, cudaStream_t st);
// 0: the step chain ran (db: column sums of dA are the caller's); 1: the persistent BPTT ran and wrote
// p.dbpart (rec_step_bwd_db_groups() partial groups per direction); < 0: error
int rec_step_bwd(const RecStepBwd &p, cudaStream_t st);
int rec_step_bwd_db_groups();
// CTAs of the persistent BPTT for this shape, 0 when it does not apply (then the chain runs)
int rec_step_bwd_persist_ctas(int B, int Hq, int ndir);

}  // namespace blstm
