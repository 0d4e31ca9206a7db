// mdlstm.h -- multi-directional 2-D LSTM layer (§4.2; SURVEY.md §8(f) NEXT-2;
// DESIGN.md §5.8, reading R21).  Internal interface of mdlstm.cu.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

namespace blstm {

struct MdGeo {
    int U, V, B, D, H, stable;
    int Hp, Dp;       // H padded to 16, D padded to 64 (GEMM operand alignment)
    long cells;       // U * V * B (physical order (u, v, b))
    long prow;        // (U + 1) * (V + 1) * B rows of the padded direction-frame grids
};

struct MdWS {  // carved from the caller's workspace / reserve
    size_t x16, x16lo, w16, w16lo, z, hf, cs, dap, rt, dcu, dcv, daf, gW, gR, gb, gsk, dxs, bar, total;  // workspace
    size_t da16;                                                                   // (workspace)
    size_t act, c, h16, rtotal;                                                    // reserve
};

MdGeo md_geo(int U, int V, int B, int D, int H, int stable);
MdWS md_ws(const MdGeo &g);
size_t md_param_count(const MdGeo &g);

// theta / grad: per direction k = 0..3: W [D, 5H], Ru [H, 5H], Rv [H, 5H], b [5H] (fp32)
int md_forward(const MdGeo &g, const float *theta, const float *x, const uint8_t *mask, float *y, uint8_t *ws,
               uint8_t *res, cudaStream_t st);
int md_backward(const MdGeo &g, const float *theta, const float *x, const uint8_t *mask, const float *dy, float *dx,
                float *grad, uint8_t *ws, uint8_t *res, cudaStream_t st);

}  // namespace blstm
