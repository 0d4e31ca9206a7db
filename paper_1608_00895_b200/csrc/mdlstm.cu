// mdlstm.cu -- multi-directional 2-D LSTM layer (§4.2: "the activations for all
// positions on a common diagonal can be computed at the same time ... we process multiple images
// and also the four directions ... simultaneously", R21).
//
// Direction k = 0..3 runs on the grid flipped by (fu, fv) = (k & 1, k >> 1) (identity, flip-u,
// flip-v, both); its state lives in its own frame (u', v').  Per call:
//   Z = X W_all + b_all                 one tcgen05 GEMM for every cell and all four directions
//   for d = 0 .. U+V-2:                 one fused launch per anti-diagonal, all directions, images
//     a = Z + h(u'-1,v') Ru + h(u',v'-1) Rv;  gates, cell (two-forget or stable), mask
// Backward: the reverse wavefront (dh from the successors' dA through R^T, dc from the successors),
// then dX = dA W_all^T, dW^T = dA^T X, dRu^T / dRv^T = dA^T H_pred (tcgen05 GEMMs; the predecessor
// pairing is a fixed row shift of a zero-bordered [(U+1) x (V+1) x B] grid), db = column sums.
#include "common.cuh"
#include "gemm.h"
#include "graph.h"
#include "lstm_rec.h"
#include "mdlstm.h"
#include "ops.h"
#include "prof.h"

namespace blstm {

namespace {

DEVI float msg(float z) { return __fdividef(1.f, 1.f + __expf(-z)); }
DEVI float mth(float z) { return 2.f * msg(2.f * z) - 1.f; }

inline size_t al(size_t b) { return (b + 255) & ~(size_t)255; }
int rup(int a, int b) { return (a + b - 1) / b * b; }
int grid1(long n) {
    long g = (n + 255) / 256;
    return (int)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

struct MdK {  // kernel arguments
    int U, V, B, D, H, Hp, stable;
    long P1;                 // parameters per direction
    const float *theta;
    const float *z;          // [cells][20Hp]
    const uint8_t *mask;     // [cells]
    float *y;                // [cells][4H]
    float *hf;               // [4][U][V][B][H] fp32 h (forward state)
    float *act, *c;          // [4][U][V][B][5H], [4][U][V][B][H]
    __half *h16;             // [4][prow][Hp]
    // backward
    const float *dy;         // [cells][4H]
    const float *rt;         // [4][2][5H][H]  Ru^T, Rv^T
    float *daf;              // [4][U][V][B][5H]
    float *dcu, *dcv;        // [4][U][V][B][H]: dc this cell passes to its u- / v-predecessor
    __half *da16;            // [4][prow][5Hp]
    __half *dap;             // [cells][20Hp]
    unsigned long long *trace;  // debug (BLSTM_TRACE builds): per-diagonal phase clocks of CTA 0
};
#ifdef BLSTM_TRACE
#define WTRACE(s, k) \
    if (trace) trace[(size_t)(s) * 16 + (k)] = (unsigned long long)clock64()
#else
#define WTRACE(s, k)
#endif

// Tile decomposition of one anti-diagonal: block = (direction k, 32-unit tile, group of 32 rows),
// row = (cell on the diagonal, image); warp w of the block owns rows w, w+8, w+16, w+24 of its group
// (warp-uniform), lane = unit.  The recurrent weights of the unit tile are staged in shared memory
// 32 rows of K at a time; the predecessor states are warp-broadcast loads.
constexpr int MT_J = 32, MT_RL = 8, MT_RPT = 2, MT_ROWS = MT_RL * MT_RPT, MT_MC = 32;
constexpr int MT_MCF = 16;  // K chunk of the forward (5 gates x 2 predecessors of R per chunk row)

struct MdRow {
    long cp, ck;
    int up, vp;
    bool live, on;  // row exists on this diagonal; its pixel is in the image
};
DEVI MdRow md_row(const MdK &a, int d, int k, int r) {
    MdRow w;
    const int u0 = d - a.V + 1 > 0 ? d - a.V + 1 : 0;
    const int u1 = d < a.U - 1 ? d : a.U - 1;
    w.live = r < (u1 - u0 + 1) * a.B;
    if (!w.live) r = 0;
    const int i = r / a.B, b = r - i * a.B;
    w.up = u0 + i; w.vp = d - w.up;
    const int u = (k & 1) ? a.U - 1 - w.up : w.up, v = (k & 2) ? a.V - 1 - w.vp : w.vp;
    w.cp = ((long)u * a.V + v) * a.B + b;
    w.ck = (((long)k * a.U + w.up) * a.V + w.vp) * a.B + b;
    w.on = w.live && a.mask[w.cp] != 0;
    return w;
}
__host__ DEVI int md_blocks(int U, int V, int B, int H, int d) {
    const int u0 = d - V + 1 > 0 ? d - V + 1 : 0;
    const int u1 = d < U - 1 ? d : U - 1;
    const int nrows = (u1 - u0 + 1) * B;
    return 4 * ((H + MT_J - 1) / MT_J) * ((nrows + MT_ROWS - 1) / MT_ROWS);
}
DEVI long slot(const MdK &a, int up, int vp, int b) { return ((long)(up + 1) * (a.V + 1) + vp + 1) * a.B + b; }

__global__ void __launch_bounds__(256) md_fwd_diag_kernel(MdK a, int d) {
    __shared__ float Rs[2][MT_MCF][5][MT_J];
    __shared__ float Hs[2][MT_ROWS][MT_MCF + 1];   // predecessor h chunk of the block's rows (u, v)
    __shared__ long rowpred[2][MT_ROWS];           // h index of each row's predecessors (-1: none)
    const int H = a.H, G = 5 * H, Hp = a.Hp;
    const long VB = (long)a.V * a.B;
    const int u0 = d - a.V + 1 > 0 ? d - a.V + 1 : 0;
    const int u1 = d < a.U - 1 ? d : a.U - 1;
    const int nrg = ((u1 - u0 + 1) * a.B + MT_ROWS - 1) / MT_ROWS, njt = (H + MT_J - 1) / MT_J;
    int bid = blockIdx.x;
    const int rg = bid % nrg; bid /= nrg;
    const int jt = bid % njt, k = bid / njt;
    const int jj = threadIdx.x & 31, rl = threadIdx.x >> 5, j = jt * MT_J + jj;
    const bool jok = j < H;
    const float *Ru = a.theta + k * a.P1 + (long)a.D * G, *Rv = Ru + (long)H * G;
    MdRow rw[MT_RPT];
    float acc[MT_RPT][5];
#pragma unroll
    for (int t = 0; t < MT_RPT; ++t) {
        rw[t] = md_row(a, d, k, rg * MT_ROWS + rl + MT_RL * t);
        const float *zc = a.z + rw[t].cp * 20 * Hp + (long)k * 5 * Hp;
#pragma unroll
        for (int q = 0; q < 5; ++q) acc[t][q] = (rw[t].on && jok) ? zc[q * Hp + j] : 0.f;
        if (jj == 0) {  // row rl + 8t of the block
            rowpred[0][rl + MT_RL * t] = (rw[t].on && rw[t].up > 0) ? (rw[t].ck - VB) * H : -1;
            rowpred[1][rl + MT_RL * t] = (rw[t].on && rw[t].vp > 0) ? (rw[t].ck - a.B) * H : -1;
        }
    }
    for (int m0 = 0; m0 < H; m0 += MT_MCF) {
        __syncthreads();
        // all copies of the chunk in flight at once (cp.async, zero-filled out of range): a load ->
        // store loop serializes ~20 L2 round trips per thread (measured: half the stall samples)
        for (int e = threadIdx.x; e < 2 * MT_MCF * 5 * MT_J; e += blockDim.x) {
            const int jx = e % MT_J, q = (e / MT_J) % 5, mm = (e / (5 * MT_J)) % MT_MCF, w = e / (MT_MCF * 5 * MT_J);
            const int m = m0 + mm, jg = jt * MT_J + jx;
            const bool ok = m < H && jg < H;
            cp_async4_zfill(smem_u32(&Rs[w][mm][q][jx]), ok ? (w ? Rv : Ru) + (long)m * G + q * H + jg : Ru, ok ? 4 : 0);
        }
        for (int e = threadIdx.x; e < 2 * MT_ROWS * MT_MCF; e += blockDim.x) {  // coalesced per row
            const int mm = e % MT_MCF, rr = (e / MT_MCF) % MT_ROWS, w = e / (MT_ROWS * MT_MCF);
            const long src = rowpred[w][rr];
            const bool ok = src >= 0 && m0 + mm < H;
            cp_async4_zfill(smem_u32(&Hs[w][rr][mm]), ok ? a.hf + src + m0 + mm : a.hf, ok ? 4 : 0);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        const int mlen = H - m0 < MT_MCF ? H - m0 : MT_MCF;
#pragma unroll
        for (int t = 0; t < MT_RPT; ++t) {
            if (!rw[t].on) continue;  // warp-uniform
            const int rr = rl + MT_RL * t;
            for (int mm = 0; mm < mlen; ++mm) {
                const float hu = Hs[0][rr][mm], hv = Hs[1][rr][mm];
#pragma unroll
                for (int q = 0; q < 5; ++q)
                    acc[t][q] = fmaf(hv, Rs[1][mm][q][jj], fmaf(hu, Rs[0][mm][q][jj], acc[t][q]));
            }
        }
    }
    const long prow = (long)(a.U + 1) * (a.V + 1) * a.B;
#pragma unroll
    for (int t = 0; t < MT_RPT; ++t) {
        const MdRow &w = rw[t];
        if (!w.live || !jok) continue;
        const long ck = w.ck;
        const int b = (int)(w.cp % a.B);
        const float cu = w.up > 0 ? a.c[(ck - VB) * H + j] : 0.f;
        const float cv = w.vp > 0 ? a.c[(ck - a.B) * H + j] : 0.f;
        float *ac = a.act + ck * G;
        float h = 0.f, cn;
        if (!w.on) {
            cn = w.up > 0 ? cu : cv;  // carried (0 when neither predecessor exists)
#pragma unroll
            for (int q = 0; q < 5; ++q) ac[q * H + j] = 0.f;
        } else if (!a.stable) {  // [i, fu, fv, g, o]
            const float gi = msg(acc[t][0]), fu = msg(acc[t][1]), fv = msg(acc[t][2]), gg = mth(acc[t][3]),
                        go = msg(acc[t][4]);
            cn = fu * cu + fv * cv + gi * gg;
            h = go * mth(cn);
            ac[j] = gi; ac[H + j] = fu; ac[2 * H + j] = fv; ac[3 * H + j] = gg; ac[4 * H + j] = go;
        } else {                 // [i, f, g, o, lambda]
            const float gi = msg(acc[t][0]), f = msg(acc[t][1]), gg = mth(acc[t][2]), go = msg(acc[t][3]),
                        lam = msg(acc[t][4]);
            cn = f * (lam * cu + (1.f - lam) * cv) + gi * gg;
            h = go * mth(cn);
            ac[j] = gi; ac[H + j] = f; ac[2 * H + j] = gg; ac[3 * H + j] = go; ac[4 * H + j] = lam;
        }
        a.c[ck * H + j] = cn;
        a.hf[ck * H + j] = h;
        a.h16[((long)k * prow + slot(a, w.up, w.vp, b)) * Hp + j] = __float2half_rn(h);
        a.y[w.cp * 4 * H + (long)k * H + j] = h;
    }
}

__global__ void __launch_bounds__(256) md_bwd_diag_kernel(MdK a, int d) {
    __shared__ float Rs[2][MT_MC][MT_J];
    __shared__ float Ds[2][MT_ROWS][MT_MC + 1];  // successor dA chunk of the block's rows (u, v)
    __shared__ long rowsucc[2][MT_ROWS];          // dA index of each row's successors (-1: none)
    const int H = a.H, G = 5 * H, Hp = a.Hp;
    const long VB = (long)a.V * a.B;
    const long prow = (long)(a.U + 1) * (a.V + 1) * a.B;
    const float scale = (float)(1 << DA_SHIFT);
    const int u0 = d - a.V + 1 > 0 ? d - a.V + 1 : 0;
    const int u1 = d < a.U - 1 ? d : a.U - 1;
    const int nrg = ((u1 - u0 + 1) * a.B + MT_ROWS - 1) / MT_ROWS, njt = (H + MT_J - 1) / MT_J;
    int bid = blockIdx.x;
    const int rg = bid % nrg; bid /= nrg;
    const int jt = bid % njt, k = bid / njt;
    const int jj = threadIdx.x & 31, rl = threadIdx.x >> 5, j = jt * MT_J + jj;
    const bool jok = j < H;
    const float *RuT = a.rt + (long)k * 2 * G * H, *RvT = RuT + (long)G * H;
    MdRow rw[MT_RPT];
    float dh[MT_RPT];
#pragma unroll
    for (int t = 0; t < MT_RPT; ++t) {
        rw[t] = md_row(a, d, k, rg * MT_ROWS + rl + MT_RL * t);
        dh[t] = (rw[t].on && jok) ? a.dy[rw[t].cp * 4 * H + (long)k * H + j] : 0.f;
        if (jj == 0) {
            rowsucc[0][rl + MT_RL * t] = (rw[t].on && rw[t].up + 1 < a.U) ? (rw[t].ck + VB) * G : -1;
            rowsucc[1][rl + MT_RL * t] = (rw[t].on && rw[t].vp + 1 < a.V) ? (rw[t].ck + a.B) * G : -1;
        }
    }
    // dh += dA(u'+1, v') Ru^T + dA(u', v'+1) Rv^T
    for (int n0 = 0; n0 < G; n0 += MT_MC) {
        __syncthreads();
        for (int e = threadIdx.x; e < 2 * MT_MC * MT_J; e += blockDim.x) {
            const int jx = e % MT_J, nn = (e / MT_J) % MT_MC, w = e / (MT_MC * MT_J);
            const int n = n0 + nn, jg = jt * MT_J + jx;
            const bool ok = n < G && jg < H;
            cp_async4_zfill(smem_u32(&Rs[w][nn][jx]), ok ? (w ? RvT : RuT) + (long)n * H + jg : RuT, ok ? 4 : 0);
        }
        for (int e = threadIdx.x; e < 2 * MT_ROWS * MT_MC; e += blockDim.x) {
            const int nn = e % MT_MC, rr = (e / MT_MC) % MT_ROWS, w = e / (MT_ROWS * MT_MC);
            const long src = rowsucc[w][rr];
            const bool ok = src >= 0 && n0 + nn < G;
            cp_async4_zfill(smem_u32(&Ds[w][rr][nn]), ok ? a.daf + src + n0 + nn : a.daf, ok ? 4 : 0);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        const int nlen = G - n0 < MT_MC ? G - n0 : MT_MC;
#pragma unroll
        for (int t = 0; t < MT_RPT; ++t) {
            if (!rw[t].on) continue;  // warp-uniform
            const int rr = rl + MT_RL * t;
            for (int nn = 0; nn < nlen; ++nn)
                dh[t] = fmaf(Ds[1][rr][nn], Rs[1][nn][jj], fmaf(Ds[0][rr][nn], Rs[0][nn][jj], dh[t]));
        }
    }
#pragma unroll
    for (int t = 0; t < MT_RPT; ++t) {
        const MdRow &w = rw[t];
        if (!w.live || !jok) continue;
        const long ck = w.ck, cp = w.cp;
        const int b = (int)(cp % a.B);
        const bool su = w.up + 1 < a.U, sv = w.vp + 1 < a.V;
        const float dc = (su ? a.dcu[(ck + VB) * H + j] : 0.f) + (sv ? a.dcv[(ck + a.B) * H + j] : 0.f);
        float *df = a.daf + ck * G;
        __half *d16 = a.da16 + ((long)k * prow + slot(a, w.up, w.vp, b)) * 5 * Hp;
        __half *dp = a.dap + cp * 20 * Hp + (long)k * 5 * Hp;
        if (!w.on) {
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                df[q * H + j] = 0.f;
                d16[q * Hp + j] = __float2half_rn(0.f);
                dp[q * Hp + j] = __float2half_rn(0.f);
            }
            a.dcu[ck * H + j] = w.up > 0 ? dc : 0.f;                 // the carried c came from the
            a.dcv[ck * H + j] = (w.up == 0 && w.vp > 0) ? dc : 0.f;  // u-, else the v-predecessor
            continue;
        }
        const float *ac = a.act + ck * G;
        const float c = a.c[ck * H + j];
        const float cu = w.up > 0 ? a.c[(ck - VB) * H + j] : 0.f;
        const float cv = w.vp > 0 ? a.c[(ck - a.B) * H + j] : 0.f;
        const float tc = mth(c);
        float da[5];
        if (!a.stable) {
            const float gi = ac[j], fu = ac[H + j], fv = ac[2 * H + j], gg = ac[3 * H + j], go = ac[4 * H + j];
            const float dct = dc + dh[t] * go * (1.f - tc * tc);
            da[0] = dct * gg * gi * (1.f - gi);
            da[1] = dct * cu * fu * (1.f - fu);
            da[2] = dct * cv * fv * (1.f - fv);
            da[3] = dct * gi * (1.f - gg * gg);
            da[4] = dh[t] * tc * go * (1.f - go);
            a.dcu[ck * H + j] = dct * fu;
            a.dcv[ck * H + j] = dct * fv;
        } else {
            const float gi = ac[j], f = ac[H + j], gg = ac[2 * H + j], go = ac[3 * H + j], lam = ac[4 * H + j];
            const float dct = dc + dh[t] * go * (1.f - tc * tc);
            const float m = lam * cu + (1.f - lam) * cv;
            da[0] = dct * gg * gi * (1.f - gi);
            da[1] = dct * m * f * (1.f - f);
            da[2] = dct * gi * (1.f - gg * gg);
            da[3] = dh[t] * tc * go * (1.f - go);
            da[4] = dct * f * (cu - cv) * lam * (1.f - lam);
            a.dcu[ck * H + j] = dct * f * lam;
            a.dcv[ck * H + j] = dct * f * (1.f - lam);
        }
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            df[q * H + j] = da[q];
            const __half sv16 = __float2half_rn(da[q] * scale);
            d16[q * Hp + j] = sv16;
            dp[q * Hp + j] = sv16;
        }
    }
}

// ---------------------------------------------------------------------------------------------
// Persistent forward wavefront (one launch per pass): block (direction k, unit tile jt, lane g) keeps its
// tile of the recurrent weights in shared memory for the whole pass and processes row groups
// g, g + NG, ... of every anti-diagonal; a grid barrier (monotonic counter, release / acquire)
// separates the diagonals.  State written by other blocks is read with L1-bypassing loads.  Launched
// cooperatively (all blocks co-resident, else the launch fails and the per-diagonal kernels run).
// ---------------------------------------------------------------------------------------------
DEVI void grid_barrier(uint32_t *count, uint32_t target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        red_release_gpu_add(count, 1u);
        while (ld_acquire_gpu(count) < target) __nanosleep(64);
    }
    __syncthreads();
}
DEVI int md_nrows(const MdK &a, int d) {
    const int u0 = d - a.V + 1 > 0 ? d - a.V + 1 : 0;
    const int u1 = d < a.U - 1 ? d : a.U - 1;
    return (u1 - u0 + 1) * a.B;
}

__global__ void __launch_bounds__(256) md_fwd_persist_kernel(MdK a, uint32_t *bar, int NG) {
    extern __shared__ float dsm[];
    __shared__ long rowpred[2][MT_ROWS];
    const int H = a.H, G = 5 * H, Hp = a.Hp, njt = (H + MT_J - 1) / MT_J, HS = H + 1;
    const long VB = (long)a.V * a.B;
    const long prow = (long)(a.U + 1) * (a.V + 1) * a.B;
    float *Rs = dsm;                   // [2][H][5][32]: Ru, Rv columns of the unit tile
    float *Hs = Rs + 2 * H * 5 * MT_J; // [2][MT_ROWS][H+1]: predecessor h of the block's rows
    int bid = blockIdx.x;
    const int g = bid % NG; bid /= NG;
    const int jt = bid % njt, k = bid / njt;
    const int jj = threadIdx.x & 31, rl = threadIdx.x >> 5, j = jt * MT_J + jj;
    const bool jok = j < H;
    const float *Ru = a.theta + k * a.P1 + (long)a.D * G, *Rv = Ru + (long)H * G;
    for (int e = threadIdx.x; e < 2 * H * 5 * MT_J; e += blockDim.x) {
        const int jx = e % MT_J, q = (e / MT_J) % 5, m = (e / (5 * MT_J)) % H, w = e / (H * 5 * MT_J);
        const int jg = jt * MT_J + jx;
        Rs[e] = jg < H ? (w ? Rv : Ru)[(long)m * G + q * H + jg] : 0.f;
    }
    const int ND = a.U + a.V - 1;
    for (int d = 0; d < ND; ++d) {
        const int nrg = (md_nrows(a, d) + MT_ROWS - 1) / MT_ROWS;
        for (int rg = g; rg < nrg; rg += NG) {
            MdRow rw[MT_RPT];
            float acc[MT_RPT][5];
#pragma unroll
            for (int t = 0; t < MT_RPT; ++t) {
                rw[t] = md_row(a, d, k, rg * MT_ROWS + rl + MT_RL * t);
                const float *zc = a.z + rw[t].cp * 20 * Hp + (long)k * 5 * Hp;
#pragma unroll
                for (int q = 0; q < 5; ++q) acc[t][q] = (rw[t].on && jok) ? zc[q * Hp + j] : 0.f;
                if (jj == 0) {
                    rowpred[0][rl + MT_RL * t] = (rw[t].on && rw[t].up > 0) ? (rw[t].ck - VB) * H : -1;
                    rowpred[1][rl + MT_RL * t] = (rw[t].on && rw[t].vp > 0) ? (rw[t].ck - a.B) * H : -1;
                }
            }
            __syncthreads();
            for (int e = threadIdx.x; e < 2 * MT_ROWS * H; e += blockDim.x) {
                const int m = e % H, rr = (e / H) % MT_ROWS, w = e / (MT_ROWS * H);
                const long src = rowpred[w][rr];
                Hs[(w * MT_ROWS + rr) * HS + m] = src >= 0 ? __ldcg(a.hf + src + m) : 0.f;
            }
            __syncthreads();
#pragma unroll
            for (int t = 0; t < MT_RPT; ++t) {
                if (!rw[t].on) continue;  // warp-uniform
                const float *hu = Hs + (rl + MT_RL * t) * HS, *hv = Hs + (MT_ROWS + rl + MT_RL * t) * HS;
                for (int m = 0; m < H; ++m) {
                    const float u = hu[m], v = hv[m];
                    const float *r0 = Rs + (m * 5) * MT_J + jj, *r1 = Rs + ((H + m) * 5) * MT_J + jj;
#pragma unroll
                    for (int q = 0; q < 5; ++q) acc[t][q] = fmaf(v, r1[q * MT_J], fmaf(u, r0[q * MT_J], acc[t][q]));
                }
            }
#pragma unroll
            for (int t = 0; t < MT_RPT; ++t) {
                const MdRow &w = rw[t];
                if (!w.live || !jok) continue;
                const long ck = w.ck;
                const int b = (int)(w.cp % a.B);
                const float cu = w.up > 0 ? __ldcg(a.c + (ck - VB) * H + j) : 0.f;
                const float cv = w.vp > 0 ? __ldcg(a.c + (ck - a.B) * H + j) : 0.f;
                float *ac = a.act + ck * G;
                float h = 0.f, cn;
                if (!w.on) {
                    cn = w.up > 0 ? cu : cv;
#pragma unroll
                    for (int q = 0; q < 5; ++q) ac[q * H + j] = 0.f;
                } else if (!a.stable) {
                    const float gi = msg(acc[t][0]), fu = msg(acc[t][1]), fv = msg(acc[t][2]), gg = mth(acc[t][3]),
                                go = msg(acc[t][4]);
                    cn = fu * cu + fv * cv + gi * gg;
                    h = go * mth(cn);
                    ac[j] = gi; ac[H + j] = fu; ac[2 * H + j] = fv; ac[3 * H + j] = gg; ac[4 * H + j] = go;
                } else {
                    const float gi = msg(acc[t][0]), f = msg(acc[t][1]), gg = mth(acc[t][2]), go = msg(acc[t][3]),
                                lam = msg(acc[t][4]);
                    cn = f * (lam * cu + (1.f - lam) * cv) + gi * gg;
                    h = go * mth(cn);
                    ac[j] = gi; ac[H + j] = f; ac[2 * H + j] = gg; ac[3 * H + j] = go; ac[4 * H + j] = lam;
                }
                a.c[ck * H + j] = cn;
                a.hf[ck * H + j] = h;
                a.h16[((long)k * prow + slot(a, w.up, w.vp, b)) * Hp + j] = __float2half_rn(h);
                a.y[w.cp * 4 * H + (long)k * H + j] = h;
            }
            __syncthreads();  // rowpred / Hs reused by the next row group
        }
        if (d + 1 < ND) grid_barrier(bar, (uint32_t)(d + 1) * gridDim.x);
    }
}

// ---------------------------------------------------------------------------------------------
// Tensor-core wavefront: one persistent CTA per (direction k,
// image b).  Cells of different images or directions never depend on each other, so a CTA walks
// all U+V-1 anti-diagonals of its image alone -- no grid barrier, the previous diagonal's state
// stays in shared memory.  The recurrent weights are resident in TMEM as the tcgen05 A operand,
// split hi + lo (fp16 each), and every contraction is the 3-term product A_hi B_hi + A_lo B_hi +
// A_hi B_lo (operand error ~2^-22: the 2-D recurrence compounds errors along paths of up to U+V
// cells and |c| grows with u+v, so one fp16 pass is not accurate enough).
// Forward, diagonal d: Q = [Ru^T; Rv^T] . H_{d-1}^T  (M = 10 Hp gate rows in up to 5 tiles, N = the
//   <= 32 cells of diagonal d-1, K = Hp); cell (u', v') takes column (u'-1) of the Ru half and
//   column u' of the Rv half (its two predecessors on d-1), adds Z, and runs the gates and cell.
// Backward, diagonal d (reverse): P = [Ru; Rv] . dA_{d+1}^T  (M = 2 Hp, K = 5 Hp split over four
//   issuing warps into four accumulators, N = cells of d+1); dh of (u', v') = dy + P_u column of
//   its u-successor (u'+1) + P_v column of its v-successor (u').
// Requires Hp <= 64 and min(U, V) <= 32 (md_wave_ok); else the per-diagonal CUDA-core kernels run.
// ---------------------------------------------------------------------------------------------
constexpr int WV_N = 32;         // MMA N: cells of one diagonal (min(U, V) <= 32)
constexpr int WV_THREADS = 512;  // 16 warps: thread = (unit pair jp = tid % 32, cell slot tid / 32)
constexpr int WV_KW = 4;         // backward: K-split issuing warps / accumulators

// element (n, k) of a [WV_N x K] K-major no-swizzle B operand: core matrices of 8 n x 8 k (128 B),
// the WV_N / 8 of one K group contiguous, K groups WV_LBO bytes apart.  The 16-byte pad per K group
// keeps the epilogue's stores conflict-free: a warp writes one n and 64 consecutive k, i.e. 8 K
// groups, which would otherwise all start on the same bank (8-way conflicts).
constexpr int WV_LBO = WV_N * 16 + 16;
constexpr int WV_LBOH = WV_LBO / 2;  // in halves
DEVI int wv_bidx(int n, int k) { return (k >> 3) * WV_LBOH + n * 8 + (k & 7); }
__host__ DEVI int wv_bsize(int K) { return K / 8 * WV_LBOH; }  // halves of one B part
DEVI uint32_t pack_h2(__half lo16, __half hi16) {
    return (uint32_t)__half_as_ushort(lo16) | ((uint32_t)__half_as_ushort(hi16) << 16);
}
// two values at once: packed conversions (one cvt.rn.f16x2.f32 per pair instead of two scalar ones)
DEVI void split_h2(float x, float y, uint32_t &hi, uint32_t &lo) {
    const __half2 h = __floats2half2_rn(x, y);
    const float2 hf = __half22float2(h);
    const __half2 l = __floats2half2_rn(x - hf.x, y - hf.y);
    hi = *reinterpret_cast<const uint32_t *>(&h);
    lo = *reinterpret_cast<const uint32_t *>(&l);
}
DEVI void split_h(float x, __half &hi, __half &lo) {
    hi = __float2half_rn(x);
    lo = __float2half_rn(x - __half2float(hi));
}
__host__ DEVI int wv_u0(int d, int V) { return d - V + 1 > 0 ? d - V + 1 : 0; }
__host__ DEVI int wv_u1(int d, int U) { return d < U - 1 ? d : U - 1; }

// per-cell constants of one diagonal (int32 offsets; md_wave_ok bounds them)
struct WvCell {
    int ck;    // direction-frame cell index ((k U + u') V + v') B + b
    int cp;    // physical cell index (u V + v) B + b
    int slot;  // row of the zero-bordered [(U+1)(V+1)B] direction-frame grid (h16 / da16)
    int flags; // bit 0 mask, 1 has u-pred, 2 has v-pred, 3 has u-succ, 4 has v-succ
};
DEVI WvCell wv_cell(const MdK &a, int k, int b, int d, int i) {
    const int up = wv_u0(d, a.V) + i, vp = d - up;
    const int u = (k & 1) ? a.U - 1 - up : up, v = (k & 2) ? a.V - 1 - vp : vp;
    WvCell c;
    c.ck = ((k * a.U + up) * a.V + vp) * a.B + b;
    c.cp = (u * a.V + v) * a.B + b;
    c.slot = ((up + 1) * (a.V + 1) + vp + 1) * a.B + b;
    c.flags = (a.mask[c.cp] != 0) | (up > 0) << 1 | (vp > 0) << 2 | (up + 1 < a.U) << 3 | (vp + 1 < a.V) << 4;
    return c;
}

// A operand rows -> TMEM (hi at column col_hi, lo at col_lo; ncol 32-bit columns = 2 ncol K values
// per row).  row_val(r, kk) gives the fp32 value; warp w writes lanes 32 (w & 3) .. of tile mt for
// the 8-column blocks with (block % 4) == (w >> 2).
template <typename F>
DEVI void wv_load_a(uint32_t tmem, int mt, uint32_t col_hi, uint32_t col_lo, int ncol, F row_val) {
    const int w = warp_id(), l = lane_id(), q = w & 3;
    const int r = mt * 128 + 32 * q + l;
    for (int c0 = 8 * (w >> 2); c0 < ncol; c0 += 32) {
        uint32_t vh[8], vl[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int kk = 2 * (c0 + i);
            __half h0, l0, h1, l1;
            split_h(row_val(r, kk), h0, l0);
            split_h(row_val(r, kk + 1), h1, l1);
            vh[i] = pack_h2(h0, h1);
            vl[i] = pack_h2(l0, l1);
        }
        const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16);
        tmem_st8(lane_base + col_hi + c0, vh);
        tmem_st8(lane_base + col_lo + c0, vl);
    }
}
// 32 lanes x 8 columns load
DEVI void tmem_ld8f(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
// issue the three split products D (+)= A_hi B_hi + A_lo B_hi + A_hi B_lo over K steps [ks0, ks1)
DEVI void wv_mma3(uint32_t dt, uint32_t ah, uint32_t al, uint32_t bh, uint32_t bl, int ks0, int ks1, uint32_t idesc) {
    // descriptor of K step ks = that of step 0 + ks * 2 * WV_LBO bytes in the 14-bit address field
    // (shared-memory addresses < 256 KB: no carry out of the field)
    const uint64_t dh0 = sdesc_noswz(bh, WV_LBO, 128), dl0 = sdesc_noswz(bl, WV_LBO, 128);
    constexpr uint64_t DKS = 2 * WV_LBO / 16;
    for (int ks = ks0; ks < ks1; ++ks) mma_f16_ts_w(dt, ah + ks * 8, dh0 + ks * DKS, idesc, ks > ks0);
    for (int ks = ks0; ks < ks1; ++ks) mma_f16_ts_w(dt, al + ks * 8, dh0 + ks * DKS, idesc, 1);
    for (int ks = ks0; ks < ks1; ++ks) mma_f16_ts_w(dt, ah + ks * 8, dl0 + ks * DKS, idesc, 1);
}

__global__ void __launch_bounds__(WV_THREADS, 1) md_wave_fwd_kernel(MdK a) {
    extern __shared__ uint8_t wv_smem[];
    uint8_t *sm = (uint8_t *)(((uintptr_t)wv_smem + 1023) & ~(uintptr_t)1023);
    const int Hp = a.Hp, H = a.H, G5 = 5 * Hp, R10 = 10 * Hp, U = a.U, V = a.V, B = a.B;
    const int k = blockIdx.x / B, b = blockIdx.x - k * B;
    const int Mt = (R10 + 127) / 128;
    float *Zs = (float *)sm;                       // [2][WV_N][5Hp]  Z of the cells of a diagonal
    float *stg = Zs + 2 * WV_N * G5;               // [WV_N][10Hp]    Q^T (column-major staging)
    __half *Bh = (__half *)(stg + WV_N * R10);     // [Hp/8][WV_N][8] (+pad) h of the previous diagonal, hi
    __half *Bl = Bh + wv_bsize(Hp);                //                  and lo parts
    float *cst = (float *)(Bl + wv_bsize(Hp));     // [2][WV_N][Hp]   c of the previous / this diagonal
    WvCell *tab = (WvCell *)(cst + 2 * WV_N * Hp); // [2][WV_N]       cells of diagonals d, d+1
    uint64_t *bars = (uint64_t *)(tab + 2 * WV_N); // [0] mma, [1..2] Z landed
    uint32_t *tslot = (uint32_t *)(bars + 4);
    const int w = warp_id(), l = lane_id(), tid = threadIdx.x;
    const int prow = (U + 1) * (V + 1) * B;

    if (tid == 0) {
        mbar_init(&bars[0], Mt);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], 1);
        fence_mbar_init();
    }
    if (w == 0) {
        tmem_alloc(tslot, 512);
        tmem_relinquish();
    }
    for (int e = tid; e < wv_bsize(Hp); e += WV_THREADS) reinterpret_cast<uint32_t *>(Bh)[e] = 0u;  // Bh + Bl
    if (tid < WV_N && tid <= wv_u1(0, U) - wv_u0(0, V)) tab[tid] = wv_cell(a, k, b, 0, tid);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    // TMEM columns: A_hi tile mt at [mt Hp/2, ...), A_lo at Mt Hp/2 + mt Hp/2, D tile mt at Mt Hp + 32 mt
    const uint32_t colAl = Mt * Hp / 2, colD = Mt * Hp;
    const float *Ru = a.theta + k * a.P1 + (long)a.D * 5 * H, *Rv = Ru + (long)H * 5 * H;
    for (int mt = 0; mt < Mt; ++mt)  // row r = wv 5Hp + q Hp + jj: gate column q H + jj of R_wv; K = unit
        wv_load_a(tmem, mt, mt * Hp / 2, colAl + mt * Hp / 2, Hp / 2, [&](int r, int kk) -> float {
            const int wv = r / G5, n = r - wv * G5, q = n / Hp, jj = n - q * Hp;
            return (r < R10 && jj < H && kk < H) ? (wv ? Rv : Ru)[(long)kk * 5 * H + q * H + jj] : 0.f;
        });
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    const int ND = U + V - 1;
    auto issue_z = [&](int d, int sl) {  // warp 15: lane i copies cell i's Z row (5Hp fp32)
        const int u0 = wv_u0(d, V), n = wv_u1(d, U) - u0 + 1;
        if (l == 0) mbar_arrive_expect_tx(&bars[1 + sl], (uint32_t)(n * G5 * 4));
        __syncwarp();
        if (l < n) {
            const int up = u0 + l, vp = d - up;
            const int u = (k & 1) ? U - 1 - up : up, v = (k & 2) ? V - 1 - vp : vp;
            const long cp = ((long)u * V + v) * B + b;
            bulk_g2s(smem_u32(Zs + (sl * WV_N + l) * G5), a.z + cp * 20 * Hp + (long)k * G5, (uint32_t)(G5 * 4),
                     &bars[1 + sl]);
        }
    };
    if (w == 15) issue_z(0, 0);
    const int j = 2 * (tid & 31), cs = tid >> 5;  // epilogue: units j, j+1 of cells cs, cs + 16
    const bool j0 = j < H, j1 = j + 1 < H, hodd = H & 1;
    const uint32_t idesc = idesc_f16(128, WV_N, 0, 0);
    uint32_t mph = 0;
#ifdef BLSTM_TRACE
    unsigned long long *trace = (blockIdx.x == 0 && tid == 0) ? a.trace : nullptr;
#endif
    for (int d = 0; d < ND; ++d) {
        const int sl = d & 1;
        WTRACE(d, 0);
        const int u0 = wv_u0(d, V), n = wv_u1(d, U) - u0 + 1;
        const int pu0 = d > 0 ? wv_u0(d - 1, V) : 0;
        if (d > 0 && w < Mt) {  // Q tile w = A_w . H_{d-1}^T, three products
            tc_fence_after();
            wv_mma3(tmem + colD + 32 * w, tmem + w * Hp / 2, tmem + colAl + w * Hp / 2, smem_u32(Bh), smem_u32(Bl), 0,
                    Hp / 16, idesc);
            mma_commit_w(&bars[0]);
        }
        WTRACE(d, 1);
        if (w == 15 && d + 1 < ND) {
            issue_z(d + 1, sl ^ 1);  // its slot was last read at d-1
            const int n1 = wv_u1(d + 1, U) - wv_u0(d + 1, V) + 1;
            if (l < n1) tab[(sl ^ 1) * WV_N + l] = wv_cell(a, k, b, d + 1, l);  // read after the next barriers
        }
        WTRACE(d, 2);
        // one warp waits for Z and the MMAs (spinning warps would take issue slots from the MMA
        // issue); the CTA barrier then releases the rest (hardware-blocking, no polling)
        if (w == Mt) {
            mbar_wait(&bars[1 + sl], (d >> 1) & 1);
            if (d > 0) mbar_wait(&bars[0], mph);
        }
        if (d > 0) mph ^= 1;
        WTRACE(d, 3);
        __syncthreads();
        WTRACE(d, 4);
        if (d > 0) {
            tc_fence_after();
            const int q = w & 3, cb = 8 * (w >> 2);
            float v[5][8];  // all tiles' loads in flight, one wait
#pragma unroll
            for (int mt = 0; mt < 5; ++mt)
                if (mt < Mt) tmem_ld8f(tmem + ((uint32_t)(32 * q) << 16) + colD + 32 * mt + cb, v[mt]);
            tmem_ld_wait();
#pragma unroll
            for (int mt = 0; mt < 5; ++mt) {
                const int row = mt * 128 + 32 * q + l;
                if (mt < Mt && row < R10) {
#pragma unroll
                    for (int c = 0; c < 8; ++c) stg[(cb + c) * R10 + row] = v[mt][c];
                }
            }
        }
        WTRACE(d, 5);
        tc_fence_before();
        __syncthreads();
        WTRACE(d, 6);
        const float *cprev = cst + (sl ^ 1) * WV_N * Hp;
        float *ccur = cst + sl * WV_N * Hp;
        const float *zs = Zs + sl * WV_N * G5;
        const WvCell *tb = tab + sl * WV_N;
        if (j < Hp) {
            for (int i = cs; i < n; i += 16) {
                const WvCell ce = tb[i];
                const int up = u0 + i;
                const bool hasu = ce.flags & 2, hasv = ce.flags & 4, on = ce.flags & 1;
                const int mu = up - 1 - pu0, mv = up - pu0;
                const float2 cu = hasu ? *reinterpret_cast<const float2 *>(cprev + mu * Hp + j) : make_float2(0.f, 0.f);
                const float2 cv = hasv ? *reinterpret_cast<const float2 *>(cprev + mv * Hp + j) : make_float2(0.f, 0.f);
                float2 g[5], h = make_float2(0.f, 0.f), cn;
                if (on) {
                    float2 pre[5];
#pragma unroll
                    for (int q = 0; q < 5; ++q) {
                        float2 s = *reinterpret_cast<const float2 *>(zs + i * G5 + q * Hp + j);
                        if (hasu) {
                            const float2 t = *reinterpret_cast<const float2 *>(stg + mu * R10 + q * Hp + j);
                            s.x += t.x; s.y += t.y;
                        }
                        if (hasv) {
                            const float2 t = *reinterpret_cast<const float2 *>(stg + mv * R10 + G5 + q * Hp + j);
                            s.x += t.x; s.y += t.y;
                        }
                        pre[q] = s;
                    }
                    if (!a.stable) {  // [i, fu, fv, g, o]
#pragma unroll
                        for (int q = 0; q < 5; ++q)
                            g[q] = q == 3 ? make_float2(mth(pre[q].x), mth(pre[q].y)) : make_float2(msg(pre[q].x), msg(pre[q].y));
                        cn.x = g[1].x * cu.x + g[2].x * cv.x + g[0].x * g[3].x;
                        cn.y = g[1].y * cu.y + g[2].y * cv.y + g[0].y * g[3].y;
                        h = make_float2(g[4].x * mth(cn.x), g[4].y * mth(cn.y));
                    } else {          // [i, f, g, o, lambda]
#pragma unroll
                        for (int q = 0; q < 5; ++q)
                            g[q] = q == 2 ? make_float2(mth(pre[q].x), mth(pre[q].y)) : make_float2(msg(pre[q].x), msg(pre[q].y));
                        cn.x = g[1].x * (g[4].x * cu.x + (1.f - g[4].x) * cv.x) + g[0].x * g[2].x;
                        cn.y = g[1].y * (g[4].y * cu.y + (1.f - g[4].y) * cv.y) + g[0].y * g[2].y;
                        h = make_float2(g[3].x * mth(cn.x), g[3].y * mth(cn.y));
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 5; ++q) g[q] = make_float2(0.f, 0.f);
                    cn = hasu ? cu : cv;  // masked: c carried (0 without predecessors), h = 0
                }
                if (!j0) { h.x = 0.f; cn.x = 0.f; }  // padding units stay 0 (B operand K padding)
                if (!j1) { h.y = 0.f; cn.y = 0.f; }
                *reinterpret_cast<float2 *>(ccur + i * Hp + j) = cn;
                uint32_t hh, hl;
                split_h2(h.x, h.y, hh, hl);
                *reinterpret_cast<uint32_t *>(Bh + wv_bidx(i, j)) = hh;
                *reinterpret_cast<uint32_t *>(Bl + wv_bidx(i, j)) = hl;
                // the dR GEMMs' operand, every unit (padding: 0), so only its border rows need zeroing
                *reinterpret_cast<__half2 *>(a.h16 + ((long)k * prow + ce.slot) * Hp + j) = __floats2half2_rn(h.x, h.y);
                if (j0) {  // saved state (Hp-strided rows: pairs stay 8-byte aligned) and the outputs
                    float *ac = a.act + (long)ce.ck * G5 + j;
#pragma unroll
                    for (int q = 0; q < 5; ++q) *reinterpret_cast<float2 *>(ac + q * Hp) = g[q];
                    *reinterpret_cast<float2 *>(a.c + (long)ce.ck * Hp + j) = cn;
                    float *yp = a.y + (long)ce.cp * 4 * H + k * H + j;
                    if (!hodd && j1) {
                        *reinterpret_cast<float2 *>(yp) = h;
                    } else {
                        yp[0] = h.x;
                        if (j1) yp[1] = h.y;
                    }
                }
            }
        }
        WTRACE(d, 7);
        fence_async_smem();  // B written by the generic proxy, read by the next MMAs
        tc_fence_before();
        __syncthreads();
        WTRACE(d, 8);
    }
    if (w == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

__global__ void __launch_bounds__(WV_THREADS, 1) md_wave_bwd_kernel(MdK a) {
    extern __shared__ uint8_t wv_smem[];
    uint8_t *sm = (uint8_t *)(((uintptr_t)wv_smem + 1023) & ~(uintptr_t)1023);
    const int Hp = a.Hp, H = a.H, G5 = 5 * Hp, R2 = 2 * Hp, U = a.U, V = a.V, B = a.B;
    const int k = blockIdx.x / B, b = blockIdx.x - k * B;
    float *stg = (float *)sm;                      // [WV_N][2Hp]   P^T (column-major staging), x 2^DA_SHIFT
    __half *Bh = (__half *)(stg + WV_N * R2);      // [5Hp/8][WV_N][8] (+pad) dA x 2^DA_SHIFT of diagonal d+1, hi
    __half *Bl = Bh + wv_bsize(G5);                //                   and lo parts
    float *acts = (float *)(Bl + wv_bsize(G5));    // [2][WV_N][5Hp] saved gate activations of a diagonal
    float *cr = acts + 2 * WV_N * G5;              // [3][WV_N][Hp]  c of diagonals d, d-1 (ring by d % 3)
    float *dcu = cr + 3 * WV_N * Hp;               // [2][WV_N][Hp]  dc passed to the u- / v-predecessor
    float *dcv = dcu + 2 * WV_N * Hp;
    float *dys = dcv + 2 * WV_N * Hp;              // [2][WV_N][Hp]  dy of a diagonal's cells
    WvCell *tab = (WvCell *)(dys + 2 * WV_N * Hp); // [2][WV_N]
    uint64_t *bars = (uint64_t *)(tab + 2 * WV_N); // [0] mma, [1..2] inputs landed
    uint32_t *tslot = (uint32_t *)(bars + 4);
    const int w = warp_id(), l = lane_id(), tid = threadIdx.x;
    const int prow = (U + 1) * (V + 1) * B;
    const float scale = (float)(1 << DA_SHIFT), unscale = 1.f / scale;
    const int KS = G5 / 16;  // K steps of the contraction

    if (tid == 0) {
        mbar_init(&bars[0], WV_KW);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], 1);
        fence_mbar_init();
    }
    if (w == 0) {
        tmem_alloc(tslot, 512);
        tmem_relinquish();
    }
    for (int e = tid; e < wv_bsize(G5); e += WV_THREADS) reinterpret_cast<uint32_t *>(Bh)[e] = 0u;  // Bh + Bl
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    // TMEM: A_hi [0, 5Hp/2), A_lo [5Hp/2, 5Hp), accumulator a at 5Hp + 32 a
    const uint32_t colAl = G5 / 2, colD = G5;
    const float *Ru = a.theta + k * a.P1 + (long)a.D * 5 * H, *Rv = Ru + (long)H * 5 * H;
    // row r = wv Hp + unit; K index q Hp + jj = gate column q H + jj of that unit's R_wv row
    wv_load_a(tmem, 0, 0, colAl, G5 / 2, [&](int r, int kk) -> float {
        const int wv = r / Hp, rr = r - wv * Hp, q = kk / Hp, jj = kk - q * Hp;
        return (r < R2 && rr < H && jj < H) ? (wv ? Rv : Ru)[(long)rr * 5 * H + q * H + jj] : 0.f;
    });
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    const int ND = U + V - 1;
    const bool dy_bulk = ((H * 4) & 15) == 0;  // dy rows by bulk copy when 16-byte sized
    // inputs of diagonal d2 (warp 15, lane i = cell i): the saved activations, dy and the cell table
    // of its cells, c of diagonal d2-1 (the predecessors); c of d2 itself came with d2+1 (with_c for
    // the first)
    auto issue_in = [&](int d2, bool with_c) {
        const int sl = d2 & 1;
        const int u0 = wv_u0(d2, V), n = wv_u1(d2, U) - u0 + 1;
        const int np = d2 >= 1 ? wv_u1(d2 - 1, U) - wv_u0(d2 - 1, V) + 1 : 0;
        WvCell ce{};
        if (l < n) ce = wv_cell(a, k, b, d2, l);
        uint32_t bytes = (uint32_t)(n * G5 * 4 + np * Hp * 4 + (with_c ? n * Hp * 4 : 0) + (dy_bulk ? n * H * 4 : 0));
        if (l == 0) mbar_arrive_expect_tx(&bars[1 + sl], bytes);
        __syncwarp();
        if (l < n) {
            tab[sl * WV_N + l] = ce;
            bulk_g2s(smem_u32(acts + (sl * WV_N + l) * G5), a.act + (long)ce.ck * G5, (uint32_t)(G5 * 4), &bars[1 + sl]);
            if (with_c)
                bulk_g2s(smem_u32(cr + ((d2 % 3) * WV_N + l) * Hp), a.c + (long)ce.ck * Hp, (uint32_t)(Hp * 4), &bars[1 + sl]);
            const float *dyp = a.dy + (long)ce.cp * 4 * H + k * H;
            float *dyd = dys + (sl * WV_N + l) * Hp;
            if (dy_bulk)
                bulk_g2s(smem_u32(dyd), dyp, (uint32_t)(H * 4), &bars[1 + sl]);
            else
                for (int e = 0; e < H; ++e) dyd[e] = dyp[e];  // (rare: H * 4 not a multiple of 16)
        }
        if (l < np) {
            const int up = wv_u0(d2 - 1, V) + l;
            const int ckp = ((k * U + up) * V + (d2 - 1 - up)) * B + b;
            bulk_g2s(smem_u32(cr + (((d2 + 2) % 3) * WV_N + l) * Hp), a.c + (long)ckp * Hp, (uint32_t)(Hp * 4),
                     &bars[1 + sl]);
        }
    };
    if (w == 15) issue_in(ND - 1, true);
    const int j = 2 * (tid & 31), cs = tid >> 5;
    const bool j0 = j < H, j1 = j + 1 < H;
    const uint32_t idesc = idesc_f16(128, WV_N, 0, 0);
    uint32_t mph = 0, iph = 0;
    const int ks0 = (w * KS) / WV_KW, ks1 = ((w + 1) * KS) / WV_KW;  // this warp's K range (w < WV_KW)
#ifdef BLSTM_TRACE
    unsigned long long *trace = (blockIdx.x == 0 && tid == 0) ? a.trace : nullptr;
#endif
    for (int d = ND - 1; d >= 0; --d) {
        const int sl = d & 1;
        WTRACE(ND - 1 - d, 0);
        const int u0 = wv_u0(d, V), n = wv_u1(d, U) - u0 + 1;
        const bool has_succ = d + 1 < ND;
        const int su0 = has_succ ? wv_u0(d + 1, V) : 0, pu0 = d > 0 ? wv_u0(d - 1, V) : 0;
        if (has_succ && w < WV_KW) {  // P_w = A[:, K range w] . dA_{d+1}[:, K range w]^T, three products
            tc_fence_after();
            wv_mma3(tmem + colD + 32 * w, tmem, tmem + colAl, smem_u32(Bh), smem_u32(Bl), ks0, ks1, idesc);
            mma_commit_w(&bars[0]);
        }
        WTRACE(ND - 1 - d, 1);
        if (w == 15 && d >= 1) issue_in(d - 1, false);  // its slots were last read at d+1
        WTRACE(ND - 1 - d, 2);
        if (w == WV_KW) {  // one warp waits (see the forward), the CTA barrier releases the rest
            mbar_wait(&bars[1 + sl], (iph >> sl) & 1);
            if (has_succ) mbar_wait(&bars[0], mph);
        }
        iph ^= 1u << sl;
        if (has_succ) mph ^= 1;
        WTRACE(ND - 1 - d, 3);
        __syncthreads();
        WTRACE(ND - 1 - d, 4);
        if (has_succ) {
            tc_fence_after();
            const int q = w & 3, cb = 8 * (w >> 2);
            float x[WV_KW][8], v[8];  // KS = 5Hp/16 >= 5: every K range is non-empty
#pragma unroll
            for (int aa = 0; aa < WV_KW; ++aa) tmem_ld8f(tmem + ((uint32_t)(32 * q) << 16) + colD + 32 * aa + cb, x[aa]);
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < 8; ++c) v[c] = (x[0][c] + x[1][c]) + (x[2][c] + x[3][c]);
            const int row = 32 * q + l;
            if (row < R2) {
#pragma unroll
                for (int c = 0; c < 8; ++c) stg[(cb + c) * R2 + row] = v[c];
            }
        }
        WTRACE(ND - 1 - d, 5);
        tc_fence_before();
        __syncthreads();
        WTRACE(ND - 1 - d, 6);
        const float *ac_s = acts + sl * WV_N * G5, *c_s = cr + (d % 3) * WV_N * Hp;
        const float *cp_s = cr + ((d + 2) % 3) * WV_N * Hp;  // c of diagonal d-1
        const float *dcu_p = dcu + (sl ^ 1) * WV_N * Hp, *dcv_p = dcv + (sl ^ 1) * WV_N * Hp;
        float *dcu_c = dcu + sl * WV_N * Hp, *dcv_c = dcv + sl * WV_N * Hp;
        const float *dy_s = dys + sl * WV_N * Hp;
        const WvCell *tb = tab + sl * WV_N;
        if (j < Hp) {
            for (int i = cs; i < n; i += 16) {
                const WvCell ce = tb[i];
                const int up = u0 + i;
                const bool su = ce.flags & 8, sv = ce.flags & 16, on = ce.flags & 1;
                float2 da[5], ou = make_float2(0.f, 0.f), ov = make_float2(0.f, 0.f);
#pragma unroll
                for (int q = 0; q < 5; ++q) da[q] = make_float2(0.f, 0.f);
                const int iu = up + 1 - su0, iv = up - su0;  // successor columns on d+1
                float2 dc = make_float2(0.f, 0.f);
                if (su) {
                    const float2 t = *reinterpret_cast<const float2 *>(dcu_p + iu * Hp + j);
                    dc.x += t.x; dc.y += t.y;
                }
                if (sv) {
                    const float2 t = *reinterpret_cast<const float2 *>(dcv_p + iv * Hp + j);
                    dc.x += t.x; dc.y += t.y;
                }
                if (!on) {
                    if (ce.flags & 2) ou = dc;                       // the carried c came from the u-,
                    else if (ce.flags & 4) ov = dc;                  // else the v-predecessor
                } else {
                    float2 dh = *reinterpret_cast<const float2 *>(dy_s + i * Hp + j);  // (.y unused past H)
                    if (su) {
                        const float2 t = *reinterpret_cast<const float2 *>(stg + iu * R2 + j);
                        dh.x += t.x * unscale; dh.y += t.y * unscale;
                    }
                    if (sv) {
                        const float2 t = *reinterpret_cast<const float2 *>(stg + iv * R2 + Hp + j);
                        dh.x += t.x * unscale; dh.y += t.y * unscale;
                    }
                    const float *acl = ac_s + i * G5 + j;
                    const float2 c = *reinterpret_cast<const float2 *>(c_s + i * Hp + j);
                    const float2 cu = (ce.flags & 2) ? *reinterpret_cast<const float2 *>(cp_s + (up - 1 - pu0) * Hp + j)
                                                     : make_float2(0.f, 0.f);
                    const float2 cv = (ce.flags & 4) ? *reinterpret_cast<const float2 *>(cp_s + (up - pu0) * Hp + j)
                                                     : make_float2(0.f, 0.f);
                    float2 A[5];
#pragma unroll
                    for (int q = 0; q < 5; ++q) A[q] = *reinterpret_cast<const float2 *>(acl + q * Hp);
                    auto cellg = [&](float dhv, float dcv_, float cc, float cuu, float cvv, const float *g, float *o,
                                     float &ouu, float &ovv) {
                        const float tc = mth(cc);
                        const float dct = dcv_ + dhv * (a.stable ? g[3] : g[4]) * (1.f - tc * tc);
                        if (!a.stable) {  // [i, fu, fv, g, o]
                            o[0] = dct * g[3] * g[0] * (1.f - g[0]);
                            o[1] = dct * cuu * g[1] * (1.f - g[1]);
                            o[2] = dct * cvv * g[2] * (1.f - g[2]);
                            o[3] = dct * g[0] * (1.f - g[3] * g[3]);
                            o[4] = dhv * tc * g[4] * (1.f - g[4]);
                            ouu = dct * g[1];
                            ovv = dct * g[2];
                        } else {          // [i, f, g, o, lambda]
                            const float m = g[4] * cuu + (1.f - g[4]) * cvv;
                            o[0] = dct * g[2] * g[0] * (1.f - g[0]);
                            o[1] = dct * m * g[1] * (1.f - g[1]);
                            o[2] = dct * g[0] * (1.f - g[2] * g[2]);
                            o[3] = dhv * tc * g[3] * (1.f - g[3]);
                            o[4] = dct * g[1] * (cuu - cvv) * g[4] * (1.f - g[4]);
                            ouu = dct * g[1] * g[4];
                            ovv = dct * g[1] * (1.f - g[4]);
                        }
                    };
                    float gx[5], gy[5], ox[5], oy[5];
#pragma unroll
                    for (int q = 0; q < 5; ++q) { gx[q] = A[q].x; gy[q] = A[q].y; }
                    cellg(dh.x, dc.x, c.x, cu.x, cv.x, gx, ox, ou.x, ov.x);
                    cellg(dh.y, dc.y, c.y, cu.y, cv.y, gy, oy, ou.y, ov.y);
#pragma unroll
                    for (int q = 0; q < 5; ++q) da[q] = make_float2(ox[q], oy[q]);
                    if (!j0) { ou.x = ov.x = 0.f; }
                    if (!j1) { ou.y = ov.y = 0.f; }
                }
#pragma unroll
                for (int q = 0; q < 5; ++q) {
                    if (!j0) da[q].x = 0.f;
                    if (!j1) da[q].y = 0.f;
                }
                *reinterpret_cast<float2 *>(dcu_c + i * Hp + j) = ou;
                *reinterpret_cast<float2 *>(dcv_c + i * Hp + j) = ov;
                __half2 *dpp = reinterpret_cast<__half2 *>(a.dap + (long)ce.cp * 20 * Hp + k * G5 + j);
                __half2 *d16 = reinterpret_cast<__half2 *>(a.da16 + ((long)k * prow + ce.slot) * G5 + j);
#pragma unroll
                for (int q = 0; q < 5; ++q) {
                    uint32_t hh, hl;
                    split_h2(da[q].x * scale, da[q].y * scale, hh, hl);
                    *reinterpret_cast<uint32_t *>(Bh + wv_bidx(i, q * Hp + j)) = hh;
                    *reinterpret_cast<uint32_t *>(Bl + wv_bidx(i, q * Hp + j)) = hl;
                    reinterpret_cast<uint32_t *>(dpp)[q * Hp / 2] = hh;  // (padding units: zeros)
                    reinterpret_cast<uint32_t *>(d16)[q * Hp / 2] = hh;
                }
            }
        }
        WTRACE(ND - 1 - d, 7);
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        WTRACE(ND - 1 - d, 8);
    }
    if (w == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

size_t wv_fwd_smem(int Hp) {
    return 1024 + (size_t)(2 * WV_N * 5 * Hp + WV_N * 10 * Hp + 2 * WV_N * Hp) * 4 + (size_t)2 * wv_bsize(Hp) * 2 +
           2 * WV_N * sizeof(WvCell) + 64;
}
size_t wv_bwd_smem(int Hp) {
    return 1024 + (size_t)(WV_N * 2 * Hp + 2 * WV_N * 5 * Hp + 3 * WV_N * Hp + 6 * WV_N * Hp) * 4 +
           (size_t)2 * wv_bsize(5 * Hp) * 2 + 2 * WV_N * sizeof(WvCell) + 64;
}
// ---------------------------------------------------------------------------------------------
// CTA-pair wavefront (round 2): a cluster of 2 CTAs per (direction k, image b); rank r owns the
// units [r Hh, (r+1) Hh), Hh = Hp / 2, so each SM does half of a diagonal's gate math (the single-
// CTA kernels above are bound by that epilogue) and 128 instead of 64 SMs work.
//   Forward: rank r's A operand holds the gate rows of its own units (M = 10 Hh, <= 3 tiles), K = all
//   Hp units of h_{d-1}; after its epilogue each rank writes h_d of its units (hi / lo) into its own
//   B operand and, by st.async with complete_tx, into the partner's (double-buffered by diagonal
//   parity: the partner may finish diagonal d+1 while this rank's MMA still reads diagonal d-1).
//   Backward: K split -- rank r's A operand is [Ru; Rv] (all 2 Hp rows) restricted to the gate columns
//   of its own units, its B operand its own dA_{d+1}; the partial P rows of the partner's units go
//   to the partner by st.async (8 KB at Hp = 64), and each rank sums the two partials of its own rows
//   in fixed order (rank 0's + rank 1's: deterministic).
// Applies for Hp in {32, 64} (md_wave_pair).
// ---------------------------------------------------------------------------------------------
DEVI void named_bar(int id, int nthreads) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory"); }
DEVI void st_async_b32(uint32_t dst_cluster, uint32_t v, uint32_t mbar_cluster) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(dst_cluster), "r"(v),
                 "r"(mbar_cluster)
                 : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(WV_THREADS, 1) md_wave2_fwd_kernel(MdK a) {
    extern __shared__ uint8_t wv_smem[];
    uint8_t *sm = (uint8_t *)(((uintptr_t)wv_smem + 1023) & ~(uintptr_t)1023);
    const int Hp = a.Hp, Hh = Hp / 2, H = a.H, G5 = 5 * Hp, R10 = 10 * Hh, U = a.U, V = a.V, B = a.B;
    const int r = (int)cluster_ctarank();
    const int kbi = blockIdx.x >> 1, k = kbi / B, b = kbi - k * B;
    const int Mt = (R10 + 127) / 128;
    const int BS = wv_bsize(Hp);
    float *Zs = (float *)sm;                        // [2][WV_N][5Hp]
    float *stg = Zs + 2 * WV_N * G5;                // [WV_N][10Hh]   Q^T rows of the own units
    __half *Bb = (__half *)(stg + WV_N * R10);      // [2 parity][2 part][BS]  h of a diagonal (all units)
    float *cst = (float *)(Bb + 4 * BS);            // [2][WV_N][Hh]  c of the own units
    WvCell *tab = (WvCell *)(cst + 2 * WV_N * Hh);  // [2][WV_N]
    // [0] mma, [1..2] Z landed, [3..4] partner's h half landed, [5..6] slot free (consumers -> producer)
    uint64_t *bars = (uint64_t *)(tab + 2 * WV_N);
    uint32_t *tslot = (uint32_t *)(bars + 7);
    const int w = warp_id(), l = lane_id(), tid = threadIdx.x;
    const int prow = (U + 1) * (V + 1) * B;

    if (tid == 0) {
        mbar_init(&bars[0], Mt);
        for (int i = 1; i < 7; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    if (w == 0) {
        tmem_alloc(tslot, 512);
        tmem_relinquish();
    }
    for (int e = tid; e < 2 * BS; e += WV_THREADS) reinterpret_cast<uint32_t *>(Bb)[e] = 0u;  // 4 B halves
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t colAl = Mt * Hp / 2, colD = Mt * Hp;
    const float *Ru = a.theta + k * a.P1 + (long)a.D * 5 * H, *Rv = Ru + (long)H * 5 * H;
    for (int mt = 0; mt < Mt; ++mt)  // row = wv 5Hh + q Hh + jj': gate column q H + (r Hh + jj') of R_wv
        wv_load_a(tmem, mt, mt * Hp / 2, colAl + mt * Hp / 2, Hp / 2, [&](int row, int kk) -> float {
            const int wv = row / (5 * Hh), n = row - wv * 5 * Hh, q = n / Hh, jj = r * Hh + (n - q * Hh);
            return (row < R10 && jj < H && kk < H) ? (wv ? Rv : Ru)[(long)kk * 5 * H + q * H + jj] : 0.f;
        });
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    cluster_sync();  // the partner's barriers are initialised before any remote store

    const int ND = U + V - 1;
    auto issue_z = [&](int d, int sl) {  // warp 15: lane i copies cell i's Z row (5Hp fp32)
        const int u0 = wv_u0(d, V), n = wv_u1(d, U) - u0 + 1;
        if (l == 0) mbar_arrive_expect_tx(&bars[1 + sl], (uint32_t)(n * G5 * 4));
        __syncwarp();
        if (l < n) {
            const int up = u0 + l, vp = d - up;
            const int u = (k & 1) ? U - 1 - up : up, v = (k & 2) ? V - 1 - vp : vp;
            const long cp = ((long)u * V + v) * B + b;
            bulk_g2s(smem_u32(Zs + (sl * WV_N + l) * G5), a.z + cp * 20 * Hp + (long)k * G5, (uint32_t)(G5 * 4),
                     &bars[1 + sl]);
        }
    };
    // warp 15 is the producer: Z rows and the cell table of diagonal d2 into slot d2 & 1 as soon as the
    // consumers (warps 0-14, named barrier 1) released it after diagonal d2 - 2 -- the ~32 bulk copies
    // a diagonal needs cost ~1 us of issue and stay off the consumers' per-diagonal chain
    if (w == 15) {
        for (int d2 = 0; d2 < ND; ++d2) {
            const int sl2 = d2 & 1;
            if (d2 >= 2) mbar_wait(&bars[5 + sl2], ((d2 - 2) >> 1) & 1);
            const int n2 = wv_u1(d2, U) - wv_u0(d2, V) + 1;
            if (l < n2) tab[sl2 * WV_N + l] = wv_cell(a, k, b, d2, l);
            __syncwarp();  // the table is written before lane 0's arrive (release) in issue_z
            issue_z(d2, sl2);
        }
    } else {
    // epilogue work item (unit pair pi: own units jl = 2 pi, 2 pi + 1, global j = r Hh + jl; cell ic)
    const uint32_t idesc = idesc_f16(128, WV_N, 0, 0);
    const uint32_t bb_addr = smem_u32(Bb), peer_bb = mapa_shared(bb_addr, (uint32_t)(r ^ 1));
    const uint32_t peer_x = mapa_shared(smem_u32(&bars[3]), (uint32_t)(r ^ 1));
    uint32_t mph = 0;
#ifdef BLSTM_TRACE
    unsigned long long *trace = (blockIdx.x == 0 && tid == 0) ? a.trace : nullptr;
#endif
    for (int d = 0; d < ND; ++d) {
        const int sl = d & 1;
        WTRACE(d, 0);
        const int u0 = wv_u0(d, V), n = wv_u1(d, U) - u0 + 1;
        const int pu0 = d > 0 ? wv_u0(d - 1, V) : 0;
        if (d > 0 && w < Mt) {  // h_{d-1}: the own half (CTA barrier below) and the partner's half landed
            mbar_wait_cluster(&bars[3 + (sl ^ 1)], ((d - 1) >> 1) & 1);
            tc_fence_after();
            const uint32_t bh = bb_addr + (uint32_t)((sl ^ 1) * 2) * BS * 2;
            wv_mma3(tmem + colD + 32 * w, tmem + w * Hp / 2, tmem + colAl + w * Hp / 2, bh, bh + BS * 2, 0, Hp / 16,
                    idesc);
            mma_commit_w(&bars[0]);
        }
        WTRACE(d, 1);
        // the partner's h_d: n cells x Hh units x (hi, lo) fp16
        if (w == 14 && l == 0) mbar_arrive_expect_tx(&bars[3 + sl], (uint32_t)(n * Hh * 4));
        WTRACE(d, 2);
        if (w == 0) {  // (after its MMA issue; thread 0's trace then shows the waits)
            mbar_wait(&bars[1 + sl], (d >> 1) & 1);
            if (d > 0) mbar_wait(&bars[0], mph);
        }
        if (d > 0) mph ^= 1;
        WTRACE(d, 3);
        named_bar(1, WV_THREADS - 32);
        WTRACE(d, 4);
        if (d > 0) {
            tc_fence_after();
            // lane quarter q = w & 3 (the warp's TMEM lanes); 8-column blocks: warp 11 also takes the
            // producer warp's block 3 (a 17th warp measured slower: 96 registers, spills)
            const int q = w & 3;
            for (int cbi = w >> 2; cbi < 4; cbi += (w == 11 ? 1 : 4)) {
                const int cb = 8 * cbi;
                float v[3][8];
#pragma unroll
                for (int mt = 0; mt < 3; ++mt)
                    if (mt < Mt) tmem_ld8f(tmem + ((uint32_t)(32 * q) << 16) + colD + 32 * mt + cb, v[mt]);
                tmem_ld_wait();
#pragma unroll
                for (int mt = 0; mt < 3; ++mt) {
                    const int row = mt * 128 + 32 * q + l;
                    if (mt < Mt && row < R10) {
#pragma unroll
                        for (int c = 0; c < 8; ++c) stg[(cb + c) * R10 + row] = v[mt][c];
                    }
                }
            }
        }
        WTRACE(d, 5);
        tc_fence_before();
        named_bar(1, WV_THREADS - 32);
        WTRACE(d, 6);
        const float *cprev = cst + (sl ^ 1) * WV_N * Hh;
        float *ccur = cst + sl * WV_N * Hh;
        const float *zs = Zs + sl * WV_N * G5;
        // epilogue work item = (4 own units jl = 4 qi .. 4 qi + 3, global j = r Hh + jl; cell ic): 256
        // items at Hh = 32, at most one per consumer thread (with 2-unit items, 32 threads took two)
        for (int item = tid; item < (Hh / 4) * WV_N; item += WV_THREADS - 32) {
            const int qi = item % (Hh / 4), ic = item / (Hh / 4), jl = 4 * qi, j = r * Hh + jl;
            if (ic >= n) continue;
            const int i = ic;
            const WvCell ce = tab[sl * WV_N + i];
            const int up = u0 + i;
            const bool hasu = ce.flags & 2, hasv = ce.flags & 4, on = ce.flags & 1;
            const int mu = up - 1 - pu0, mv = up - pu0;
            const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 cu4 = hasu ? *reinterpret_cast<const float4 *>(cprev + mu * Hh + jl) : z4;
            const float4 cv4 = hasv ? *reinterpret_cast<const float4 *>(cprev + mv * Hh + jl) : z4;
            const float cu[4] = {cu4.x, cu4.y, cu4.z, cu4.w}, cv[4] = {cv4.x, cv4.y, cv4.z, cv4.w};
            float g[5][4], h[4], cn[4];
            if (on) {
                float pre[5][4];
#pragma unroll
                for (int q = 0; q < 5; ++q) {
                    float4 s4 = *reinterpret_cast<const float4 *>(zs + i * G5 + q * Hp + j);
                    if (hasu) {
                        const float4 t4 = *reinterpret_cast<const float4 *>(stg + mu * R10 + q * Hh + jl);
                        s4.x += t4.x; s4.y += t4.y; s4.z += t4.z; s4.w += t4.w;
                    }
                    if (hasv) {
                        const float4 t4 = *reinterpret_cast<const float4 *>(stg + mv * R10 + 5 * Hh + q * Hh + jl);
                        s4.x += t4.x; s4.y += t4.y; s4.z += t4.z; s4.w += t4.w;
                    }
                    pre[q][0] = s4.x; pre[q][1] = s4.y; pre[q][2] = s4.z; pre[q][3] = s4.w;
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if (!a.stable) {  // [i, fu, fv, g, o]
#pragma unroll
                        for (int q = 0; q < 5; ++q) g[q][e] = q == 3 ? mth(pre[q][e]) : msg(pre[q][e]);
                        cn[e] = g[1][e] * cu[e] + g[2][e] * cv[e] + g[0][e] * g[3][e];
                        h[e] = g[4][e] * mth(cn[e]);
                    } else {          // [i, f, g, o, lambda]
#pragma unroll
                        for (int q = 0; q < 5; ++q) g[q][e] = q == 2 ? mth(pre[q][e]) : msg(pre[q][e]);
                        cn[e] = g[1][e] * (g[4][e] * cu[e] + (1.f - g[4][e]) * cv[e]) + g[0][e] * g[2][e];
                        h[e] = g[3][e] * mth(cn[e]);
                    }
                }
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
#pragma unroll
                    for (int q = 0; q < 5; ++q) g[q][e] = 0.f;
                    h[e] = 0.f;
                    cn[e] = hasu ? cu[e] : cv[e];  // masked: c carried (0 without predecessors), h = 0
                }
            }
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (j + e >= H) { h[e] = 0.f; cn[e] = 0.f; }  // padding units stay 0 (B operand K padding)
            *reinterpret_cast<float4 *>(ccur + i * Hh + jl) = make_float4(cn[0], cn[1], cn[2], cn[3]);
            uint32_t hh0, hl0, hh1, hl1;
            split_h2(h[0], h[1], hh0, hl0);
            split_h2(h[2], h[3], hh1, hl1);
            const uint32_t off = (uint32_t)((sl * 2) * BS + wv_bidx(i, j)) * 2;  // bytes, part hi (8-byte aligned)
            *reinterpret_cast<uint2 *>(reinterpret_cast<uint8_t *>(Bb) + off) = make_uint2(hh0, hh1);
            *reinterpret_cast<uint2 *>(reinterpret_cast<uint8_t *>(Bb) + off + BS * 2) = make_uint2(hl0, hl1);
            st_async_v2u(peer_bb + off, hh0, hh1, peer_x + 8 * sl);
            st_async_v2u(peer_bb + off + BS * 2, hl0, hl1, peer_x + 8 * sl);
            *reinterpret_cast<uint2 *>(a.h16 + ((long)k * prow + ce.slot) * Hp + j) = make_uint2(hh0, hh1);
            if (j < H) {
                float *ac = a.act + (long)ce.ck * G5 + j;
#pragma unroll
                for (int q = 0; q < 5; ++q) *reinterpret_cast<float4 *>(ac + q * Hp) = make_float4(g[q][0], g[q][1], g[q][2], g[q][3]);
                *reinterpret_cast<float4 *>(a.c + (long)ce.ck * Hp + j) = make_float4(cn[0], cn[1], cn[2], cn[3]);
                float *yp = a.y + (long)ce.cp * 4 * H + k * H + j;
                if ((H & 3) == 0) {
                    *reinterpret_cast<float4 *>(yp) = make_float4(h[0], h[1], h[2], h[3]);
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (j + e < H) yp[e] = h[e];
                }
            }
        }
        WTRACE(d, 7);
        fence_async_smem();
        tc_fence_before();
        named_bar(1, WV_THREADS - 32);
        if (tid == 0) mbar_arrive(&bars[5 + sl]);  // slot sl (Z, cell table of diagonal d) free
        WTRACE(d, 8);
    }
    // the partner's h of the last diagonal (never read) has landed: no remote store is outstanding
    if (tid == 0) mbar_wait_cluster(&bars[3 + ((ND - 1) & 1)], ((ND - 1) >> 1) & 1);
    }  // consumers
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (w == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(WV_THREADS, 1) md_wave2_bwd_kernel(MdK a) {
    extern __shared__ uint8_t wv_smem[];
    uint8_t *sm = (uint8_t *)(((uintptr_t)wv_smem + 1023) & ~(uintptr_t)1023);
    const int Hp = a.Hp, Hh = Hp / 2, H = a.H, G5 = 5 * Hp, K5 = 5 * Hh, R2 = 2 * Hh, U = a.U, V = a.V, B = a.B;
    const int r = (int)cluster_ctarank();
    const int kbi = blockIdx.x >> 1, k = kbi / B, b = kbi - k * B;
    const int BS = wv_bsize(K5);
    float *stg = (float *)sm;                       // [WV_N][2Hh]  this rank's partial P of its own rows (x 2^DA_SHIFT)
    float *rcv = stg + WV_N * R2;                   // [2 par][WV_N][2Hh]  the partner's partial of them
    __half *Bh = (__half *)(rcv + 2 * WV_N * R2);   // [5Hh/8][WV_N][8] (+pad): own dA of diagonal d+1, hi
    __half *Bl = Bh + BS;                           //                         and lo parts
    float *acts = (float *)(Bl + BS);               // [2][WV_N][5Hp]
    float *cr = acts + 2 * WV_N * G5;               // [3][WV_N][Hp]
    float *dcu = cr + 3 * WV_N * Hp;                // [2][WV_N][Hh]  (own units)
    float *dcv = dcu + 2 * WV_N * Hh;
    float *dys = dcv + 2 * WV_N * Hh;               // [2][WV_N][Hp]
    WvCell *tab = (WvCell *)(dys + 2 * WV_N * Hp);  // [2][WV_N]
    // [0] mma, [1..2] inputs landed, [3..4] partner's partial landed, [5..6] slot free (consumers -> producer)
    uint64_t *bars = (uint64_t *)(tab + 2 * WV_N);
    uint32_t *tslot = (uint32_t *)(bars + 7);
    const int w = warp_id(), l = lane_id(), tid = threadIdx.x;
    const int prow = (U + 1) * (V + 1) * B;
    const float scale = (float)(1 << DA_SHIFT), unscale = 1.f / scale;
    const int KS = K5 / 16;

    if (tid == 0) {
        mbar_init(&bars[0], WV_KW);
        for (int i = 1; i < 7; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    if (w == 0) {
        tmem_alloc(tslot, 512);
        tmem_relinquish();
    }
    for (int e = tid; e < BS; e += WV_THREADS) reinterpret_cast<uint32_t *>(Bh)[e] = 0u;  // Bh + Bl
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t colAl = K5 / 2, colD = K5;
    const float *Ru = a.theta + k * a.P1 + (long)a.D * 5 * H, *Rv = Ru + (long)H * 5 * H;
    // row = wv Hp + unit; K index q Hh + jj' = gate column q H + (r Hh + jj') of that unit's R_wv row
    wv_load_a(tmem, 0, 0, colAl, K5 / 2, [&](int row, int kk) -> float {
        const int wv = row / Hp, rr = row - wv * Hp, q = kk / Hh, jj = r * Hh + (kk - q * Hh);
        return (row < 2 * Hp && rr < H && jj < H) ? (wv ? Rv : Ru)[(long)rr * 5 * H + q * H + jj] : 0.f;
    });
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    cluster_sync();

    const int ND = U + V - 1;
    const bool dy_bulk = ((H * 4) & 15) == 0;
    auto issue_in = [&](int d2, bool with_c) {  // as md_wave_bwd_kernel
        const int sl = d2 & 1;
        const int u0 = wv_u0(d2, V), n = wv_u1(d2, U) - u0 + 1;
        const int np = d2 >= 1 ? wv_u1(d2 - 1, U) - wv_u0(d2 - 1, V) + 1 : 0;
        WvCell ce{};
        if (l < n) ce = wv_cell(a, k, b, d2, l);
        const float *dyp = a.dy + (long)ce.cp * 4 * H + k * H;
        float *dyd = dys + (sl * WV_N + l) * Hp;
        if (l < n) {  // generic writes first: lane 0's arrive (release) below publishes them
            tab[sl * WV_N + l] = ce;
            if (!dy_bulk)
                for (int e = 0; e < H; ++e) dyd[e] = dyp[e];  // (rare: H * 4 not a multiple of 16)
        }
        __syncwarp();
        uint32_t bytes = (uint32_t)(n * G5 * 4 + np * Hp * 4 + (with_c ? n * Hp * 4 : 0) + (dy_bulk ? n * H * 4 : 0));
        if (l == 0) mbar_arrive_expect_tx(&bars[1 + sl], bytes);
        __syncwarp();
        if (l < n) {
            bulk_g2s(smem_u32(acts + (sl * WV_N + l) * G5), a.act + (long)ce.ck * G5, (uint32_t)(G5 * 4), &bars[1 + sl]);
            if (with_c)
                bulk_g2s(smem_u32(cr + ((d2 % 3) * WV_N + l) * Hp), a.c + (long)ce.ck * Hp, (uint32_t)(Hp * 4), &bars[1 + sl]);
            if (dy_bulk) bulk_g2s(smem_u32(dyd), dyp, (uint32_t)(H * 4), &bars[1 + sl]);
        }
        if (l < np) {
            const int up = wv_u0(d2 - 1, V) + l;
            const int ckp = ((k * U + up) * V + (d2 - 1 - up)) * B + b;
            bulk_g2s(smem_u32(cr + (((d2 + 2) % 3) * WV_N + l) * Hp), a.c + (long)ckp * Hp, (uint32_t)(Hp * 4),
                     &bars[1 + sl]);
        }
    };
    // warp 15 is the producer (see md_wave2_fwd_kernel): the inputs of diagonal d2 into slot d2 & 1
    // once the consumers released it after diagonal d2 + 2
    if (w == 15) {
        for (int d2 = ND - 1; d2 >= 0; --d2) {
            if (d2 + 2 <= ND - 1) mbar_wait(&bars[5 + (d2 & 1)], ((ND - 3 - d2) >> 1) & 1);
            issue_in(d2, d2 == ND - 1);
        }
    } else {
    const uint32_t idesc = idesc_f16(128, WV_N, 0, 0);
    const uint32_t peer_rcv = mapa_shared(smem_u32(rcv), (uint32_t)(r ^ 1));
    const uint32_t peer_x = mapa_shared(smem_u32(&bars[3]), (uint32_t)(r ^ 1));
    uint32_t mph = 0, iph = 0;
    const int ks0 = (w * KS) / WV_KW, ks1 = ((w + 1) * KS) / WV_KW;
#ifdef BLSTM_TRACE
    unsigned long long *trace = (blockIdx.x == 0 && tid == 0) ? a.trace : nullptr;
#endif
    for (int d = ND - 1; d >= 0; --d) {
        const int sl = d & 1;
        WTRACE(ND - 1 - d, 0);
        const int u0 = wv_u0(d, V), n = wv_u1(d, U) - u0 + 1;
        const bool has_succ = d + 1 < ND;
        const int su0 = has_succ ? wv_u0(d + 1, V) : 0, pu0 = d > 0 ? wv_u0(d - 1, V) : 0;
        if (has_succ && w < WV_KW) {  // partial P_w over this rank's K range part w
            tc_fence_after();
            wv_mma3(tmem + colD + 32 * w, tmem, tmem + colAl, smem_u32(Bh), smem_u32(Bl), ks0, ks1, idesc);
            mma_commit_w(&bars[0]);
        }
        WTRACE(ND - 1 - d, 1);
        if (has_succ && w == 14 && l == 0) mbar_arrive_expect_tx(&bars[3 + sl], (uint32_t)(WV_N * R2 * 4));
        WTRACE(ND - 1 - d, 2);
        if (w == 0) {  // (after its MMA issue; thread 0's trace then shows the waits)
            mbar_wait(&bars[1 + sl], (iph >> sl) & 1);
            if (has_succ) mbar_wait(&bars[0], mph);
        }
        iph ^= 1u << sl;
        if (has_succ) mph ^= 1;
        WTRACE(ND - 1 - d, 3);
        named_bar(1, WV_THREADS - 32);
        WTRACE(ND - 1 - d, 4);
        if (has_succ) {  // the partial's rows: own units -> stg, the partner's -> its receive buffer
          tc_fence_after();
          const int q = w & 3;
          for (int cbi = w >> 2; cbi < 4; cbi += (w == 11 ? 1 : 4)) {
            const int cb = 8 * cbi;
            float x[WV_KW][8], v[8];
#pragma unroll
            for (int aa = 0; aa < WV_KW; ++aa) tmem_ld8f(tmem + ((uint32_t)(32 * q) << 16) + colD + 32 * aa + cb, x[aa]);
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < 8; ++c) v[c] = (x[0][c] + x[1][c]) + (x[2][c] + x[3][c]);
            const int row = 32 * q + l;
            if (row < 2 * Hp) {
                const int wv = row / Hp, unit = row - wv * Hp, owner = unit / Hh;
                const int lr = wv * Hh + (unit - owner * Hh);  // row among the owner's 2Hh
                if (owner == r) {
#pragma unroll
                    for (int c = 0; c < 8; ++c) stg[(cb + c) * R2 + lr] = v[c];
                } else {
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        st_async_b32(peer_rcv + (uint32_t)(((sl * WV_N + cb + c) * R2 + lr) * 4), __float_as_uint(v[c]),
                                     peer_x + 8 * sl);
                }
            }
          }
        }
        WTRACE(ND - 1 - d, 5);
        if (has_succ && w == 0) mbar_wait_cluster(&bars[3 + sl], ((ND - 2 - d) >> 1) & 1);
        WTRACE(ND - 1 - d, 9);
        tc_fence_before();
        named_bar(1, WV_THREADS - 32);
        WTRACE(ND - 1 - d, 6);
        const float *ac_s = acts + sl * WV_N * G5, *c_s = cr + (d % 3) * WV_N * Hp;
        const float *cp_s = cr + ((d + 2) % 3) * WV_N * Hp;
        const float *dcu_p = dcu + (sl ^ 1) * WV_N * Hh, *dcv_p = dcv + (sl ^ 1) * WV_N * Hh;
        float *dcu_c = dcu + sl * WV_N * Hh, *dcv_c = dcv + sl * WV_N * Hh;
        const float *dy_s = dys + sl * WV_N * Hp;
        const float *rv = rcv + sl * WV_N * R2;
        // work item = (4 own units jl = 4 qi .., global j = r Hh + jl; cell ic): at most one per thread
        for (int item = tid; item < (Hh / 4) * WV_N; item += WV_THREADS - 32) {
            const int qi = item % (Hh / 4), ic = item / (Hh / 4), jl = 4 * qi, j = r * Hh + jl;
            if (ic >= n) continue;
            const int i = ic;
            const WvCell ce = tab[sl * WV_N + i];
            const int up = u0 + i;
            const bool su = ce.flags & 8, sv = ce.flags & 16, on = ce.flags & 1;
            const int iu = up + 1 - su0, iv = up - su0;
            const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
            auto ld4 = [](const float *q) { return *reinterpret_cast<const float4 *>(q); };
            auto arr = [](float4 v, float (&o)[4]) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; };
            float dc[4], dcu4[4], dcv4[4];
            arr(su ? ld4(dcu_p + iu * Hh + jl) : z4, dcu4);
            arr(sv ? ld4(dcv_p + iv * Hh + jl) : z4, dcv4);
#pragma unroll
            for (int e = 0; e < 4; ++e) dc[e] = dcu4[e] + dcv4[e];
            float da[5][4], ou[4], ov[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                ou[e] = ov[e] = 0.f;
#pragma unroll
                for (int q = 0; q < 5; ++q) da[q][e] = 0.f;
            }
            if (!on) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if (ce.flags & 2) ou[e] = dc[e];       // the carried c came from the u-,
                    else if (ce.flags & 4) ov[e] = dc[e];  // else the v-predecessor
                }
            } else {
                // P of an own row = rank 0's partial + rank 1's partial (fixed order on both ranks)
                auto prow4 = [&](int col, int lr, float (&o)[4]) {
                    const float4 mine = ld4(stg + col * R2 + lr), peer = ld4(rv + col * R2 + lr);
                    if (r == 0) arr(make_float4(mine.x + peer.x, mine.y + peer.y, mine.z + peer.z, mine.w + peer.w), o);
                    else arr(make_float4(peer.x + mine.x, peer.y + mine.y, peer.z + mine.z, peer.w + mine.w), o);
                };
                float dh[4], pu[4], pv[4], c[4], cu[4], cv[4];
                arr(ld4(dy_s + i * Hp + j), dh);
                if (su) prow4(iu, jl, pu);
                if (sv) prow4(iv, Hh + jl, pv);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if (su) dh[e] += pu[e] * unscale;
                    if (sv) dh[e] += pv[e] * unscale;
                }
                arr(ld4(c_s + i * Hp + j), c);
                arr((ce.flags & 2) ? ld4(cp_s + (up - 1 - pu0) * Hp + j) : z4, cu);
                arr((ce.flags & 4) ? ld4(cp_s + (up - pu0) * Hp + j) : z4, cv);
                float gq[5][4];
                const float *acl = ac_s + i * G5 + j;
#pragma unroll
                for (int q = 0; q < 5; ++q) arr(ld4(acl + q * Hp), gq[q]);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float tc = mth(c[e]);
                    if (!a.stable) {  // [i, fu, fv, g, o]
                        const float gi = gq[0][e], fu = gq[1][e], fv = gq[2][e], gg = gq[3][e], go = gq[4][e];
                        const float dct = dc[e] + dh[e] * go * (1.f - tc * tc);
                        da[0][e] = dct * gg * gi * (1.f - gi);
                        da[1][e] = dct * cu[e] * fu * (1.f - fu);
                        da[2][e] = dct * cv[e] * fv * (1.f - fv);
                        da[3][e] = dct * gi * (1.f - gg * gg);
                        da[4][e] = dh[e] * tc * go * (1.f - go);
                        ou[e] = dct * fu;
                        ov[e] = dct * fv;
                    } else {          // [i, f, g, o, lambda]
                        const float gi = gq[0][e], f = gq[1][e], gg = gq[2][e], go = gq[3][e], lam = gq[4][e];
                        const float dct = dc[e] + dh[e] * go * (1.f - tc * tc);
                        const float m = lam * cu[e] + (1.f - lam) * cv[e];
                        da[0][e] = dct * gg * gi * (1.f - gi);
                        da[1][e] = dct * m * f * (1.f - f);
                        da[2][e] = dct * gi * (1.f - gg * gg);
                        da[3][e] = dh[e] * tc * go * (1.f - go);
                        da[4][e] = dct * f * (cu[e] - cv[e]) * lam * (1.f - lam);
                        ou[e] = dct * f * lam;
                        ov[e] = dct * f * (1.f - lam);
                    }
                }
            }
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (j + e >= H) {  // padding units: zeros
                    ou[e] = ov[e] = 0.f;
#pragma unroll
                    for (int q = 0; q < 5; ++q) da[q][e] = 0.f;
                }
            *reinterpret_cast<float4 *>(dcu_c + i * Hh + jl) = make_float4(ou[0], ou[1], ou[2], ou[3]);
            *reinterpret_cast<float4 *>(dcv_c + i * Hh + jl) = make_float4(ov[0], ov[1], ov[2], ov[3]);
            uint2 *dpp = reinterpret_cast<uint2 *>(a.dap + (long)ce.cp * 20 * Hp + k * G5 + j);
            uint2 *d16 = reinterpret_cast<uint2 *>(a.da16 + ((long)k * prow + ce.slot) * G5 + j);
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                uint32_t hh0, hl0, hh1, hl1;
                split_h2(da[q][0] * scale, da[q][1] * scale, hh0, hl0);
                split_h2(da[q][2] * scale, da[q][3] * scale, hh1, hl1);
                *reinterpret_cast<uint2 *>(Bh + wv_bidx(i, q * Hh + jl)) = make_uint2(hh0, hh1);
                *reinterpret_cast<uint2 *>(Bl + wv_bidx(i, q * Hh + jl)) = make_uint2(hl0, hl1);
                dpp[q * Hp / 4] = make_uint2(hh0, hh1);  // (padding units: zeros)
                d16[q * Hp / 4] = make_uint2(hh0, hh1);
            }
        }
        WTRACE(ND - 1 - d, 7);
        fence_async_smem();
        tc_fence_before();
        named_bar(1, WV_THREADS - 32);
        if (tid == 0) mbar_arrive(&bars[5 + sl]);  // slot sl (inputs of diagonal d) free
        WTRACE(ND - 1 - d, 8);
    }
    }  // consumers
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (w == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

size_t wv2_fwd_smem(int Hp) {
    const int Hh = Hp / 2;
    return 1024 + (size_t)(2 * WV_N * 5 * Hp + WV_N * 10 * Hh + 2 * WV_N * Hh) * 4 + (size_t)4 * wv_bsize(Hp) * 2 +
           2 * WV_N * sizeof(WvCell) + 64;
}
size_t wv2_bwd_smem(int Hp) {
    const int Hh = Hp / 2;
    return 1024 + (size_t)(3 * WV_N * 2 * Hh + 2 * WV_N * 5 * Hp + 3 * WV_N * Hp + 4 * WV_N * Hh + 2 * WV_N * Hp) * 4 +
           (size_t)2 * wv_bsize(5 * Hh) * 2 + 2 * WV_N * sizeof(WvCell) + 64;
}
// the CTA-pair wavefront applies (Hp in {32, 64}: K groups of the half split stay whole; BLSTM_MD_PAIR=0: never)
bool md_wave_pair(const MdGeo &g) {
    const bool off = getenv("BLSTM_MD_PAIR") && atoi(getenv("BLSTM_MD_PAIR")) == 0;
    return !off && (g.Hp == 32 || g.Hp == 64) && wv2_fwd_smem(g.Hp) <= 227 * 1024 && wv2_bwd_smem(g.Hp) <= 227 * 1024;
}

// the tensor-core wavefront applies (BLSTM_MD_WAVE=0: never)
bool md_wave_ok(const MdGeo &g) {
    const bool off = getenv("BLSTM_MD_WAVE") && atoi(getenv("BLSTM_MD_WAVE")) == 0;  // read per call (tests A/B)
    if (off) return false;
    const int mn = g.U < g.V ? g.U : g.V;
    // int32 cell offsets (WvCell) and grid rows
    const bool fits32 = g.cells * 20 * g.Hp < (1L << 31) && 4 * g.prow * 5 * g.Hp < (1L << 31);
    return fits32 && g.Hp <= 64 && mn <= WV_N && wv_fwd_smem(g.Hp) <= 227 * 1024 && wv_bwd_smem(g.Hp) <= 227 * 1024;
}
int md_wave_launch(bool fwd, const MdGeo &g, const MdK &a, cudaStream_t st) {
    if (md_wave_pair(g)) {  // clusters of 2 CTAs per (direction, image)
        const void *fn = fwd ? (const void *)md_wave2_fwd_kernel : (const void *)md_wave2_bwd_kernel;
        const size_t smem = fwd ? wv2_fwd_smem(g.Hp) : wv2_bwd_smem(g.Hp);
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -5;
        ProfScope ps(fwd ? PROF_REC_FWD : PROF_REC_BWD, st);
        if (fwd)
            md_wave2_fwd_kernel<<<8 * g.B, WV_THREADS, smem, st>>>(a);
        else
            md_wave2_bwd_kernel<<<8 * g.B, WV_THREADS, smem, st>>>(a);
        note_launch();
        return cudaGetLastError() == cudaSuccess ? 0 : -5;
    }
    const void *fn = fwd ? (const void *)md_wave_fwd_kernel : (const void *)md_wave_bwd_kernel;
    const size_t smem = fwd ? wv_fwd_smem(g.Hp) : wv_bwd_smem(g.Hp);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -5;
    ProfScope ps(fwd ? PROF_REC_FWD : PROF_REC_BWD, st);
    if (fwd)
        md_wave_fwd_kernel<<<4 * g.B, WV_THREADS, smem, st>>>(a);
    else
        md_wave_bwd_kernel<<<4 * g.B, WV_THREADS, smem, st>>>(a);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

// W16 [20Hp][Dp]: row k*5Hp + q*Hp + j <- W_k[f][q*H + j] as hi + lo fp16 parts (w16lo may be
// null); bq [20Hp] <- b_k
__global__ void md_pack_kernel(const float *theta, long P1, int D, int H, int Hp, int Dp, __half *w16, __half *w16lo,
                               float *bq) {
    const long n = 20L * Hp * Dp;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) {
        const int f = (int)(e % Dp);
        const int row = (int)(e / Dp), k = row / (5 * Hp), q = (row / Hp) % 5, j = row % Hp;
        const bool ok = j < H;
        const float v = (ok && f < D) ? theta[k * P1 + (long)f * 5 * H + q * H + j] : 0.f;
        const __half hi = __float2half_rn(v);
        w16[e] = hi;
        if (w16lo) w16lo[e] = __float2half_rn(v - __half2float(hi));
        if (f == 0) bq[row] = ok ? theta[k * P1 + (long)D * 5 * H + 2L * H * 5 * H + q * H + j] : 0.f;
    }
}
// the split-precision projection as ONE GEMM over a tripled K (Z written once):
//   xcat [cells][3Dp] = [x_hi | x_hi | x_lo],  wcat [20Hp][3Dp] = [W_hi | W_lo | W_hi]
//   Z = xcat wcat^T = x_hi W_hi + x_hi W_lo + x_lo W_hi  (zero padded past D)
__global__ void md_split_x_kernel(const float *x, int D, int Dp, long cells, __half *xcat) {
    const long n = cells * Dp;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) {
        const long r = e / Dp;
        const int f = (int)(e - r * Dp);
        const float v = f < D ? x[r * D + f] : 0.f;
        const __half h = __float2half_rn(v);
        __half *row = xcat + r * 3 * Dp;
        row[f] = h;
        row[Dp + f] = h;
        row[2 * Dp + f] = __float2half_rn(v - __half2float(h));
    }
}
__global__ void md_pack_cat_kernel(const float *theta, long P1, int D, int H, int Hp, int Dp, __half *wcat, float *bq) {
    const long n = 20L * Hp * Dp;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) {
        const int f = (int)(e % Dp);
        const int row = (int)(e / Dp), k = row / (5 * Hp), q = (row / Hp) % 5, j = row % Hp;
        const bool ok = j < H;
        const float v = (ok && f < D) ? theta[k * P1 + (long)f * 5 * H + q * H + j] : 0.f;
        const __half hi = __float2half_rn(v);
        __half *r = wcat + (long)row * 3 * Dp;
        r[f] = hi;
        r[Dp + f] = __float2half_rn(v - __half2float(hi));
        r[2 * Dp + f] = hi;
        if (f == 0) bq[row] = ok ? theta[k * P1 + (long)D * 5 * H + 2L * H * 5 * H + q * H + j] : 0.f;
    }
}
// rt [4][2][5H][H] <- Ru_k^T, Rv_k^T
__global__ void md_pack_rt_kernel(const float *theta, long P1, int D, int H, float *rt) {
    const int G = 5 * H;
    const long n = 8L * G * H;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) {
        const int j = (int)(e % H);
        const long r = e / H;
        const int q = (int)(r % G), w = (int)((r / G) % 2), k = (int)(r / (2L * G));
        rt[e] = theta[k * P1 + (long)D * G + (long)w * H * G + (long)j * G + q];
    }
}
// zero the border rows (u' = -1 or v' = -1) of a zero-bordered [4][(U+1)(V+1)B][width] fp16 grid
// (h16, da16): the tensor-core wavefront writes every interior row, so no full memset is needed
__global__ void md_zero_border_kernel(__half *grid, int U, int V, int B, int width) {
    const long per = (long)(V + 1 + U) * B, prow = (long)(U + 1) * (V + 1) * B;
    const long n = 4 * per * (width / 2);
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) {
        const long row = e / (width / 2);
        const int col = (int)(e - row * (width / 2)) * 2;
        const int k = (int)(row / per);
        const long br = row - k * per;
        // border row br: the first (V+1) B rows (u' = -1), then rows ((up+1)(V+1)) B + b (v' = -1)
        const long slot = br < (long)(V + 1) * B ? br : ((br / B - (V + 1) + 1) * (long)(V + 1)) * B + br % B;
        *reinterpret_cast<__half2 *>(grid + (k * prow + slot) * width + col) = __floats2half2_rn(0.f, 0.f);
    }
}
// x16 [cells][Dp] column D <- 1: the dW GEMM's column D is then db = the column sums of dA (D < Dp)
__global__ void md_ones_col_kernel(__half *x16, long cells, int Dp, int D) {
    for (long r = blockIdx.x * (long)blockDim.x + threadIdx.x; r < cells; r += (long)gridDim.x * blockDim.x)
        x16[r * Dp + D] = __float2half_rn(1.f);
}
// grad W_k[f][q*H + j] += gW[k*5Hp + q*Hp + j][f]; Ru, Rv from gR [4][2][5Hp][Hp]; b from gb[row * gbs]
__global__ void md_scatter_kernel(float *grad, long P1, int D, int H, int Hp, int Dp, const float *gW, const float *gR,
                                  const float *gb, int gbs) {
    const int G = 5 * H;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < 4 * P1; e += (long)gridDim.x * blockDim.x) {
        const int k = (int)(e / P1);
        long o = e - k * P1;
        float v;
        if (o < (long)D * G) {
            const int f = (int)(o / G), n = (int)(o % G), q = n / H, j = n % H;
            v = gW[((long)k * 5 * Hp + q * Hp + j) * Dp + f];
        } else if (o < (long)D * G + 2L * H * G) {
            o -= (long)D * G;
            const int w = (int)(o / ((long)H * G));
            const long oo = o - (long)w * H * G;
            const int m = (int)(oo / G), n = (int)(oo % G), q = n / H, j = n % H;
            v = gR[(((long)k * 2 + w) * 5 * Hp + q * Hp + j) * Hp + m];
        } else {
            const int n = (int)(o - (long)D * G - 2L * H * G), q = n / H, j = n % H;
            v = gb[((long)k * 5 * Hp + q * Hp + j) * gbs];
        }
        grad[e] += v;
    }
}

}  // namespace

MdGeo md_geo(int U, int V, int B, int D, int H, int stable) {
    MdGeo g;
    g.U = U; g.V = V; g.B = B; g.D = D; g.H = H; g.stable = stable;
    g.Hp = rup(H, 16);
    g.Dp = rup(D, 64);
    g.cells = (long)U * V * B;
    g.prow = (long)(U + 1) * (V + 1) * B;
    return g;
}
size_t md_param_count(const MdGeo &g) { return 4 * ((size_t)g.D * 5 * g.H + 2 * (size_t)g.H * 5 * g.H + 5 * g.H); }

MdWS md_ws(const MdGeo &g) {
    MdWS w{};
    size_t o = 0;
    auto take = [&](size_t b) { size_t r = o; o += al(b); return r; };
    const size_t cells = g.cells, st = 4 * cells;  // direction-frame elements per unit
    w.x16 = take(cells * g.Dp * 2);
    w.x16lo = take(cells * 3 * g.Dp * 2);          // forward: xcat [cells][3Dp]
    w.w16 = take((size_t)20 * g.Hp * g.Dp * 2);
    w.w16lo = take((size_t)20 * g.Hp * 3 * g.Dp * 2);  // forward: wcat [20Hp][3Dp]
    w.z = take(cells * 20 * g.Hp * 4);
    w.hf = take(st * g.H * 4);
    w.gb = take((size_t)20 * g.Hp * 4);  // bias vector in the forward, db in the backward
    w.dap = take(cells * 20 * g.Hp * 2);
    w.rt = take((size_t)8 * 5 * g.H * g.H * 4);
    w.dcu = take(st * g.H * 4);
    w.dcv = take(st * g.H * 4);
    w.daf = take(st * 5 * g.H * 4);
    w.gW = take((size_t)20 * g.Hp * g.Dp * 4);
    w.gR = take((size_t)8 * 5 * g.Hp * g.Hp * 4);
    w.cs = take(colsum_scratch_bytes(cells, 20 * g.Hp));
    w.gsk = take((size_t)(8L << 20) * 4);
    w.da16 = take((size_t)4 * g.prow * 5 * g.Hp * 2);
    w.dxs = take(cells * g.Dp * 4);
    w.bar = take(256);
    w.total = o;
    size_t r = 0;
    auto rtake = [&](size_t b) { size_t q = r; r += al(b); return q; };
    w.act = rtake(st * 5 * g.Hp * 4);  // row stride 5H (per-diagonal kernels) or 5Hp (wavefront)
    w.c = rtake(st * g.Hp * 4);
    w.h16 = rtake((size_t)4 * g.prow * g.Hp * 2);
    w.rtotal = r;
    return w;
}

static MdK md_args(const MdGeo &g, const float *theta, const uint8_t *mask, uint8_t *ws, uint8_t *res) {
    const MdWS w = md_ws(g);
    MdK a{};
    a.U = g.U; a.V = g.V; a.B = g.B; a.D = g.D; a.H = g.H; a.Hp = g.Hp; a.stable = g.stable;
    a.P1 = (long)(md_param_count(g) / 4);
    a.theta = theta; a.mask = mask;
    a.z = (const float *)(ws + w.z);
    a.hf = (float *)(ws + w.hf);
    a.act = (float *)(res + w.act); a.c = (float *)(res + w.c); a.h16 = (__half *)(res + w.h16);
    a.rt = (const float *)(ws + w.rt);
    a.daf = (float *)(ws + w.daf); a.dcu = (float *)(ws + w.dcu); a.dcv = (float *)(ws + w.dcv);
    a.da16 = (__half *)(ws + w.da16); a.dap = (__half *)(ws + w.dap);
    a.trace = nullptr;
    return a;
}

// Persistent forward wavefront launch: 0 = done, 1 = not possible here (per-diagonal path instead),
// < 0 error.  BLSTM_MD_PERSIST=0 forces the per-diagonal path.  (A persistent backward -- the R^T
// tile plus the successors' dA staged per row group -- measured slower than the per-diagonal
// kernels: 17.2 vs 11.1 ms at H = 64, one block per SM.)
static int md_persist(bool fwd, MdK &a, const MdGeo &g, uint32_t *bar, cudaStream_t st) {
    if (!fwd) return 1;
    const bool env_off = getenv("BLSTM_MD_PERSIST") && atoi(getenv("BLSTM_MD_PERSIST")) == 0;
    if (env_off) return 1;
    const int H = g.H, G = 5 * H;
    const size_t smem = fwd ? (size_t)(2 * H * 5 * MT_J + 2 * MT_ROWS * (H + 1)) * 4
                            : (size_t)(2 * G * MT_J + 2 * MT_ROWS * (G + 1)) * 4;
    if (smem > 200 * 1024) return 1;
    const void *fn = (const void *)md_fwd_persist_kernel;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return 1;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem) != cudaSuccess || per_sm < 1) {
        cudaGetLastError();
        return 1;
    }
    const int njt = (H + MT_J - 1) / MT_J;
    const int maxrows = (g.U < g.V ? g.U : g.V) * g.B;
    const int maxrg = (maxrows + MT_ROWS - 1) / MT_ROWS;
    int NG = num_sms() * per_sm / (4 * njt);
    if (NG > maxrg) NG = maxrg;
    if (NG < 1) return 1;
    if (cudaMemsetAsync(bar, 0, sizeof(uint32_t), st) != cudaSuccess) return -5;
    void *args[] = {(void *)&a, (void *)&bar, (void *)&NG};
    ProfScope ps(fwd ? PROF_REC_FWD : PROF_REC_BWD, st);
    if (cudaLaunchCooperativeKernel(fn, dim3(4 * njt * NG), dim3(256), args, smem, st) != cudaSuccess) {
        cudaGetLastError();
        return 1;
    }
    note_launch();
    return 0;
}

int md_forward(const MdGeo &g, const float *theta, const float *x, const uint8_t *mask, float *y, uint8_t *ws,
               uint8_t *res, cudaStream_t st) {
    const MdWS w = md_ws(g);
    MdK a = md_args(g, theta, mask, ws, res);
    a.y = y;
    __half *xcat = (__half *)(ws + w.x16lo), *wcat = (__half *)(ws + w.w16lo);
    float *bq = (float *)(ws + w.gb);
    {
        ProfScope ps(PROF_OTHER, st);
        md_pack_cat_kernel<<<grid1(20L * g.Hp * g.Dp), 256, 0, st>>>(theta, a.P1, g.D, g.H, g.Hp, g.Dp, wcat, bq);
        md_split_x_kernel<<<grid1(g.cells * g.Dp), 256, 0, st>>>(x, g.D, g.Dp, g.cells, xcat);
        note_launch(2);
    }
    if (md_wave_ok(g)) {  // the wavefront writes every interior row (all Hp units): zero the borders only
        ProfScope ps(PROF_OTHER, st);
        md_zero_border_kernel<<<grid1(4L * (g.U + g.V + 1) * g.B * g.Hp / 2), 256, 0, st>>>(
            (__half *)(res + w.h16), g.U, g.V, g.B, g.Hp);
        note_launch();
    } else if (cudaMemsetAsync(res + w.h16, 0, (size_t)4 * g.prow * g.Hp * 2, st) != cudaSuccess) {
        return -5;
    }
    // Z = x W + b in split precision: x_hi W_hi + x_hi W_lo + x_lo W_hi (fp16 tensor-core operands,
    // fp32 accumulate; operand error ~2^-22 instead of 2^-11: the 2-D recurrence compounds the input
    // error along paths of up to U+V cells), one GEMM over K = 3 Dp
    GemmParams gz{(int)g.cells, 20 * g.Hp, 3 * g.Dp, (float *)(ws + w.z), 20L * g.Hp, 1.f, 0, bq, 0, 0};
    if (gemm_f16({xcat, 3L * g.Dp, 0}, {wcat, 3L * g.Dp, 0}, gz, 0, st)) return -5;
    a.trace = rec_trace_fwd();
    if (md_wave_ok(g)) return md_wave_launch(true, g, a, st);
    {
        const int rc = md_persist(true, a, g, (uint32_t *)(ws + w.bar), st);
        if (rc <= 0) return rc;
    }
    // the U+V-1 wavefront launches, captured once into a CUDA graph (graph.h) and replayed
    const std::vector<uint64_t> key{3, (uint64_t)g.U, (uint64_t)g.V, (uint64_t)g.B, (uint64_t)g.D, (uint64_t)g.H,
                                    (uint64_t)g.stable, u64(theta), u64(mask), u64(y), u64(ws), u64(res)};
    return graph_run(key, PROF_REC_FWD, st, {(const void *)md_fwd_diag_kernel}, [&](cudaStream_t s0) -> int {
        for (int d = 0; d < g.U + g.V - 1; ++d) {
            md_fwd_diag_kernel<<<md_blocks(g.U, g.V, g.B, g.H, d), 256, 0, s0>>>(a, d);
            note_launch();
        }
        return cudaGetLastError() == cudaSuccess ? 0 : -5;
    });
}

int md_backward(const MdGeo &g, const float *theta, const float *x, const uint8_t *mask, const float *dy, float *dx,
                float *grad, uint8_t *ws, uint8_t *res, cudaStream_t st) {
    const MdWS w = md_ws(g);
    MdK a = md_args(g, theta, mask, ws, res);
    a.dy = dy;
    const float alpha = 1.f / (float)(1 << DA_SHIFT);
    __half *x16 = (__half *)(ws + w.x16), *w16 = (__half *)(ws + w.w16);
    const bool wave = md_wave_ok(g);
    {
        ProfScope ps(PROF_OTHER, st);
        md_pack_kernel<<<grid1(20L * g.Hp * g.Dp), 256, 0, st>>>(theta, a.P1, g.D, g.H, g.Hp, g.Dp, w16, nullptr,
                                                                 (float *)(ws + w.gb));
        note_launch();
        if (!wave) {
            md_pack_rt_kernel<<<grid1(8L * 5 * g.H * g.H), 256, 0, st>>>(theta, a.P1, g.D, g.H, (float *)(ws + w.rt));
            note_launch();
        }
    }
    if (cast_x_f16(x, g.D, g.D, x16, g.Dp, g.cells, st)) return -5;
    const bool ones = g.D < g.Dp;  // db through the dW GEMM (a column of ones in x), else column sums
    if (ones) {
        ProfScope ps(PROF_OTHER, st);
        md_ones_col_kernel<<<grid1(g.cells), 256, 0, st>>>(x16, g.cells, g.Dp, g.D);
        note_launch();
    }
    if (wave) {  // every interior row and every unit of dap / da16 is written: zero da16's borders only
        ProfScope ps(PROF_OTHER, st);
        md_zero_border_kernel<<<grid1(4L * (g.U + g.V + 1) * g.B * 5 * g.Hp / 2), 256, 0, st>>>(
            (__half *)(ws + w.da16), g.U, g.V, g.B, 5 * g.Hp);
        note_launch();
    } else {
        if (cudaMemsetAsync(ws + w.da16, 0, (size_t)4 * g.prow * 5 * g.Hp * 2, st) != cudaSuccess) return -5;
        if (cudaMemsetAsync(ws + w.dap, 0, (size_t)g.cells * 20 * g.Hp * 2, st) != cudaSuccess) return -5;
    }
    a.trace = rec_trace_bwd();
    if (wave && md_wave_launch(false, g, a, st)) return -5;
    const int prc = wave ? 0 : md_persist(false, a, g, (uint32_t *)(ws + w.bar), st);
    if (prc < 0) return prc;
    const std::vector<uint64_t> key{4, (uint64_t)g.U, (uint64_t)g.V, (uint64_t)g.B, (uint64_t)g.D, (uint64_t)g.H,
                                    (uint64_t)g.stable, u64(theta), u64(mask), u64(dy), u64(ws), u64(res)};
    if (prc == 1 && graph_run(key, PROF_REC_BWD, st, {(const void *)md_bwd_diag_kernel}, [&](cudaStream_t s0) -> int {
            for (int d = g.U + g.V - 2; d >= 0; --d) {
                md_bwd_diag_kernel<<<md_blocks(g.U, g.V, g.B, g.H, d), 256, 0, s0>>>(a, d);
                note_launch();
            }
            return cudaGetLastError() == cudaSuccess ? 0 : -5;
        }))
        return -5;
    const __half *dap = (const __half *)(ws + w.dap);
    float *gsk = (float *)(ws + w.gsk);
    if (dx) {  // dX = dA W_all^T (the four directions sum in the contraction)
        GemmParams gx{(int)g.cells, g.Dp, 20 * g.Hp, (float *)(ws + w.dxs), (long)g.Dp, alpha, 0, nullptr, 0, 0};
        if (gemm_f16({dap, 20L * g.Hp, 0}, {w16, g.Dp, 1}, gx, 0, st)) return -5;
        if (store_dx(dx, g.D, (const float *)(ws + w.dxs), g.Dp, g.D, g.cells, 0, st)) return -5;
    }
    {   // dW_all^T [20Hp, Dp] = dA^T X
        GemmParams gw{20 * g.Hp, g.Dp, (int)g.cells, (float *)(ws + w.gW), (long)g.Dp, alpha, 0, nullptr, 0, 0};
        gw.splitk_ws = gsk; gw.splitk_elems = 8L << 20;
        if (gemm_f16({dap, 20L * g.Hp, 1}, {x16, g.Dp, 1}, gw, 0, st)) return -5;
    }
    const __half *da16 = (const __half *)(ws + w.da16), *h16 = (const __half *)(res + w.h16);
    for (int k = 0; k < 4; ++k)
        for (int wv = 0; wv < 2; ++wv) {  // dRu (shift one u-row of the padded grid) / dRv (one v-step)
            const long shift = wv == 0 ? (long)(g.V + 1) * g.B : (long)g.B;
            const __half *A = da16 + ((long)k * g.prow + shift) * 5 * g.Hp;
            const __half *Hb = h16 + (long)k * g.prow * g.Hp;
            GemmParams gr{5 * g.Hp, g.Hp, (int)(g.prow - shift), (float *)(ws + w.gR) + (size_t)(k * 2 + wv) * 5 * g.Hp * g.Hp,
                          (long)g.Hp, alpha, 0, nullptr, 0, 0};
            gr.splitk_ws = gsk; gr.splitk_elems = 8L << 20;
            if (gemm_f16({A, 5L * g.Hp, 1}, {Hb, g.Hp, 1}, gr, 0, st)) return -5;
        }
    if (!ones) {
        if (cudaMemsetAsync(ws + w.gb, 0, (size_t)20 * g.Hp * 4, st) != cudaSuccess) return -5;
        if (colsum_f16_add(dap, g.cells, 20 * g.Hp, 20L * g.Hp, alpha, (float *)(ws + w.gb), (float *)(ws + w.cs), st))
            return -5;
    }
    {
        ProfScope ps(PROF_OTHER, st);
        const float *gb = ones ? (const float *)(ws + w.gW) + g.D : (const float *)(ws + w.gb);
        md_scatter_kernel<<<grid1(4 * a.P1), 256, 0, st>>>(grad, a.P1, g.D, g.H, g.Hp, g.Dp, (const float *)(ws + w.gW),
                                                           (const float *)(ws + w.gR), gb, ones ? g.Dp : 1);
        note_launch();
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

}  // namespace blstm
