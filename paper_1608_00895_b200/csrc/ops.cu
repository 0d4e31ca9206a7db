// ops.cu -- HBM-bound helper kernels of the path: operand packing (fp32 master
// parameters -> fp16 tensor-core operands in the kernel-private gate-interleaved
// layout), the softmax-CE head (§3.2, summed over valid frames,
// P:253-254), deterministic reductions, gradient scatter-add back to the flat
// theta layout, and SGD (§4.3).  All grid-stride, coalesced on the
// large side of each mapping.
#include <algorithm>
#include "common.cuh"
#include "ops.h"
#include "prof.h"

namespace blstm {

static int grid_for(long n, int block = 256, int cap = 148 * 16) {
    long g = (n + block - 1) / block;
    if (g > cap) g = cap;
    return g < 1 ? 1 : (int)g;
}

// --- input dropout draw (R20): lowbias32 finalizer over (seed, site, element) --------
DEVI uint32_t mix32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}
DEVI bool drop_keep(uint32_t seed, int site, unsigned long long i, uint32_t thr) {
    uint32_t h = mix32(seed + 0x9E3779B9u * (uint32_t)(site + 1));
    h = mix32(h ^ (uint32_t)i);
    h = mix32(h ^ (uint32_t)(i >> 32));
    return h >= thr;
}

// --- x [rows, ldx] fp32 -> X16 [rows, Dp] fp16 (zero pad; site-0 dropout when dr.on) ---------
__global__ void cast_x_kernel(const float *__restrict__ x, long ldx, int D, __half *__restrict__ x16, int Dp,
                              long rows, Dropout dr) {
    const long n = rows * Dp;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const long r = i / Dp;
        const int k = (int)(i - r * Dp);
        float v = k < D ? x[r * ldx + k] : 0.f;
        if (dr.on && k < D) v = drop_keep(dr.seed, 0, (unsigned long long)r * D + k, dr.thr) ? v * dr.scale : 0.f;
        x16[i] = __float2half_rn(v);
    }
}
int cast_x_f16(const float *x, long ldx, int D, __half *x16, int Dp, long rows, cudaStream_t st, const Dropout &dr) {
    ProfScope ps_(PROF_OTHER, st);
    cast_x_kernel<<<grid_for(rows * Dp), 256, 0, st>>>(x, ldx, D, x16, Dp, rows, dr);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

// --- in-place dropout of a layer output (next layer's input) / its gradient -------------------
// element keep draw with the (seed, site) part precomputed: h0 = mix32(seed + 0x9E3779B9 (site+1))
DEVI bool drop_keep_h0(uint32_t h0, unsigned long long i, uint32_t thr) {
    uint32_t h = mix32(h0 ^ (uint32_t)i);
    h = mix32(h ^ (uint32_t)(i >> 32));
    return h >= thr;
}
// VEC elements (16 bytes) per thread per iteration over the padded row [2Hq]; physical column
// c holds logical feature c (c < H) or H + c - Hq (Hq <= c < Hq + H); padding columns are 0 and
// stay 0 either way.  Blocks stride over rows: no integer division.
template <typename V>
__global__ void dropout_kernel(V *__restrict__ y, long rows, int H, int Hq, int site, Dropout dr, int lg_nv) {
    constexpr int VEC = 16 / sizeof(V);
    const uint32_t h0 = mix32(dr.seed + 0x9E3779B9u * (uint32_t)(site + 1));
    const long total = rows << lg_nv;  // 16-byte vectors; a row holds 2^lg_nv of them (Hq = 2^k)
    const int W = 2 * H;
    uint4 *y4 = reinterpret_cast<uint4 *>(y);
    for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < total; q += (long)gridDim.x * blockDim.x) {
        const long r = q >> lg_nv;
        const int v = (int)(q & ((1 << lg_nv) - 1));
        uint4 pk = y4[q];
        V *e = reinterpret_cast<V *>(&pk);
        const unsigned long long base = (unsigned long long)r * W;
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            const int c = v * VEC + k, dd = c >= Hq, u = c - dd * Hq;
            const bool keep = u < H && drop_keep_h0(h0, base + dd * H + u, dr.thr);
            if constexpr (sizeof(V) == 2) e[k] = keep ? __float2half_rn(__half2float(e[k]) * dr.scale) : __float2half_rn(0.f);
            else e[k] = keep ? e[k] * dr.scale : 0.f;
        }
        y4[q] = pk;
    }
}
static int lg2(int v) {
    int k = 0;
    while ((1 << k) < v) ++k;
    return (1 << k) == v ? k : -1;
}
int dropout_f16(__half *y, long rows, int H, int Hq, int site, const Dropout &dr, cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    const int lg = lg2(2 * Hq / 8);
    if (lg < 0) return -1;  // Hq is a power of two (rec_supported)
    dropout_kernel<__half><<<grid_for(rows << lg, 256, 148 * 8), 256, 0, st>>>(y, rows, H, Hq, site, dr, lg);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}
int dropout_f32(float *y, long rows, int H, int Hq, int site, const Dropout &dr, cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    const int lg = lg2(2 * Hq / 4);
    if (lg < 0) return -1;
    dropout_kernel<float><<<grid_for(rows << lg, 256, 148 * 8), 256, 0, st>>>(y, rows, H, Hq, site, dr, lg);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

// internal input row r of layer input -> source row of W (or -1 for padding)
DEVI int src_row(int r, int Drows, int H, int Hq, int rowmode) {
    if (rowmode == 0) return r < Drows ? r : -1;
    const int half = r / Hq, jj = r - half * Hq;
    return (half < 2 && jj < H) ? half * H + jj : -1;
}

// --- W_d [Drows, 4H] -> W16 [Dn, ndir*4Hq] with column 4j+gamma (+ d*4Hq) ------------------
// one thread per (row, direction, unit j): the four gate reads are each coalesced across the warp
// (consecutive j), the four fp16 results one 8-byte store
// split_w (BLSTM_PREC_FP16X2W, R9): four fp32 gate values -> fp16 hi (round to nearest) and
// lo = fp16(v - hi), so hi + lo carries ~22 bits of v
DEVI void store_w4(__half *out, const float v[4], __half *out_lo) {
    __half2 a = __floats2half2_rn(v[0], v[1]), b = __floats2half2_rn(v[2], v[3]);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t *>(&a);
    pk.y = *reinterpret_cast<uint32_t *>(&b);
    *reinterpret_cast<uint2 *>(out) = pk;
    if (out_lo) {
        const float2 fa = __half22float2(a), fb = __half22float2(b);
        __half2 la = __floats2half2_rn(v[0] - fa.x, v[1] - fa.y), lb = __floats2half2_rn(v[2] - fb.x, v[3] - fb.y);
        pk.x = *reinterpret_cast<uint32_t *>(&la);
        pk.y = *reinterpret_cast<uint32_t *>(&lb);
        *reinterpret_cast<uint2 *>(out_lo) = pk;
    }
}

__global__ void pack_w_kernel(const float *__restrict__ W0, const float *__restrict__ W1, int Drows, int H, int Hq,
                              int ndir, int Dn, int rowmode, __half *__restrict__ W16, int lo_rows) {
    const int r = blockIdx.y, d = blockIdx.z;
    const int sr = src_row(r, Drows, H, Hq, rowmode);
    const float *W = d == 0 ? W0 : W1;
    __half *out = W16 + (long)r * ndir * 4 * Hq + (long)d * 4 * Hq;
    __half *out_lo = lo_rows ? out + (long)lo_rows * ndir * 4 * Hq : nullptr;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < Hq; j += gridDim.x * blockDim.x) {
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (sr >= 0 && j < H) {
#pragma unroll
            for (int gam = 0; gam < 4; ++gam) v[gam] = W[(long)sr * 4 * H + gam * H + j];
        }
        store_w4(out + 4 * j, v, out_lo ? out_lo + 4 * j : nullptr);
    }
}
int pack_w(const float *W0, const float *W1, int Drows, int H, int Hq, int ndir, int Dn, int rowmode, __half *W16,
           cudaStream_t st, int lo_rows) {
    ProfScope ps_(PROF_OTHER, st);
    dim3 grid((Hq + 255) / 256, Dn, ndir);
    pack_w_kernel<<<grid, 256, 0, st>>>(W0, W1, Drows, H, Hq, ndir, Dn, rowmode, W16, lo_rows);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

// --- R_d [H, 4H] -> RT16 [ndir][4Hq][Hq]: row 4j+gamma, col k --------------------------------
// a transpose: 32 k x 32 j tiles through shared memory, reads coalesced along j (R's rows) and
// writes coalesced along k (RT16's rows)
__global__ void __launch_bounds__(256) pack_rt_kernel(const float *__restrict__ R0, const float *__restrict__ R1, int H,
                                                      int Hq, int ndir, __half *__restrict__ RT16) {
    __shared__ float tile[4][32][33];
    const int k0 = blockIdx.x * 32, j0 = blockIdx.y * 32, d = blockIdx.z;
    const float *R = d == 0 ? R0 : R1;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int kk = ty; kk < 32; kk += 8) {
        const int k = k0 + kk, j = j0 + tx;
#pragma unroll
        for (int gam = 0; gam < 4; ++gam)
            tile[gam][kk][tx] = (k < H && j < H) ? R[(long)k * 4 * H + gam * H + j] : 0.f;
    }
    __syncthreads();
    // output rows 4j + gam for j in the tile (128 rows), 32 k each
    for (int rr = ty; rr < 128; rr += 8) {
        const int jj = rr >> 2, gam = rr & 3;
        RT16[((long)d * 4 * Hq + 4 * (j0 + jj) + gam) * Hq + k0 + tx] = __float2half_rn(tile[gam][tx][jj]);
    }
}
int pack_rt(const float *R0, const float *R1, int H, int Hq, int ndir, __half *RT16, cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    dim3 grid(Hq / 32, Hq / 32, ndir);
    pack_rt_kernel<<<grid, 256, 0, st>>>(R0, R1, H, Hq, ndir, RT16);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

__global__ void pack_bias_kernel(const float *__restrict__ b0, const float *__restrict__ b1, int H, int Hq, int ndir,
                                 float *__restrict__ bq) {
    const int n = ndir * 4 * Hq;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int d = i / (4 * Hq), qq = i - d * 4 * Hq, j = qq >> 2, gam = qq & 3;
        const float *b = d == 0 ? b0 : b1;
        bq[i] = j < H ? b[gam * H + j] : 0.f;
    }
}
int pack_bias(const float *b0, const float *b1, int H, int Hq, int ndir, float *bq, cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    pack_bias_kernel<<<grid_for(ndir * 4 * Hq), 256, 0, st>>>(b0, b1, H, Hq, ndir, bq);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

// --- every layer's pack_w / pack_rt / pack_bias in one launch each (the step's preamble was
// 3L launch-bound kernels of a few us each) ------------------------------------------------------
__global__ void pack_w_all_kernel(PackLayers a) {
    const int r = blockIdx.y, l = blockIdx.z >> 1, d = blockIdx.z & 1;
    if (r >= a.Dn[l]) return;
    const int H = a.H, Hq = a.Hq;
    const int sr = src_row(r, a.Drows[l], H, Hq, a.rowmode[l]);
    const float *W = a.W[l][d];
    __half *out = a.W16[l] + (long)r * 2 * 4 * Hq + (long)d * 4 * Hq;
    __half *out_lo = a.lo_rows[l] ? out + (long)a.lo_rows[l] * 2 * 4 * Hq : nullptr;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < Hq; j += gridDim.x * blockDim.x) {
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (sr >= 0 && j < H) {
#pragma unroll
            for (int gam = 0; gam < 4; ++gam) v[gam] = W[(long)sr * 4 * H + gam * H + j];
        }
        store_w4(out + 4 * j, v, out_lo ? out_lo + 4 * j : nullptr);
    }
}
__global__ void __launch_bounds__(256) pack_rt_all_kernel(PackLayers a) {
    __shared__ float tile[4][32][33];
    const int H = a.H, Hq = a.Hq;
    const int k0 = blockIdx.x * 32, j0 = blockIdx.y * 32, l = blockIdx.z >> 1, d = blockIdx.z & 1;
    const float *R = a.R[l][d];
    __half *RT16 = a.RT16[l];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int kk = ty; kk < 32; kk += 8) {
        const int k = k0 + kk, j = j0 + tx;
#pragma unroll
        for (int gam = 0; gam < 4; ++gam)
            tile[gam][kk][tx] = (k < H && j < H) ? R[(long)k * 4 * H + gam * H + j] : 0.f;
    }
    __syncthreads();
    for (int rr = ty; rr < 128; rr += 8) {
        const int jj = rr >> 2, gam = rr & 3;
        RT16[((long)d * 4 * Hq + 4 * (j0 + jj) + gam) * Hq + k0 + tx] = __float2half_rn(tile[gam][tx][jj]);
    }
}
__global__ void pack_bias_all_kernel(PackLayers a) {
    const int Hq = a.Hq, H = a.H, per = 2 * 4 * Hq;
    const long n = (long)a.L * per;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) {
        const int l = (int)(e / per), i = (int)(e - (long)l * per);
        const int d = i / (4 * Hq), qq = i - d * 4 * Hq, j = qq >> 2, gam = qq & 3;
        a.bq[l][i] = j < H ? a.b[l][d][gam * H + j] : 0.f;
    }
}
int pack_layers(const PackLayers &a, cudaStream_t st) {
    if (a.L < 1 || a.L > PACK_MAXL) return -3;
    ProfScope ps_(PROF_OTHER, st);
    int maxDn = 0;
    for (int l = 0; l < a.L; ++l) maxDn = a.Dn[l] > maxDn ? a.Dn[l] : maxDn;
    pack_w_all_kernel<<<dim3((a.Hq + 255) / 256, maxDn, 2 * a.L), 256, 0, st>>>(a);
    pack_rt_all_kernel<<<dim3(a.Hq / 32, a.Hq / 32, 2 * a.L), 256, 0, st>>>(a);
    pack_bias_all_kernel<<<grid_for((long)a.L * 8 * a.Hq), 256, 0, st>>>(a);
    note_launch(3);
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

// --- head weights: W_out [2H, K] -> Wo16 [2Hq, Kp] (rows = padded [fwd | bwd] halves) --------
__global__ void pack_wout_kernel(const float *__restrict__ Wo, const float *__restrict__ bo, int H, int Hq, int K,
                                 int Kp, __half *__restrict__ Wo16, float *__restrict__ boq) {
    const long n = (long)2 * Hq * Kp;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const int r = (int)(i / Kp), k = (int)(i - (long)r * Kp);
        const int sr = src_row(r, 2 * H, H, Hq, 1);
        Wo16[i] = __float2half_rn((sr >= 0 && k < K) ? Wo[(long)sr * K + k] : 0.f);
        if (r == 0) boq[k] = k < K ? bo[k] : 0.f;
    }
}
int pack_wout(const float *Wo, const float *bo, int H, int Hq, int K, int Kp, __half *Wo16, float *boq,
              cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    pack_wout_kernel<<<grid_for((long)2 * Hq * Kp), 256, 0, st>>>(Wo, bo, H, Hq, K, Kp, Wo16, boq);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

// --- initial history slot (h0 or 0) for each direction -------------------------------------
__global__ void init_hist_kernel(__half *__restrict__ hist, const float *__restrict__ h0, int T, int B, int H,
                                 int Hq, int ndir, int dir0) {
    const long n = (long)ndir * B * Hq;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const int d = (int)(i / ((long)B * Hq));
        const long rem = i - (long)d * B * Hq;
        const int b = (int)(rem / Hq), j = (int)(rem - (long)b * Hq);
        const int dir = d == 0 ? dir0 : -1;
        const int slot = dir > 0 ? 0 : T;
        const float v = (h0 && j < H) ? h0[(long)d * B * H + (long)b * H + j] : 0.f;
        hist[(((long)d * (T + 1) + slot) * B + b) * Hq + j] = __float2half_rn(v);
    }
}
int init_hist(__half *hist, const float *h0, int T, int B, int H, int Hq, int ndir, int dir0, cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    init_hist_kernel<<<grid_for((long)ndir * B * Hq), 256, 0, st>>>(hist, h0, T, B, H, Hq, ndir, dir0);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

// --- softmax cross-entropy over one frame per CTA ------------------------------------------
// logits [rows, ldl] fp32 (K valid columns); writes dlog16 [rows, Kp] = 2^shift (softmax - onehot)
// at valid frames (0 elsewhere), rowloss (double) and rowerr (argmax != label, lowest index on ties).
constexpr int CE_THREADS = 256;  // 8 warps, one frame (row) per warp
// one warp per frame: coalesced 128-byte reads of the logits row (re-reads hit L1), warp-shuffle
// max / argmax (ties: lowest index) and sum, 16-byte fp16 stores of dlogits.  Per row:
//   loss = lse - logit[label],  err = argmax != label,  dlog = (softmax - onehot) * scale
template <int CE_CHUNKS>
__global__ void __launch_bounds__(CE_THREADS) ce_head_kernel(const float *__restrict__ logits, long ldl, int K, int Kp,
                                                             const uint8_t *__restrict__ mask,
                                                             const int32_t *__restrict__ labels, float scale,
                                                             __half *__restrict__ dlog16, double *__restrict__ rowloss,
                                                             int32_t *__restrict__ rowerr, long rows) {
    const long r = (long)blockIdx.x * (CE_THREADS / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    __half *drow = dlog16 + r * Kp;
    if (!mask[r]) {
        for (int k = lane * 8; k < Kp; k += 256) *reinterpret_cast<uint4 *>(drow + k) = make_uint4(0, 0, 0, 0);
        if (lane == 0) { rowloss[r] = 0.0; rowerr[r] = 0; }
        return;
    }
    // the row is read once into registers: lane owns columns [256c + 8 lane, +8) of chunk c
    // (float4 loads; every warp access is 1 KB contiguous), exp is evaluated once per logit
    const float *lrow = logits + r * ldl;
    float v[CE_CHUNKS][8];
    float mv = -INFINITY;
    int mi = 0x7fffffff;
#pragma unroll
    for (int c = 0; c < CE_CHUNKS; ++c) {
        const int k0 = 256 * c + 8 * lane;
        if (k0 < Kp) {
            const float4 a = *reinterpret_cast<const float4 *>(lrow + k0);
            const float4 b = *reinterpret_cast<const float4 *>(lrow + k0 + 4);
            v[c][0] = a.x; v[c][1] = a.y; v[c][2] = a.z; v[c][3] = a.w;
            v[c][4] = b.x; v[c][5] = b.y; v[c][6] = b.z; v[c][7] = b.w;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (k0 + u >= K) v[c][u] = -INFINITY;
            if (v[c][u] > mv) { mv = v[c][u]; mi = k0 + u; }  // ascending k per lane: first max = lowest index
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, mv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, mi, o);
        if (ov > mv || (ov == mv && oi < mi)) { mv = ov; mi = oi; }
    }
    float se = 0.f;
#pragma unroll
    for (int c = 0; c < CE_CHUNKS; ++c)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            v[c][u] = __expf(v[c][u] - mv);  // exp(-inf) = 0 past K
            se += v[c][u];
        }
    for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    const float lse = mv + __logf(se), inv = 1.f / se;
    const int lab = labels[r];
#pragma unroll
    for (int c = 0; c < CE_CHUNKS; ++c) {
        const int k0 = 256 * c + 8 * lane;
        if (k0 >= Kp) continue;
        uint32_t hv[4];
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
            const bool l0 = k0 + u == lab, l1 = k0 + u + 1 == lab;
            const float p0 = v[c][u] * inv - (l0 ? 1.f : 0.f), p1 = v[c][u + 1] * inv - (l1 ? 1.f : 0.f);
            __half2 h2 = __floats2half2_rn(p0 * scale, p1 * scale);
            hv[u / 2] = *reinterpret_cast<uint32_t *>(&h2);
        }
        *reinterpret_cast<uint4 *>(drow + k0) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
    }
    if (lane == 0) {
        rowloss[r] = (double)lse - (double)lrow[lab];
        rowerr[r] = mi != lab;
    }
}
// generic width (Kp > 2048): three passes over the row
__global__ void __launch_bounds__(CE_THREADS) ce_head_any_kernel(const float *__restrict__ logits, long ldl, int K, int Kp,
                                                             const uint8_t *__restrict__ mask,
                                                             const int32_t *__restrict__ labels, float scale,
                                                             __half *__restrict__ dlog16, double *__restrict__ rowloss,
                                                             int32_t *__restrict__ rowerr, long rows) {
    const long r = (long)blockIdx.x * (CE_THREADS / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    __half *drow = dlog16 + r * Kp;
    if (!mask[r]) {
        for (int k = lane * 8; k < Kp; k += 256) *reinterpret_cast<uint4 *>(drow + k) = make_uint4(0, 0, 0, 0);
        if (lane == 0) { rowloss[r] = 0.0; rowerr[r] = 0; }
        return;
    }
    const float *lrow = logits + r * ldl;
    float mv = -INFINITY;
    int mi = 0x7fffffff;
    for (int k = lane; k < K; k += 32) {
        const float v = lrow[k];
        if (v > mv) { mv = v; mi = k; }  // k ascends per lane: the first max is the lowest index
    }
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, mv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, mi, o);
        if (ov > mv || (ov == mv && oi < mi)) { mv = ov; mi = oi; }
    }
    float se = 0.f;
    for (int k = lane; k < K; k += 32) se += expf(lrow[k] - mv);
    for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    const float lse = mv + logf(se);
    const int lab = labels[r];
    for (int k0 = lane * 8; k0 < Kp; k0 += 256) {
        uint32_t hv[4];
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
            float v0 = 0.f, v1 = 0.f;
            if (k0 + u < K) v0 = expf(lrow[k0 + u] - lse) - (k0 + u == lab ? 1.f : 0.f);
            if (k0 + u + 1 < K) v1 = expf(lrow[k0 + u + 1] - lse) - (k0 + u + 1 == lab ? 1.f : 0.f);
            __half2 h2 = __floats2half2_rn(v0 * scale, v1 * scale);
            hv[u / 2] = *reinterpret_cast<uint32_t *>(&h2);
        }
        *reinterpret_cast<uint4 *>(drow + k0) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
    }
    if (lane == 0) {
        rowloss[r] = (double)lse - (double)lrow[lab];
        rowerr[r] = mi != lab;
    }
}
int ce_head(const float *logits, long ldl, int K, int Kp, const uint8_t *mask, const int32_t *labels, float scale,
            __half *dlog16, double *rowloss, int32_t *rowerr, long rows, cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    if (rows <= 0) return 0;
    const long blocks = (rows + CE_THREADS / 32 - 1) / (CE_THREADS / 32);
    const int ch = (Kp + 255) / 256;
#define CE_CASE(C)                                                                                             \
    if (ch <= C)                                                                                               \
        ce_head_kernel<C><<<(unsigned)blocks, CE_THREADS, 0, st>>>(logits, ldl, K, Kp, mask, labels, scale, dlog16, \
                                                                   rowloss, rowerr, rows);                     \
    else
    CE_CASE(1) CE_CASE(2) CE_CASE(4) CE_CASE(8)
    ce_head_any_kernel<<<(unsigned)blocks, CE_THREADS, 0, st>>>(logits, ldl, K, Kp, mask, labels, scale, dlog16,
                                                                rowloss, rowerr, rows);
#undef CE_CASE
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

// --- deterministic loss / error reduction (one CTA, fixed order) ---------------------------
__global__ void __launch_bounds__(1024) reduce_loss_kernel(const double *__restrict__ rowloss,
                                                           const int32_t *__restrict__ rowerr, long rows,
                                                           double *__restrict__ loss, int32_t *__restrict__ ferr) {
    __shared__ double sl[1024];
    __shared__ long se[1024];
    double a = 0.0;
    long e = 0;
    for (long r = threadIdx.x; r < rows; r += 1024) { a += rowloss[r]; e += rowerr[r]; }
    sl[threadIdx.x] = a;
    se[threadIdx.x] = e;
    __syncthreads();
    for (int s = 512; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) { sl[threadIdx.x] += sl[threadIdx.x + s]; se[threadIdx.x] += se[threadIdx.x + s]; }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *loss = sl[0];
        if (ferr) *ferr = (int32_t)se[0];
    }
}
int reduce_loss(const double *rowloss, const int32_t *rowerr, long rows, double *loss, int32_t *ferr,
                cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    reduce_loss_kernel<<<1, 1024, 0, st>>>(rowloss, rowerr, rows, loss, ferr);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

// --- column sums of an fp16 matrix, two deterministic passes: out[k] += alpha * sum_r src[r,k] ----
constexpr int CS_ROWS = 256;
__global__ void colsum_pass1(const __half *__restrict__ src, long rows, int cols, long ld, float *__restrict__ part) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const long r0 = (long)blockIdx.y * CS_ROWS;
    if (k >= cols) return;
    float a = 0.f;
    const long r1 = r0 + CS_ROWS < rows ? r0 + CS_ROWS : rows;
    for (long r = r0; r < r1; ++r) a += __half2float(src[r * ld + k]);
    part[(long)blockIdx.y * cols + k] = a;
}
__global__ void colsum_pass2(const float *__restrict__ part, int nchunks, int cols, float alpha,
                             float *__restrict__ out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= cols) return;
    float a = 0.f;
    for (int c = 0; c < nchunks; ++c) a += part[(long)c * cols + k];
    out[k] += alpha * a;
}
size_t colsum_scratch_bytes(long rows, int cols) { return (size_t)((rows + CS_ROWS - 1) / CS_ROWS) * cols * 4; }
int colsum_f16_add(const __half *src, long rows, int cols, long ld, float alpha, float *out, float *scratch,
                   cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    const int nch = (int)((rows + CS_ROWS - 1) / CS_ROWS);
    if (nch == 0) return 0;
    dim3 g1((cols + 127) / 128, nch);
    colsum_pass1<<<g1, 128, 0, st>>>(src, rows, cols, ld, scratch);
    colsum_pass2<<<(cols + 127) / 128, 128, 0, st>>>(scratch, nch, cols, alpha, out);
    note_launch(2);
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

// --- gradient scatter-add from kernel-private layouts to the flat theta layout ---------------
// gW [Drows, 4H] += dWT[(d*4Hq + 4j+gamma) * ldw + r(src_row)]
__global__ void scatter_w_kernel(float *__restrict__ gW, int Drows, int H, int Hq, const float *__restrict__ dWT,
                                 long ldw, int d, int rowmode) {
    const long n = (long)Drows * 4 * H;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const int sr = (int)(i / (4 * H)), col = (int)(i - (long)sr * 4 * H);
        const int gam = col / H, j = col - gam * H;
        const int r = rowmode == 0 ? sr : (sr / H) * Hq + (sr % H);
        gW[i] += dWT[((long)d * 4 * Hq + 4 * j + gam) * ldw + r];
    }
}
int scatter_w(float *gW, int Drows, int H, int Hq, const float *dWT, long ldw, int d, int rowmode, cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    scatter_w_kernel<<<grid_for((long)Drows * 4 * H), 256, 0, st>>>(gW, Drows, H, Hq, dWT, ldw, d, rowmode);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}
// gR [H, 4H] += dRT[(4j+gamma) * Hq + k]
__global__ void scatter_r_kernel(float *__restrict__ gR, int H, int Hq, const float *__restrict__ dRT) {
    const long n = (long)H * 4 * H;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const int k = (int)(i / (4 * H)), col = (int)(i - (long)k * 4 * H);
        const int gam = col / H, j = col - gam * H;
        gR[i] += dRT[(long)(4 * j + gam) * Hq + k];
    }
}
int scatter_r(float *gR, int H, int Hq, const float *dRT, cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    scatter_r_kernel<<<grid_for((long)H * 4 * H), 256, 0, st>>>(gR, H, Hq, dRT);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}
// gb [4H] += sum_g dbpart[(d*G + g)*4Hq + 4j+gamma]
__global__ void scatter_b_kernel(float *__restrict__ gb, int H, int Hq, const float *__restrict__ dbpart, int G,
                                 int d) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 4 * H; i += gridDim.x * blockDim.x) {
        const int gam = i / H, j = i - gam * H;
        float a = 0.f;
        for (int g = 0; g < G; ++g) a += dbpart[((long)d * G + g) * 4 * Hq + 4 * j + gam];
        gb[i] += a;
    }
}
int scatter_b(float *gb, int H, int Hq, const float *dbpart, int G, int d, cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    scatter_b_kernel<<<grid_for(4 * H), 256, 0, st>>>(gb, H, Hq, dbpart, G, d);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}
// gWo [2H, K] += dWoT[k * ldw + r(src)]
__global__ void scatter_wout_kernel(float *__restrict__ gWo, int H, int Hq, int K, const float *__restrict__ dWoT,
                                    long ldw) {
    const long n = (long)2 * H * K;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const int sr = (int)(i / K), k = (int)(i - (long)sr * K);
        const int r = (sr / H) * Hq + (sr % H);
        gWo[i] += dWoT[(long)k * ldw + r];
    }
}
int scatter_wout(float *gWo, int H, int Hq, int K, const float *dWoT, long ldw, cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    scatter_wout_kernel<<<grid_for((long)2 * H * K), 256, 0, st>>>(gWo, H, Hq, K, dWoT, ldw);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

// --- dy_top [rows, 2H] -> dY [rows, 2Hq] (padded halves) ------------------------------------
// --- mask validation (blstm.h: an entry outside {0,1} -> BLSTM_ERR_ARG, read back lazily) ------
// One flag per process in mapped pinned host memory: kernels that read the caller's mask OR 1 into
// it on a bad byte; the host reads it at the next API call (mask_flag_take), after the kernel ran.
static unsigned *g_mask_flag = nullptr;
unsigned *mask_flag() {
    if (!g_mask_flag) {
        void *p = nullptr;
        if (cudaHostAlloc(&p, 16, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) return nullptr;
        *(volatile unsigned *)p = 0;
        g_mask_flag = (unsigned *)p;
    }
    return g_mask_flag;
}
// --- the stack step's preamble in one launch (ops.h StackPrep) -----------------------------
// Each job is the body of its single-purpose kernel above with (blockIdx, gridDim) replaced by the
// job-local block index and block count.
__global__ void __launch_bounds__(256) stack_prep_kernel(StackPrep p) {
    __shared__ float tile[4][32][33];  // pack_rt's transpose tile
    int b = blockIdx.x;
    const long t = threadIdx.x, nt = blockDim.x;
    if (b < p.nb[0]) {  // cast_x_kernel
        const long n = p.rows * p.Dp, stride = (long)p.nb[0] * nt;
        for (long i = b * nt + t; i < n; i += stride) {
            const long r = i / p.Dp;
            const int k = (int)(i - r * p.Dp);
            float v = k < p.D ? p.x[r * p.ldx + k] : 0.f;
            if (p.dr.on && k < p.D) v = drop_keep(p.dr.seed, 0, (unsigned long long)r * p.D + k, p.dr.thr) ? v * p.dr.scale : 0.f;
            p.x16[i] = __float2half_rn(v);
        }
        return;
    }
    b -= p.nb[0];
    const PackLayers &a = p.pk;
    if (b < p.nb[1]) {  // pack_w_all_kernel: block (bx, r, z) of grid (ceil(Hq/256), maxDn, 2L)
        const int gx = (a.Hq + 255) / 256;
        const int bx = b % gx, r = (b / gx) % p.maxDn, z = b / (gx * p.maxDn);
        const int l = z >> 1, d = z & 1;
        if (r >= a.Dn[l]) return;
        const int H = a.H, Hq = a.Hq;
        const int sr = src_row(r, a.Drows[l], H, Hq, a.rowmode[l]);
        const float *W = a.W[l][d];
        __half *out = a.W16[l] + (long)r * 2 * 4 * Hq + (long)d * 4 * Hq;
        __half *out_lo = a.lo_rows[l] ? out + (long)a.lo_rows[l] * 2 * 4 * Hq : nullptr;
        for (int j = bx * (int)nt + (int)t; j < Hq; j += gx * (int)nt) {
            float v[4] = {0.f, 0.f, 0.f, 0.f};
            if (sr >= 0 && j < H) {
#pragma unroll
                for (int gam = 0; gam < 4; ++gam) v[gam] = W[(long)sr * 4 * H + gam * H + j];
            }
            store_w4(out + 4 * j, v, out_lo ? out_lo + 4 * j : nullptr);
        }
        return;
    }
    b -= p.nb[1];
    if (b < p.nb[2]) {  // pack_rt_all_kernel: block (bx, by, z) of grid (Hq/32, Hq/32, 2L)
        const int H = a.H, Hq = a.Hq, g32 = Hq / 32;
        const int bx = b % g32, by = (b / g32) % g32, z = b / (g32 * g32);
        const int k0 = bx * 32, j0 = by * 32, l = z >> 1, d = z & 1;
        const float *R = a.R[l][d];
        __half *RT16 = a.RT16[l];
        const int tx = (int)t & 31, ty = (int)t >> 5;
        for (int kk = ty; kk < 32; kk += 8) {
            const int k = k0 + kk, j = j0 + tx;
#pragma unroll
            for (int gam = 0; gam < 4; ++gam)
                tile[gam][kk][tx] = (k < H && j < H) ? R[(long)k * 4 * H + gam * H + j] : 0.f;
        }
        __syncthreads();
        for (int rr = ty; rr < 128; rr += 8) {
            const int jj = rr >> 2, gam = rr & 3;
            RT16[((long)d * 4 * Hq + 4 * (j0 + jj) + gam) * Hq + k0 + tx] = __float2half_rn(tile[gam][tx][jj]);
        }
        return;
    }
    b -= p.nb[2];
    if (b < p.nb[3]) {  // pack_bias_all_kernel
        const int Hq = a.Hq, H = a.H, per = 2 * 4 * Hq;
        const long n = (long)a.L * per, stride = (long)p.nb[3] * nt;
        for (long e = b * nt + t; e < n; e += stride) {
            const int l = (int)(e / per), i = (int)(e - (long)l * per);
            const int d = i / (4 * Hq), qq = i - d * 4 * Hq, j = qq >> 2, gam = qq & 3;
            a.bq[l][i] = j < H ? a.b[l][d][gam * H + j] : 0.f;
        }
        return;
    }
    b -= p.nb[3];
    if (b < p.nb[4]) {  // pack_mask_kernel (mode 1) / check_mask_kernel (mode 2)
        bool bad = false;
        const long stride = (long)p.nb[4] * nt;
        if (p.mask_mode == 1) {
            const long n = (long)p.T * p.G * p.N;
            for (long i = b * nt + t; i < n; i += stride) {
                const long tg = i / p.N;
                const int c = (int)(i - tg * p.N), g = (int)(tg % p.G);
                const long tt = tg / p.G;
                const int bb = g * p.Bg + c;
                const uint8_t v = (c < p.Bg && bb < p.B) ? p.mask[tt * p.B + bb] : 0;
                bad |= v > 1;
                p.maskN[i] = v;
            }
        } else {
            const long n = p.mask_n, n16 = n / 16;
            for (long i = b * nt + t; i < n16; i += stride) {
                const uint4 v = __ldg((const uint4 *)p.mask + i);
                bad |= ((v.x | v.y | v.z | v.w) & 0xFEFEFEFEu) != 0;
            }
            for (long i = n16 * 16 + b * nt + t; i < n; i += stride) bad |= p.mask[i] > 1;
        }
        if (bad && p.err) *(volatile unsigned *)p.err = 1u;
        return;
    }
    b -= p.nb[4];
    if (b < p.nb[5]) {  // zero words
        for (long i = b * nt + t; i < p.zero_n; i += (long)p.nb[5] * nt) p.zero[i] = 0u;
        return;
    }
    b -= p.nb[5];
    if (b < p.nb[6]) {  // the zero h0 history slots (init_hist_kernel without h0): block (bx, layer)
        const int per = p.nb[6] / p.hist_L, l = b / per, bx = b - l * per;
        __half *hist = p.hl.hist[l];
        const long n = 2L * p.hB * p.hHq;
        for (long i = bx * nt + t; i < n; i += (long)per * nt) {
            const int d = (int)(i / ((long)p.hB * p.hHq));
            const long rem = i - (long)d * p.hB * p.hHq;
            const int slot = d == 0 ? 0 : p.hT;
            hist[((long)d * (p.hT + 1) + slot) * p.hB * p.hHq + rem] = __float2half_rn(0.f);
        }
        return;
    }
    b -= p.nb[6];
    if (b < p.nb[7]) {  // pack_wout_kernel
        const int H = p.pk.H, Hq = p.pk.Hq;
        const long n = (long)2 * Hq * p.Kp;
        for (long i = b * nt + t; i < n; i += (long)p.nb[7] * nt) {
            const int r = (int)(i / p.Kp), k = (int)(i - (long)r * p.Kp);
            const int sr = src_row(r, 2 * H, H, Hq, 1);
            p.Wo16[i] = __float2half_rn((sr >= 0 && k < p.K) ? p.Wo[(long)sr * p.K + k] : 0.f);
            if (r == 0) p.boq[k] = k < p.K ? p.bo[k] : 0.f;
        }
    }
}
int stack_prep(StackPrep &p, cudaStream_t st) {
    auto cap = [](long work, long lim) { long g = (work + 255) / 256; return (int)(g < 1 ? 1 : (g > lim ? lim : g)); };
    p.err = mask_flag();
    p.nb[0] = p.rows * p.Dp > 0 ? cap(p.rows * p.Dp, 148 * 4) : 0;
    p.maxDn = 0;
    for (int l = 0; l < p.pk.L; ++l) p.maxDn = p.pk.Dn[l] > p.maxDn ? p.pk.Dn[l] : p.maxDn;
    p.nb[1] = p.pk.L ? ((p.pk.Hq + 255) / 256) * p.maxDn * 2 * p.pk.L : 0;
    p.nb[2] = p.pk.L ? (p.pk.Hq / 32) * (p.pk.Hq / 32) * 2 * p.pk.L : 0;
    p.nb[3] = p.pk.L ? cap((long)p.pk.L * 8 * p.pk.Hq, 148 * 4) : 0;
    const long mwork = p.mask_mode == 1 ? (long)p.T * p.G * p.N : p.mask_mode == 2 ? (p.mask_n + 15) / 16 : 0;
    p.nb[4] = mwork > 0 ? cap(mwork, 148 * 4) : 0;
    p.nb[5] = p.zero_n > 0 ? cap(p.zero_n, 148) : 0;
    p.nb[6] = p.hist_L > 0 ? p.hist_L * cap(2L * p.hB * p.hHq, 64) : 0;
    p.nb[7] = p.Wo16 ? cap((long)2 * p.pk.Hq * p.Kp, 148 * 2) : 0;
    long total = 0;
    for (int i = 0; i < 8; ++i) total += p.nb[i];
    if (total == 0) return 0;
    if (total > 0x7fffffffL || p.hist_L > PACK_MAXL || p.pk.L > PACK_MAXL) return -3;
    ProfScope ps_(PROF_OTHER, st);
    stack_prep_kernel<<<(unsigned)total, 256, 0, st>>>(p);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

int mask_flag_take() {
    if (!g_mask_flag || *(volatile unsigned *)g_mask_flag == 0) return 0;
    *(volatile unsigned *)g_mask_flag = 0;
    return 1;
}

__global__ void pack_mask_kernel(const uint8_t *__restrict__ mask, int T, int B, int G, int Bg, int N,
                                 uint8_t *__restrict__ maskN, unsigned *err) {
    const long n = (long)T * G * N;
    bool bad = false;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const long tg = i / N;
        const int c = (int)(i - tg * N), g = (int)(tg % G);
        const long t = tg / G;
        const int b = g * Bg + c;
        const uint8_t v = (c < Bg && b < B) ? mask[t * B + b] : 0;
        bad |= v > 1;
        maskN[i] = v;
    }
    if (bad && err) *(volatile unsigned *)err = 1u;
}
int pack_mask(const uint8_t *mask, int T, int B, int G, int Bg, int N, uint8_t *maskN, cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    if (T == 0) return 0;
    pack_mask_kernel<<<grid_for((long)T * G * N), 256, 0, st>>>(mask, T, B, G, Bg, N, maskN, mask_flag());
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

__global__ void check_mask_kernel(const uint8_t *__restrict__ mask, long n, unsigned *err) {
    bool bad = false;
    const long n16 = n / 16;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n16; i += (long)gridDim.x * blockDim.x) {
        const uint4 v = __ldg((const uint4 *)mask + i);
        bad |= ((v.x | v.y | v.z | v.w) & 0xFEFEFEFEu) != 0;
    }
    for (long i = n16 * 16 + blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        bad |= mask[i] > 1;
    if (bad && err) *(volatile unsigned *)err = 1u;
}
int check_mask(const uint8_t *mask, long n, cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    if (n <= 0) return 0;
    const long work = (n + 15) / 16;
    check_mask_kernel<<<(unsigned)std::min<long>((work + 255) / 256, 148 * 4), 256, 0, st>>>(mask, n, mask_flag());
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

__global__ void copy_rows_kernel(const float *__restrict__ src, long lds, long rows, int cols,
                                 float *__restrict__ dst, long ldd) {
    const long n = rows * cols;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const long r = i / cols;
        const int j = (int)(i - r * cols);
        dst[r * ldd + j] = src[r * lds + j];
    }
}
int copy_rows(const float *src, long lds, long rows, int cols, float *dst, long ldd, cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    if (rows * cols == 0) return 0;
    copy_rows_kernel<<<grid_for(rows * cols), 256, 0, st>>>(src, lds, rows, cols, dst, ldd);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

__global__ void pad_halves_kernel(const float *__restrict__ src, int H, int Hq, long rows, float *__restrict__ dst) {
    const long n = rows * 2 * Hq;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const long r = i / (2 * Hq);
        const int c = (int)(i - r * 2 * Hq), half = c / Hq, j = c - half * Hq;
        dst[i] = j < H ? src[r * 2 * H + half * H + j] : 0.f;
    }
}
int pad_halves(const float *src, int H, int Hq, long rows, float *dst, cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    pad_halves_kernel<<<grid_for(rows * 2 * Hq), 256, 0, st>>>(src, H, Hq, rows, dst);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

// --- dx [rows, ldx] (=|+=) dX [rows, ldX] for k < D ------------------------------------------
__global__ void store_dx_kernel(float *__restrict__ dx, long ldx, const float *__restrict__ dX, long ldX, int D,
                                long rows, int accum) {
    const long n = rows * D;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const long r = i / D;
        const int k = (int)(i - r * D);
        const float v = dX[r * ldX + k];
        if (accum) dx[r * ldx + k] += v;
        else dx[r * ldx + k] = v;
    }
}
int store_dx(float *dx, long ldx, const float *dX, long ldX, int D, long rows, int accum, cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    store_dx_kernel<<<grid_for(rows * D), 256, 0, st>>>(dx, ldx, dX, ldX, D, rows, accum);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

// --- chunk gather (NEXT-4): batch tensors from a device-resident corpus -----------------------
// one warp per batch row (t, b): lanes copy the row's D features (float4 when D % 4 == 0);
// x = 0, mask = 0, label = 0 past the chunk's valid length
__global__ void gather_chunks_kernel(const float *__restrict__ frames, const int32_t *__restrict__ flab, int D,
                                     const int64_t *__restrict__ cstart, const int32_t *__restrict__ clen, int B,
                                     int T, float *__restrict__ x, uint8_t *__restrict__ mask,
                                     int32_t *__restrict__ labels) {
    const int lane = threadIdx.x & 31;
    const long rows = (long)T * B;
    const long nw = (long)gridDim.x * (blockDim.x >> 5);
    for (long tb = blockIdx.x * (long)(blockDim.x >> 5) + (threadIdx.x >> 5); tb < rows; tb += nw) {
        const int t = (int)(tb / B), b = (int)(tb - (long)t * B);
        const bool ok = t < clen[b];
        const long f = cstart[b] + t;
        float *xo = x + tb * D;
        if ((D & 3) == 0) {
            const float4 *src = reinterpret_cast<const float4 *>(frames + f * D);
            float4 *dst = reinterpret_cast<float4 *>(xo);
            for (int k = lane; k < D / 4; k += 32) dst[k] = ok ? src[k] : make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
            for (int k = lane; k < D; k += 32) xo[k] = ok ? frames[f * D + k] : 0.f;
        }
        if (lane == 0) {
            mask[tb] = ok ? 1 : 0;
            if (labels) labels[tb] = (ok && flab) ? flab[f] : 0;
        }
    }
}
int gather_chunks(const float *frames, const int32_t *flab, int D, const int64_t *cstart, const int32_t *clen, int B,
                  int T, float *x, uint8_t *mask, int32_t *labels, cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    gather_chunks_kernel<<<grid_for((long)T * B * 32, 256, 148 * 8), 256, 0, st>>>(frames, flab, D, cstart, clen, B, T,
                                                                                  x, mask, labels);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

// --- placement guard: hold a stream until *flag >= target (or timeout_ns passed) -------------
__global__ void wait_count_kernel(const uint32_t *flag, uint32_t target, unsigned long long timeout_ns) {
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_gpu(flag) < target) {
        if (globaltimer_ns() - t0 > timeout_ns) break;  // never a deadlock: only placement is at stake
        __nanosleep(200);
    }
}
int wait_count(const uint32_t *flag, uint32_t target, cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    wait_count_kernel<<<1, 32, 0, st>>>(flag, target, 2000000ull);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

// --- SGD (§4.3): theta -= lr * grad; optional grad = 0 ------------------------------
__global__ void sgd_kernel(float *__restrict__ th, float *__restrict__ gr, long n, float lr, int zero) {
    const long n4 = n >> 2;
    float4 *t4 = reinterpret_cast<float4 *>(th);
    float4 *g4 = reinterpret_cast<float4 *>(gr);
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
        float4 t = t4[i];
        const float4 g = g4[i];
        t.x -= lr * g.x; t.y -= lr * g.y; t.z -= lr * g.z; t.w -= lr * g.w;
        t4[i] = t;
        if (zero) g4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (long i = (n4 << 2) + blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        th[i] -= lr * gr[i];
        if (zero) gr[i] = 0.f;
    }
}
int sgd(float *theta, float *grad, long n, float lr, int zero, cudaStream_t st) {
    ProfScope ps_(PROF_OTHER, st);
    sgd_kernel<<<grid_for(n / 4 + 1, 256, 148 * 8), 256, 0, st>>>(theta, grad, n, lr, zero);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

}  // namespace blstm
