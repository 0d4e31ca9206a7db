// optim.cu -- the on-device update rules (§4.3).
//
// One step of a rule over the flat parameter vector theta[n] and its gradient grad[n]:
//   g_i = grad_i (+ 2*l2*theta_i on weight entries: the L2 penalty on weight matrices)
//   g  <- g * max_norm/||g||_2 if max_norm > 0 and ||g||_2 > max_norm  (norm constraint)
//   then the rule (R19 restates the formulas):
//     sgd       theta -= lr*g
//     momentum  v = mu*v - lr*g;  theta += v                       (classical momentum)
//     nesterov  v = mu*v - lr*g;  theta += mu*v - lr*g             (simplified Nesterov)
//     adagrad   a += g^2;  theta -= lr*g/(sqrt(a) + eps)
//     adadelta  Eg = rho*Eg + (1-rho)*g^2;  u = g*sqrt(Eu + eps)/sqrt(Eg + eps);
//               Eu = rho*Eu + (1-rho)*u^2;  theta -= lr*u
//     adam      m = b1*m + (1-b1)*g;  v = b2*v + (1-b2)*g^2;
//               theta -= lr*(m/(1-b1^t)) / (sqrt(v/(1-b2^t)) + eps)
//   and grad <- 0 when asked (the next step accumulates into it).
// Gradients are not scaled by the batch.
//
// Kernels: HBM-bound streams.  The update is one fused pass (float4 loads/stores of theta,
// grad and the rule's state, two per thread per 2048-element CTA tile, grid-stride over
// 8 CTAs per SM).  The norm needs the whole
// conditioned gradient first, so with max_norm > 0 a first pass writes one fp64 partial sum of
// squares per CTA of a fixed grid (fixed tree order inside the CTA); every CTA of the update
// pass sums those partials in the same fixed order, so the scale -- and the result -- is
// bitwise reproducible run to run.
#include "ops.h"
#include "optim.h"
#include "prof.h"

namespace blstm {

namespace {

constexpr int OPT_THREADS = 256;
constexpr int OPT_VEC = 2;                          // float4 per thread per tile
constexpr int TILE4 = OPT_THREADS * OPT_VEC;        // float4 per CTA tile (2048 elements)

// number of boundaries <= i in the sorted table: odd <=> i lies in a bias range
__device__ __forceinline__ int count_le(const OptBiasTable &tab, long i) {
    int pos = 0;
#pragma unroll
    for (int step = OPT_MAX_BOUNDS / 2; step > 0; step >>= 1)
        if (tab.bnd[pos + step - 1] <= i) pos += step;
    return pos;
}

// The L2 term's factor (2*l2 on weight entries, 0 on bias entries) over one CTA tile
// [e0, e1]: decided once per tile with block-uniform lookups (constant-cache broadcasts);
// only a tile that straddles a range boundary falls back to a per-element lookup.
struct L2Tile {
    float f;
    bool mixed;
};
__device__ __forceinline__ L2Tile l2_tile(const OptArgs &a, const OptBiasTable &tab, long e0, long e1) {
    L2Tile r{2.f * a.l2, false};
    if (a.l2 > 0.f && tab.nb > 0) {
        const int p0 = count_le(tab, e0), p1 = count_le(tab, e1);
        r.mixed = p0 != p1;
        if (p0 & 1) r.f = 0.f;
    }
    return r;
}
__device__ __forceinline__ float cond_grad(float g, float th, long i, const OptArgs &a, const OptBiasTable &tab,
                                           const L2Tile &lt) {
    if (a.l2 > 0.f) {
        const float f = lt.mixed ? ((count_le(tab, i) & 1) ? 0.f : 2.f * a.l2) : lt.f;
        g = fmaf(f, th, g);
    }
    return g;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// fixed-order CTA reduction of one double per thread; result valid in thread 0
__device__ double block_sum(double v) {
    __shared__ double red[OPT_THREADS / 32];
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < OPT_THREADS / 32; ++w) s += red[w];
    return s;
}

__device__ __forceinline__ float4 ld4(const float *p, long q) { return reinterpret_cast<const float4 *>(p)[q]; }
__device__ __forceinline__ void st4(float *p, long q, float4 v) { reinterpret_cast<float4 *>(p)[q] = v; }
__device__ __forceinline__ float &el(float4 &v, int k) { return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w; }

__global__ void __launch_bounds__(OPT_THREADS) opt_sumsq_kernel(const float *__restrict__ th,
                                                                const float *__restrict__ gr, long n, OptArgs a,
                                                                const __grid_constant__ OptBiasTable tab,
                                                                double *__restrict__ partial) {
    const long n4 = n >> 2;
    const long ntile = (n4 + TILE4 - 1) / TILE4;
    double acc = 0.0;
    for (long tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
        const long q0 = tile * TILE4 + threadIdx.x;
        const long e1 = ((tile + 1) * TILE4 < n4 ? (tile + 1) * TILE4 : n4) * 4 - 1;
        const L2Tile lt = l2_tile(a, tab, tile * TILE4 * 4, e1);
        float4 g[OPT_VEC], t[OPT_VEC];
#pragma unroll
        for (int k = 0; k < OPT_VEC; ++k) {
            const long q = q0 + k * OPT_THREADS;
            g[k] = q < n4 ? ld4(gr, q) : make_float4(0.f, 0.f, 0.f, 0.f);
            t[k] = (a.l2 > 0.f && q < n4) ? ld4(th, q) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < OPT_VEC; ++k) {
            const long i = (q0 + k * OPT_THREADS) * 4;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float x = cond_grad(el(g[k], j), el(t[k], j), i + j, a, tab, lt);
                acc = fma((double)x, (double)x, acc);
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {  // ragged tail (< 4 elements)
        const long i = (n4 << 2) + threadIdx.x;
        const float x = cond_grad(gr[i], th[i], i, a, tab, L2Tile{0.f, true});
        acc = fma((double)x, (double)x, acc);
    }
    const double s = block_sum(acc);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

template <int RULE>
__device__ __forceinline__ void rule_step(float &th, float g, float &s0, float &s1, const OptArgs &a) {
    if (RULE == OPT_SGD) {
        th -= a.lr * g;
    } else if (RULE == OPT_MOMENTUM) {
        const float v = a.mu * s0 - a.lr * g;
        s0 = v;
        th += v;
    } else if (RULE == OPT_NESTEROV) {
        const float v = a.mu * s0 - a.lr * g;
        s0 = v;
        th += a.mu * v - a.lr * g;
    } else if (RULE == OPT_ADAGRAD) {
        const float acc = s0 + g * g;
        s0 = acc;
        th -= __fdividef(a.lr * g, sqrtf(acc) + a.eps);
    } else if (RULE == OPT_ADADELTA) {
        const float eg = a.rho * s0 + a.rho1 * g * g;
        const float u = g * sqrtf(s1 + a.eps) * rsqrtf(eg + a.eps);
        s0 = eg;
        s1 = a.rho * s1 + a.rho1 * u * u;
        th -= a.lr * u;
    } else {  // OPT_ADAM
        const float m = a.b1 * s0 + a.b1c * g;
        const float v = a.b2 * s1 + a.b2c * g * g;
        s0 = m;
        s1 = v;
        th -= __fdividef(a.lr * (m * a.c1), sqrtf(v * a.c2) + a.eps);
    }
}

template <int RULE>
__global__ void __launch_bounds__(OPT_THREADS) opt_apply_kernel(float *__restrict__ th, float *__restrict__ gr,
                                                                float *__restrict__ s0, float *__restrict__ s1,
                                                                long n, OptArgs a,
                                                                const __grid_constant__ OptBiasTable tab,
                                                                const double *__restrict__ partial, int npartial,
                                                                double max_norm, int zero) {
    __shared__ float s_scale;
    float scale = 1.f;
    if (npartial > 0) {  // every CTA sums the norm partials in the same fixed order
        if (threadIdx.x < 32) {
            double ss = 0.0;
            for (int k = threadIdx.x; k < npartial; k += 32) ss += partial[k];
            ss = warp_sum(ss);
            if (threadIdx.x == 0) {
                const double norm = sqrt(ss);
                s_scale = norm > max_norm ? (float)(max_norm / norm) : 1.f;
            }
        }
        __syncthreads();
        scale = s_scale;
    }
    constexpr bool ONE = RULE == OPT_MOMENTUM || RULE == OPT_NESTEROV || RULE == OPT_ADAGRAD;
    constexpr bool TWO = RULE == OPT_ADADELTA || RULE == OPT_ADAM;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    const long n4 = n >> 2;
    const long ntile = (n4 + TILE4 - 1) / TILE4;
    for (long tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
        const long q0 = tile * TILE4 + threadIdx.x;
        const long e1 = ((tile + 1) * TILE4 < n4 ? (tile + 1) * TILE4 : n4) * 4 - 1;
        const L2Tile lt = l2_tile(a, tab, tile * TILE4 * 4, e1);
        float4 t[OPT_VEC], g[OPT_VEC], u[OPT_VEC], v[OPT_VEC];
#pragma unroll
        for (int k = 0; k < OPT_VEC; ++k) {  // all loads of the tile first (memory-level parallelism)
            const long q = q0 + k * OPT_THREADS;
            const bool ok = q < n4;
            t[k] = ok ? ld4(th, q) : z4;
            g[k] = ok ? ld4(gr, q) : z4;
            u[k] = (ONE || TWO) && ok ? ld4(s0, q) : z4;
            v[k] = TWO && ok ? ld4(s1, q) : z4;
        }
#pragma unroll
        for (int k = 0; k < OPT_VEC; ++k) {
            const long q = q0 + k * OPT_THREADS;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float gj = cond_grad(el(g[k], j), el(t[k], j), q * 4 + j, a, tab, lt) * scale;
                rule_step<RULE>(el(t[k], j), gj, el(u[k], j), el(v[k], j), a);
            }
            if (q < n4) {
                st4(th, q, t[k]);
                if (ONE || TWO) st4(s0, q, u[k]);
                if (TWO) st4(s1, q, v[k]);
                if (zero) st4(gr, q, z4);
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {  // ragged tail (< 4 elements)
        const long i = (n4 << 2) + threadIdx.x;
        float t = th[i];
        float u = (ONE || TWO) ? s0[i] : 0.f, v = TWO ? s1[i] : 0.f;
        const float g = cond_grad(gr[i], t, i, a, tab, L2Tile{0.f, true}) * scale;
        rule_step<RULE>(t, g, u, v, a);
        th[i] = t;
        if (ONE || TWO) s0[i] = u;
        if (TWO) s1[i] = v;
        if (zero) gr[i] = 0.f;
    }
}

int grid_for_tiles(long n4) {
    const long want = (n4 + TILE4 - 1) / TILE4;
    const long cap = 148L * 8;  // 8 CTAs of 256 threads per SM: full occupancy, grid-stride beyond
    return (int)(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace

int opt_norm_partials() { return 148 * 8; }

// --- replicas on one device: x_r <- scale * sum_q x_q for every r (§4.1 P:209-211:
// "combined into a single set of parameters by averaging"; scale = 1/n).  Summed in fixed
// replica order 0..n-1 in fp32, so every replica receives the same bits.
__global__ void __launch_bounds__(OPT_THREADS) reduce_replicas_kernel(const __grid_constant__ ReplicaPtrs rp, int n,
                                                                      long len, float scale) {
    const long n4 = len >> 2;
    const long stride = (long)gridDim.x * OPT_THREADS;
    for (long q = blockIdx.x * (long)OPT_THREADS + threadIdx.x; q < n4; q += stride) {
        float4 acc = ld4(rp.p[0], q);
        for (int r = 1; r < n; ++r) {
            const float4 v = ld4(rp.p[r], q);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        acc.x *= scale; acc.y *= scale; acc.z *= scale; acc.w *= scale;
        for (int r = 0; r < n; ++r) st4(rp.p[r], q, acc);
    }
    for (long i = (n4 << 2) + blockIdx.x * (long)OPT_THREADS + threadIdx.x; i < len; i += stride) {
        float acc = rp.p[0][i];
        for (int r = 1; r < n; ++r) acc += rp.p[r][i];
        acc *= scale;
        for (int r = 0; r < n; ++r) rp.p[r][i] = acc;
    }
}

int reduce_replicas(const ReplicaPtrs &rp, int n, long len, float scale, cudaStream_t st) {
    const long n4 = len >> 2;
    long grid = (n4 + OPT_THREADS - 1) / OPT_THREADS;
    grid = grid < 1 ? 1 : (grid > 148L * 8 ? 148L * 8 : grid);
    reduce_replicas_kernel<<<(int)grid, OPT_THREADS, 0, st>>>(rp, n, len, scale);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

int opt_update(int rule, float *theta, float *grad, float *s0, float *s1, long n, const OptArgs &a,
               double max_norm, const OptBiasTable &tab, double *partial, int zero, cudaStream_t st) {
    int npartial = 0;
    if (max_norm > 0.0) {
        npartial = opt_norm_partials();
        opt_sumsq_kernel<<<npartial, OPT_THREADS, 0, st>>>(theta, grad, n, a, tab, partial);
        note_launch();
    }
    const int grid = grid_for_tiles(n >> 2);
    switch (rule) {
#define OPT_CASE(R)                                                                                          \
    case R:                                                                                                  \
        opt_apply_kernel<R><<<grid, OPT_THREADS, 0, st>>>(theta, grad, s0, s1, n, a, tab, partial, npartial, \
                                                          max_norm, zero);                                             \
        break;
        OPT_CASE(OPT_SGD) OPT_CASE(OPT_MOMENTUM) OPT_CASE(OPT_NESTEROV) OPT_CASE(OPT_ADAGRAD)
        OPT_CASE(OPT_ADADELTA) OPT_CASE(OPT_ADAM)
#undef OPT_CASE
    default:
        return -1;
    }
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

}  // namespace blstm
