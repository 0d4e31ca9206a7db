// lstm_rec.cu -- persistent recurrence kernels of the LSTM layer (§4.2):
// the recurrent matmul h_{t-1} R on tcgen05 tensor cores, fused with the gating
// ("custom CUDA kernels for the LSTM gating mechanism"), the cell update and
// the mask, one launch for the whole sequence (no launch per time step).
//
// Decomposition: CTA (d, g, c) owns hidden units [32c, 32c+32) of
// direction d for batch group g.  Its 128 gate rows of R^T (gate-interleaved, row 4*jl+gamma)
// stay resident in shared memory for the whole sequence as the tcgen05 A operand.
// 16 warps: warp w reads TMEM lane quarter q = w%4 (8 units x 4 gates) for the batch
// columns of block cb = w/4 (N/4 columns), so the per-step epilogue is spread over 4 warps
// per scheduler.  Per step:
//   forward : D[128 x N] = R^T_slice[128 x Hq] . h_{t-1}^T  (h from the group's history buffer,
//             TMA-loaded after the group barrier), + Z_t, gates, cell update, mask in registers,
//             h_t published to the history buffer, group barrier (gpu-scope counter).
//   backward: dA_t for the CTA's 128 gate columns (fp16, scaled), partial
//             P_c[Hq x N] = R[:, cols_c] . dA_t^T on tcgen05 (same smem tile read MN-major),
//             P published, group barrier, each CTA sums the NC partials of its own units
//             (fixed order -> deterministic) to get dh_{t-1}.
#include "common.cuh"
#include "gemm.h"
#include "lstm_rec.h"
#include "prof.h"

namespace blstm {

constexpr int REC_THREADS = 512;

static DEVI uint8_t *align1024(uint8_t *p) { return (uint8_t *)(((uintptr_t)p + 1023) & ~(uintptr_t)1023); }

static __host__ __device__ constexpr uint32_t tmem_cols_for(int cols) {
    return cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
}

// 32 lanes x NC columns of TMEM -> registers (thread i: lane base+i)
template <int NC>
DEVI void tmem_ld(uint32_t taddr, float (&v)[NC]) {
    uint32_t r[NC];
    if constexpr (NC == 4) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                     : "r"(taddr));
    } else if constexpr (NC == 8) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                       "=r"(r[7])
                     : "r"(taddr));
    } else {
        static_assert(NC == 16, "tmem_ld: 4, 8 or 16 columns");
        float t[16];
        tmem_ld16(taddr, t);
#pragma unroll
        for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(t[i]);
    }
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < NC; ++i) v[i] = __uint_as_float(r[i]);
}

// 4x4 transpose inside each group of 4 lanes: lane gam holds a[k] = gate gam at batch column
// 4m+k; afterwards b[k] = gate k at batch column 4m+gam.
DEVI float sel4(const float (&a)[4], int i) { return i == 0 ? a[0] : i == 1 ? a[1] : i == 2 ? a[2] : a[3]; }
DEVI void xpose4(const float (&a)[4], float (&b)[4], int gam) {
    b[0] = b[1] = b[2] = b[3] = 0.f;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int k = gam ^ r;
        const float send = sel4(a, k);
        const float recv = r == 0 ? send : __shfl_xor_sync(0xffffffffu, send, r);
        if (k == 0) b[0] = recv;
        if (k == 1) b[1] = recv;
        if (k == 2) b[2] = recv;
        if (k == 3) b[3] = recv;
    }
}

// Gate nonlinearities in fp32 with the hardware exp2 (relative error ~1e-7, far inside the
// fp16-operand budget; R9): sigmoid(z) = 1/(1+e^-z), tanh(z) = 2 sigmoid(2z) - 1.
DEVI float sigm_f(float z) { return __fdividef(1.f, 1.f + __expf(-z)); }
DEVI float tanh_f(float z) { return 2.f * sigm_f(2.f * z) - 1.f; }
// activation of gate row gam (tanh for g, sigmoid otherwise) without lane divergence
DEVI float gate_act(float pre, int gam) {
    const bool is_g = gam == 2;
    const float s = sigm_f(is_g ? 2.f * pre : pre);
    return is_g ? 2.f * s - 1.f : s;
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
template <int NT>
__global__ void __launch_bounds__(REC_THREADS, 1)
    lstm_rec_fwd_kernel(const __grid_constant__ CUtensorMap tmR, const __grid_constant__ CUtensorMap tmH,
                        RecParams p) {
    constexpr int N = 16 * NT;   // MMA N = padded batch columns of the group
    constexpr int NQ = N / 4;    // columns handled by one warp
    constexpr int NMQ = NQ / 4;  // columns owned (cell state) by one thread
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    const int Hq = p.Hq, KB = Hq / 64;
    uint8_t *Rs = smem;
    uint8_t *Hs = smem + KB * 16384;
    uint64_t *bars = (uint64_t *)(Hs + KB * N * 128);
    uint32_t *tslot = (uint32_t *)(bars + 2);

    const int c = blockIdx.x % p.NC;
    const int g = (blockIdx.x / p.NC) % p.G;
    const int d = blockIdx.x / (p.NC * p.G);
    const int dir = d == 0 ? p.dir0 : -1;
    const int w = warp_id(), q = w & 3, cb = w >> 2, l = lane_id();
    const int jl = 8 * q + (l >> 2), gam = l & 3;
    const int j = c * REC_UNITS + jl;
    const bool unit_ok = j < p.H;
    const int B = p.B, T = p.T, H = p.H;
    const int b0 = g * p.Bg;        // first batch row of the group
    const int nq0 = cb * NQ;        // first column of this warp
    const int bq0 = b0 + nq0;       // its first batch row
    uint32_t *counter = p.counters + d * p.G + g;
    constexpr uint32_t TCOLS = tmem_cols_for(N);

    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    if (w == 0) {
        tmem_alloc(tslot, TCOLS);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t idesc = idesc_f16(128, N, 0, 0);

    // valid columns of this warp (bit i <-> column nq0 + i)
    uint32_t cm = 0;
#pragma unroll
    for (int i = 0; i < NQ; ++i)
        if (nq0 + i < p.Bg && bq0 + i < B) cm |= 1u << i;

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmR);
        tma_prefetch_desc(&tmH);
        mbar_arrive_expect_tx(&bars[0], KB * 16384);
        for (int kb = 0; kb < KB; ++kb) tma_load_2d(Rs + kb * 16384, &tmR, &bars[0], kb * 64, d * 4 * Hq + c * 128);
        mbar_wait(&bars[0], 0);
    }
    uint32_t tma_phase = 1, mma_phase = 0;

    float c_st[NMQ], h_st[NMQ];
#pragma unroll
    for (int m = 0; m < NMQ; ++m) {
        const int i = 4 * m + gam, b = bq0 + i;
        const bool ok = ((cm >> i) & 1) && unit_ok;
        c_st[m] = (ok && p.c0) ? p.c0[(long)d * B * H + (long)b * H + j] : 0.f;
        h_st[m] = (ok && p.h0) ? p.h0[(long)d * B * H + (long)b * H + j] : 0.f;
    }

    // CTA-native layout of Z and of the saved gates: this thread's NQ values of step t are
    // contiguous, and the warp's 32 x NQ values form one contiguous block
    const long nat_step = (long)p.ndir * p.G * p.NC * 512 * NQ;
    const long nat_off = (((long)d * p.G + g) * p.NC + c) * 512 * NQ + ((long)cb * 128 + 32 * q + l) * NQ;
    float zv[NQ];
    auto prefetch_z = [&](int t) {
        const float4 *zp = reinterpret_cast<const float4 *>(p.Z + t * nat_step + nat_off);
#pragma unroll
        for (int i = 0; i < NQ / 4; ++i) {
            const float4 v = __ldg(zp + i);
            zv[4 * i] = v.x; zv[4 * i + 1] = v.y; zv[4 * i + 2] = v.z; zv[4 * i + 3] = v.w;
        }
    };
    if (T > 0) prefetch_z(dir > 0 ? 0 : T - 1);

    const uint32_t rs_addr = smem_u32(Rs), hs_addr = smem_u32(Hs);
#ifdef BLSTM_TRACE
    unsigned long long *trace = (blockIdx.x == 0 && threadIdx.x == 0) ? p.trace : nullptr;
#define TRACE(k) \
    if (trace) trace[(size_t)s * 8 + (k)] = globaltimer_ns()
#else
#define TRACE(k)
#endif
    for (int s = 0; s < T; ++s) {
        const int t = dir > 0 ? s : T - 1 - s;
        TRACE(0);
        if (threadIdx.x == 0) {
            if (s > 0) spin_until_geq(counter, (uint32_t)(p.NC * s));
            TRACE(1);
            fence_async_global();
            const int rslot = t + (dir < 0 ? 1 : 0);
            const int row0 = (d * (T + 1) + rslot) * B + b0;
            mbar_arrive_expect_tx(&bars[0], KB * N * 128);
            for (int kb = 0; kb < KB; ++kb) tma_load_2d(Hs + kb * N * 128, &tmH, &bars[0], kb * 64, row0);
            mbar_wait(&bars[0], tma_phase);
            TRACE(2);
            tc_fence_after();
            for (int kb = 0; kb < KB; ++kb)
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    mma_f16_ss(tmem, sdesc_sw128(rs_addr + kb * 16384 + kk * 32, 16, 1024),
                               sdesc_sw128(hs_addr + kb * N * 128 + kk * 32, 16, 1024), idesc, (kb | kk) != 0);
            mma_commit(&bars[1]);
        }
        tma_phase ^= 1;
        // frame-valid bits of this warp's columns (lane i reads the mask of column i)
        const uint32_t frm =
            __ballot_sync(0xffffffffu, l < NQ && ((cm >> l) & 1) && p.mask[(long)t * B + bq0 + l]);
        const int wslot = t + (dir > 0 ? 1 : 0);
        mbar_wait(&bars[1], mma_phase);
        mma_phase ^= 1;
        tc_fence_after();
        TRACE(3);

        float act[NQ];
        {
            float v[NQ];
            tmem_ld<NQ>(tmem + ((uint32_t)(32 * q) << 16) + nq0, v);
#pragma unroll
            for (int i = 0; i < NQ; ++i) act[i] = gate_act(v[i] + zv[i], gam);
        }
        tc_fence_before();
        uint32_t fmq = 0;  // bit m: owned column 4m+gam is a valid frame
#pragma unroll
        for (int m = 0; m < NMQ; ++m) {
            float a4[4] = {act[4 * m], act[4 * m + 1], act[4 * m + 2], act[4 * m + 3]};
            float gv[4];
            xpose4(a4, gv, gam);  // gv = (i, f, g, o) of unit j at column 4m + gam
            const int i = 4 * m + gam;
            const bool fm = ((frm >> i) & 1) && unit_ok;
            if (fm) {
                const float cn = gv[1] * c_st[m] + gv[0] * gv[2];
                c_st[m] = cn;
                h_st[m] = gv[3] * tanh_f(cn);
                fmq |= 1u << m;
            }
            // h_t to the history buffer first: the only store the group barrier publishes
            if ((cm >> i) & 1)
                p.hist[(((long)d * (T + 1) + wslot) * B + bq0 + i) * Hq + j] = __float2half_rn(h_st[m]);
        }
        TRACE(4);
        __syncthreads();
        TRACE(5);
        if (threadIdx.x == 0) red_release_gpu_add(counter, 1u);
        TRACE(6);
        // off the critical path: saved activations (CTA-native, one vector store), c, y, y16
        {
            uint32_t hv[NQ / 2];
#pragma unroll
            for (int i = 0; i < NQ; i += 2) {
                const float a0 = (((frm >> i) & 1) && unit_ok) ? act[i] : 0.f;
                const float a1 = (((frm >> (i + 1)) & 1) && unit_ok) ? act[i + 1] : 0.f;
                __half2 h2 = __floats2half2_rn(a0, a1);
                hv[i / 2] = *reinterpret_cast<uint32_t *>(&h2);
            }
            __half *gp = p.gates + t * nat_step + nat_off;
            if constexpr (NQ == 4) {
                *reinterpret_cast<uint2 *>(gp) = make_uint2(hv[0], hv[1]);
            } else {
#pragma unroll
                for (int i = 0; i < NQ / 8; ++i)
                    reinterpret_cast<uint4 *>(gp)[i] = make_uint4(hv[4 * i], hv[4 * i + 1], hv[4 * i + 2], hv[4 * i + 3]);
            }
        }
#pragma unroll
        for (int m = 0; m < NMQ; ++m) {
            const int i = 4 * m + gam;
            if (((cm >> i) & 1)) {
                const bool fm = (fmq >> m) & 1;
                const long row = (long)t * B + bq0 + i;
                if (unit_ok) {
                    if (p.y) p.y[row * p.ldy + d * p.y_doff + j] = fm ? h_st[m] : 0.f;
                    p.C[row * p.ldc + d * p.c_doff + j] = c_st[m];
                }
                if (p.y16) p.y16[row * p.ldy16 + (long)d * Hq + j] = __float2half_rn(fm ? h_st[m] : 0.f);
            }
        }
        if (s + 1 < T) prefetch_z(dir > 0 ? t + 1 : t - 1);
        TRACE(7);
    }
#pragma unroll
    for (int m = 0; m < NMQ; ++m) {
        const int i = 4 * m + gam, b = bq0 + i;
        if (((cm >> i) & 1) && unit_ok) {
            if (p.hT) p.hT[(long)d * B * H + (long)b * H + j] = h_st[m];
            if (p.cT) p.cT[(long)d * B * H + (long)b * H + j] = c_st[m];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (w == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, TCOLS);
    }
}

// ---------------------------------------------------------------------------
// backward through time
// ---------------------------------------------------------------------------
template <int NT>
__global__ void __launch_bounds__(REC_THREADS, 1)
    lstm_rec_bwd_kernel(const __grid_constant__ CUtensorMap tmR, RecParams p) {
    constexpr int N = 16 * NT;
    constexpr int NQ = N / 4;
    constexpr int NMQ = NQ / 4;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    const int Hq = p.Hq, KB = Hq / 64, MT = Hq / 128;
    uint8_t *Rs = smem;
    uint8_t *dAs = smem + KB * 16384;  // [2][N][128 B] K-major SW128
    uint64_t *bars = (uint64_t *)(dAs + 2 * N * 128);
    uint32_t *tslot = (uint32_t *)(bars + 2);

    const int c = blockIdx.x % p.NC;
    const int g = (blockIdx.x / p.NC) % p.G;
    const int d = blockIdx.x / (p.NC * p.G);
    const int dir = d == 0 ? p.dir0 : -1;
    const int w = warp_id(), q = w & 3, cb = w >> 2, l = lane_id();
    const int jl = 8 * q + (l >> 2), gam = l & 3;
    const int j = c * REC_UNITS + jl;
    const bool unit_ok = j < p.H;
    const int B = p.B, T = p.T, H = p.H, NC = p.NC;
    const int b0 = g * p.Bg;
    const int nq0 = cb * NQ;
    const int bq0 = b0 + nq0;
    uint32_t *counter = p.counters + d * p.G + g;
    const uint32_t TCOLS = tmem_cols_for(MT * N);
    const float inv_scale = 1.f / (float)(1 << DA_SHIFT);
    const float scale = (float)(1 << DA_SHIFT);

    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    if (w == 0) {
        tmem_alloc(tslot, TCOLS);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t idesc = idesc_f16(128, N, 1, 0);

    uint32_t cm = 0;
#pragma unroll
    for (int i = 0; i < NQ; ++i)
        if (nq0 + i < p.Bg && bq0 + i < B) cm |= 1u << i;

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmR);
        mbar_arrive_expect_tx(&bars[0], KB * 16384);
        for (int kb = 0; kb < KB; ++kb) tma_load_2d(Rs + kb * 16384, &tmR, &bars[0], kb * 64, d * 4 * Hq + c * 128);
        mbar_wait(&bars[0], 0);
    }
    __syncthreads();

    float dh[NMQ], dc[NMQ], dbp[4] = {0.f, 0.f, 0.f, 0.f};
    uint32_t pfm = 0;  // bit m: the previous step's frame was valid for owned column 4m+gam
#pragma unroll
    for (int m = 0; m < NMQ; ++m) {
        const int i = 4 * m + gam, b = bq0 + i;
        const bool ok = ((cm >> i) & 1) && unit_ok;
        dh[m] = (ok && p.dhT) ? p.dhT[(long)d * B * H + (long)b * H + j] : 0.f;
        dc[m] = (ok && p.dcT) ? p.dcT[(long)d * B * H + (long)b * H + j] : 0.f;
    }
    // P (partial dh) exchange in a CTA-native layout [buf][d][g][c_src][mt][cb][128][NQ]: the
    // writer's warp stores one contiguous block per M tile; the reader sums its units' rows
    const size_t p_src = (size_t)MT * 512 * NQ;             // one source CTA
    const size_t pstride_buf = (size_t)p.ndir * p.G * NC * p_src;
    const size_t p_grp = (((size_t)d * p.G + g) * NC) * p_src;
    auto gather = [&](int buf) {
        const float *Pb = p.P + buf * pstride_buf + p_grp + (size_t)(j >> 7) * 512 * NQ +
                          ((size_t)cb * 128 + (j & 127)) * NQ;
#pragma unroll
        for (int m = 0; m < NMQ; ++m) {
            if ((pfm >> m) & 1) {
                float acc = 0.f;
                for (int cc = 0; cc < NC; ++cc) acc += Pb[(size_t)cc * p_src + 4 * m + gam];
                dh[m] = acc * inv_scale;
            }
        }
    };
    const long nat_step = (long)p.ndir * p.G * NC * 512 * NQ;
    const long nat_off = (((long)d * p.G + g) * NC + c) * 512 * NQ + ((long)cb * 128 + 32 * q + l) * NQ;

    uint32_t mma_phase = 0;
    const uint32_t rs_addr = smem_u32(Rs), das_addr = smem_u32(dAs);
#ifdef BLSTM_TRACE
    unsigned long long *trace = (blockIdx.x == 0 && threadIdx.x == 0) ? p.trace : nullptr;
#endif
    for (int s = T - 1; s >= 0; --s) {
        const int t = dir > 0 ? s : T - 1 - s;
        const int k_done = T - 1 - s;
        TRACE(0);
        // ---- this step's saved state (independent of the recurrence: issue first) ----
        float graw[NQ];
        {
            const __half *gp = p.gates + t * nat_step + nat_off;
            uint32_t hv[NQ / 2];
            if constexpr (NQ == 4) {
                const uint2 u = *reinterpret_cast<const uint2 *>(gp);
                hv[0] = u.x; hv[1] = u.y;
            } else {
#pragma unroll
                for (int i = 0; i < NQ / 8; ++i) {
                    const uint4 u = reinterpret_cast<const uint4 *>(gp)[i];
                    hv[4 * i] = u.x; hv[4 * i + 1] = u.y; hv[4 * i + 2] = u.z; hv[4 * i + 3] = u.w;
                }
            }
#pragma unroll
            for (int i = 0; i < NQ; i += 2) {
                const float2 f2 = __half22float2(*reinterpret_cast<const __half2 *>(&hv[i / 2]));
                graw[i] = f2.x;
                graw[i + 1] = f2.y;
            }
        }
        float ct[NMQ], cp[NMQ], dyv[NMQ];
        const int tp = t - dir;
#pragma unroll
        for (int m = 0; m < NMQ; ++m) {
            const int i = 4 * m + gam, b = bq0 + i;
            const bool ok = ((cm >> i) & 1) && unit_ok;
            const long row = (long)t * B + b;
            ct[m] = ok ? p.C[row * p.ldc + d * p.c_doff + j] : 0.f;
            if (ok && tp >= 0 && tp < T) cp[m] = p.C[((long)tp * B + b) * p.ldc + d * p.c_doff + j];
            else cp[m] = (ok && p.c0) ? p.c0[(long)d * B * H + (long)b * H + j] : 0.f;
            dyv[m] = ok ? p.dy[row * p.lddy + d * p.dy_doff + j] : 0.f;
        }
        const uint32_t frm =
            __ballot_sync(0xffffffffu, l < NQ && ((cm >> l) & 1) && p.mask[(long)t * B + bq0 + l]);
        // ---- dh_t from the previous step's partials ----
        TRACE(1);
        if (k_done > 0) {
            if (threadIdx.x == 0) spin_until_geq(counter, (uint32_t)(NC * k_done));
            TRACE(2);
            __syncthreads();
            gather((k_done - 1) & 1);
        }
        TRACE(3);
        // ---- gate gradients ----
        pfm = 0;
        uint2 pks[NMQ];
#pragma unroll
        for (int m = 0; m < NMQ; ++m) {
            float a4[4] = {graw[4 * m], graw[4 * m + 1], graw[4 * m + 2], graw[4 * m + 3]};
            float gv[4];
            xpose4(a4, gv, gam);
            const int i = 4 * m + gam, n = nq0 + i;
            const bool fm = ((frm >> i) & 1) && unit_ok;
            float da0 = 0.f, da1 = 0.f, da2 = 0.f, da3 = 0.f;
            if (fm) {
                const float ig = gv[0], f = gv[1], gg = gv[2], o = gv[3];
                const float th = tanh_f(ct[m]);
                const float dH = dh[m] + dyv[m];
                const float dC = dc[m] + dH * o * (1.f - th * th);
                da0 = dC * gg * ig * (1.f - ig);
                da1 = dC * cp[m] * f * (1.f - f);
                da2 = dC * ig * (1.f - gg * gg);
                da3 = dH * th * o * (1.f - o);
                dc[m] = dC * f;
                dbp[0] += da0; dbp[1] += da1; dbp[2] += da2; dbp[3] += da3;
                pfm |= 1u << m;
            }
            __half2 lo = __floats2half2_rn(da0 * scale, da1 * scale);
            __half2 hi = __floats2half2_rn(da2 * scale, da3 * scale);
            uint2 pk;
            pk.x = *reinterpret_cast<uint32_t *>(&lo);
            pk.y = *reinterpret_cast<uint32_t *>(&hi);
            *reinterpret_cast<uint2 *>(dAs + sw128_offset(n, 4 * jl, N)) = pk;
            pks[m] = pk;
        }
        fence_async_smem();
        tc_fence_before();
        TRACE(4);
        __syncthreads();
        if (threadIdx.x == 0) {
            TRACE(5);
            tc_fence_after();
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_f16_ss(tmem + mt * N, sdesc_sw128(rs_addr + 2 * mt * 16384 + kk * 2048, 16384, 1024),
                               sdesc_sw128(das_addr + (kk >> 2) * N * 128 + (kk & 3) * 32, 16, 1024), idesc, kk != 0);
            mma_commit(&bars[1]);
        }
        // while the MMA runs: dA of this step to global memory for the weight / input GEMMs
#pragma unroll
        for (int m = 0; m < NMQ; ++m) {
            const int i = 4 * m + gam;
            if ((cm >> i) & 1)
                *reinterpret_cast<uint2 *>(p.dA + ((long)t * B + bq0 + i) * p.ldda + (long)d * 4 * Hq + 4 * j) = pks[m];
        }
        mbar_wait(&bars[1], mma_phase);
        mma_phase ^= 1;
        tc_fence_after();
        TRACE(6);
        float *Pw = p.P + (size_t)(k_done & 1) * pstride_buf + p_grp + (size_t)c * p_src +
                    ((size_t)cb * 128 + 32 * q + l) * NQ;
        for (int mt = 0; mt < MT; ++mt) {
            float v[NQ];
            tmem_ld<NQ>(tmem + ((uint32_t)(32 * q) << 16) + mt * N + nq0, v);
            float4 *dst = reinterpret_cast<float4 *>(Pw + (size_t)mt * 512 * NQ);
#pragma unroll
            for (int i = 0; i < NQ / 4; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
        tc_fence_before();
        __syncthreads();
        if (threadIdx.x == 0) red_release_gpu_add(counter, 1u);
        TRACE(7);
    }
#undef TRACE
    if (T > 0) {
        if (threadIdx.x == 0) spin_until_geq(counter, (uint32_t)(NC * T));
        __syncthreads();
        gather((T - 1) & 1);
    }
#pragma unroll
    for (int m = 0; m < NMQ; ++m) {
        const int i = 4 * m + gam, b = bq0 + i;
        if (((cm >> i) & 1) && unit_ok) {
            if (p.dh0) p.dh0[(long)d * B * H + (long)b * H + j] = dh[m];
            if (p.dc0) p.dc0[(long)d * B * H + (long)b * H + j] = dc[m];
        }
    }
    // bias gradient: sum over the thread's columns, the 4 lanes of the unit, then the 4 column
    // blocks (fixed order through shared memory)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        dbp[k] += __shfl_xor_sync(0xffffffffu, dbp[k], 1);
        dbp[k] += __shfl_xor_sync(0xffffffffu, dbp[k], 2);
    }
    float *dbs = reinterpret_cast<float *>(dAs);  // [4 cb][128 rows]
    __syncthreads();
    dbs[cb * 128 + 4 * jl + gam] = sel4(dbp, gam);
    __syncthreads();
    if (cb == 0) {
        const int r = 4 * jl + gam;
        p.dbpart[((long)d * p.G + g) * 4 * Hq + 4 * j + gam] = ((dbs[r] + dbs[128 + r]) + dbs[256 + r]) + dbs[384 + r];
    }
    tc_fence_before();
    __syncthreads();
    if (w == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, TCOLS);
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int round_up(int a, int b) { return (a + b - 1) / b * b; }
static int mma_n(int Bg) { return Bg <= 16 ? 16 : Bg <= 32 ? 32 : round_up(Bg, 64); }

RecPlan rec_plan(int T, int B, int H, int ndir, int sms) {
    (void)T;
    RecPlan pl{};
    pl.Hq = round_up(H, 128);
    pl.NC = pl.Hq / REC_UNITS;
    pl.ndir = ndir;
    int bestG = 1, bestN = 1 << 30;
    for (int G = 1; G <= B; ++G) {
        if (ndir * G * pl.NC > sms) break;
        const int N = mma_n((B + G - 1) / G);
        if (N < bestN) { bestN = N; bestG = G; }
    }
    pl.G = bestG;
    pl.Bg = (B + bestG - 1) / bestG;
    pl.N = mma_n(pl.Bg);
    return pl;
}

static size_t fwd_smem(const RecPlan &pl) { return (size_t)pl.Hq / 64 * (16384 + pl.N * 128) + 1024 + 64; }
static size_t bwd_smem(const RecPlan &pl) { return (size_t)pl.Hq / 64 * 16384 + 2 * pl.N * 128 + 1024 + 64; }

bool rec_supported(const RecPlan &pl, int H) {
    if (H < 1 || (pl.N != 16 && pl.N != 32 && pl.N != 64)) return false;
    if (fwd_smem(pl) > 227 * 1024 || bwd_smem(pl) > 227 * 1024) return false;
    if (pl.ndir * pl.G * pl.NC > num_sms()) return false;
    if (pl.Hq / 128 * pl.N > 512) return false;
    return pl.Hq % 128 == 0;
}

size_t rec_P_bytes(const RecPlan &pl) {
    return (size_t)2 * pl.ndir * pl.G * pl.NC * pl.Hq * pl.N * sizeof(float);
}

template <typename Kern, typename... Args>
static cudaError_t launch_coop(Kern kern, int grid, size_t smem, cudaStream_t st, Args... args) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(REC_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

static unsigned long long *g_trace_fwd = nullptr, *g_trace_bwd = nullptr;
void rec_set_trace(unsigned long long *fwd, unsigned long long *bwd) {
    g_trace_fwd = fwd;
    g_trace_bwd = bwd;
}

int lstm_rec_fwd(const RecParams &p_in, const __half *RT16, cudaStream_t st) {
    RecParams p = p_in;
    if (g_trace_fwd) p.trace = g_trace_fwd;
    if (p.T == 0) return 0;
    CUtensorMap tmR, tmH;
    if (make_tmap_f16(&tmR, RT16, p.Hq, (uint64_t)p.ndir * 4 * p.Hq, p.Hq, 128)) return -2;
    if (make_tmap_f16(&tmH, p.hist, p.Hq, (uint64_t)p.ndir * (p.T + 1) * p.B, p.Hq, p.N)) return -2;
    RecPlan pl{p.Hq, p.NC, p.G, p.Bg, p.N, p.ndir};
    const int grid = p.ndir * p.G * p.NC;
    const size_t smem = fwd_smem(pl);
    cudaError_t e = cudaMemsetAsync(p.counters, 0, sizeof(uint32_t) * p.ndir * p.G, st);
    if (e != cudaSuccess) return -5;
    ProfScope ps(PROF_REC_FWD, st);
    note_launch();
    switch (p.N) {
        case 16: e = launch_coop(lstm_rec_fwd_kernel<1>, grid, smem, st, tmR, tmH, p); break;
        case 32: e = launch_coop(lstm_rec_fwd_kernel<2>, grid, smem, st, tmR, tmH, p); break;
        case 64: e = launch_coop(lstm_rec_fwd_kernel<4>, grid, smem, st, tmR, tmH, p); break;
        default: return -6;
    }
    return e == cudaSuccess ? 0 : -5;
}

int lstm_rec_bwd(const RecParams &p_in, const __half *RT16, cudaStream_t st) {
    RecParams p = p_in;
    if (g_trace_bwd) p.trace = g_trace_bwd;
    CUtensorMap tmR;
    if (make_tmap_f16(&tmR, RT16, p.Hq, (uint64_t)p.ndir * 4 * p.Hq, p.Hq, 128)) return -2;
    RecPlan pl{p.Hq, p.NC, p.G, p.Bg, p.N, p.ndir};
    const int grid = p.ndir * p.G * p.NC;
    const size_t smem = bwd_smem(pl);
    cudaError_t e = cudaMemsetAsync(p.counters, 0, sizeof(uint32_t) * p.ndir * p.G, st);
    if (e != cudaSuccess) return -5;
    ProfScope ps(PROF_REC_BWD, st);
    note_launch();
    switch (p.N) {
        case 16: e = launch_coop(lstm_rec_bwd_kernel<1>, grid, smem, st, tmR, p); break;
        case 32: e = launch_coop(lstm_rec_bwd_kernel<2>, grid, smem, st, tmR, p); break;
        case 64: e = launch_coop(lstm_rec_bwd_kernel<4>, grid, smem, st, tmR, p); break;
        default: return -6;
    }
    return e == cudaSuccess ? 0 : -5;
}

}  // namespace blstm
