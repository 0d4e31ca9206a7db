// lstm_rec.cu -- persistent recurrence kernels of the LSTM layer (§4.2):
// the recurrent matmul h_{t-1} R on tcgen05 tensor cores, fused with the gating
// ("custom CUDA kernels for the LSTM gating mechanism"), the cell update and
// the mask, one launch for the whole sequence (no launch per time step).
//
// Decomposition: one thread-block cluster of NC = Hq/32 CTAs per
// (direction d, batch group g); cluster rank c owns hidden units [32c, 32c+32).  The CTA's
// slice of the recurrent weights stays resident in TMEM for the whole sequence as the
// tcgen05 A operand (forward: R^T rows of its 128 gate columns; BPTT: R rows, all Hq units x
// its 128 gate columns).  16 warps: warp w reads TMEM lane quarter q = w%4 (8 units x 4 gates)
// for the batch columns of block cb = w/4 (N/4 columns).
// Per step, all exchange is on chip, through distributed shared memory and mbarriers:
//   forward : D[128 x N] = R^T_slice . h_{t-1}^T (B operand = the cluster's h, double-buffered
//             in smem), + Z_t, gates, cell update, mask in registers; the CTA's h_t slice is
//             staged in smem and bulk-copied into every peer's next B buffer (complete_tx on
//             the peer's mbarrier).
//   backward: dA_t for the CTA's 128 gate columns (fp16, scaled) -> smem B operand;
//             P_c[Hq x N] = R[:, cols_c] . dA_t^T; each warp st.async's the 32 rows owned by
//             peer c' straight from registers into c''s slot for source c; every CTA sums its
//             NC slots in fixed order (deterministic) -> dh_{t-1} of its units.
#include "common.cuh"
#include "gemm.h"
#include "lstm_rec.h"
#include "prof.h"

namespace blstm {

constexpr int REC_THREADS = 512;

// pointer arithmetic on the shared array (not an integer round trip) keeps the shared address
// space visible to the compiler, so accesses through the result compile to LDS/STS
static DEVI uint8_t *align1024(uint8_t *p) { return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u); }

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

// 32 lanes x NC columns, issued without waiting (pair with tmem_wait_regs on the same registers)
template <int NC>
DEVI void tmem_ld_nowait(uint32_t taddr, uint32_t (&r)[NC]) {
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
        static_assert(NC == 16, "tmem_ld_nowait: 4, 8 or 16 columns");
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
    }
}
// after tcgen05.wait::ld: "redefine" the loaded registers so no consumer is scheduled before the wait
template <int NC>
DEVI void pin_regs(uint32_t (&r)[NC]) {
#pragma unroll
    for (int i = 0; i < NC; ++i) asm volatile("" : "+r"(r[i]));
}

// 4x4 transpose inside each group of 4 lanes: lane gam holds a[k] = gate gam at batch column
// 4m+k; afterwards b[k] = gate k at batch column 4m+gam.  Two butterfly stages (lane bit 0 /
// element bit 0, then lane bit 1 / element bit 1), selects only: a lane-dependent array index
// would compile to divergent branch trees.
DEVI float sel4(const float (&a)[4], int i) {
    const float lo = (i & 1) ? a[1] : a[0], hi = (i & 1) ? a[3] : a[2];
    return (i & 2) ? hi : lo;
}
DEVI void xpose4(const float (&a)[4], float (&b)[4], int gam) {
    const bool o1 = gam & 1, o2 = gam & 2;
    float v0 = a[0], v1 = a[1], v2 = a[2], v3 = a[3];
    float s0 = __shfl_xor_sync(0xffffffffu, o1 ? v0 : v1, 1);
    float s1 = __shfl_xor_sync(0xffffffffu, o1 ? v2 : v3, 1);
    v0 = o1 ? s0 : v0; v1 = o1 ? v1 : s0;
    v2 = o1 ? s1 : v2; v3 = o1 ? v3 : s1;
    s0 = __shfl_xor_sync(0xffffffffu, o2 ? v0 : v2, 2);
    s1 = __shfl_xor_sync(0xffffffffu, o2 ? v1 : v3, 2);
    v0 = o2 ? s0 : v0; v2 = o2 ? v2 : s0;
    v1 = o2 ? s1 : v1; v3 = o2 ? v3 : s1;
    b[0] = v0; b[1] = v1; b[2] = v2; b[3] = v3;
}

// Gate nonlinearities in fp32 with the hardware exp2 (R9): sigmoid(z) = 1/(1+e^-z) has
// ~1e-7 relative error; tanh(z) = 2 sigmoid(2z) - 1 has ~1e-7 ABSOLUTE error (so up to ~1e-3
// relative near |z| ~ 1e-4, where tanh itself is tiny).  Both are far inside the normwise fp16-operand
// budget, which is what R10 measures.
DEVI float sigm_f(float z) { return __fdividef(1.f, 1.f + __expf(-z)); }
DEVI float tanh_f(float z) { return 2.f * sigm_f(2.f * z) - 1.f; }
// activation of gate row gam (tanh for g, sigmoid otherwise) without lane divergence
DEVI float gate_act(float pre, int gam) {
    const bool is_g = gam == 2;
    const float s = sigm_f(is_g ? 2.f * pre : pre);
    return is_g ? 2.f * s - 1.f : s;
}

#ifndef BLSTM_TRACE_CTA
#define BLSTM_TRACE_CTA 0  // the CTA whose thread 0 records the trace (build.py: BLSTM_TRACE_CTA env)
#endif
#ifdef BLSTM_TRACE
#define TRACE(k) \
    if (trace) trace[(size_t)s * 16 + (k)] = (unsigned long long)clock64()
#else
#define TRACE(k)
#endif

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
// CTA pairs: cluster ranks (2p, 2p+1) run each step's MMA as one cta_group::2 MMA (M = 256: the
// pair's 2 x 128 gate rows), issued by the even CTA.  The B operand h_{t-1}^T is split by batch
// column: CTA 2p holds columns [0, N/2), CTA 2p+1 columns [N/2, N).  Every CTA therefore receives
// and sends half the bytes of a full all-gather (the DSMEM port, ~18 B/clk/SM, bounds the step).
// smem: [region0: R^T slice (TMA, start only) | aliased later by hbuf[2] + stg[2][2]] [barriers]
//   hbuf[b]: this CTA's half of the B operand [N/2 x Hq] fp16, no-swizzle K-major: element (n', k)
//            at ((k/8)*N/2 + n')*16 + (k%8)*2, so CTA c's units [32c, 32c+32) are one contiguous
//            32N-byte block
//   stg[b][h]: this CTA's h slice, column half h, in that block format (sent to the CTAs of parity h)
//   zin[2]: the CTA's Z block of a step (CTA-native, 512N bytes) + its mask row (N bytes, padded
//           to 128), bulk-copied by one thread one step ahead (per-thread loads cost ~0.27 us/step)
static __host__ __device__ size_t fwd_region0(int Hq, int N) {
    const size_t rs = (size_t)Hq / 64 * 16384,
                 hb = (size_t)Hq * N * 2 + 2 * 64 * (size_t)N + 2 * (512 * (size_t)N + 128);
    return rs > hb ? rs : hb;
}

template <int NT>
__global__ void __launch_bounds__(REC_THREADS, 1)
    lstm_rec_fwd_kernel(const __grid_constant__ CUtensorMap tmR, RecParams p) {
    constexpr int N = 16 * NT;   // MMA N = padded batch columns of the group
    constexpr int NQ = N / 4;    // columns handled by one warp
    constexpr int NMQ = NQ / 4;  // columns owned (cell state) by one thread
    constexpr int NH = N / 2;          // B-operand columns held by each CTA of a pair
    constexpr uint32_t SGh = 64 * NH;  // bytes of one column half of a CTA's h slice
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    const int Hq = p.Hq, KB = Hq / 64, NC = p.NC;
    const uint32_t HB = (uint32_t)Hq * NH * 2;
    uint8_t *Rs = smem;
    uint8_t *hbuf = smem;            // aliases Rs after the TMEM load
    uint8_t *stg = smem + 2 * HB;    // [2 b][2 halves][SGh]
    constexpr uint32_t ZB = 512 * N, ZSLOT = ZB + 128;  // Z block + mask row
    uint8_t *zin = stg + 4 * SGh;    // [2][ZSLOT]
    // [0] tma, [1] mma (arrived by the pair's commits), [2..3] full[b] (own half of h landed),
    // [4..5] pfull[b] (even CTA: the odd CTA's half landed), [6..7] zfull[slot] (Z + mask landed)
    uint64_t *bars = (uint64_t *)(smem + fwd_region0(Hq, N));
    uint32_t *tslot = (uint32_t *)(bars + 8);

    // the conditional re-launch after an aborted start (RecParams::rerun), a programmatic dependent
    // of the Z GEMM: wait for the GEMM grid (and through its own wait, the primary recurrence) to
    // complete, then a uniform early exit unless the primary aborted
    if (p.rerun) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (*(volatile const uint32_t *)(p.rerun + 1) != ARB_ABORT) return;
    }
    // this CTA is resident: a programmatically dependent launch (the concurrent Z GEMM, gemm.h pdl)
    // may start on the SMs left free once every CTA of this grid got here
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int c = (int)cluster_ctarank();
    const int pr = c & 1;                                   // 0: issues the pair's MMAs
    const uint16_t pair_mask = (uint16_t)(3u << (c & ~1));  // both CTAs of the pair
    const int grp = blockIdx.x / NC;  // cluster index = d*G + g
    const int g = grp % p.G;
    const int d = grp / p.G;
    const int dir = d == 0 ? p.dir0 : -1;
    const int w = warp_uniform(warp_id()), q = w & 3, cb = w >> 2, l = lane_id();
    const int jl = 8 * q + (l >> 2), gam = l & 3;
    const int j = c * REC_UNITS + jl;
    const bool unit_ok = j < p.H;
    const int B = p.B, T = p.T, H = p.H;
    const int b0 = g * p.Bg;        // first batch row of the group
    const int nq0 = cb * NQ;        // first column of this warp
    const int bq0 = b0 + nq0;       // its first batch row
    constexpr uint32_t TCOLS = 512;
    // TMEM: columns [0, Hq/2) hold the CTA's R^T slice (A operand, 128 lanes = gate rows, two
    // fp16 of K per 32-bit column); from column Hq/2, NISSUE K-split accumulators D_w[128 x N]
    // (warps 0..NISSUE-1 each issue a 1/NISSUE share of K).
    const uint32_t DCOL = Hq / 2;
    // four issuing warps: even with warp-collective uniform-register issue one warp sustains only
    // ~1 MMA per ~45 cycles (measured: 32 MMAs 0.77 us from one warp vs 0.26 us from four)
    constexpr int NISSUE = 4;

    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], NISSUE);
        mbar_init(&bars[2], 1);
        mbar_init(&bars[3], 1);
        mbar_init(&bars[4], 1);
        mbar_init(&bars[5], 1);
        mbar_init(&bars[6], 1);
        mbar_init(&bars[7], 1);
        fence_mbar_init();
    }
    if (w == 0) {  // one warp of each CTA of the pair
        tmem_alloc2(tslot, TCOLS);
        tmem_relinquish2();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t idesc = idesc_f16(256, N, 0, 0);

    // valid columns of this warp (bit i <-> column nq0 + i)
    uint32_t cm = 0;
#pragma unroll
    for (int i = 0; i < NQ; ++i)
        if (nq0 + i < p.Bg && bq0 + i < B) cm |= 1u << i;

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmR);
        mbar_arrive_expect_tx(&bars[0], KB * 16384);
        for (int kb = 0; kb < KB; ++kb) tma_load_2d(Rs + kb * 16384, &tmR, &bars[0], kb * 64, d * 4 * Hq + c * 128);
    }
    mbar_wait(&bars[0], 0);
    // R^T slice: shared memory (SW128 K-major) -> registers -> TMEM, once per launch.
    // Warp (q, cb) writes lanes 32q.. and columns [cb*Hq/8, (cb+1)*Hq/8).
    {
        const int r = 32 * q + l;
        const int cw = Hq / 8;
        for (int col = cb * cw; col < (cb + 1) * cw; col += 16) {
            uint32_t v[16];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int kc = col / 4 + u;  // 8 K-elements = 4 columns
                const uint4 x = *reinterpret_cast<const uint4 *>(Rs + (kc >> 3) * 16384 + r * 128 +
                                                                  (((kc & 7) ^ (r & 7)) << 4));
                v[4 * u] = x.x; v[4 * u + 1] = x.y; v[4 * u + 2] = x.z; v[4 * u + 3] = x.w;
            }
            tmem_st16(tmem + ((uint32_t)(32 * q) << 16) + col, v);
        }
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // h_{-1} = h0 (or 0) into hbuf[0]: all Hq units of this CTA's column half
    for (int e = threadIdx.x; e < NH * Hq / 2; e += REC_THREADS) {
        const int nn = e / (Hq / 2), k = 2 * (e - nn * (Hq / 2)), n = pr * NH + nn, b = b0 + n;
        float v0 = 0.f, v1 = 0.f;
        if (p.h0 && n < p.Bg && b < B) {
            const float *hp = p.h0 + (long)d * B * H + (long)b * H;
            if (k < H) v0 = hp[k];
            if (k + 1 < H) v1 = hp[k + 1];
        }
        __half2 h2 = __floats2half2_rn(v0, v1);
        *reinterpret_cast<__half2 *>(hbuf + ((k >> 3) * NH + nn) * 16 + (k & 7) * 2) = h2;
    }
    fence_async_smem();
    if (threadIdx.x == 0) {
        if (T > 1) mbar_arrive_expect_tx(&bars[3], NC * SGh);  // h_0 from the cluster -> step 1
        if (T > 2) mbar_arrive_expect_tx(&bars[2], NC * SGh);  // h_1 -> step 2
    }
    // Z of step t2 may still be in flight from the concurrent Z GEMM (p.zflags): one thread (lane 0
    // of the first non-issuing warp) verifies the M-tiles holding frames t2*B .. t2*B+B-1 in this
    // direction's time order, advancing a frontier; the CTA barrier that follows publishes it to
    // the threads that then load Z (acquire -> bar.sync -> ld.global.cg)
    constexpr int ZPOLL = 32 * NISSUE;
    const uint32_t *zf = p.zflags ? p.zflags + (size_t)d * p.zflag_nm : nullptr;
    int zfront = dir > 0 ? 0 : p.zflag_nm - 1;  // next M-tile to verify (polling thread only)
    auto z_tile_of = [&](int t2) {  // last M-tile (in time order) that step t2 needs
        return dir > 0 ? (int)(((long)t2 * B + B - 1) / GEMM_BM_ROWS) : (int)(((long)t2 * B) / GEMM_BM_ROWS);
    };
    auto z_wait = [&](int t2) {
        const int need = z_tile_of(t2);
        while (dir > 0 ? zfront <= need : zfront >= need) {
            spin_until_geq(zf + zfront, (uint32_t)p.zflag_target);
            zfront += dir;
        }
    };
    uint32_t *go = tslot + 1;  // the start arbitration's decision (RecParams::arb), CTA-wide
    if (threadIdx.x == ZPOLL) {
        const bool ok = p.arb ? arb_decide(p.arb, p.arb_target) : true;
        *go = ok ? 1u : 0u;
        if (ok && zf && T > 0) {
            z_wait(dir > 0 ? 0 : T - 1);
            if (T > 1) z_wait(dir > 0 ? 1 : T - 2);
        }
    }
    cluster_sync();  // every CTA done with its R staging before peers write into hbuf / stg
    if (*go == 0) {  // the Z GEMM never became resident: the re-launch after it does the layer
        tc_fence_before();
        __syncthreads();
        if (w == 0) {
            tc_fence_after();
            tmem_dealloc2(tmem, TCOLS);
        }
        return;
    }

    float c_st[NMQ], h_st[NMQ];
#pragma unroll
    for (int m = 0; m < NMQ; ++m) {
        const int i = 4 * m + gam, b = bq0 + i;
        const bool ok = ((cm >> i) & 1) && unit_ok;
        c_st[m] = (ok && p.c0) ? p.c0[(long)d * B * H + (long)b * H + j] : 0.f;
        h_st[m] = (ok && p.h0) ? p.h0[(long)d * B * H + (long)b * H + j] : 0.f;
    }

    // CTA-native layout of Z and of the saved gates (lstm_rec.h): this thread's NQ values of step t
    // are contiguous, and the warp's 32 x NQ values form one contiguous block
    const long nat_step = (long)p.ndir * p.G * NC * 512 * NQ;
    const long nat_cta = (((long)d * p.G + g) * NC + c) * 512 * NQ;
    const long nat_off = nat_cta + ((long)cb * 128 + 32 * q + l) * NQ;
    // step s2's Z block + mask row -> zin[s2 & 1] (thread 0); the slot was last read at step s2-2.
    // The bulk copy engine serves these behind this CTA's h sends of the previous step.
    auto issue_z = [&](int s2) {
        const int t2 = dir > 0 ? s2 : T - 1 - s2, sl = s2 & 1;
        mbar_arrive_expect_tx(&bars[6 + sl], ZB + N);
        bulk_g2s(smem_u32(zin + sl * ZSLOT), p.Z + t2 * nat_step + nat_cta, ZB, &bars[6 + sl]);
        bulk_g2s(smem_u32(zin + sl * ZSLOT + ZB), p.maskN + ((long)t2 * p.G + g) * N, N, &bars[6 + sl]);
    };
    if (threadIdx.x == ZPOLL && T > 0) {  // verified ready above (zf)
        fence_proxy_async_global();
        issue_z(0);
        if (T > 1) issue_z(1);
    }

    const uint32_t hbuf_addr = smem_u32(hbuf), stg_addr = smem_u32(stg);
    const uint32_t full_addr = smem_u32(&bars[2]);
    uint32_t fph = 0, mma_phase = 0;  // fph bit b: phase parity of full[b]
#ifdef BLSTM_TRACE
    unsigned long long *trace = (blockIdx.x == BLSTM_TRACE_CTA && threadIdx.x == 0) ? p.trace : nullptr;
#endif
    // HBM stores of a step (saved activations in CTA-native layout, c, y, y16, h history): off the
    // critical path, so they are issued at the start of the NEXT step, behind its MMA issue
    float act[NQ];
    auto store_step = [&](int t, uint32_t frm, uint32_t fmq) {
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
        const int wslot = t + (dir > 0 ? 1 : 0);
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
                p.hist[(((long)d * (T + 1) + wslot) * B + bq0 + i) * Hq + j] = __float2half_rn(h_st[m]);
            }
        }
    };
    int t_prev = 0;
    uint32_t frm_prev = 0, fmq_prev = 0;
    for (int s = 0; s < T; ++s) {
        const int t = dir > 0 ? s : T - 1 - s;
        const int b = s & 1;
        TRACE(0);
        // Z of step s+1 (verified during step s-1) -> its ring slot, last read at step s-1
        if (threadIdx.x == ZPOLL && s >= 1 && s + 1 < T) {
            fence_proxy_async_global();  // generic writes acquired from the GEMM -> bulk-copy reads
            issue_z(s + 1);
        }
        // Z of step s+2: issue the acquire load of the frontier M-tile now, check it before this
        // step's __syncthreads (its latency hides behind the step)
        const bool zcheck = zf && threadIdx.x == ZPOLL && s + 2 < T &&
                            (dir > 0 ? zfront <= z_tile_of(t + 2) : zfront >= z_tile_of(t - 2));
        uint32_t zseen = 0;
        if (zcheck) zseen = ld_acquire_gpu(zf + zfront);
        if (pr == 0 && w < NISSUE) {  // warp-collective issue of the pair MMA (one elected lane)
            if (s > 0) {  // h_{s-1}: this CTA's half and the odd CTA's half have landed
                mbar_wait(&bars[2 + b], (fph >> b) & 1);
                TRACE(11);
                mbar_wait_cluster(&bars[4 + b], (fph >> b) & 1);
            }
            TRACE(1);
            tc_fence_after();
            const uint32_t hb = hbuf_addr + b * HB;
            const int ks0 = w * (Hq / 16 / NISSUE), ks1 = ks0 + Hq / 16 / NISSUE;
            for (int ks = ks0; ks < ks1; ++ks)  // K step = 16N bytes of the half B buffer
                mma_f16_ts2_w(tmem + DCOL + w * N, tmem + ks * 8, sdesc_noswz(hb + ks * 32 * NH, 16 * NH, 128), idesc,
                              ks != ks0);
            mma_commit2_w(&bars[1], pair_mask);
            TRACE(2);
        } else if (pr == 1 && threadIdx.x == 0 && s > 0) {
            // odd CTA: its half of h_{s-1} landed -> tell the even CTA, which reads it in the MMA
            mbar_wait(&bars[2 + b], (fph >> b) & 1);
            TRACE(11);
            mbar_remote_arrive(mapa_shared(smem_u32(&bars[4 + b]), c ^ 1));
            TRACE(1);
            TRACE(2);
        }
        if (s > 0) fph ^= 1u << b;
        if (s > 0) store_step(t_prev, frm_prev, fmq_prev);
        TRACE(12);
        // this step's Z block and mask row (issued two steps ahead)
        mbar_wait(&bars[6 + b], (s >> 1) & 1);
        const uint8_t *zs = zin + b * ZSLOT;
        // frame-valid bits of this warp's columns (lane i reads the mask byte of column i)
        const uint32_t frm = __ballot_sync(0xffffffffu, l < NQ && zs[ZB + nq0 + l] != 0);
        TRACE(13);
        mbar_wait(&bars[1], mma_phase);
        mma_phase ^= 1;
        tc_fence_after();
        TRACE(3);

        {
            uint32_t v[NISSUE][NQ];
            float zv[NQ];
#pragma unroll
            for (int i = 0; i < NQ / 4; ++i) {
                const float4 z4 = reinterpret_cast<const float4 *>(zs)[((cb * 128 + 32 * q + l) * NQ) / 4 + i];
                zv[4 * i] = z4.x; zv[4 * i + 1] = z4.y; zv[4 * i + 2] = z4.z; zv[4 * i + 3] = z4.w;
            }
            const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + DCOL + nq0;
#pragma unroll
            for (int k4 = 0; k4 < NISSUE; ++k4) tmem_ld_nowait<NQ>(ta + k4 * N, v[k4]);
            tmem_ld_wait();
#pragma unroll
            for (int k4 = 0; k4 < NISSUE; ++k4) pin_regs<NQ>(v[k4]);
            TRACE(8);
#pragma unroll
            for (int i = 0; i < NQ; ++i) {
                float pre = __uint_as_float(v[0][i]);
#pragma unroll
                for (int k4 = 1; k4 < NISSUE; ++k4) pre += __uint_as_float(v[k4][i]);
                act[i] = gate_act(pre + zv[i], gam);
            }
        }
        TRACE(9);
        tc_fence_before();
        uint32_t fmq = 0;  // bit m: owned column 4m+gam is a valid frame
        // this warp's columns lie in one column half (NQ divides N/2)
        const int hh = nq0 / NH;
        uint8_t *sg = stg + (b * 2 + hh) * SGh;
#pragma unroll
        for (int m = 0; m < NMQ; ++m) {
            float a4[4] = {act[4 * m], act[4 * m + 1], act[4 * m + 2], act[4 * m + 3]};
            float gv[4];
            xpose4(a4, gv, gam);  // gv = (i, f, g, o) of unit j at column 4m + gam
            const int i = 4 * m + gam;
            const bool fm = ((frm >> i) & 1) && unit_ok;
            // computed for every lane, kept by select (no divergent branch; padded columns may
            // hold garbage, which the select discards)
            const float cn = gv[1] * c_st[m] + gv[0] * gv[2];
            const float hn = gv[3] * tanh_f(cn);
            c_st[m] = fm ? cn : c_st[m];
            h_st[m] = fm ? hn : h_st[m];
            fmq |= (uint32_t)fm << m;
            // staged slice in the B-operand block format: unit jl -> k chunk q, byte (jl%8)*2
            *reinterpret_cast<__half *>(sg + (q * NH + nq0 - hh * NH + i) * 16 + (jl & 7) * 2) = __float2half_rn(h_st[m]);
        }
        TRACE(10);
        fence_async_smem();
        TRACE(7);
        if (zcheck) {
            if (zseen < (uint32_t)p.zflag_target) spin_until_geq(zf + zfront, (uint32_t)p.zflag_target);
            zfront += dir;
            z_wait(dir > 0 ? t + 2 : t - 2);  // rare: the step spans a further M-tile
        }
        // the previous step's bulk copies (of the other staging buffer) have long finished reading;
        // this __syncthreads orders that before the rewrite of that buffer at the next step
        if (l == 0 && w < NC) bulk_wait_read<0>();
        __syncthreads();
        TRACE(4);
        if (l == 0 && w < NC && s + 1 < T) {
            // h_s of this CTA, the column half CTA w holds -> hbuf[b^1] (block c) of CTA w
            // (16 warps send in parallel)
            bulk_s2c(mapa_shared(hbuf_addr + (b ^ 1) * HB + c * SGh, w), stg_addr + (b * 2 + (w & 1)) * SGh, SGh,
                     mapa_shared(full_addr + 8 * (b ^ 1), w));
            bulk_commit();
        }
        if (threadIdx.x == 0 && s > 0 && s + 2 < T) mbar_arrive_expect_tx(&bars[2 + b], NC * SGh);  // full[b]: step s+2
        TRACE(5);
        t_prev = t;
        frm_prev = frm;
        fmq_prev = fmq;
        TRACE(6);
    }
    if (T > 0) store_step(t_prev, frm_prev, fmq_prev);
#pragma unroll
    for (int m = 0; m < NMQ; ++m) {
        const int i = 4 * m + gam, b = bq0 + i;
        if (((cm >> i) & 1) && unit_ok) {
            if (p.hT) p.hT[(long)d * B * H + (long)b * H + j] = h_st[m];
            if (p.cT) p.cT[(long)d * B * H + (long)b * H + j] = c_st[m];
        }
    }
    if (l == 0 && w < NC) bulk_wait_read<0>();  // outgoing copies done with the staging buffers
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // both CTAs of every pair are done (the pair MMAs wrote both TMEMs)
    if (w == 0) {
        tc_fence_after();
        tmem_dealloc2(tmem, TCOLS);
    }
}

// ---------------------------------------------------------------------------
// backward through time
// ---------------------------------------------------------------------------
// CTA pairs (cluster ranks 2p, 2p+1; see the forward): the pair owns the 256 gate columns of its
// 64 units.  Per step it computes P_p[Hq x N] = R[:, cols_p] . dA_p^T as cta_group::2 MMAs with
// K = those 256 columns and M = 256-unit tiles, CTA r of the pair holding unit rows
// 256mt + 128r + [0, 128) of tile mt (in TMEM, A operand) and batch columns [rN/2, (r+1)N/2) of
// dA (smem, B operand).  Each CTA computes dA for its own 128 gate columns and all N batch columns
// and st.async's the half its partner holds (4 KB at N=32).  P rows are partial sums over the
// pair's 256 gate columns, so every owner gathers NC/2 partials (not NC) and every CTA sends NC/2
// blocks: half the DSMEM bytes of a per-CTA decomposition.
// smem: [region0: R slices (TMA, start only) | aliased later by slots[2] + stg[2]] [dAs] [in ring]
//       [barriers]
//   slots[b][src pair][32 rows][N] fp16: partial dh (x 2^DA_SHIFT x P_SCALE) of this CTA's 32
//   units from source pair src, 16-byte chunks swizzled by row (pswz): conflict-free gather
constexpr float P_SCALE = 1.f / 16.f;  // keeps the fp16 partials far from overflow
//   stg[b][block][32 rows][N] fp16: this CTA's partial rows per destination owner (same swizzle)
//   dAs[4 x 64-column blocks][N/2 rows][128 B] fp16, K-major SW128: the pair's 256 gate columns
//   (the even CTA's first) for this CTA's batch-column half
static __host__ __device__ size_t bwd_region0(int Hq, int N, int NC) {
    const size_t rs = (size_t)Hq / 64 * 16384, sl = 2 * (size_t)NC * 32 * N * 2;
    return rs > sl ? rs : sl;
}
// byte offset of element (row r, column n) in a P block [32 rows][N] fp16: the 16-byte chunk index
// is XORed with a row function, so the gather's warp access (8 rows x 4 adjacent columns) hits 8
// distinct 4-bank groups
template <int N>
DEVI uint32_t pswz(int r, int n) {
    constexpr int RB = 2 * N, CH = RB / 16, RPL = 128 / RB > 1 ? 128 / RB : 1;
    const int f = (r / RPL) % CH;
    return (uint32_t)(r * RB + ((((2 * n) >> 4) ^ f) << 4) + ((2 * n) & 15));
}

template <int NT, int MT2>
__global__ void __launch_bounds__(REC_THREADS, 1)
    lstm_rec_bwd_kernel(const __grid_constant__ CUtensorMap tmR, const __grid_constant__ CUtensorMap tmC,
                        const __grid_constant__ CUtensorMap tmDY, RecParams p) {
    constexpr int N = 16 * NT;
    constexpr int NH = N / 2;  // batch columns of the B operand held by each CTA of a pair
    constexpr int NQ = N / 4;
    constexpr int NMQ = NQ / 4;
    if (p.started && threadIdx.x == 0) atomicAdd(p.started, 1u);
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    const int Hq = p.Hq, NC = p.NC;
    // MT2 = Hq / 256 pair M tiles (256 units); KP K parts per tile: 4 issuing warps, one
    // accumulator each
    constexpr int KP = 4 / MT2;
    const int NSRC = NC / 2;       // source pairs = P blocks per slot buffer = blocks sent per CTA
    constexpr uint32_t BLK = 32 * N * 2;  // one (owner, source) block
    const uint32_t SLOTB = (uint32_t)NSRC * BLK;
    const uint32_t SLOT_TX = SLOTB;
    constexpr uint32_t DA_TX = 128 * NH * 2;  // dA bytes the partner sends per step
    uint8_t *Rs = smem;
    uint8_t *slots = smem;               // [2][NSRC][BLK], aliases Rs after the TMEM load
    uint8_t *stgp = smem + 2 * SLOTB;    // [2][NSRC][BLK]
    uint8_t *dAs = smem + bwd_region0(Hq, N, NC);  // [4][NH][128 B]
    // per-step inputs, loaded by one thread with bulk / TMA copies one step ahead (bwd_in_bytes); a
    // per-thread cp.async of these scattered values cost ~0.7 us of issue per step:
    //   inr[2]: dy tile [N rows][32 units] fp32 (TMA, SW128), the CTA's gate block (512 x NQ fp16,
    //           CTA-native), the mask row (N bytes); slot k&1 for processing index k
    //   cring[3]: c tile [N rows][32 units] fp32 (TMA, SW128); slot k%3 holds c(t_k), so step k reads
    //           c_t from slot k%3 and c_{t-dir} = c(t_{k+1}) from slot (k+1)%3: one c tile per step
    constexpr uint32_t TILE = N * 128, IN_G = 512 * NQ * 2, IN_SLOT = TILE + IN_G + 1024;
    uint8_t *inr = dAs + 4 * NH * 128;
    uint8_t *cring = inr + 2 * IN_SLOT;
    // [0] tma, [1] mma (pair commits), [2..3] slots full[b], [4] dfull (partner's dA half landed),
    // [5] dpair (even CTA: the odd CTA's B operand is complete), [6..7] inb[slot] (inputs landed)
    uint64_t *bars = (uint64_t *)(cring + 3 * TILE);
    uint32_t *tslot = (uint32_t *)(bars + 8);

    const int c = (int)cluster_ctarank();
    const int pr = c & 1;
    const uint16_t pair_mask = (uint16_t)(3u << (c & ~1));
    const int grp = blockIdx.x / NC;
    const int g = grp % p.G;
    const int d = grp / p.G;
    const int dir = d == 0 ? p.dir0 : -1;
    const int w = warp_uniform(warp_id()), q = w & 3, cb = w >> 2, l = lane_id();
    const int jl = 8 * q + (l >> 2), gam = l & 3;
    const int j = c * REC_UNITS + jl;
    const bool unit_ok = j < p.H;
    const int B = p.B, T = p.T, H = p.H;
    const int b0 = g * p.Bg;
    const int nq0 = cb * NQ;
    const int bq0 = b0 + nq0;
    constexpr uint32_t TCOLS = 512;
    // TMEM: pair tile mt of A at columns [128mt, 128mt+128): lanes = this CTA's units 256mt+128pr+lane,
    // two fp16 gate columns (pair K order) per 32-bit column.  Accumulators D_w[128 x N] at
    // Hq/2 + w*N: warp w issues tile w / KP, K part w % KP.
    const uint32_t DCOL = Hq / 2;
    const float inv_scale = 1.f / ((float)(1 << DA_SHIFT) * P_SCALE);
    const float scale = (float)(1 << DA_SHIFT);

    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 4);
        mbar_init(&bars[2], 1);
        mbar_init(&bars[3], 1);
        mbar_init(&bars[4], 1);
        mbar_init(&bars[5], 1);
        mbar_init(&bars[6], 1);
        mbar_init(&bars[7], 1);
        fence_mbar_init();
    }
    if (w == 0) {  // one warp of each CTA of the pair
        tmem_alloc2(tslot, TCOLS);
        tmem_relinquish2();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t idesc = idesc_f16(256, N, 0, 0);

    uint32_t cm = 0;
#pragma unroll
    for (int i = 0; i < NQ; ++i)
        if (nq0 + i < p.Bg && bq0 + i < B) cm |= 1u << i;

    // R^T rows of both slices of the pair (gate columns), unit columns of this CTA's rows:
    // box (si, mt, h) = slice si (0: even CTA), units 256mt + 128pr + 64h .. +64
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmR);
        mbar_arrive_expect_tx(&bars[0], (uint32_t)(2 * MT2 * 2) * 16384);
        for (int si = 0; si < 2; ++si)
            for (int mt = 0; mt < MT2; ++mt)
                for (int h = 0; h < 2; ++h)
                    tma_load_2d(Rs + ((si * MT2 + mt) * 2 + h) * 16384, &tmR, &bars[0], 256 * mt + 128 * pr + 64 * h,
                                d * 4 * Hq + ((c & ~1) + si) * 128);
    }
    mbar_wait(&bars[0], 0);
    // -> TMEM: lane u = unit 256mt + 128pr + u, column 128mt + kk/2 holds gate columns kk, kk+1 of
    // the pair (kk < 128: the even CTA's slice)
    {
        const int u = 32 * q + l;
        const int cw = Hq / 8;
        for (int col = cb * cw; col < (cb + 1) * cw; col += 16) {
            const int mt = col >> 7, kk0 = (col & 127) * 2, si = kk0 >> 7, r0 = kk0 & 127;
            const uint8_t *rk = Rs + ((si * MT2 + mt) * 2 + (u >> 6)) * 16384 + (u & 7) * 2;
            const int chunk = (u & 63) >> 3;
            uint32_t v[16];
#pragma unroll
            for (int uu = 0; uu < 16; ++uu) {
                const int r = r0 + 2 * uu;
                const uint16_t lo = *reinterpret_cast<const uint16_t *>(rk + r * 128 + ((chunk ^ (r & 7)) << 4));
                const uint16_t hi =
                    *reinterpret_cast<const uint16_t *>(rk + (r + 1) * 128 + ((chunk ^ ((r + 1) & 7)) << 4));
                v[uu] = (uint32_t)lo | ((uint32_t)hi << 16);
            }
            tmem_st16(tmem + ((uint32_t)(32 * q) << 16) + col, v);
        }
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // P produced at processing index k lands in slots[k&1] and is consumed at index k+1
    // (index T = the final gather for dh0)
    if (threadIdx.x == 0) {
        if (T >= 1) mbar_arrive_expect_tx(&bars[2], SLOT_TX);  // index 1 <- P of index 0
        if (T >= 2) mbar_arrive_expect_tx(&bars[3], SLOT_TX);  // index 2 <- P of index 1
        if (T >= 1) mbar_arrive_expect_tx(&bars[4], DA_TX);    // the partner's dA of index 0
    }
    cluster_sync();  // every CTA done with its R staging before peers write into the slots

    float dh[NMQ], dc[NMQ], dbp[4] = {0.f, 0.f, 0.f, 0.f};
    uint32_t pfm = 0;  // bit m: the previous step's frame was valid for owned column 4m+gam
#pragma unroll
    for (int m = 0; m < NMQ; ++m) {
        const int i = 4 * m + gam, b = bq0 + i;
        const bool ok = ((cm >> i) & 1) && unit_ok;
        dh[m] = (ok && p.dhT) ? p.dhT[(long)d * B * H + (long)b * H + j] : 0.f;
        dc[m] = (ok && p.dcT) ? p.dcT[(long)d * B * H + (long)b * H + j] : 0.f;
    }
    uint32_t fph = 0;
    // wait for the cluster's partials of index k-1 and sum this CTA's rows in fixed order
    auto gather = [&](int k) {
        const int b = (k - 1) & 1;
        mbar_wait(&bars[2 + b], (fph >> b) & 1);
        fph ^= 1u << b;
        if (threadIdx.x == 0 && k + 2 <= T) mbar_arrive_expect_tx(&bars[2 + b], SLOT_TX);  // index k+2
#pragma unroll
        for (int m = 0; m < NMQ; ++m) {
            if ((pfm >> m) & 1) {
                const uint8_t *sl = slots + b * SLOTB + pswz<N>(jl, nq0 + 4 * m + gam);
                float acc = 0.f;
                for (int src = 0; src < NSRC; ++src)
                    acc += __half2float(*reinterpret_cast<const __half *>(sl + src * BLK));
                dh[m] = acc * inv_scale;
            }
        }
    };
    const long nat_step = (long)p.ndir * p.G * NC * 512 * NQ;

    // saved state of one step (independent of the recurrence), one step ahead: one thread issues the
    // copies for processing index k into ring slot k&1, and c(t_{k+1}) into cring[(k+1)%3]
    const int tid = threadIdx.x;
    const long nat_cta = (((long)d * p.G + g) * NC + c) * 512 * NQ;
    const int crows = p.ldc ? (int)(p.c_doff / p.ldc) : 0;  // rows per direction of the C array
    auto t_of = [&](int k) { return dir > 0 ? T - 1 - k : k; };
    auto issue_in = [&](int k, bool with_c0) {
        const int tk = t_of(k), sl = k & 1;
        uint8_t *slot = inr + sl * IN_SLOT;
        const bool cnext = k + 1 < T;
        mbar_arrive_expect_tx(&bars[6 + sl], TILE + IN_G + N + (cnext ? TILE : 0) + (with_c0 ? TILE : 0));
        tma_load_2d(slot, &tmDY, &bars[6 + sl], d * (int)p.dy_doff + 32 * c, tk * B + b0);
        bulk_g2s(smem_u32(slot + TILE), p.gates + tk * nat_step + nat_cta, IN_G, &bars[6 + sl]);
        bulk_g2s(smem_u32(slot + TILE + IN_G), p.maskN + ((long)tk * p.G + g) * N, N, &bars[6 + sl]);
        if (with_c0) tma_load_2d(cring + (k % 3) * TILE, &tmC, &bars[6 + sl], 32 * c, d * crows + tk * B + b0);
        if (cnext) tma_load_2d(cring + ((k + 1) % 3) * TILE, &tmC, &bars[6 + sl], 32 * c, d * crows + t_of(k + 1) * B + b0);
    };
    constexpr int IN_THREAD = 128;  // lane 0 of warp 4: not an MMA-issuing warp
    if (threadIdx.x == IN_THREAD && T > 0) {
        tma_prefetch_desc(&tmC);
        tma_prefetch_desc(&tmDY);
        issue_in(0, true);
    }
    // element (row n, unit jl) of a [N rows][32 fp32] SW128 tile
    auto tile_f32 = [&](const uint8_t *tile, int n) {
        return *reinterpret_cast<const float *>(tile + n * 128 + ((((jl >> 2) ^ n) & 7) << 4) + (jl & 3) * 4);
    };
    // c before the sequence (for the last processed frame): c0 or 0
    float c0v[NMQ];
#pragma unroll
    for (int m = 0; m < NMQ; ++m) {
        const int i = 4 * m + gam, b = bq0 + i;
        c0v[m] = (((cm >> i) & 1) && unit_ok && p.c0) ? p.c0[(long)d * B * H + (long)b * H + j] : 0.f;
    }
    float graw[NQ], ct[NMQ], cp[NMQ], dyv[NMQ];

    uint32_t mma_phase = 0;
    const uint32_t das_addr = smem_u32(dAs);
    const uint32_t slots_addr = smem_u32(slots), full_addr = smem_u32(&bars[2]);
    const uint32_t das_peer = mapa_shared(das_addr, c ^ 1), dfull_peer = mapa_shared(smem_u32(&bars[4]), c ^ 1);
    // this warp's batch columns lie in one column half (NQ divides N/2): local or the partner's
    const int hh = nq0 / NH;
#ifdef BLSTM_TRACE
    unsigned long long *trace = (blockIdx.x == BLSTM_TRACE_CTA && threadIdx.x == 0) ? p.trace : nullptr;
#endif
    for (int s = T - 1; s >= 0; --s) {
        const int t = dir > 0 ? s : T - 1 - s;
        const int k_done = T - 1 - s;
        TRACE(0);
        // the next step's inputs: its ring slots were last read one step ago
        if (threadIdx.x == IN_THREAD && k_done + 1 < T) issue_in(k_done + 1, false);
        TRACE(1);
        // ---- dh_t from the previous step's partials ----
        if (k_done > 0) gather(k_done);
        TRACE(2);
        // ---- this step's saved state (issued one step ago) ----
        mbar_wait(&bars[6 + (k_done & 1)], (k_done >> 1) & 1);
        uint32_t mraw;
        {
            const uint8_t *in = inr + (k_done & 1) * IN_SLOT;
            const __half2 *gh = reinterpret_cast<const __half2 *>(in + TILE + tid * NQ * 2);
#pragma unroll
            for (int i = 0; i < NQ; i += 2) {
                const float2 f2 = __half22float2(gh[i / 2]);
                graw[i] = f2.x;
                graw[i + 1] = f2.y;
            }
            const uint8_t *ctile = cring + (k_done % 3) * TILE, *ptile = cring + ((k_done + 1) % 3) * TILE;
#pragma unroll
            for (int m = 0; m < NMQ; ++m) {
                const int n = nq0 + 4 * m + gam;
                ct[m] = tile_f32(ctile, n);
                cp[m] = k_done + 1 < T ? tile_f32(ptile, n) : c0v[m];
                dyv[m] = tile_f32(in, n);
            }
            mraw = l < NQ ? in[TILE + IN_G + nq0 + l] : 0;
        }
        // ---- gate gradients ----
        const uint32_t frm = __ballot_sync(0xffffffffu, mraw != 0);
        pfm = 0;
        TRACE(8);
        uint2 pks[NMQ];
#pragma unroll
        for (int m = 0; m < NMQ; ++m) {
            float a4[4] = {graw[4 * m], graw[4 * m + 1], graw[4 * m + 2], graw[4 * m + 3]};
            float gv[4];
            xpose4(a4, gv, gam);
            const int i = 4 * m + gam, n = nq0 + i;
            const bool fm = ((frm >> i) & 1) && unit_ok;
            // computed for every lane, kept by select (no divergent branch)
            const float ig = gv[0], f = gv[1], gg = gv[2], o = gv[3];
            const float th = tanh_f(ct[m]);
            const float dH = dh[m] + dyv[m];
            const float dC = dc[m] + dH * o * (1.f - th * th);
            const float da0 = fm ? dC * gg * ig * (1.f - ig) : 0.f;
            const float da1 = fm ? dC * cp[m] * f * (1.f - f) : 0.f;
            const float da2 = fm ? dC * ig * (1.f - gg * gg) : 0.f;
            const float da3 = fm ? dH * th * o * (1.f - o) : 0.f;
            dc[m] = fm ? dC * f : dc[m];
            dbp[0] += da0; dbp[1] += da1; dbp[2] += da2; dbp[3] += da3;
            pfm |= (uint32_t)fm << m;
            __half2 lo = __floats2half2_rn(da0 * scale, da1 * scale);
            __half2 hi = __floats2half2_rn(da2 * scale, da3 * scale);
            uint2 pk;
            pk.x = *reinterpret_cast<uint32_t *>(&lo);
            pk.y = *reinterpret_cast<uint32_t *>(&hi);
            // B operand position: row n - hh*NH of the CTA holding half hh, pair K column 128pr + 4jl
            const uint32_t off = sw128_offset(n - hh * NH, 128 * pr + 4 * jl, NH);
            if (hh == pr) *reinterpret_cast<uint2 *>(dAs + off) = pk;
            else st_async_v2u(das_peer + off, pk.x, pk.y, dfull_peer);
            pks[m] = pk;
        }
        TRACE(9);
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        TRACE(3);
        if (pr == 0 && w < 4) {  // even CTA: warp-collective issue of tile w / KP, K part w % KP
            // the partner's dA half has landed here, and the partner's own B operand is complete
            mbar_wait_cluster(&bars[4], k_done & 1);
            TRACE(12);
            mbar_wait_cluster(&bars[5], k_done & 1);
            TRACE(13);
            if (threadIdx.x == 0 && k_done + 1 < T) mbar_arrive_expect_tx(&bars[4], DA_TX);
            tc_fence_after();
            const int mt = w / KP, kp = w % KP, kpn = 16 / KP;  // K steps of 16 per part
#pragma unroll 1
            for (int ks = kp * kpn; ks < (kp + 1) * kpn; ++ks)  // 64 gate columns per SW128 block
                mma_f16_ts2_w(tmem + DCOL + w * N, tmem + 128 * mt + ks * 8,
                              sdesc_sw128(das_addr + (ks >> 2) * NH * 128 + (ks & 3) * 32, 16, 1024), idesc,
                              ks != kp * kpn);
            mma_commit2_w(&bars[1], pair_mask);
        } else if (pr == 1 && threadIdx.x == 0) {
            // odd CTA: the even CTA's dA half landed and this CTA's own part is written -> relay
            mbar_wait_cluster(&bars[4], k_done & 1);
            if (k_done + 1 < T) mbar_arrive_expect_tx(&bars[4], DA_TX);
            mbar_remote_arrive(mapa_shared(smem_u32(&bars[5]), c ^ 1));
        }
        // while the MMA runs: dA of this step to global memory for the weight / input GEMMs
#pragma unroll
        for (int m = 0; m < NMQ; ++m) {
            const int i = 4 * m + gam;
            if ((cm >> i) & 1)
                *reinterpret_cast<uint2 *>(p.dA + ((long)t * B + bq0 + i) * p.ldda + (long)d * 4 * Hq + 4 * j) = pks[m];
        }
        TRACE(10);
        mbar_wait(&bars[1], mma_phase);
        mma_phase ^= 1;
        tc_fence_after();
        TRACE(4);
        // rows of tile mt, lane quarter q = units 256mt + 128pr + 32q + l belong to owner
        // c' = 8mt + 4pr + q (its local row l): stage P = sum of the tile's K parts (fp16) per owner,
        // then warp w (< NSRC) bulk-copies block w into its owner's slot for this pair
        {
            const int kb = k_done & 1;
            constexpr int NACC = 4;
            uint32_t v[NACC][NQ];
#pragma unroll
            for (int a = 0; a < NACC; ++a) tmem_ld_nowait<NQ>(tmem + ((uint32_t)(32 * q) << 16) + DCOL + a * N + nq0, v[a]);
            tmem_ld_wait();
#pragma unroll
            for (int a = 0; a < NACC; ++a) pin_regs<NQ>(v[a]);
            TRACE(11);
#pragma unroll
            for (int mt = 0; mt < MT2; ++mt) {
                uint32_t hv[NQ / 2];
#pragma unroll
                for (int i = 0; i < NQ; i += 2) {
                    float s0 = 0.f, s1 = 0.f;
#pragma unroll
                    for (int a = 0; a < NACC; ++a)
                        if (a / KP == mt) {
                            s0 += __uint_as_float(v[a][i]);
                            s1 += __uint_as_float(v[a][i + 1]);
                        }
                    __half2 h2 = __floats2half2_rn(s0 * P_SCALE, s1 * P_SCALE);
                    hv[i / 2] = *reinterpret_cast<uint32_t *>(&h2);
                }
                uint8_t *blk = stgp + ((uint32_t)kb * NSRC + 4 * mt + q) * BLK;
                if constexpr (NQ == 4) {
                    *reinterpret_cast<uint2 *>(blk + pswz<N>(l, nq0)) = make_uint2(hv[0], hv[1]);
                } else {
#pragma unroll
                    for (int i = 0; i < NQ / 8; ++i)
                        *reinterpret_cast<uint4 *>(blk + pswz<N>(l, nq0 + 8 * i)) =
                            make_uint4(hv[4 * i], hv[4 * i + 1], hv[4 * i + 2], hv[4 * i + 3]);
                }
            }
            tc_fence_before();
            fence_async_smem();
            TRACE(6);
            // the previous step's bulk copies (other staging buffer) are done reading; this
            // __syncthreads orders that before the rewrite of that buffer at the next step
            if (l == 0 && w < NSRC) bulk_wait_read<0>();
            __syncthreads();
            TRACE(7);
            if (l == 0 && w < NSRC) {
                const int owner = 8 * (w >> 2) + 4 * pr + (w & 3);
                bulk_s2c(mapa_shared(slots_addr + kb * SLOTB + (c >> 1) * BLK, owner),
                         smem_u32(stgp) + ((uint32_t)kb * NSRC + w) * BLK, BLK, mapa_shared(full_addr + 8 * kb, owner));
                bulk_commit();
            }
        }
        TRACE(5);
    }
#undef TRACE
    if (T > 0) gather(T);
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
    float *dbs = reinterpret_cast<float *>(dAs);  // [4 cb][128 rows] (2 KB <= dAs); the last MMA is done
    cluster_sync();  // the partner's last st.async into dAs (and its MMA reads) are complete
    dbs[cb * 128 + 4 * jl + gam] = sel4(dbp, gam);
    __syncthreads();
    if (cb == 0) {
        const int r = 4 * jl + gam;
        p.dbpart[((long)d * p.G + g) * 4 * Hq + 4 * j + gam] = ((dbs[r] + dbs[128 + r]) + dbs[256 + r]) + dbs[384 + r];
    }
    if (l == 0 && w < NSRC) bulk_wait_read<0>();  // outgoing copies done with the staging buffers
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // no peer still writes into this CTA's slots; both CTAs of the pair are done
    if (w == 0) {
        tc_fence_after();
        tmem_dealloc2(tmem, TCOLS);
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
    pl.Hq = round_up(H, 256);  // BPTT pair tiles are 256 units (two CTAs x 128)
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

static size_t fwd_smem(const RecPlan &pl) { return fwd_region0(pl.Hq, pl.N) + 1024 + 128; }
// per-step input rings of the BPTT kernel (see IN_SLOT / cring there)
static size_t bwd_in_bytes(int N) { return 2 * ((size_t)N * 128 + 512 * (N / 4) * 2 + 1024) + 3 * (size_t)N * 128; }
static size_t bwd_smem(const RecPlan &pl) {
    return bwd_region0(pl.Hq, pl.N, pl.NC) + 2 * pl.N * 128 + bwd_in_bytes(pl.N) + 1024 + 64;
}

bool rec_supported(const RecPlan &pl, int H) {
    if (H < 1 || (pl.N != 16 && pl.N != 32 && pl.N != 64)) return false;
    if (pl.NC > 16) return false;  // one cluster (<= 16 CTAs, non-portable size) per group
    if (fwd_smem(pl) > 227 * 1024 || bwd_smem(pl) > 227 * 1024) return false;
    if (pl.ndir * pl.G * pl.NC > num_sms()) return false;
    if (pl.Hq / 2 + 4 * pl.N > 512) return false;  // TMEM: resident R + 4 accumulators (both kernels)
    return pl.Hq == 256 || pl.Hq == 512;  // one cluster of <= 16 CTAs; BPTT tiles of 256 units
}

size_t rec_P_bytes(const RecPlan &pl) {
    (void)pl;
    return 256;  // partials travel through distributed shared memory
}

template <typename Kern, typename... Args>
static cudaError_t launch_cluster_ex(Kern kern, int grid, int cluster, size_t smem, cudaStream_t st, bool pdl,
                                     Args... args) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (cluster > 8) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(REC_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}
template <typename Kern, typename... Args>
static cudaError_t launch_cluster(Kern kern, int grid, int cluster, size_t smem, cudaStream_t st, Args... args) {
    return launch_cluster_ex(kern, grid, cluster, smem, st, false, args...);
}

static unsigned long long *g_trace_fwd = nullptr, *g_trace_bwd = nullptr;
unsigned long long *rec_trace_fwd() { return g_trace_fwd; }
unsigned long long *rec_trace_bwd() { return g_trace_bwd; }
void rec_set_trace(unsigned long long *fwd, unsigned long long *bwd) {
    g_trace_fwd = fwd;
    g_trace_bwd = bwd;
}

int lstm_rec_fwd(const RecParams &p_in, const __half *RT16, cudaStream_t st) {
    RecParams p = p_in;
    if (g_trace_fwd) p.trace = g_trace_fwd;
    if (p.T == 0) return 0;
    CUtensorMap tmR;
    if (make_tmap_f16(&tmR, RT16, p.Hq, (uint64_t)p.ndir * 4 * p.Hq, p.Hq, 128)) return -2;
    RecPlan pl{p.Hq, p.NC, p.G, p.Bg, p.N, p.ndir};
    const int grid = p.ndir * p.G * p.NC;
    const size_t smem = fwd_smem(pl);
    ProfScope ps(PROF_REC_FWD, st);
    note_launch();
    cudaError_t e;
    switch (p.N) {
        case 16: e = launch_cluster_ex(lstm_rec_fwd_kernel<1>, grid, p.NC, smem, st, p.rerun != nullptr, tmR, p); break;
        case 32: e = launch_cluster_ex(lstm_rec_fwd_kernel<2>, grid, p.NC, smem, st, p.rerun != nullptr, tmR, p); break;
        case 64: e = launch_cluster_ex(lstm_rec_fwd_kernel<4>, grid, p.NC, smem, st, p.rerun != nullptr, tmR, p); break;
        default: return -6;
    }
    return e == cudaSuccess ? 0 : -5;
}

int lstm_rec_bwd(const RecParams &p_in, const __half *RT16, cudaStream_t st) {
    RecParams p = p_in;
    if (g_trace_bwd) p.trace = g_trace_bwd;
    if (p.T == 0) return 0;
    CUtensorMap tmR, tmC, tmDY;
    if (make_tmap_f16(&tmR, RT16, p.Hq, (uint64_t)p.ndir * 4 * p.Hq, p.Hq, 128)) return -2;
    // c and dy tiles [N rows][32 units] by TMA: C rows = ndir blocks of c_doff/ldc rows (or T*B)
    const uint64_t crows = p.c_doff ? (uint64_t)(p.ndir - 1) * (p.c_doff / p.ldc) + (uint64_t)p.T * p.B
                                    : (uint64_t)p.T * p.B;
    if (make_tmap_f32_rows(&tmC, p.C, p.ldc, crows, p.ldc, p.N)) return -3;
    if (make_tmap_f32_rows(&tmDY, p.dy, p.lddy, (uint64_t)p.T * p.B, p.lddy, p.N)) return -3;
    RecPlan pl{p.Hq, p.NC, p.G, p.Bg, p.N, p.ndir};
    const int grid = p.ndir * p.G * p.NC;
    const size_t smem = bwd_smem(pl);
    ProfScope ps(PROF_REC_BWD, st);
    note_launch();
    cudaError_t e;
#define BWD_CASE(n, mt2)                                                                                  \
    if (p.N == 16 * (n) && p.Hq == 256 * (mt2)) {                                                         \
        e = launch_cluster(lstm_rec_bwd_kernel<n, mt2>, grid, p.NC, smem, st, tmR, tmC, tmDY, p);         \
    } else
    BWD_CASE(1, 1) BWD_CASE(2, 1) BWD_CASE(4, 1) BWD_CASE(1, 2) BWD_CASE(2, 2) BWD_CASE(4, 2) { return -6; }
#undef BWD_CASE
    return e == cudaSuccess ? 0 : -5;
}

}  // namespace blstm
