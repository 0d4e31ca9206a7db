// rec_step.cu -- step-launched recurrence (rec_step.h).
//
// Forward step s (both directions; direction d processes frame t_d = s or T-1-s):
//   P_d = h_{t-1,d} R_d^T            tcgen05 GEMM, M = B, N = 4Hq, K = Hq (A = the h history slot)
//   a = P_d + Z[t_d]; i, f, o = sigma(a); g = tanh(a); c = f c_prev + i g; h = o tanh(c);
//   masked frame: state carried, outputs 0 (R2).
// BPTT step s (reverse order per direction):
//   dH = dh_in + dy_t; dc~ = dc + dH o (1 - tanh^2 c); dA = [dc~ g i(1-i), dc~ c_prev f(1-f),
//   dc~ i (1-g^2), dH tanh(c) o(1-o)]; dc <- dc~ f; masked: dA = 0, dh and dc pass through (R4);
//   dh_in of the next step = dA_t R_d (GEMM, M = B, N = Hq, K = 4Hq, split-K), or the carried dh
//   where frame t was masked.
#include "common.cuh"
#include "gemm.h"
#include "lstm_rec.h"
#include "prof.h"
#include "graph.h"
#include "rec_step.h"

namespace blstm {

// per-step GEMMs split K this many ways into fp32 partials, summed (fixed order) by the gate kernel
// that consumes them: 4x / 8x the CTAs of the unsplit GEMM and no reduction launch
constexpr int SF = 2;  // forward  h R^T: K = Hq (a multiple of 256); 2 x 2 directions x 32 tiles <= 148 SMs
constexpr int SB = 4;  // BPTT     dA R:  K = 4Hq; 2 dirs x 8 tiles x 4 = 64 CTAs beside the side GEMMs (BLSTM_STEP_SIDE_CTAS)

namespace {

DEVI float sg(float z) { return __fdividef(1.f, 1.f + __expf(-z)); }
DEVI float th(float z) { return 2.f * sg(2.f * z) - 1.f; }

// thread per (d, b, u), u < Hq
// every kernel of the step chain waits for its predecessor here (see launch_chain); before this
// point a kernel reads only data produced before the graph (Z, the mask, the forward's saved
// activations, dy), never anything the chain writes
DEVI void chain_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__global__ void step_fwd_gate_kernel(RecStepFwd p, int s) {
    const int Hq = p.Hq, B = p.B, T = p.T, G4 = p.ndir * 4 * Hq;
    // grid: x over units, y over (direction, batch row): no 64-bit index division
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    const int db = blockIdx.y, b = db % B, d = db / B;
    const int dir = d == 0 ? p.dir0 : -1;
    const int t = dir > 0 ? s : T - 1 - s;
    const long r = (long)t * B + b;
    const bool valid = u < Hq && p.mask[r] != 0 && u < p.H;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    if (valid) a = reinterpret_cast<const float4 *>(p.Z + r * G4 + (long)d * 4 * Hq)[u];  // before the wait
    chain_enter();
    if (u < Hq) {
        const int slot_prev = t + (dir < 0), slot_next = slot_prev + dir;
        __half *hn = p.hist + (((long)d * (T + 1) + slot_next) * B + b) * Hq + u;
        const float c_prev = s == 0 ? ((p.c0 && u < p.H) ? p.c0[((long)d * B + b) * p.H + u] : 0.f)
                                    : p.C[d * p.c_doff + (r - (long)dir * B) * p.ldc + u];
        // the fp32 state carried across masked frames (the history holds it in fp16 only)
        float *hc = p.P + (size_t)2 * SF * B * 4 * Hq + db * Hq + u;
        const float h_prev = s == 0 ? ((p.h0 && u < p.H) ? p.h0[((long)d * B + b) * p.H + u] : 0.f) : *hc;
        float c = c_prev, h = h_prev;
        float4 act = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid) {
            if (s > 0 || p.h0) {  // h_{t-1} R^T (at s = 0 from the h0 slot of the history)
#pragma unroll
                for (int k = 0; k < SF; ++k) {
                    const float4 q = reinterpret_cast<const float4 *>(p.P + (((long)d * SF + k) * B + b) * 4 * Hq)[u];
                    a.x += q.x; a.y += q.y; a.z += q.z; a.w += q.w;
                }
            }
            act = make_float4(sg(a.x), sg(a.y), th(a.z), sg(a.w));
            c = act.y * c_prev + act.x * act.z;
            h = act.w * th(c);
        }
        if (u < p.H) p.C[d * p.c_doff + r * p.ldc + u] = c;
        *hc = h;
        *hn = __float2half_rn(h);
        if (s == T - 1 && u < p.H) {  // state after the whole scan
            if (p.hT) p.hT[((long)d * B + b) * p.H + u] = h;
            if (p.cT) p.cT[((long)d * B + b) * p.H + u] = c;
        }
        if (p.y && u < p.H) p.y[r * p.ldy + d * p.y_doff + u] = valid ? h : 0.f;
        if (p.y16) p.y16[r * 2 * Hq + (long)d * Hq + u] = __float2half_rn(valid ? h : 0.f);
        __half2 *gp = reinterpret_cast<__half2 *>(p.gates + r * G4 + (long)d * 4 * Hq + 4 * u);
        gp[0] = __floats2half2_rn(act.x, act.y);
        gp[1] = __floats2half2_rn(act.z, act.w);
    }
}

__global__ void step_bwd_gate_kernel(RecStepBwd p, int s) {
    const int Hq = p.Hq, B = p.B, T = p.T, G4 = p.ndir * 4 * Hq;
    const float scale = (float)(1 << DA_SHIFT);
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    const int db = blockIdx.y, b = db % B, d = db / B;
    const int dir = d == 0 ? p.dir0 : -1;
    const int t = dir > 0 ? T - 1 - s : s;       // this step's frame (reverse of the forward scan)
    const long r = (long)t * B + b;
    const long sidx = db * Hq + u;               // [ndir][B][Hq] state index
    const bool valid = u < Hq && p.mask[r] != 0 && u < p.H;
    const bool prev_valid = s > 0 && p.mask[r + (long)dir * B] != 0;  // the frame of step s-1
    // the forward's saved activations and dy: produced before the graph, loaded before the wait
    float gi = 0.f, gf = 0.f, gg = 0.f, go = 0.f, c = 0.f, c_prev = 0.f, dy = 0.f;
    if (valid) {
        const __half2 *gp = reinterpret_cast<const __half2 *>(p.gates + r * G4 + (long)d * 4 * Hq + 4 * u);
        const float2 g01 = __half22float2(gp[0]), g23 = __half22float2(gp[1]);
        gi = g01.x; gf = g01.y; gg = g23.x; go = g23.y;
        c = p.C[d * p.c_doff + r * p.ldc + u];
        const int tp = t - dir;                  // the frame before t in the forward scan
        c_prev = (tp >= 0 && tp < T) ? p.C[d * p.c_doff + ((long)tp * B + b) * p.ldc + u]
                                     : (p.c0 ? p.c0[((long)d * B + b) * p.H + u] : 0.f);
        dy = p.dy[r * p.lddy + d * p.dy_doff + u];
    }
    chain_enter();
    if (u < Hq) {
        float dh_in = 0.f, dc = 0.f;
        if (s == 0 && u < p.H) {  // gradients at the end of the scan
            if (p.dhT) dh_in = p.dhT[((long)d * B + b) * p.H + u];
            if (p.dcT) dc = p.dcT[((long)d * B + b) * p.H + u];
        }
        if (s > 0) {
            if (prev_valid) {
                const long pb = (long)d * SB * B * Hq + (long)b * Hq + u;
#pragma unroll
                for (int k = 0; k < SB; ++k) dh_in += p.dhR[pb + (long)k * B * Hq];
            } else {
                dh_in = p.dhc[sidx];
            }
            dc = p.dcc[sidx];
        }
        __half2 *dap = reinterpret_cast<__half2 *>(p.dA + r * G4 + (long)d * 4 * Hq + 4 * u);
        if (!valid) {
            dap[0] = __floats2half2_rn(0.f, 0.f);
            dap[1] = __floats2half2_rn(0.f, 0.f);
            p.dhc[sidx] = dh_in;                 // pass through; dc unchanged
            if (s == 0) p.dcc[sidx] = dc;
            return;
        }
        const float dH = dh_in + dy;
        const float tc = th(c);
        const float dct = dc + dH * go * (1.f - tc * tc);
        const float da_i = dct * gg * gi * (1.f - gi);
        const float da_f = dct * c_prev * gf * (1.f - gf);
        const float da_g = dct * gi * (1.f - gg * gg);
        const float da_o = dH * tc * go * (1.f - go);
        dap[0] = __floats2half2_rn(da_i * scale, da_f * scale);
        dap[1] = __floats2half2_rn(da_g * scale, da_o * scale);
        p.dcc[sidx] = dct * gf;
    }
}

// dh0 / dc0 after the last BPTT step: dh = dA R of the last processed frame (its partials) where
// that frame was valid, else the carried dh; dc = the carried dc
__global__ void step_bwd_final_kernel(RecStepBwd p) {
    const int Hq = p.Hq, B = p.B, T = p.T;
    const long n = (long)p.ndir * B * p.H;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) {
        const int u = (int)(e % p.H);
        const long db = e / p.H;
        const int b = (int)(db % B), d = (int)(db / B);
        const int dir = d == 0 ? p.dir0 : -1;
        const int t = dir > 0 ? 0 : T - 1;  // the frame processed last
        const long sidx = db * Hq + u;
        if (p.dh0) {
            float v = 0.f;
            if (p.mask[(long)t * B + b]) {
                const long pb = (long)d * SB * B * Hq + (long)b * Hq + u;
#pragma unroll
                for (int k = 0; k < SB; ++k) v += p.dhR[pb + (long)k * B * Hq];
            } else {
                v = p.dhc[sidx];
            }
            p.dh0[e] = v;
        }
        if (p.dc0) p.dc0[e] = p.dcc[sidx];
    }
}

// The per-step kernels form one chain on one stream (gate kernel -> GEMM of both directions ->
// gate kernel ...).  With pdl each is a programmatic dependent of its predecessor: it is launched
// while the predecessor runs, and its prologue (for the GEMM: barriers, TMEM allocation, tensor-map
// prefetch) overlaps the predecessor's tail.  Every kernel waits for the predecessor's completion
// (griddepcontrol.wait) before it reads anything the chain produced or writes anything, so the
// reuse of P / dhR, the history and the state buffers from step to step stays ordered.
bool step_pdl() {
    const char *e = getenv("BLSTM_STEP_PDL");
    return !(e && e[0] == '0');
}
template <typename K, typename P>
int launch_chain(K kern, dim3 grid, cudaStream_t st, bool pdl, const P &p, int s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    note_launch();
    return cudaLaunchKernelEx(&cfg, kern, p, s) == cudaSuccess ? 0 : -5;
}

int grid_of(long n) {
    long g = (n + 255) / 256;
    return (int)(g < 1 ? 1 : (g > 148 * 8 ? 148 * 8 : g));
}

}  // namespace

// ---------------------------------------------------------------------------------------------
// Persistent forward (Hq <= 1024, B <= 128): the step chain above pays two launches and two grid
// completions per step.  Here one cooperative launch runs the whole scan.  Thread-block clusters of
// two CTAs, one cluster per (direction d, 128-column gate tile nt); cluster rank kh holds the K half
// [kh Hq/2, (kh+1) Hq/2) of the tile's R^T rows in shared memory for the whole scan (TMA, once).
// Per step s:
//   1. the TMA warp waits until every CTA of direction d published h_{s-1} (a per-direction counter,
//      release / acquire at gpu scope), then streams its K half of h_{t-1} (the history slot, the
//      MMA A operand, M = 128 batch rows) through a PF_S-stage ring;
//   2. one warp issues the tcgen05 MMAs: D[128 rows x 128 gate columns] = h_{t-1} R^T (K half);
//   3. the pair exchanges half of D through distributed shared memory: CTA kh finalizes gate columns
//      [64 kh, 64 kh + 64) of the tile (its 16 units) for all 128 rows and receives the partner's
//      partial sums for them, so all 8 warps finalize (8 cells per thread);
//   4. a = Z + P_0 + P_1 (the step chain's order), gates, cell update and mask as in
//      step_fwd_gate_kernel, with c and the fp32 h carried in registers; h_t -> the history (the
//      next step's A operand);
//   5. arrive on the direction's counter, then store C, y, y16 and the gates (off the critical path:
//      the counter's release covers only the history stores).
// ---------------------------------------------------------------------------------------------
#ifndef BLSTM_PF_THREADS
#define BLSTM_PF_THREADS 256  // 512 (4 units per thread) measured slower: C5 forward 33.4 vs 31.3 ms
#endif
constexpr int PF_THREADS = BLSTM_PF_THREADS;  // 256 or 512
#ifndef BLSTM_PTRACE_CTA
#define BLSTM_PTRACE_CTA 0  // the persistent step kernels' traced CTA (-1: the last, i.e. direction 1)
#endif
constexpr int PF_CH = PF_THREADS / 128;       // column chunks per TMEM lane quarter
constexpr int PF_CW = 64 / PF_CH;             // tile columns a thread finalizes (32 or 16)
constexpr int PF_UPT = PF_CW / 4;             // units a thread finalizes (8 or 4)
constexpr int PF_S = 4;                  // h ring stages (16 KB each: 128 rows x 64 K)
constexpr uint32_t PF_CHUNK = 16384;
constexpr uint32_t PF_RECV = 64 * 128 * 4;  // the partner's partial sums of this CTA's 64 columns
static size_t pf_smem(int Hq) { return (size_t)(Hq / 2 / 64) * PF_CHUNK + PF_S * PF_CHUNK + PF_RECV + 1024 + 256; }

__global__ void __launch_bounds__(PF_THREADS, 1)
    step_fwd_persist_kernel(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmR,
                            RecStepFwd p, uint32_t *cnt, unsigned long long *trace) {
#ifdef BLSTM_TRACE
#define PTR(k) \
    if (tr) tr[(size_t)s * 16 + (k)] = (unsigned long long)clock64()
    unsigned long long *tr = (blockIdx.x == (BLSTM_PTRACE_CTA < 0 ? gridDim.x - 1 : BLSTM_PTRACE_CTA) && threadIdx.x == 0)
                                 ? trace : nullptr;
    if (tr) tr[15] = (unsigned long long)clock64();  // kernel entry (slot 15 of step 0)
    if (tr) tr[14] = globaltimer_ns();                // (slot 14: entry / exit in globaltimer ns)
#else
#define PTR(k)
#endif
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int Hq = p.Hq, B = p.B, T = p.T, H = p.H, G4 = p.ndir * 4 * Hq;
    const int KC = Hq / 2 / 64;                   // 64-wide K chunks of the half
    uint8_t *Rs = smem;                           // [KC][128 rows][128 B] SW128
    uint8_t *ring = Rs + KC * PF_CHUNK;           // [PF_S][128 rows][128 B] SW128
    float4 *recv = reinterpret_cast<float4 *>(ring + PF_S * PF_CHUNK);  // [16 float4 columns][128 rows]
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + PF_S * PF_CHUNK + PF_RECV);
    uint64_t *empty = full + PF_S;
    uint64_t *mma_done = empty + PF_S;
    uint64_t *rbar = mma_done + 1;
    uint64_t *xbar = rbar + 1;  // the partner's partial sums landed (st.async complete_tx)
    uint32_t *tslot = reinterpret_cast<uint32_t *>(xbar + 1);

    const int kh = (int)cluster_ctarank();        // K half (cluster rank)
    const int tile = blockIdx.x >> 1;
    const int NT = 4 * Hq / 128;
    const int d = tile / NT, nt = tile - d * NT;
    const int dir = d == 0 ? p.dir0 : -1;
    const int w = warp_uniform(warp_id()), l = lane_id(), q = w & 3, ch = w >> 2;
    const int m = 32 * q + l;                     // batch row (TMEM lane) this thread reads
    // this thread finalizes row m, tile columns [64 kh + CW ch, +CW) = UPT units from u0, and sends
    // the partner its partial sums of columns [64 (1 - kh) + CW ch, +CW)
    constexpr int CW = PF_CW, UPT = PF_UPT;
    const int u0 = nt * 32 + 16 * kh + UPT * ch;
    uint32_t *cnt_d = cnt + 32 * d;
    const uint32_t cpd = 2 * NT;                  // CTAs per direction

    if (threadIdx.x == 0) {
        for (int i = 0; i < PF_S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(mma_done, 1);
        mbar_init(rbar, 1);
        mbar_init(xbar, 1);
        fence_mbar_init();
        tma_prefetch_desc(&tmH);
        tma_prefetch_desc(&tmR);
    }
    if (w == 1) {
        tmem_alloc(tslot, 128);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    if (threadIdx.x == 0) {  // the tile's R^T rows, this CTA's K half: resident for the whole scan
        mbar_arrive_expect_tx(rbar, KC * PF_CHUNK);
        for (int kc = 0; kc < KC; ++kc)
            tma_load_2d(Rs + kc * PF_CHUNK, &tmR, rbar, kh * (Hq / 2) + kc * 64, d * 4 * Hq + nt * 128);
    }
    mbar_wait(rbar, 0);
    cluster_sync();  // the partner's barriers are initialised before any remote store

    // state of the UPT cells this thread finalizes (row m, units u0..u0+UPT-1)
    float c_st[UPT], h_st[UPT];
    const bool row_ok = m < B;
#pragma unroll
    for (int i = 0; i < UPT; ++i) {
        const int u = u0 + i;
        c_st[i] = (row_ok && p.c0 && u < H) ? p.c0[((long)d * B + m) * H + u] : 0.f;
        h_st[i] = (row_ok && p.h0 && u < H) ? p.h0[((long)d * B + m) * H + u] : 0.f;
    }
    const bool cvec = (p.ldc & 3) == 0 && (p.c_doff & 3) == 0 && ((uintptr_t)p.C & 15) == 0 && u0 + UPT <= H;
    const bool yvec = p.y && (p.ldy & 3) == 0 && (p.y_doff & 3) == 0 && ((uintptr_t)p.y & 15) == 0 && u0 + UPT <= H;
    const uint32_t idesc = idesc_f16(128, 128, 0, 0);
    const uint32_t partner_recv = mapa_shared(smem_u32(recv), (uint32_t)(kh ^ 1));
    const uint32_t partner_xbar = mapa_shared(smem_u32(xbar), (uint32_t)(kh ^ 1));
    int stage = 0;
    uint32_t phase = 0, mph = 0, xph = 0;
    // a step's outputs other than the history (read only after the launch completes)
    float yv[UPT];
    __half2 ga[2 * UPT];  // (packed conversions: one cvt per pair)
    long r_pend = -1;
    auto store_outputs = [&](long rr) {
        uint4 *gp = reinterpret_cast<uint4 *>(p.gates + rr * G4 + (long)d * 4 * Hq + 4 * u0);
#pragma unroll
        for (int j = 0; j < UPT / 2; ++j) gp[j] = *reinterpret_cast<const uint4 *>(&ga[4 * j]);
        if (p.y16) {
            __half2 yh[UPT / 2];
#pragma unroll
            for (int i = 0; i < UPT / 2; ++i) yh[i] = __floats2half2_rn(yv[2 * i], yv[2 * i + 1]);
            __half *yd = p.y16 + rr * 2 * Hq + (long)d * Hq + u0;
            if constexpr (UPT == 8) *reinterpret_cast<uint4 *>(yd) = *reinterpret_cast<const uint4 *>(yh);
            else *reinterpret_cast<uint2 *>(yd) = *reinterpret_cast<const uint2 *>(yh);
        }
        float *cp = p.C + d * p.c_doff + rr * p.ldc + u0;
        if (cvec) {
#pragma unroll
            for (int v = 0; v < UPT / 4; ++v)
                reinterpret_cast<float4 *>(cp)[v] = make_float4(c_st[4 * v], c_st[4 * v + 1], c_st[4 * v + 2], c_st[4 * v + 3]);
        } else {
#pragma unroll
            for (int i = 0; i < UPT; ++i)
                if (u0 + i < H) cp[i] = c_st[i];
        }
        if (p.y) {
            float *yq = p.y + rr * p.ldy + d * p.y_doff + u0;
            if (yvec) {
#pragma unroll
                for (int v = 0; v < UPT / 4; ++v)
                    reinterpret_cast<float4 *>(yq)[v] = make_float4(yv[4 * v], yv[4 * v + 1], yv[4 * v + 2], yv[4 * v + 3]);
            } else {
#pragma unroll
                for (int i = 0; i < UPT; ++i)
                    if (u0 + i < H) yq[i] = yv[i];
            }
        }
    };
    for (int s = 0; s < T; ++s) {
        const int t = dir > 0 ? s : T - 1 - s;
        const long r = (long)t * B + m;
        const bool need_mma = s > 0 || p.h0 != nullptr;
        const int slot_prev = t + (dir < 0);
        PTR(0);
        float acc[CW];
        if (need_mma) {
            if (threadIdx.x == 0) mbar_arrive_expect_tx(xbar, PF_RECV);  // this step's partial sums
            if (w == 0) {
                if (elect_one()) {  // h_{t-1}: wait for the direction's step s-1, then stream it
                    PTR(1);
                    if (s > 0) spin_until_geq(cnt_d, (uint32_t)s * cpd);
                    PTR(2);
                    fence_proxy_async_global();
                    const int row0 = (d * (T + 1) + slot_prev) * B;
                    int st2 = stage;
                    uint32_t ph2 = phase;
                    for (int kc = 0; kc < KC; ++kc) {
                        mbar_wait(&empty[st2], ph2 ^ 1);
                        mbar_arrive_expect_tx(&full[st2], PF_CHUNK);
                        tma_load_2d(ring + st2 * PF_CHUNK, &tmH, &full[st2], kh * (Hq / 2) + kc * 64, row0);
                        if (++st2 == PF_S) { st2 = 0; ph2 ^= 1; }
                    }
                    PTR(3);
                }
                __syncwarp();
            } else if (w == 1) {
                int st2 = stage;
                uint32_t ph2 = phase;
                for (int kc = 0; kc < KC; ++kc) {
                    mbar_wait(&full[st2], ph2);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(ring + st2 * PF_CHUNK), sb = smem_u32(Rs + kc * PF_CHUNK);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        mma_f16_ss_w(tmem, sdesc_sw128(sa + kk * 32, 16, 1024), sdesc_sw128(sb + kk * 32, 16, 1024), idesc,
                                     (kc | kk) != 0);
                    mma_commit_w(&empty[st2]);
                    __syncwarp();
                    if (++st2 == PF_S) { st2 = 0; ph2 ^= 1; }
                }
                mma_commit_w(mma_done);
                __syncwarp();
            }
            {  // ring position after this step (identical in every thread)
                const int adv = stage + KC;
                phase ^= (uint32_t)((adv / PF_S) & 1);
                stage = adv % PF_S;
            }
        }
        // the previous step's other outputs, deferred to here: off the TMA / MMA warps' path to this
        // step's loads, overlapping the MMAs
        if (r_pend >= 0) store_outputs(r_pend);
        // Z and the mask of this step (produced before the launch): in flight during the MMA
        float z[CW];
#pragma unroll
        for (int i = 0; i < CW; ++i) z[i] = 0.f;
        bool valid_row = false;
        if (row_ok) {
            valid_row = p.mask[r] != 0;
            const float4 *zp = reinterpret_cast<const float4 *>(p.Z + r * G4 + (long)d * 4 * Hq + 4 * u0);
#pragma unroll
            for (int j = 0; j < CW / 4; ++j) {
                const float4 v = zp[j];
                z[4 * j] = v.x; z[4 * j + 1] = v.y; z[4 * j + 2] = v.z; z[4 * j + 3] = v.w;
            }
        }
        if (need_mma) {
            mbar_wait(mma_done, mph);
            PTR(4);
            mph ^= 1;
            tc_fence_after();
            const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16);
            {  // the partner's columns of row m: partial sums -> its receive buffer
                float v[CW];
#pragma unroll
                for (int k16 = 0; k16 < CW / 16; ++k16) {
                    tmem_ld16(ta + 64 * (kh ^ 1) + CW * ch + 16 * k16, *reinterpret_cast<float(*)[16]>(&v[16 * k16]));
                    tmem_ld16(ta + 64 * kh + CW * ch + 16 * k16, *reinterpret_cast<float(*)[16]>(&acc[16 * k16]));
                }
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < CW / 4; ++j)
                    st_async_v4(partner_recv + (uint32_t)(((ch * (CW / 4) + j) * 128 + m) * 16), v[4 * j], v[4 * j + 1],
                                v[4 * j + 2], v[4 * j + 3], partner_xbar);
            }
            PTR(5);
            mbar_wait(xbar, xph);  // the partner's partial sums of this CTA's columns have landed
            xph ^= 1;
            PTR(6);
        } else {
#pragma unroll
            for (int i = 0; i < CW; ++i) acc[i] = 0.f;
        }
        // a = (Z + P_0) + P_1: the step chain's summation order (P_k = K half k)
#pragma unroll
        for (int j = 0; j < CW / 4; ++j) {
            const float4 o = need_mma ? recv[(ch * (CW / 4) + j) * 128 + m] : make_float4(0.f, 0.f, 0.f, 0.f);
            const float ov[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float p0 = kh == 0 ? acc[4 * j + e] : ov[e], p1 = kh == 0 ? ov[e] : acc[4 * j + e];
                acc[4 * j + e] = (z[4 * j + e] + p0) + p1;
            }
        }
        if (row_ok) {
            float hv[UPT];
#pragma unroll
            for (int i = 0; i < UPT; ++i) {
                const bool valid = valid_row && u0 + i < H;
                float ai = 0.f, af = 0.f, ag = 0.f, ao = 0.f;
                if (valid) {
                    ai = sg(acc[4 * i]); af = sg(acc[4 * i + 1]); ag = th(acc[4 * i + 2]); ao = sg(acc[4 * i + 3]);
                    const float cn = af * c_st[i] + ai * ag;
                    c_st[i] = cn;
                    h_st[i] = ao * th(cn);
                }
                hv[i] = h_st[i];
                yv[i] = valid ? h_st[i] : 0.f;
                ga[2 * i] = __floats2half2_rn(ai, af);
                ga[2 * i + 1] = __floats2half2_rn(ag, ao);
            }
            __half2 hh[UPT / 2];
#pragma unroll
            for (int i = 0; i < UPT / 2; ++i) hh[i] = __floats2half2_rn(hv[2 * i], hv[2 * i + 1]);
            // h_t -> the history slot the next step's TMA reads
            __half *hd = p.hist + (((long)d * (T + 1) + slot_prev + dir) * B + m) * Hq + u0;
            if constexpr (UPT == 8) *reinterpret_cast<uint4 *>(hd) = *reinterpret_cast<const uint4 *>(hh);
            else *reinterpret_cast<uint2 *>(hd) = *reinterpret_cast<const uint2 *>(hh);
        }
        // publish h_t of this CTA's columns to the direction: the CTA barrier orders every thread's
        // history store before thread 0's release (cumulative), which the next step's acquire pairs with
        PTR(7);
        tc_fence_before();
        __syncthreads();
        PTR(8);
        if (threadIdx.x == 0) red_release_gpu_add(cnt_d, 1u);
        PTR(9);
        r_pend = row_ok ? r : -1;  // its other outputs: stored during the next step
    }
    if (r_pend >= 0) store_outputs(r_pend);
    if (row_ok) {  // state after the whole scan
#pragma unroll
        for (int i = 0; i < UPT; ++i) {
            const int u = u0 + i;
            if (u < H) {
                if (p.hT) p.hT[((long)d * B + m) * H + u] = h_st[i];
                if (p.cT) p.cT[((long)d * B + m) * H + u] = c_st[i];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // no remote store into this CTA's shared memory is outstanding
#ifdef BLSTM_TRACE
    if (tr) tr[(size_t)(T - 1) * 16 + 14] = globaltimer_ns();
#endif
    if (w == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 128);
    }
}

// 1: launched; 0: not used (the caller runs the step chain); < 0: error.  Used where it applies
// (B <= 128, Hq <= 1024, all CTAs co-resident); BLSTM_STEP_PERSIST=0 turns it off, =1 forces it
// (then an inapplicable size or a failed launch is an error instead of the fallback).
static int rec_step_fwd_persist(const RecStepFwd &p, cudaStream_t st) {
    const char *e = getenv("BLSTM_STEP_PERSIST");
    if (e && e[0] == '0') return 0;
    const bool force = e && e[0] == '1';
    const int no = force ? -6 : 0;
    const int Hq = p.Hq;
    if (p.B > 128 || Hq > 1024 || Hq % 128 || p.T < 1) return no;
    const int ctas = p.ndir * 2 * (4 * Hq / 128);
    if (ctas > num_sms()) return no;
    const size_t smem = pf_smem(Hq);
    if (cudaFuncSetAttribute(step_fwd_persist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess) {
        cudaGetLastError();
        return force ? -5 : 0;
    }
    CUtensorMap tmH, tmR;
    if (make_tmap_f16(&tmH, p.hist, Hq, (uint64_t)p.ndir * (p.T + 1) * p.B, Hq, 128)) return -5;
    if (make_tmap_f16(&tmR, p.RT16, Hq, (uint64_t)p.ndir * 4 * Hq, Hq, 128)) return -5;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(PF_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, step_fwd_persist_kernel, &cfg) != cudaSuccess ||
        nclusters < ctas / 2) {
        cudaGetLastError();
        return no;
    }
    uint32_t *cnt = reinterpret_cast<uint32_t *>(p.P);  // the partials scratch is unused here
    if (cudaMemsetAsync(cnt, 0, 64 * sizeof(uint32_t), st) != cudaSuccess) return -5;
    // a cooperative cluster launch can be refused (e.g. under a profiler that replays kernels):
    // then the launched chain runs instead, unless forced
    bool ok;
    {
        ProfScope ps(PROF_REC_FWD, st);
        ok = cudaLaunchKernelEx(&cfg, step_fwd_persist_kernel, tmH, tmR, p, cnt, rec_trace_fwd()) == cudaSuccess;
    }
    if (!ok) {
        cudaGetLastError();
        return force ? -5 : 0;
    }
    note_launch();
    return 1;
}

// ---------------------------------------------------------------------------------------------
// Persistent BPTT (Hq in {512, 1024}, B <= 128): the mirror of the persistent forward, with the
// recurrent weights resident on chip for the whole reverse scan and no launch per time step
// (north_star: "the mirrored BPTT kernel").
//   dh_{t'}[b, k] = sum_n dA_t[b, n] R[k, n]   (k: hidden unit, n: gate column 4u + gamma)
// Thread-block clusters of PB_KS = 4 CTAs, one cluster per (direction d, 128-unit tile ut); cluster
// rank ks holds the K-split n in [ks Hq, (ks+1) Hq) of the tile's R rows as the tcgen05 A operand
// (M = 128 units): the first PB_TK columns in TMEM (A-from-TMEM MMAs), the rest in shared memory
// (SW128, TMA once).  2 * (Hq / 128) * 4 CTAs: 64 at C5, which leaves the other SMs to the
// weight-gradient GEMMs of the layer above (side stream).
// Per step s (frame t; the reverse of the forward scan):
//   1. the TMA warp waits until the unit tiles whose gate columns form this CTA's K-split have
//      published dA of step s-1 (per-(direction, tile) counters, release / acquire at gpu scope),
//      then streams dA_{s-1}[128 batch rows][K-split] (the B operand, N = batch) through a ring;
//   2. one warp issues the MMAs: D[128 units x 128 batch] (fp32, TMEM) = R[tile, K-split] dA^T;
//   3. reduce-scatter of D over the cluster through distributed shared memory: rank j owns batch
//      columns [32 j, 32 j + 32) and receives the other three ranks' partial sums of them
//      (st.async, complete_tx on its mbarrier); dh = P_0 + P_1 + P_2 + P_3 (fixed order);
//   4. the gate gradients of frame t as in step_bwd_gate_kernel (dH, dc~, dA, dc; masked frames
//      pass dh and dc through, R4), dA -> HBM (scaled fp16, the next step's B operand and the
//      weight-gradient GEMMs' input), db accumulated in registers;
//   5. arrive on the tile's counter.
// After the last step, with dh0 requested, one more MMA + reduction gives dh0.
// ---------------------------------------------------------------------------------------------
constexpr int PB_THREADS = 256;
constexpr int PB_KS = 4;                 // K-splits = cluster size
constexpr int PB_S = 7;                  // dA ring stages (16 KB: 128 batch rows x 64 gate columns)
constexpr int PB_TK = 768;               // K columns of the A operand held in TMEM (384 columns)
constexpr uint32_t PB_CHUNK = 16384;
constexpr uint32_t PB_RECV = (PB_KS - 1) * 32 * 128 * 2;  // three ranks' partial sums of 32 batch columns,
                                                          // fp16 (x2: double-buffered by step parity)
constexpr uint32_t PB_DCOL = 384;        // TMEM column of D [128 lanes x 128 batch columns]
constexpr int PB_DBG = 2 * PB_KS;        // db partial groups per direction (rank x column half)
static int pb_tk(int Hq) { return Hq < PB_TK ? Hq : PB_TK; }
static size_t pb_smem(int Hq) {
    return (size_t)((Hq - pb_tk(Hq)) / 64) * PB_CHUNK + PB_S * PB_CHUNK + 2 * PB_RECV + 1024 + 256;
}

__global__ void __launch_bounds__(PB_THREADS, 1)
    step_bwd_persist_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmR,
                            RecStepBwd p, const __half *__restrict__ R16, uint32_t *cnt, float *dbpart,
                            unsigned long long *trace) {
#ifdef BLSTM_TRACE
#define PTB(k) \
    if (trb) trb[(size_t)s * 16 + (k)] = (unsigned long long)clock64()
    unsigned long long *trb = (blockIdx.x == 0 && threadIdx.x == 0) ? trace : nullptr;
#else
#define PTB(k)
#endif
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int Hq = p.Hq, B = p.B, T = p.T, H = p.H, G4 = p.ndir * 4 * Hq;
    const int TK = Hq < PB_TK ? Hq : PB_TK;      // K in TMEM
    const int KCT = TK / 64, KC = Hq / 64;        // 64-wide K chunks: in TMEM, in total
    uint8_t *Rs = smem;                           // [KC - KCT][128 rows][128 B] SW128 (K-major A)
    uint8_t *ring = Rs + (KC - KCT) * PB_CHUNK;   // [PB_S][128 batch rows][128 B] SW128 (K-major B)
    uint4 *recv = reinterpret_cast<uint4 *>(ring + PB_S * PB_CHUNK);  // [2 parity][3 slots][4 col groups][128 units][8 fp16]
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + PB_S * PB_CHUNK + 2 * PB_RECV);
    uint64_t *empty = full + PB_S;
    uint64_t *mma_done = empty + PB_S;
    uint64_t *rbar = mma_done + 1;
    uint64_t *xbar = rbar + 1;                    // [2 parity]
    uint32_t *tslot = reinterpret_cast<uint32_t *>(xbar + 2);

    const int ks = (int)cluster_ctarank();
    const int NUT = Hq / 128;
    const int cl = blockIdx.x / PB_KS;
    const int d = cl / NUT, ut = cl - d * NUT;
    const int dir = d == 0 ? p.dir0 : -1;
    const int w = warp_uniform(warp_id()), l = lane_id(), q = w & 3, ch = w >> 2;
    const int m = 32 * q + l;                     // unit row of the tile (TMEM lane)
    const int u = ut * 128 + m;                   // hidden unit
    const int b0 = 32 * ks + 16 * ch;             // this thread's 16 batch columns (owner role)
    // the unit tiles whose gate columns [ks Hq, (ks+1) Hq) this CTA's K-split covers
    const int tlo = ks * Hq / 4 / 128;  // (through ((ks + 1) Hq / 4 - 1) / 128: two tiles at Hq = 1024)
    uint32_t *cnt_d = cnt + 16 * d;
    const float scale = (float)(1 << DA_SHIFT), alpha = 1.f / scale;

    if (threadIdx.x == 0) {
        for (int i = 0; i < PB_S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(mma_done, 1);
        mbar_init(rbar, 1);
        mbar_init(&xbar[0], 1);
        mbar_init(&xbar[1], 1);
        fence_mbar_init();
        tma_prefetch_desc(&tmA);
        if (KC > KCT) tma_prefetch_desc(&tmR);
    }
    if (w == 1) {
        tmem_alloc(tslot, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    if (p.started && threadIdx.x == 0) red_release_gpu_add(p.started, 1u);  // placed (side-stream guard)
    const int col0 = d * 4 * Hq + ks * Hq;        // first gate column of the K-split in R16 / dA
    if (threadIdx.x == 0 && KC > KCT) {            // the K-split's columns beyond TK: shared memory
        mbar_arrive_expect_tx(rbar, (KC - KCT) * PB_CHUNK);
        for (int kc = KCT; kc < KC; ++kc) tma_load_2d(Rs + (kc - KCT) * PB_CHUNK, &tmR, rbar, col0 + kc * 64, ut * 128);
    }
    {   // the first TK columns -> TMEM columns [0, TK/2) (two fp16 per 32-bit column, lane = unit row);
        // warps w and w + 4 share lane quarter q and split the columns
        const __half *row = R16 + (size_t)(ut * 128 + m) * (p.ndir * 4 * Hq) + col0;
        const int half = TK / 2;                  // fp16 per warp group
        const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16);
        for (int c0 = ch * half; c0 < ch * half + half; c0 += 32) {
            uint32_t v[16];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint4 x = *reinterpret_cast<const uint4 *>(row + c0 + 8 * j);
                v[4 * j] = x.x; v[4 * j + 1] = x.y; v[4 * j + 2] = x.z; v[4 * j + 3] = x.w;
            }
            tmem_st16(tq + (uint32_t)(c0 / 2), v);
        }
        tmem_st_wait();
    }
    if (KC > KCT) mbar_wait(rbar, 0);
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // every rank's barriers are initialised before any remote store
    tc_fence_after();

    const uint32_t idesc = idesc_f16(128, 128, 0, 0);
    const uint32_t dq = tmem + ((uint32_t)(32 * q) << 16) + PB_DCOL;
    // The reduction's receive buffer and its mbarrier are double-buffered by step parity.  Rank j
    // sends its step-s partial sums (buffer s & 1) only after it received every other rank's step-(s-1)
    // sums, each sent after that rank had consumed its step-(s-2) buffer (same parity) and re-armed
    // its barrier: the all-to-all exchange itself orders the reuse, no cluster barrier per step.
    if (threadIdx.x == 0) {  // steps 1 and 2 (parities 1 and 0)
        mbar_arrive_expect_tx(&xbar[1], PB_RECV);
        mbar_arrive_expect_tx(&xbar[0], PB_RECV);
    }

    // per-cell state of the 16 cells (unit u, batch b0 + i) this thread owns
    float dc[16], dhc[16], db[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int b = b0 + i;
        const bool ok = b < B && u < H;
        dc[i] = (ok && p.dcT) ? p.dcT[((long)d * B + b) * H + u] : 0.f;
        dhc[i] = (ok && p.dhT) ? p.dhT[((long)d * B + b) * H + u] : 0.f;
    }
    int stage = 0;
    uint32_t phase = 0, mph = 0, xph[2] = {0, 0};
    uint32_t mprev = 0;  // mask bits (cell i) of the frame of the previous step
    const int S_END = T + (p.dh0 ? 1 : 0);        // step T: dh0 only
    for (int s = 0; s < S_END; ++s) {
        const bool last = s == T;
        const int t = dir > 0 ? T - 1 - s : s;   // this step's frame (unused when last)
        const int tp = dir > 0 ? T - s : s - 1;  // the frame of step s-1
        const bool need_mma = s > 0;
        PTB(0);
        float dh[16];
        PTB(1);
        if (need_mma) {
            if (w == 0) {
                if (elect_one()) {  // dA of step s-1 (frame tp), this CTA's K-split of it
                    // per source tile: a chunk's loads wait only for the tile that owns its columns,
                    // so the first tile's chunks stream (and their MMAs run) while the last publishes
                    int waited = tlo - 1;
                    int st2 = stage;
                    uint32_t ph2 = phase;
                    for (int kc = 0; kc < KC; ++kc) {
                        const int tt = (ks * Hq + kc * 64) / 512;  // unit tile of gate columns col0 + kc*64
                        if (tt > waited) {
                            spin_until_geq(cnt_d + tt, (uint32_t)s * PB_KS);
                            fence_proxy_async_global();
                            waited = tt;
                            if (tt == tlo) PTB(2);
                        }
                        mbar_wait(&empty[st2], ph2 ^ 1);
#ifdef BLSTM_TRACE
                        if (p.exp == 1) { mbar_arrive(&full[st2]); if (++st2 == PB_S) { st2 = 0; ph2 ^= 1; } continue; }
#endif
                        mbar_arrive_expect_tx(&full[st2], PB_CHUNK);
                        tma_load_2d(ring + st2 * PB_CHUNK, &tmA, &full[st2], col0 + kc * 64, tp * B);
                        if (++st2 == PB_S) { st2 = 0; ph2 ^= 1; }
                    }
                    PTB(3);
                }
                __syncwarp();
            } else if (w == 1) {
                int st2 = stage;
                uint32_t ph2 = phase;
                for (int kc = 0; kc < KC; ++kc) {
                    mbar_wait(&full[st2], ph2);
                    tc_fence_after();
                    const uint32_t sb = smem_u32(ring + st2 * PB_CHUNK);
#ifdef BLSTM_TRACE
                    if (p.exp == 2) {
                    } else
#endif
                    if (kc < KCT) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            mma_f16_ts_w(tmem + PB_DCOL, tmem + (uint32_t)(kc * 32 + kk * 8),
                                         sdesc_sw128(sb + kk * 32, 16, 1024), idesc, (kc | kk) != 0);
                    } else {
                        const uint32_t sa = smem_u32(Rs + (kc - KCT) * PB_CHUNK);
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            mma_f16_ss_w(tmem + PB_DCOL, sdesc_sw128(sa + kk * 32, 16, 1024),
                                         sdesc_sw128(sb + kk * 32, 16, 1024), idesc, 1);
                    }
                    mma_commit_w(&empty[st2]);
                    __syncwarp();
                    if (++st2 == PB_S) { st2 = 0; ph2 ^= 1; }
                }
                mma_commit_w(mma_done);
                __syncwarp();
            }
            {
                const int adv = stage + KC;
                phase ^= (uint32_t)((adv / PB_S) & 1);
                stage = adv % PB_S;
            }
        }
        // saved state of this step's frame (produced before the launch), loaded while the MMAs run:
        // issued after the TMA / MMA warps' role work (a load that stalls those warps would stall
        // the chain), all independent (no load feeds an address or a branch), kept packed (gates as
        // fp16 pairs) so the 16 cells' state fits in registers; cells beyond B read row B - 1
        uint2 gq[16];
        float cc[16], cp[16], dy[16];
        uint32_t mbits = 0;
        if (!last) {
            const int tpf = t - dir;              // the frame before t in the forward scan
            const bool tpf_in = tpf >= 0 && tpf < T;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int b = min(b0 + i, B - 1);
                const long r = (long)t * B + b;
                mbits |= (p.mask[r] != 0 && b0 + i < B) ? (1u << i) : 0u;
                gq[i] = *reinterpret_cast<const uint2 *>(p.gates + r * G4 + (long)d * 4 * Hq + 4 * u);
                // (rows are read Hq wide: the callers pass ldc, lddy >= Hq; unguarded loads, since a
                // u < H guard on them measured 7 % slower BPTT at C5)
                cc[i] = p.C[d * p.c_doff + r * p.ldc + u];
                cp[i] = tpf_in ? p.C[d * p.c_doff + ((long)tpf * B + b) * p.ldc + u]
                               : (p.c0 && u < H ? p.c0[((long)d * B + b) * H + u] : 0.f);
                dy[i] = p.dy[r * p.lddy + d * p.dy_doff + u];
            }
        }
        if (need_mma) {
            mbar_wait(mma_done, mph);
            PTB(4);
            mph ^= 1;
            tc_fence_after();
            // reduce-scatter: columns [64 ch, 64 ch + 64) of row m belong to ranks 2ch and 2ch + 1
            const int par = s & 1;
            const uint32_t pofs = (uint32_t)par * PB_RECV;
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
                const int j = 2 * ch + jj;
                if (j == ks) continue;
                const uint32_t slot = (uint32_t)(ks < j ? ks : ks - 1);
                const uint32_t rbase = mapa_shared(smem_u32(recv), (uint32_t)j) + pofs;
                const uint32_t rbar = mapa_shared(smem_u32(&xbar[par]), (uint32_t)j);
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {  // 16 columns at a time (registers), as fp16
                    float v[16];
                    tmem_ld16(dq + 32 * j + 16 * hh, v);
                    tmem_ld_wait();
                    uint32_t hv[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        __half2 h2 = __floats2half2_rn(v[2 * e], v[2 * e + 1]);
                        hv[e] = *reinterpret_cast<uint32_t *>(&h2);
                    }
#pragma unroll
                    for (int cg = 0; cg < 2; ++cg)
                        st_async_v4u(rbase + (uint32_t)(((slot * 4 + 2 * hh + cg) * 128 + m) * 16), hv[4 * cg],
                                     hv[4 * cg + 1], hv[4 * cg + 2], hv[4 * cg + 3], rbar);
                }
            }
            float own[16];
            tmem_ld16(dq + b0, own);
            tmem_ld_wait();
            PTB(5);
            mbar_wait(&xbar[par], xph[par]);  // the three other ranks' partial sums of this CTA's columns
            PTB(6);
            xph[par] ^= 1;
            const uint4 *rv = recv + par * (PB_RECV / 16);
            // dh = P_0 + P_1 + P_2 + P_3 (rank order; the other ranks' partials as fp16), unscaled
            float pr[PB_KS - 1][16];
#pragma unroll
            for (int sl = 0; sl < PB_KS - 1; ++sl)
#pragma unroll
                for (int cg = 0; cg < 2; ++cg) {
                    const uint4 x = rv[(sl * 4 + 2 * ch + cg) * 128 + m];
                    const uint32_t xw[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&xw[e]));
                        pr[sl][8 * cg + 2 * e] = f.x;
                        pr[sl][8 * cg + 2 * e + 1] = f.y;
                    }
                }
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                float a = 0.f;
#pragma unroll
                for (int j = 0; j < PB_KS; ++j) {  // rank j's partial: own, or slot j (j < ks) / j - 1 (j > ks)
                    const float lo = pr[j < PB_KS - 1 ? j : PB_KS - 2][i], hi = pr[j > 0 ? j - 1 : 0][i];
                    const float v = j == ks ? own[i] : (j < ks ? lo : hi);
                    a = j == 0 ? v : a + v;
                }
                dh[i] = a * alpha;
            }
            tc_fence_before();
            // buffer par is reused at step s + 2: its barrier is re-armed by thread 0 after the CTA
            // barrier at the end of this step (every thread has read the buffer by then)
        }
        PTB(7);
        if (last) {  // dh0 / dc0: the gradient w.r.t. the state before the scan
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int b = b0 + i;
                if (b >= B || u >= H) continue;
                p.dh0[((long)d * B + b) * H + u] = ((mprev >> i) & 1u) ? dh[i] : dhc[i];
                if (p.dc0) p.dc0[((long)d * B + b) * H + u] = dc[i];
            }
            break;
        }
        // gate gradients of frame t
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int b = b0 + i;
            if (b >= B) continue;
            float dh_in = dhc[i];
            if (need_mma && ((mprev >> i) & 1u)) dh_in = dh[i];
            // masked frame or padding unit: dA = 0, dh passes through, dc unchanged (R4).  Branch-free,
            // selects on `valid` (the unselected arithmetic may see the padding's values), and one
            // 8-byte store of the four fp16 gate gradients per cell
            const bool valid = ((mbits >> i) & 1u) && u < H;
            const float2 g01 = __half22float2(*reinterpret_cast<const __half2 *>(&gq[i].x));
            const float2 g23 = __half22float2(*reinterpret_cast<const __half2 *>(&gq[i].y));
            const float gi = g01.x, gf = g01.y, gg = g23.x, go = g23.y;
            const float dH = dh_in + dy[i];
            const float tc = th(cc[i]);
            const float dct = dc[i] + dH * go * (1.f - tc * tc);
            const float da_i = valid ? dct * gg * gi * (1.f - gi) : 0.f;
            const float da_f = valid ? dct * cp[i] * gf * (1.f - gf) : 0.f;
            const float da_g = valid ? dct * gi * (1.f - gg * gg) : 0.f;
            const float da_o = valid ? dH * tc * go * (1.f - go) : 0.f;
            __half2 h01 = __floats2half2_rn(da_i * scale, da_f * scale), h23 = __floats2half2_rn(da_g * scale, da_o * scale);
            *reinterpret_cast<uint2 *>(p.dA + ((long)t * B + b) * G4 + (long)d * 4 * Hq + 4 * u) =
                make_uint2(*reinterpret_cast<uint32_t *>(&h01), *reinterpret_cast<uint32_t *>(&h23));
            db[0] += da_i; db[1] += da_f; db[2] += da_g; db[3] += da_o;
            dc[i] = valid ? dct * gf : dc[i];
            dhc[i] = dh_in;
        }
        // publish dA_t of this tile: the CTA barrier orders every thread's stores before thread 0's
        // release (cumulative), which the consumers' acquire pairs with
        mprev = mbits;
        PTB(8);
        tc_fence_before();
        __syncthreads();
        PTB(9);
        if (threadIdx.x == 0) {
            red_release_gpu_add(cnt_d + ut, 1u);
            if (need_mma) mbar_arrive_expect_tx(&xbar[s & 1], PB_RECV);  // for step s + 2
        }
    }
    if (dbpart) {  // db partials: [d][rank * 2 + column half][4Hq] (0 for padding units)
        float *dp = dbpart + ((long)d * PB_DBG + ks * 2 + ch) * 4 * Hq + 4 * u;
        dp[0] = db[0]; dp[1] = db[1]; dp[2] = db[2]; dp[3] = db[3];
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // no remote store into this CTA's shared memory is outstanding
    if (w == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// 1: the persistent BPTT ran (db partials, PB_DBG groups per direction, written to p.dbpart when
// given); 0: not used (the caller runs the step chain); < 0: error.  BLSTM_STEP_PERSIST_BWD=0 turns it
// off, =1 forces it.
static int rec_step_bwd_persist(const RecStepBwd &p, cudaStream_t st) {
    const char *e = getenv("BLSTM_STEP_PERSIST_BWD");
    if (e && e[0] == '0') return 0;
    const bool force = e && e[0] == '1';
    const int no = force ? -6 : 0;
    const int Hq = p.Hq;
    if (p.B > 128 || (Hq != 512 && Hq != 1024) || p.T < 1 || p.ndir < 1 || p.ndir > 2 || !p.R16) return no;
    const int ctas = p.ndir * (Hq / 128) * PB_KS;
    if (ctas > num_sms()) return no;
    const size_t smem = pb_smem(Hq);
    if (cudaFuncSetAttribute(step_bwd_persist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess) {
        cudaGetLastError();
        return force ? -5 : 0;
    }
    CUtensorMap tmA, tmR;
    if (make_tmap_f16(&tmA, p.dA, (uint64_t)p.ndir * 4 * Hq, (uint64_t)p.T * p.B, (uint64_t)p.ndir * 4 * Hq, 128))
        return -5;
    if (make_tmap_f16(&tmR, p.R16, (uint64_t)p.ndir * 4 * Hq, (uint64_t)Hq, (uint64_t)p.ndir * 4 * Hq, 128)) return -5;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(PB_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = PB_KS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, step_bwd_persist_kernel, &cfg) != cudaSuccess ||
        nclusters < ctas / PB_KS) {
        cudaGetLastError();
        return no;
    }
    uint32_t *cnt = reinterpret_cast<uint32_t *>(p.dhR);  // the chain's partials scratch is unused here
    if (cudaMemsetAsync(cnt, 0, 32 * sizeof(uint32_t), st) != cudaSuccess) return -5;
    RecStepBwd q = p;
#ifdef BLSTM_TRACE
    if (getenv("BLSTM_PB_EXP")) q.exp = atoi(getenv("BLSTM_PB_EXP"));  // timing isolation
#endif
    bool ok;
    {
        ProfScope ps(PROF_REC_BWD, st);
        ok = cudaLaunchKernelEx(&cfg, step_bwd_persist_kernel, tmA, tmR, q, p.R16, cnt, p.dbpart, rec_trace_bwd()) ==
             cudaSuccess;
    }
    if (!ok) {
        cudaGetLastError();
        return force ? -5 : 0;
    }
    note_launch();
    return 1;
}
int rec_step_bwd_db_groups() { return PB_DBG; }
int rec_step_bwd_persist_ctas(int B, int Hq, int ndir) {
    const char *e = getenv("BLSTM_STEP_PERSIST_BWD");
    if (e && e[0] == '0') return 0;
    if (B > 128 || (Hq != 512 && Hq != 1024) || ndir < 1 || ndir > 2) return 0;
    const int ctas = ndir * (Hq / 128) * PB_KS;
    return ctas <= num_sms() ? ctas : 0;
}

size_t rec_step_fwd_scratch_bytes(int B, int Hq) { return (size_t)2 * SF * B * 4 * Hq * 4 + (size_t)2 * B * Hq * 4; }
size_t rec_step_bwd_partial_floats(int B, int Hq) { return (size_t)2 * SB * B * Hq; }
size_t rec_step_bwd_scratch_bytes(int B, int Hq) { return (rec_step_bwd_partial_floats(B, Hq) + (size_t)4 * B * Hq) * 4; }

// The T-step loop of a layer is captured once into a CUDA graph (graph.h) and replayed: a loop of
// ~3T small launches is otherwise bound by the host's launch rate.  Inside the graph the two
// directions' per-step GEMMs are parallel branches.

int rec_step_fwd(const RecStepFwd &p, cudaStream_t st) {
    if (const int rc = rec_step_fwd_persist(p, st)) return rc < 0 ? rc : 0;
    const int Hq = p.Hq, B = p.B, T = p.T;
    const bool pdl = step_pdl();
    const std::vector<uint64_t> key{1, (uint64_t)T, (uint64_t)B, (uint64_t)p.H, (uint64_t)Hq, (uint64_t)p.ndir,
                                    (uint64_t)(p.dir0 + 2), u64(p.h0), u64(p.c0), u64(p.hT), u64(p.cT), u64(p.Z), u64(p.mask),
                                    u64(p.RT16), u64(p.P), u64(p.C), (uint64_t)p.ldc, (uint64_t)p.c_doff, u64(p.y),
                                    (uint64_t)p.ldy, (uint64_t)p.y_doff, u64(p.y16), u64(p.gates), u64(p.hist),
                                    (uint64_t)pdl};
    return graph_run(key, PROF_REC_FWD, st, {(const void *)step_fwd_gate_kernel}, [&](cudaStream_t s0) -> int {
        bool first = true;  // the first kernel of the graph has no kernel to depend on
        auto hprev = [&](int d, int s) {  // h_{t-1} of direction d at step s: its history slot
            const int dir = d == 0 ? p.dir0 : -1;
            const int t = dir > 0 ? s : T - 1 - s;
            return p.hist + ((long)d * (T + 1) + t + (dir < 0)) * B * Hq;
        };
        for (int s = 0; s < T; ++s) {
            if (s > 0 || p.h0) {  // (no h0: h_{-1} = 0, nothing to multiply)
                // P_d = h_{t-1,d} R_d^T for both directions in one launch (gemm.h a2): R^T of
                // direction 1 follows direction 0's 4Hq rows, its partials follow direction 0's
                GemmParams g{B, 4 * Hq, Hq, nullptr, 4L * Hq, 1.f, 0, nullptr, 0, 0};
                g.bn = 128;
                g.partials = SF;
                g.splitk_ws = p.P;
                g.splitk_elems = (long)SF * B * 4 * Hq;
                if (p.ndir == 2) {
                    g.a2 = hprev(1, s);
                    g.b_boff = 4L * Hq;
                    g.c_bstride = (long)SF * B * 4 * Hq;
                }
                g.pdl_chain = pdl && !first;
                if (gemm_f16({hprev(0, s), Hq, 0}, {p.RT16, Hq, 0}, g, 0, s0)) return -5;
                first = false;
            }
            if (launch_chain(step_fwd_gate_kernel, dim3((Hq + 255) / 256, p.ndir * B), s0, pdl && !first, p, s))
                return -5;
            first = false;
        }
        return 0;
    });
}

int rec_step_bwd(const RecStepBwd &p, cudaStream_t st) {
    if (const int rc = rec_step_bwd_persist(p, st)) return rc;
    const int Hq = p.Hq, B = p.B, T = p.T;
    const float alpha = 1.f / (float)(1 << DA_SHIFT);
    const bool pdl = step_pdl();
    const std::vector<uint64_t> key{2, (uint64_t)T, (uint64_t)B, (uint64_t)p.H, (uint64_t)Hq, (uint64_t)p.ndir,
                                    (uint64_t)(p.dir0 + 2), u64(p.c0), u64(p.dhT), u64(p.dcT), u64(p.dh0),
                                    u64(p.dc0), u64(p.mask), u64(p.RT16),
                                    u64(p.C), (uint64_t)p.ldc, (uint64_t)p.c_doff, u64(p.gates), u64(p.dy),
                                    (uint64_t)p.lddy, (uint64_t)p.dy_doff, u64(p.dA), u64(p.dhR), u64(p.dhc),
                                    u64(p.dcc), u64(p.splitk_ws), (uint64_t)p.splitk_elems, (uint64_t)pdl};
    return graph_run(key, PROF_REC_BWD, st, {(const void *)step_bwd_gate_kernel, (const void *)step_bwd_final_kernel},
                     [&](cudaStream_t s0) -> int {
        auto dA_of = [&](int d, int s) {  // dA of the frame direction d processed at step s
            const int dir = d == 0 ? p.dir0 : -1;
            const int t = dir > 0 ? T - 1 - s : s;
            return p.dA + ((size_t)t * B) * p.ndir * 4 * Hq + (size_t)d * 4 * Hq;
        };
        for (int s = 0; s < T; ++s) {
            if (launch_chain(step_bwd_gate_kernel, dim3((Hq + 255) / 256, p.ndir * B), s0, pdl && s > 0, p, s))
                return -5;
            if (s + 1 == T && !p.dh0) break;  // (dh0 needs the last frame's dA R)
            // dh_d = dA_{t,d} R_d for both directions in one launch: R of direction 1 (MN-major)
            // follows direction 0's 4Hq rows along K, its partials follow direction 0's
            GemmParams g{B, Hq, 4 * Hq, nullptr, (long)Hq, alpha, 0, nullptr, 0, 0};
            g.bn = 128;
            g.partials = SB;
            g.splitk_ws = p.dhR;
            g.splitk_elems = (long)SB * B * Hq;
            if (p.ndir == 2) {
                g.a2 = dA_of(1, s);
                g.b_boff = 4L * Hq;
                g.c_bstride = (long)SB * B * Hq;
            }
            g.pdl_chain = pdl;
            if (gemm_f16({dA_of(0, s), (long)p.ndir * 4 * Hq, 0}, {p.RT16, Hq, 1}, g, 0, s0)) return -5;
        }
        if (p.dh0 || p.dc0) {
            step_bwd_final_kernel<<<grid_of((long)p.ndir * B * p.H), 256, 0, s0>>>(p);
            note_launch();
        }
        return cudaGetLastError() == cudaSuccess ? 0 : -5;
    });
}

}  // namespace blstm
