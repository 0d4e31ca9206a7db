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
constexpr int SB = 8;  // BPTT     dA R:  K = 4Hq

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

size_t rec_step_fwd_scratch_bytes(int B, int Hq) { return (size_t)2 * SF * B * 4 * Hq * 4 + (size_t)2 * B * Hq * 4; }
size_t rec_step_bwd_scratch_bytes(int B, int Hq) { return (size_t)(2 * SB + 4) * B * Hq * 4; }

// The T-step loop of a layer is captured once into a CUDA graph (graph.h) and replayed: a loop of
// ~3T small launches is otherwise bound by the host's launch rate.  Inside the graph the two
// directions' per-step GEMMs are parallel branches.

int rec_step_fwd(const RecStepFwd &p, cudaStream_t st) {
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
