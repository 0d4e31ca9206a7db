// lstm_rec.h -- internal interface of the persistent recurrence kernels (lstm_rec.cu).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace blstm {

constexpr int REC_UNITS = 32;   // hidden units per CTA -> 128 gate rows = one tcgen05 M tile
constexpr int DA_SHIFT = 10;    // dA is scaled by 2^10 before its fp16 cast

// Kernel-private layouts:
//   Hq = round_up(H, 128); gate column of (unit j, gate gamma in i,f,g,o) = 4*j + gamma
//   ("gate-interleaved"), direction d adds d*4*Hq.
struct RecPlan {
    int Hq, NC;     // padded units, CTAs per (direction, batch group) = Hq / 32
    int G, Bg, N;   // batch groups, rows per group, MMA N (= round_up(Bg, 16))
    int ndir;
};

struct RecParams {
    int T, B, H, Hq, NC, G, Bg, N, ndir;
    int dir0;                    // direction (+1/-1) of direction index 0; index 1 is always -1
    const uint8_t *mask;         // [T, B]
    const uint8_t *maskN;        // [T][G][N] mask rows per batch group (pack_mask)
    // forward
    const float *Z;              // time-major transposed [T][ndir*4Hq][B] (gate row d*4Hq + 4j+gamma)
    long ldz;                    // unused (kept for ABI stability of the struct)
    // != nullptr: Z is still being written by a concurrent GEMM (GemmParams::flags); step t may be
    // read once zflags[d*zflag_nm + m] >= zflag_target for every 128-row M-tile m holding its frames
    const uint32_t *zflags;
    int zflag_target, zflag_nm;
    float *y;                    // [T*B, ldy] (+ d*y_doff), j < H; nullable
    long ldy, y_doff;
    __half *y16;                 // [T*B, ldy16] (+ d*Hq), all j < Hq; nullable
    long ldy16;
    float *C;                    // cell state after frame t: [T*B, ldc] (+ d*c_doff), j < H
    long ldc, c_doff;
    __half *gates;               // saved activations, [T][ndir*4Hq][B] like Z
    long ldg;                    // unused
    __half *hist;                // [ndir][T+1][B][Hq]: h before frame t at slot t + (dir<0)
    const float *c0, *h0;        // [B, H] (+ d*B*H) or nullptr
    float *hT, *cT;              // [B, H] (+ d*B*H) or nullptr
    // backward
    const float *dy;             // [T*B, lddy] (+ d*dy_doff), j < H
    long lddy, dy_doff;
    const float *dhT, *dcT;      // [B, H] or nullptr
    __half *dA;                  // [T*B, ldda] (+ d*4Hq), scaled by 2^DA_SHIFT
    long ldda;
    float *dbpart;               // [ndir][G][4Hq] partial bias gradient (unscaled)
    float *P;                    // [2][ndir][G][NC][Hq][N] partial dh exchange
    float *dh0, *dc0;            // [B, H] (+ d*B*H) or nullptr
    uint32_t *counters;          // [ndir][G], zeroed before each launch
    // != nullptr (BPTT): each CTA adds 1 at entry, so a side-stream kernel can hold back work
    // that would otherwise take SMs before every recurrence cluster is placed (wait_count)
    uint32_t *started;
    // forward overlapped with its Z GEMM (common.cuh arb_decide): != nullptr in the primary launch,
    // which goes ahead only once all arb_target GEMM CTAs are resident and otherwise exits at once;
    // rerun != nullptr (a second launch, a programmatic dependent of the GEMM): wait for the GEMM
    // grid, then exit unless that word carries the abort bit, else run the layer (Z complete)
    uint32_t *arb;
    uint32_t arb_target;
    const uint32_t *rerun;
    unsigned long long *trace;   // debug: per-step phase timestamps of CTA 0 / thread 0, or nullptr
};

// debug hook: per-step phase timestamps (globaltimer ns, 8 per step) of the next launches
void rec_set_trace(unsigned long long *fwd, unsigned long long *bwd);
unsigned long long *rec_trace_fwd();
unsigned long long *rec_trace_bwd();  // the forward trace buffer (nullptr unless set)

// CTA-native layout of Z and of the saved gate activations (one time step = one block per
// (direction, batch group, CTA)): element (t, d, g, c, column block cb, gate row r, i) at
//   ((((t*ndir + d)*G + g)*NC + c)*4 + cb)*128*NQ + r*NQ + i,   NQ = N/4,
// for batch row b = g*Bg + cb*NQ + i and gate column d*4Hq + 128c + r.  Each thread of the
// recurrence kernels reads/writes NQ contiguous values; each warp one contiguous block.
inline size_t rec_mask_bytes(const RecPlan &pl, int T) { return (size_t)T * pl.G * pl.N; }
inline size_t rec_native_elems(const RecPlan &pl, int T) {
    return (size_t)T * pl.ndir * 4 * pl.Hq * pl.G * pl.N;
}
RecPlan rec_plan(int T, int B, int H, int ndir, int num_sms);
bool rec_supported(const RecPlan &pl, int H);
size_t rec_P_bytes(const RecPlan &pl);
// RT16: [ndir][4Hq][Hq] fp16 (row = gate column 4j+gamma, col = k)
int lstm_rec_fwd(const RecParams &p, const __half *RT16, cudaStream_t st);
int lstm_rec_bwd(const RecParams &p, const __half *RT16, cudaStream_t st);

}  // namespace blstm
