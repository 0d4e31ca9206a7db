// api.cu -- the C-ABI of libblstm.so (include/blstm.h): argument validation,
// workspace / reserve carving and the launch sequence of one layer and of the
// BLSTM stack's training step.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "blstm.h"
#include "gemm.h"
#include "lstm_rec.h"
#include "ops.h"
#include "optim.h"
#include "prof.h"
#include "mdlstm.h"
#include "rec_step.h"

using namespace blstm;

// scatter-add output of a weight-gradient GEMM whose rows are the gate-interleaved columns
// d 4Hq + 4u + gamma of dA (gemm.h GemmScatter): row (u, gamma) of direction d -> d dstride +
// gamma H + u; column n -> n ld (colmode 0, n < ncols) or, for padded halves of width Hq, (h H + u) ld
static GemmScatter scatter_gate_rows(float *dst, int H, int Hq, long dstride, int colmode, int ncols, long ld) {
    GemmScatter s;
    s.dst = dst; s.rowmode = 1; s.colmode = colmode; s.H = H; s.Hq = Hq; s.ncols = ncols;
    s.dstride = dstride; s.ld = ld;
    return s;
}

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local char g_err[512] = "";
static int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}
#define TRY(expr, what)                                                                                   \
    do {                                                                                                  \
        int _rc = (expr);                                                                                 \
        if (_rc != 0) {                                                                                   \
            cudaError_t _e = cudaGetLastError();                                                          \
            return fail(BLSTM_ERR_CUDA, "%s failed (rc=%d, cuda: %s)", what, _rc, cudaGetErrorString(_e)); \
        }                                                                                                 \
    } while (0)

extern "C" const char *blstm_last_error(void) { return g_err; }
int blstm_set_error(int code, const char *msg) { return fail(code, "%s", msg); }
extern "C" int blstm_version(void) { return 100; }

// blstm.h: a mask entry outside {0,1} is detected on device (pack_mask / check_mask) and reported
// lazily: by the first API call after the kernel that saw it has completed, or by blstm_check_errors.
static int mask_pending() {
    return mask_flag_take() ? fail(BLSTM_ERR_ARG, "a mask entry outside {0,1} was passed to an earlier call") : 0;
}
extern "C" int blstm_check_errors(void) { return mask_pending(); }

static inline size_t al256(size_t b) { return (b + 255) & ~(size_t)255; }
struct Carve {
    size_t off = 0;
    size_t take(size_t bytes) {
        size_t o = off;
        off += al256(bytes);
        return o;
    }
};
static inline int rup(int a, int b) { return (a + b - 1) / b * b; }
static inline bool al16(const void *p) { return ((uintptr_t)p & 15u) == 0; }
static inline bool al4(const void *p) { return ((uintptr_t)p & 3u) == 0; }

// the Z GEMM writes its output in the recurrence kernels' CTA-native layout (lstm_rec.h)
static void set_native(GemmParams &gp, const RecPlan &pl, int B) {
    gp.natB = B; gp.natBg = pl.Bg; gp.natG = pl.G; gp.natNQ = pl.N / 4; gp.natNC = pl.NC;
    gp.natHq4 = 4 * pl.Hq; gp.natNdir = pl.ndir;
}

// ---------------------------------------------------------------------------
// one layer, one direction
// ---------------------------------------------------------------------------
struct LayerGeo {
    int T, B, D, H, Hq, Dp;
    long TB;
    RecPlan pl;
    bool step = false;  // beyond the persistent kernels' capacity: step-launched recurrence (§5.7)
    int x2w = 0;        // BLSTM_PREC_FP16X2W: the input projection with W split hi + lo (R9)
};
// precision modes (blstm.h): FP16, or FP16X2W (the a1 GEMM reads [W_hi; W_lo] along a doubled K)
static int precision_x2w(int prec, int *x2w) {
    if (prec == BLSTM_PREC_FP16 || prec == BLSTM_PREC_FP16X2W) {
        *x2w = prec == BLSTM_PREC_FP16X2W;
        return 0;
    }
    return fail(BLSTM_ERR_UNSUPPORTED, "precision %d not supported (FP16 = 0, FP16X2W = 1; DESIGN.md R9)", prec);
}
// split-K scratch of the weight-gradient GEMMs (GemmParams::splitk_ws): 32 MB
constexpr long GSK_ELEMS = 8L << 20;

struct FwdWS {
    size_t x16, w16, rt16, bq, Z, maskN, cnt, stepF, total;
};
struct BwdWS {
    size_t x16, w16, rt16, dA, dX, dWT, dRT, dbp, P, maskN, cpk, dypk, gsk, cnt, stepB, cs2, r16, total;
};
struct Reserve {
    size_t gates, hist, total;
};

static int layer_geo(const lstm_desc *d, LayerGeo &g) {
    if (!d) return fail(BLSTM_ERR_ARG, "null lstm_desc");
    if (d->T < 0 || d->B < 1 || d->D < 1 || d->H < 1)
        return fail(BLSTM_ERR_SHAPE, "need T>=0, B>=1, D>=1, H>=1 (got T=%d B=%d D=%d H=%d)", d->T, d->B, d->D, d->H);
    if (d->direction != 1 && d->direction != -1) return fail(BLSTM_ERR_ARG, "direction must be +1 or -1");
    if (d->ldx < d->D || d->ldy < d->H) return fail(BLSTM_ERR_SHAPE, "need ldx >= D and ldy >= H");
    if (int rc = precision_x2w(d->precision, &g.x2w)) return rc;
    g.T = d->T; g.B = d->B; g.D = d->D; g.H = d->H;
    g.TB = (long)d->T * d->B;
    g.pl = rec_plan(d->T, d->B, d->H, 1, num_sms());
    g.Hq = g.pl.Hq;
    g.Dp = rup(d->D, 64);
    const bool force_step = getenv("BLSTM_FORCE_STEP") && atoi(getenv("BLSTM_FORCE_STEP")) != 0;
    g.step = force_step || !rec_supported(g.pl, d->H);
    if (g.step && (long)g.B * 4 * g.Hq * 2 > GSK_ELEMS)
        return fail(BLSTM_ERR_UNSUPPORTED, "H=%d B=%d: no recurrence path for this size", d->H, d->B);
    return 0;
}
static FwdWS fwd_ws(const LayerGeo &g) {
    Carve c;
    FwdWS w;
    w.x16 = c.take((size_t)g.TB * g.Dp * 2);
    w.w16 = c.take((size_t)(g.x2w ? 2 : 1) * g.Dp * 4 * g.Hq * 2);
    w.rt16 = c.take((size_t)4 * g.Hq * g.Hq * 2);
    w.bq = c.take((size_t)4 * g.Hq * 4);
    w.Z = c.take(g.step ? (size_t)g.TB * 4 * g.Hq * 4 : rec_native_elems(g.pl, g.T) * 4);
    w.maskN = c.take(rec_mask_bytes(g.pl, g.T));
    w.cnt = c.take(256);
    w.stepF = c.take(g.step ? rec_step_fwd_scratch_bytes(g.B, g.Hq) : 0);
    w.total = c.off;
    return w;
}
static BwdWS bwd_ws(const LayerGeo &g) {
    Carve c;
    BwdWS w;
    w.x16 = c.take((size_t)g.TB * g.Dp * 2);
    w.w16 = c.take((size_t)(g.x2w ? 2 : 1) * g.Dp * 4 * g.Hq * 2);
    w.rt16 = c.take((size_t)4 * g.Hq * g.Hq * 2);
    w.dA = c.take((size_t)g.TB * 4 * g.Hq * 2);
    w.dX = c.take((size_t)g.TB * g.Dp * 4);
    w.dWT = c.take((size_t)4 * g.Hq * g.Dp * 4);
    w.dRT = c.take((size_t)4 * g.Hq * g.Hq * 4);
    w.dbp = c.take((size_t)g.pl.G * 4 * g.Hq * 4);
    w.P = c.take(rec_P_bytes(g.pl));
    w.maskN = c.take(rec_mask_bytes(g.pl, g.T));
    // c and dy repacked with a 16-byte row pitch when the caller's is not (the BPTT kernel reads
    // them by TMA)
    w.cpk = c.take((size_t)g.TB * g.Hq * 4);
    w.dypk = c.take((size_t)g.TB * g.Hq * 4);
    w.gsk = c.take((size_t)GSK_ELEMS * 4);
    w.cnt = c.take(256);
    w.stepB = c.take(g.step ? rec_step_bwd_scratch_bytes(g.B, g.Hq) : 0);
    w.cs2 = c.take(g.step ? colsum_scratch_bytes(g.TB, 4 * g.Hq) : 0);
    // step mode: R in pack_w's K-major layout, the persistent BPTT's A operand (rec_step.h R16)
    w.r16 = c.take(g.step && rec_step_bwd_persist_ctas(g.B, g.Hq, 1) ? (size_t)4 * g.Hq * g.Hq * 2 : 0);
    w.total = c.off;
    return w;
}
static Reserve reserve_of(const LayerGeo &g) {
    Carve c;
    Reserve r;
    r.gates = c.take(g.step ? (size_t)g.TB * 4 * g.Hq * 2 : rec_native_elems(g.pl, g.T) * 2);
    r.hist = c.take((size_t)(g.T + 1) * g.B * g.Hq * 2);
    r.total = c.off;
    return r;
}

extern "C" size_t lstm_workspace_bytes(const lstm_desc *d) {
    LayerGeo g;
    if (layer_geo(d, g)) return 0;
    const size_t a = fwd_ws(g).total, b = bwd_ws(g).total;
    return a > b ? a : b;
}
extern "C" size_t lstm_reserve_bytes(const lstm_desc *d) {
    LayerGeo g;
    if (layer_geo(d, g)) return 0;
    return reserve_of(g).total;
}

static RecParams base_params(const LayerGeo &g, int ndir, int dir0, const uint8_t *mask) {
    RecParams p;
    memset(&p, 0, sizeof(p));
    p.T = g.T; p.B = g.B; p.H = g.H; p.Hq = g.Hq;
    p.NC = g.pl.NC; p.G = g.pl.G; p.Bg = g.pl.Bg; p.N = g.pl.N; p.ndir = ndir;
    p.dir0 = dir0;
    p.mask = mask;
    return p;
}

extern "C" int lstm_fwd(const lstm_desc *d, const float *x, const uint8_t *mask, const float *W, const float *R,
                        const float *b, const float *h0, const float *c0, float *y, float *c, float *hT, float *cT,
                        void *reserve, void *workspace, size_t workspace_bytes, void *stream) {
    if (int rc = mask_pending()) return rc;
    LayerGeo g;
    if (int rc = layer_geo(d, g)) return rc;
    if (!x || !mask || !W || !R || !b || !y || !c || !reserve || !workspace)
        return fail(BLSTM_ERR_ARG, "lstm_fwd: null required pointer");
    if (!al4(x) || !al4(W) || !al4(R) || !al4(b) || !al4(y) || !al4(c)) return fail(BLSTM_ERR_ALIGN, "misaligned fp32 pointer");
    if (!al16(reserve) || !al16(workspace)) return fail(BLSTM_ERR_ALIGN, "reserve/workspace must be 16-byte aligned");
    const FwdWS w = fwd_ws(g);
    const Reserve rv = reserve_of(g);
    if (workspace_bytes < w.total) return fail(BLSTM_ERR_WORKSPACE, "workspace %zu < %zu bytes", workspace_bytes, w.total);
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *ws = (uint8_t *)workspace, *res = (uint8_t *)reserve;
    if (g.T == 0) {
        const size_t bytes = sizeof(float) * g.B * g.H;
        if (hT) { if (h0) cudaMemcpyAsync(hT, h0, bytes, cudaMemcpyDeviceToDevice, st); else cudaMemsetAsync(hT, 0, bytes, st); }
        if (cT) { if (c0) cudaMemcpyAsync(cT, c0, bytes, cudaMemcpyDeviceToDevice, st); else cudaMemsetAsync(cT, 0, bytes, st); }
        return cudaGetLastError() == cudaSuccess ? 0 : fail(BLSTM_ERR_CUDA, "copy failed");
    }
    __half *x16 = (__half *)(ws + w.x16), *w16 = (__half *)(ws + w.w16), *rt16 = (__half *)(ws + w.rt16);
    float *bq = (float *)(ws + w.bq), *Z = (float *)(ws + w.Z);
    TRY(cast_x_f16(x, d->ldx, g.D, x16, g.Dp, g.TB, st), "cast_x");
    TRY(pack_w(W, nullptr, g.D, g.H, g.Hq, 1, g.Dp, 0, w16, st, g.x2w ? g.Dp : 0), "pack_w");
    TRY(pack_rt(R, nullptr, g.H, g.Hq, 1, rt16, st), "pack_rt");
    TRY(pack_bias(b, nullptr, g.H, g.Hq, 1, bq, st), "pack_bias");
    GemmParams gp{(int)g.TB, 4 * g.Hq, (g.x2w ? 2 : 1) * g.Dp, Z, 4L * g.Hq, 1.f, 0, bq, 0, 0};
    gp.a_kwrap = g.x2w ? g.Dp / GEMM_BK_ELEMS : 0;
    if (!g.step) set_native(gp, g.pl, g.B);  // Z in the recurrence kernels' CTA-native layout
    TRY(gemm_f16({x16, g.Dp, 0}, {w16, 4L * g.Hq, 1}, gp, 0, st), "gemm Z");
    __half *hist = (__half *)(res + rv.hist);
    TRY(init_hist(hist, h0, g.T, g.B, g.H, g.Hq, 1, d->direction, st), "init_hist");
    if (g.step) {  // one launch group per time step (rec_step.h)
        RecStepFwd q{};
        q.T = g.T; q.B = g.B; q.H = g.H; q.Hq = g.Hq; q.ndir = 1; q.dir0 = d->direction;
        q.Z = Z; q.mask = mask; q.RT16 = rt16;
        q.P = (float *)(ws + w.stepF);
        q.C = c; q.ldc = g.H; q.c_doff = 0;
        q.y = y; q.ldy = d->ldy; q.y_doff = 0;
        q.gates = (__half *)(res + rv.gates);
        q.hist = hist;
        q.h0 = h0; q.c0 = c0; q.hT = hT; q.cT = cT;
        TRY(check_mask(mask, g.TB, st), "check_mask");
        TRY(rec_step_fwd(q, st), "rec_step_fwd");
        return 0;
    }
    uint8_t *maskN = ws + w.maskN;
    TRY(pack_mask(mask, g.T, g.B, g.pl.G, g.pl.Bg, g.pl.N, maskN, st), "pack_mask");
    RecParams p = base_params(g, 1, d->direction, mask);
    p.maskN = maskN;
    p.Z = Z; p.ldz = 4L * g.Hq;
    p.y = y; p.ldy = d->ldy; p.y_doff = 0;
    p.C = c; p.ldc = g.H; p.c_doff = 0;
    p.gates = (__half *)(res + rv.gates); p.ldg = 4L * g.Hq;
    p.hist = hist;
    p.c0 = c0; p.h0 = h0; p.hT = hT; p.cT = cT;
    p.counters = (uint32_t *)(ws + w.cnt);
    TRY(lstm_rec_fwd(p, rt16, st), "lstm_rec_fwd");
    return 0;
}

extern "C" int lstm_bwd(const lstm_desc *d, const float *x, const uint8_t *mask, const float *W, const float *R,
                        const float *h0, const float *c0, const float *c, const void *reserve, const float *dy,
                        const float *dhT, const float *dcT, float *dx, float *dW, float *dR, float *db, float *dh0,
                        float *dc0, void *workspace, size_t workspace_bytes, void *stream) {
    (void)h0;  // h0 enters through the saved history (reserve)
    if (int rc = mask_pending()) return rc;
    LayerGeo g;
    if (int rc = layer_geo(d, g)) return rc;
    const bool want_dx = !(d->flags & BLSTM_NO_DX);
    if (!x || !mask || !W || !R || !c || !reserve || !dy || !dW || !dR || !db || !workspace || (want_dx && !dx))
        return fail(BLSTM_ERR_ARG, "lstm_bwd: null required pointer");
    if (!al16(reserve) || !al16(workspace)) return fail(BLSTM_ERR_ALIGN, "reserve/workspace must be 16-byte aligned");
    const BwdWS w = bwd_ws(g);
    const Reserve rv = reserve_of(g);
    if (workspace_bytes < w.total) return fail(BLSTM_ERR_WORKSPACE, "workspace %zu < %zu bytes", workspace_bytes, w.total);
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *ws = (uint8_t *)workspace;
    const uint8_t *res = (const uint8_t *)reserve;
    if (g.T == 0) {
        const size_t bytes = sizeof(float) * g.B * g.H;
        if (dh0) { if (dhT) cudaMemcpyAsync(dh0, dhT, bytes, cudaMemcpyDeviceToDevice, st); else cudaMemsetAsync(dh0, 0, bytes, st); }
        if (dc0) { if (dcT) cudaMemcpyAsync(dc0, dcT, bytes, cudaMemcpyDeviceToDevice, st); else cudaMemsetAsync(dc0, 0, bytes, st); }
        return cudaGetLastError() == cudaSuccess ? 0 : fail(BLSTM_ERR_CUDA, "copy failed");
    }
    __half *x16 = (__half *)(ws + w.x16), *w16 = (__half *)(ws + w.w16), *rt16 = (__half *)(ws + w.rt16);
    __half *dA = (__half *)(ws + w.dA);
    float *dX = (float *)(ws + w.dX), *dWT = (float *)(ws + w.dWT), *dRT = (float *)(ws + w.dRT);
    float *dbp = (float *)(ws + w.dbp);
    TRY(cast_x_f16(x, d->ldx, g.D, x16, g.Dp, g.TB, st), "cast_x");
    TRY(pack_w(W, nullptr, g.D, g.H, g.Hq, 1, g.Dp, 0, w16, st), "pack_w");
    TRY(pack_rt(R, nullptr, g.H, g.Hq, 1, rt16, st), "pack_rt");
    if (g.step) {  // one launch group per time step (rec_step.h); db = column sums of dA
        RecStepBwd q{};
        q.T = g.T; q.B = g.B; q.H = g.H; q.Hq = g.Hq; q.ndir = 1; q.dir0 = d->direction;
        q.mask = mask; q.RT16 = rt16;
        q.C = c; q.ldc = g.H; q.c_doff = 0;
        q.gates = (const __half *)(res + rv.gates);
        q.dy = dy; q.lddy = d->ldy; q.dy_doff = 0;
        q.dA = dA;
        float *sb = (float *)(ws + w.stepB);
        q.dhR = sb;
        q.dhc = sb + rec_step_bwd_partial_floats(g.B, g.Hq);
        q.dcc = q.dhc + 2L * g.B * g.Hq;
        q.c0 = c0; q.dhT = dhT; q.dcT = dcT; q.dh0 = dh0; q.dc0 = dc0;
        if (rec_step_bwd_persist_ctas(g.B, g.Hq, 1)) {  // the persistent BPTT (no launch per time step)
            __half *r16 = (__half *)(ws + w.r16);
            TRY(pack_w(R, nullptr, g.H, g.H, g.Hq, 1, g.Hq, 0, r16, st), "pack_w R16");
            q.R16 = r16;
            if (g.H < g.Hq) {  // it reads c and dy rows Hq wide (padding units: masked out, never stored)
                float *cp = (float *)(ws + w.cpk), *dyp = (float *)(ws + w.dypk);
                TRY(copy_rows(c, g.H, g.TB, g.H, cp, g.Hq, st), "copy_rows c");
                TRY(copy_rows(dy, d->ldy, g.TB, g.H, dyp, g.Hq, st), "copy_rows dy");
                q.C = cp; q.ldc = g.Hq;
                q.dy = dyp; q.lddy = g.Hq;
            }
        }
        TRY(check_mask(mask, g.TB, st), "check_mask");
        if (const int rc = rec_step_bwd(q, st); rc < 0) TRY(rc, "rec_step_bwd");  // 1: the persistent BPTT ran
        if (cudaMemsetAsync(dbp, 0, (size_t)4 * g.Hq * 4, st) != cudaSuccess) return fail(BLSTM_ERR_CUDA, "memset");
        TRY(colsum_f16_add(dA, g.TB, 4 * g.Hq, 4L * g.Hq, 1.f / (float)(1 << DA_SHIFT), dbp, (float *)(ws + w.cs2), st),
            "db colsum");
    } else {
    uint8_t *maskN = ws + w.maskN;
    TRY(pack_mask(mask, g.T, g.B, g.pl.G, g.pl.Bg, g.pl.N, maskN, st), "pack_mask");
    RecParams p = base_params(g, 1, d->direction, mask);
    p.maskN = maskN;
    p.C = const_cast<float *>(c); p.ldc = g.H; p.c_doff = 0;  // read-only in the backward kernel
    if (((uintptr_t)c & 15) || (g.H & 3)) {  // TMA rows need a 16-byte pitch
        float *cpk = (float *)(ws + w.cpk);
        TRY(copy_rows(c, g.H, g.TB, g.H, cpk, g.Hq, st), "copy c");
        p.C = cpk; p.ldc = g.Hq;
    }
    p.gates = (__half *)(res + rv.gates); p.ldg = 4L * g.Hq;
    p.c0 = c0;
    p.dy = dy; p.lddy = d->ldy; p.dy_doff = 0;
    if (((uintptr_t)dy & 15) || (d->ldy & 3)) {
        float *dypk = (float *)(ws + w.dypk);
        TRY(copy_rows(dy, d->ldy, g.TB, g.H, dypk, g.Hq, st), "copy dy");
        p.dy = dypk; p.lddy = g.Hq;
    }
    p.dhT = dhT; p.dcT = dcT;
    p.dA = dA; p.ldda = 4L * g.Hq;
    p.dbpart = dbp;
    p.P = (float *)(ws + w.P);
    p.dh0 = dh0; p.dc0 = dc0;
    p.counters = (uint32_t *)(ws + w.cnt);
    TRY(lstm_rec_bwd(p, rt16, st), "lstm_rec_bwd");
    }
    const float a = 1.f / (float)(1 << DA_SHIFT);
    if (want_dx) {
        GemmParams gp{(int)g.TB, g.Dp, 4 * g.Hq, dX, g.Dp, a, 0, nullptr, 0, 0};
        TRY(gemm_f16({dA, 4L * g.Hq, 0}, {w16, 4L * g.Hq, 0}, gp, 0, st), "gemm dX");
        TRY(store_dx(dx, d->ldx, dX, g.Dp, g.D, g.TB, (d->flags & BLSTM_ACCUM_DX) ? 1 : 0, st), "store_dx");
    }
    {
        // dW [D, 4H] += (dA^T x)^T, scattered from the gate-interleaved rows by the GEMM itself
        GemmParams gp{4 * g.Hq, g.Dp, (int)g.TB, dWT, g.Dp, a, 0, nullptr, 0, 0};
        gp.splitk_ws = (float *)(ws + w.gsk); gp.splitk_elems = GSK_ELEMS;
        gp.scat = scatter_gate_rows(dW, g.H, g.Hq, 0, 0, g.D, 4L * g.H);
        TRY(gemm_f16({dA, 4L * g.Hq, 1}, {x16, g.Dp, 1}, gp, 0, st), "gemm dW");
    }
    {
        const __half *hprev = (const __half *)(res + rv.hist) + (d->direction < 0 ? (long)g.B * g.Hq : 0);
        GemmParams gp{4 * g.Hq, g.Hq, (int)g.TB, dRT, g.Hq, a, 0, nullptr, 0, 0};
        gp.splitk_ws = (float *)(ws + w.gsk); gp.splitk_elems = GSK_ELEMS;
        gp.scat = scatter_gate_rows(dR, g.H, g.Hq, 0, 0, g.H, 4L * g.H);
        TRY(gemm_f16({dA, 4L * g.Hq, 1}, {hprev, g.Hq, 1}, gp, 0, st), "gemm dR");
    }
    TRY(scatter_b(db, g.H, g.Hq, dbp, g.step ? 1 : g.pl.G, 0, st), "scatter db");
    return 0;
}

// ---------------------------------------------------------------------------
// BLSTM stack
// ---------------------------------------------------------------------------
struct StackGeo {
    int L, D, H, K, T, B, Hq, Dp0, Kp;
    long TB;
    RecPlan pl;
    std::vector<int> Dn, Drows, rowmode;
    Dropout dr;  // input dropout of the training step (R20); dr.on == 0: off
    // beyond the persistent kernels' on-chip capacity (e.g. H = 1024): step-launched recurrence
    // (rec_step.h); BLSTM_FORCE_STEP=1 selects it for any size (tests)
    bool step = false;
    int x2w = 0;  // BLSTM_PREC_FP16X2W (LayerGeo::x2w)
    int dbs = 0;  // db partial groups per direction and parity in the dbp buffer
};
struct StackWS {
    size_t x16, Z, maskN, zflags, dA, dY0, dY1, dWT, dRT, dbp, P, cnt, wo16, boq, dlog16, dWoT, rowloss, rowerr, cs, gsk,
        stepF, stepB, cs2, optp, tsk, total;
    size_t maxDn;
    std::vector<size_t> y16, w16, rt16, bq, gates, C, hist, r16;
};

static int stack_geo(const blstm_stack_desc *d, StackGeo &g) {
    if (!d) return fail(BLSTM_ERR_ARG, "null blstm_stack_desc");
    if (d->L < 1 || d->D < 1 || d->H < 1 || d->K < 0 || d->T < 1 || d->B < 1)
        return fail(BLSTM_ERR_SHAPE, "need L,D,H,T,B >= 1 and K >= 0");
    if (int rc = precision_x2w(d->precision, &g.x2w)) return rc;
    g.L = d->L; g.D = d->D; g.H = d->H; g.K = d->K; g.T = d->T; g.B = d->B;
    g.TB = (long)d->T * d->B;
    g.pl = rec_plan(d->T, d->B, d->H, 2, num_sms());
    g.Hq = g.pl.Hq;
    g.Dp0 = rup(d->D, 64);
    g.Kp = d->K > 0 ? rup(d->K, 64) : 0;
    const bool force_step = getenv("BLSTM_FORCE_STEP") && atoi(getenv("BLSTM_FORCE_STEP")) != 0;
    g.step = force_step || !rec_supported(g.pl, d->H);
    if (g.step && (g.Hq % 256 != 0 || (long)g.B * 4 * g.Hq * 2 > GSK_ELEMS))
        return fail(BLSTM_ERR_UNSUPPORTED, "H=%d B=%d: no recurrence path for this size", d->H, d->B);
    if (!(d->dropout >= 0.f && d->dropout < 1.f)) return fail(BLSTM_ERR_ARG, "dropout must be in [0, 1)");
    g.dr.on = d->dropout > 0.f;
    g.dr.thr = (uint32_t)floor((double)d->dropout * 4294967296.0);
    g.dr.seed = d->dropout_seed;
    g.dr.scale = (float)(1.0 / (1.0 - (double)d->dropout));
    g.dbs = g.step ? (g.pl.G > rec_step_bwd_db_groups() ? g.pl.G : rec_step_bwd_db_groups()) : g.pl.G;
    g.Dn.resize(g.L); g.Drows.resize(g.L); g.rowmode.resize(g.L);
    for (int l = 0; l < g.L; ++l) {
        g.Dn[l] = l == 0 ? g.Dp0 : 2 * g.Hq;
        g.Drows[l] = l == 0 ? g.D : 2 * g.H;
        g.rowmode[l] = l == 0 ? 0 : 1;
    }
    return 0;
}
// Z GEMM completion counters [L][2 directions][M tiles], then one BPTT "CTAs started" counter per
// layer, then two start-arbitration words per layer (forward recurrence vs its Z GEMM, common.cuh)
static size_t zflag_words(const StackGeo &g) {
    return (size_t)g.L * 2 * ((g.TB + GEMM_BM_ROWS - 1) / GEMM_BM_ROWS) + 3 * g.L;
}
// true when something may serialize kernels or withhold SMs from a concurrent launch: a profiler
// or sanitizer injected into the process (ncu, compute-sanitizer: CUDA_INJECTION64_PATH),
// CUDA_LAUNCH_BLOCKING=1, or an MPS SM cap.  The Z-GEMM overlap is then not attempted at all
// (the start arbitration would also keep it correct, after a 20 ms wait per layer).
static bool tool_injected() {  // a profiler / sanitizer library mapped into this process
    FILE *f = fopen("/proc/self/maps", "r");
    if (!f) return false;
    char line[1024];
    bool hit = false;
    while (!hit && fgets(line, sizeof line, f))
        hit = strstr(line, "Injection") || strstr(line, "nsight-compute") || strstr(line, "libsanitizer") ||
              strstr(line, "compute-sanitizer");
    fclose(f);
    return hit;
}
static bool serialized_env() {
    const char *inj = getenv("CUDA_INJECTION64_PATH");
    const char *lb = getenv("CUDA_LAUNCH_BLOCKING");
    const char *mps = getenv("CUDA_MPS_ACTIVE_THREAD_PERCENTAGE");
    return (inj && *inj) || (lb && atoi(lb) != 0) || (mps && *mps) || tool_injected();
}
static StackWS stack_ws(const StackGeo &g) {
    Carve c;
    StackWS w;
    const long TB = g.TB;
    const int Hq = g.Hq;
    int maxDn = 0;
    for (int v : g.Dn) maxDn = v > maxDn ? v : maxDn;
    w.x16 = c.take((size_t)TB * g.Dp0 * 2);
    for (int l = 0; l < g.L; ++l) {
        w.y16.push_back(c.take((size_t)TB * 2 * Hq * 2));
        w.w16.push_back(c.take((size_t)(g.x2w ? 2 : 1) * g.Dn[l] * 8 * Hq * 2));
        w.rt16.push_back(c.take((size_t)2 * 4 * Hq * Hq * 2));
        w.bq.push_back(c.take((size_t)8 * Hq * 4));
        const size_t ge = g.step ? (size_t)TB * 8 * Hq : rec_native_elems(g.pl, g.T);
        w.gates.push_back(c.take(ge * 2));
        w.C.push_back(c.take((size_t)2 * TB * Hq * 4));
        w.hist.push_back(c.take((size_t)2 * (g.T + 1) * g.B * Hq * 2));
        // step mode: R in pack_w's K-major layout [Hq][8Hq] (the persistent BPTT's A operand)
        w.r16.push_back(c.take(g.step ? (size_t)Hq * 8 * Hq * 2 : 0));
    }
    const size_t zn = g.step ? (size_t)TB * 8 * Hq : rec_native_elems(g.pl, g.T), zl = (size_t)TB * g.Kp;  // Z / logits
    w.Z = c.take((zn > zl ? zn : zl) * 4);
    w.maskN = c.take(rec_mask_bytes(g.pl, g.T));
    w.zflags = c.take(zflag_words(g) * 4);
    w.maxDn = maxDn;
    // dA / dWT / dRT / dbpart: two copies (layer parity) so layer l's weight gradients can run on a
    // side stream while BPTT of layer l-1 writes the other copy
    w.dA = c.take((size_t)2 * TB * 8 * Hq * 2);
    w.dY0 = c.take((size_t)TB * 2 * Hq * 4);
    w.dY1 = c.take((size_t)TB * 2 * Hq * 4);
    w.dWT = c.take((size_t)2 * 8 * Hq * maxDn * 4);
    w.dRT = c.take((size_t)2 * 2 * 4 * Hq * Hq * 4);
    w.dbp = c.take((size_t)2 * 2 * g.dbs * 4 * Hq * 4);
    w.P = c.take(rec_P_bytes(g.pl));
    w.cnt = c.take(256);
    w.wo16 = c.take((size_t)2 * Hq * (g.Kp ? g.Kp : 64) * 2);
    w.boq = c.take((size_t)(g.Kp ? g.Kp : 64) * 4);
    w.dlog16 = c.take((size_t)TB * (g.Kp ? g.Kp : 64) * 2);
    w.dWoT = c.take((size_t)(g.K ? g.K : 1) * 2 * Hq * 4);
    w.rowloss = c.take((size_t)TB * 8);
    w.rowerr = c.take((size_t)TB * 4);
    w.cs = c.take(colsum_scratch_bytes(TB, g.K ? g.K : 1));
    w.gsk = c.take((size_t)GSK_ELEMS * 4);
    w.tsk = c.take((size_t)gemm_tail_elems() * 4);  // s_main GEMMs' tail-wave partials (gemm.h tail_ws)
    // step mode: per-step scratch and the column-sum scratch of db (dbpart from dA)
    w.stepF = c.take(g.step ? rec_step_fwd_scratch_bytes(g.B, Hq) : 0);
    w.stepB = c.take(g.step ? rec_step_bwd_scratch_bytes(g.B, Hq) : 0);
    w.cs2 = c.take(g.step ? colsum_scratch_bytes(TB, 8 * Hq) : 0);
    w.optp = c.take(sizeof(double) * (size_t)opt_norm_partials());  // norm partials of a fused update
    w.total = c.off;
    return w;
}

static size_t param_layout(const blstm_stack_desc *d, size_t *offs) {
    size_t o = 0;
    const size_t H = d->H;
    for (int l = 0; l < d->L; ++l) {
        const size_t Dl = l == 0 ? (size_t)d->D : 2 * H;
        for (int dd = 0; dd < 2; ++dd) {
            const int e = 6 * l + 3 * dd;
            if (offs) {
                offs[e] = o;
                offs[e + 1] = o + Dl * 4 * H;
                offs[e + 2] = o + Dl * 4 * H + 4 * H * H;
            }
            o += Dl * 4 * H + 4 * H * H + 4 * H;
        }
    }
    if (offs) {
        offs[6 * d->L] = o;
        offs[6 * d->L + 1] = o + (d->K > 0 ? 2 * H * d->K : 0);
    }
    if (d->K > 0) o += 2 * H * d->K + d->K;
    return o;
}

// The sync-mode exchange buckets of one step, in the order stack_step_impl issues them: the head
// [offs[6L], P) first (when K > 0), then layer L-1 down to layer 0, layer l = [offs[6l], next).
// They partition [0, P).  Returns the bucket count (<= L + 1).
static int dp_buckets(const blstm_stack_desc *d, size_t *lo, size_t *hi) {
    std::vector<size_t> offs(6 * d->L + 2);
    const size_t n = param_layout(d, offs.data());
    int k = 0;
    if (d->K > 0) { lo[k] = offs[6 * d->L]; hi[k] = n; ++k; }
    for (int l = d->L - 1; l >= 0; --l) {
        lo[k] = offs[6 * l];
        hi[k] = l + 1 < d->L ? offs[6 * (l + 1)] : offs[6 * d->L];
        ++k;
    }
    return k;
}
extern "C" int blstm_dp_buckets(const blstm_stack_desc *d, size_t *lo, size_t *hi, int max_buckets) {
    if (!d || d->L < 1 || d->H < 1 || d->D < 1 || d->K < 0 || !lo || !hi) return fail(BLSTM_ERR_ARG, "bad argument");
    if (max_buckets < d->L + (d->K > 0 ? 1 : 0)) return fail(BLSTM_ERR_ARG, "need room for %d buckets", d->L + 1);
    return dp_buckets(d, lo, hi);
}

extern "C" size_t blstm_param_count(const blstm_stack_desc *d) {
    if (!d || d->L < 1 || d->H < 1 || d->D < 1 || d->K < 0) return 0;
    return param_layout(d, nullptr);
}
extern "C" size_t blstm_param_offsets(const blstm_stack_desc *d, size_t *offs) {
    if (!d || d->L < 1 || d->H < 1 || d->D < 1 || d->K < 0) return 0;
    return param_layout(d, offs);
}
extern "C" size_t blstm_stack_workspace_bytes(const blstm_stack_desc *d) {
    StackGeo g;
    if (stack_geo(d, g)) return 0;
    return stack_ws(g).total;
}

// forward of the whole stack; Yout [L,T,B,2H] / Cout [L,2,T,B,H] optional (parity view).
// train: apply the input dropout of g.dr (sites 0..L-1 on the layer inputs, site L on the head's)
// side / packed (train step): the operand packs of layers 1..L-1 run on `side`
// beside layer 0 (recorded on `packed`; layer 1 waits for it); pack_head: the CE head's operands
// are packed in the preamble launch too
static int stack_forward(const blstm_stack_desc *d, const StackGeo &g, const StackWS &w, uint8_t *ws,
                         const float *theta, const float *x, const uint8_t *mask, float *Yout, float *Cout,
                         cudaStream_t st, bool train = false, cudaStream_t side = nullptr, cudaEvent_t packed = nullptr,
                         bool pack_head = false, cudaEvent_t z0done = nullptr, bool *r16_on_side = nullptr) {
    const bool drop = train && g.dr.on;
    std::vector<size_t> offs(6 * g.L + 2);
    param_layout(d, offs.data());
    const int Hq = g.Hq;
    __half *x16 = (__half *)(ws + w.x16);
    // layers 1..L-1's packs on the side stream beside layer 0 (C3: 7.17 vs 7.21 ms per step with every
    // pack in the preamble launch); BLSTM_PREP_SPLIT=0: all in the preamble launch
    static const bool prep_split = !(getenv("BLSTM_PREP_SPLIT") && atoi(getenv("BLSTM_PREP_SPLIT")) == 0);
    // (step mode: deferred until layer 0's Z GEMM is done -- beside it they slowed that HBM-bound
    // GEMM -- and with the persistent BPTT's R16 packs of every layer, which then leave the critical
    // path too: *r16_on_side)
    const bool split_pack = prep_split && !g.step && side && side != st && packed && g.L > 1 && g.L <= PACK_MAXL;
    const bool step_defer = prep_split && g.step && train && side && side != st && packed && z0done &&
                            g.L <= PACK_MAXL && (g.L > 1 || r16_on_side);
    const bool defer_r16 = step_defer && r16_on_side && rec_step_bwd_persist_ctas(g.B, g.Hq, 2) > 0;
    if (r16_on_side) *r16_on_side = defer_r16;
    auto pack_range = [&](int l0, int l1, PackLayers &pk) {
        pk.L = l1 - l0; pk.H = g.H; pk.Hq = Hq;
        for (int l = l0; l < l1; ++l) {
            const int i = l - l0;
            for (int dd = 0; dd < 2; ++dd) {
                pk.W[i][dd] = theta + offs[6 * l + 3 * dd];
                pk.R[i][dd] = theta + offs[6 * l + 3 * dd + 1];
                pk.b[i][dd] = theta + offs[6 * l + 3 * dd + 2];
            }
            pk.Drows[i] = g.Drows[l]; pk.Dn[i] = g.Dn[l]; pk.rowmode[i] = g.rowmode[l];
            pk.lo_rows[i] = g.x2w ? g.Dn[l] : 0;
            pk.W16[i] = (__half *)(ws + w.w16[l]); pk.RT16[i] = (__half *)(ws + w.rt16[l]);
            pk.bq[i] = (float *)(ws + w.bq[l]);
        }
    };
    float *Z = (float *)(ws + w.Z);
    uint8_t *maskN = ws + w.maskN;  // shared by every layer, forward and BPTT
    const int num_m = (int)((g.TB + GEMM_BM_ROWS - 1) / GEMM_BM_ROWS);
    uint32_t *zflags = (uint32_t *)(ws + w.zflags);
    // the preamble in one launch (ops.h StackPrep): x16, the operand packs of layer 0 (every layer
    // without the side stream), the mask, the Z flags and every layer's h0 history slots
    {
        StackPrep pr{};
        pr.x = x; pr.ldx = g.D; pr.D = g.D; pr.x16 = x16; pr.Dp = g.Dp0; pr.rows = g.TB;
        pr.dr = drop ? g.dr : Dropout{0, 0, 0, 1.f};
        if (g.L <= PACK_MAXL) pack_range(0, (split_pack || step_defer) ? 1 : g.L, pr.pk);
        pr.pk.H = g.H; pr.pk.Hq = Hq;
        if (pack_head && g.K > 0) {  // the CE head's operands (pack_wout)
            pr.Wo = theta + offs[6 * g.L]; pr.bo = theta + offs[6 * g.L + 1]; pr.K = g.K; pr.Kp = g.Kp;
            pr.Wo16 = (__half *)(ws + w.wo16); pr.boq = (float *)(ws + w.boq);
        }
        pr.mask_mode = g.step ? 2 : 1; pr.mask = mask; pr.T = g.T; pr.B = g.B;
        pr.G = g.pl.G; pr.Bg = g.pl.Bg; pr.N = g.pl.N; pr.maskN = maskN; pr.mask_n = g.TB;
        pr.zero = zflags; pr.zero_n = (long)zflag_words(g);
        if (g.L <= PACK_MAXL) {
            pr.hist_L = g.L; pr.hT = g.T; pr.hB = g.B; pr.hHq = Hq;
            for (int l = 0; l < g.L; ++l) pr.hl.hist[l] = (__half *)(ws + w.hist[l]);
        }
        TRY(stack_prep(pr, st), "stack_prep");
    }
    if (split_pack) {  // layers 1..L-1's operand copies on the side stream (after s_main's launch)
        PackLayers pk{};
        pack_range(1, g.L, pk);
        TRY(pack_layers(pk, side), "pack_layers (side)");
        TRY((int)cudaEventRecord(packed, side), "cudaEventRecord");
    }
    if (g.L > PACK_MAXL) {  // (beyond the one-launch tables: per layer)
        for (int l = 0; l < g.L; ++l) {
            const float *Wf = theta + offs[6 * l], *Rf = theta + offs[6 * l + 1], *bf = theta + offs[6 * l + 2];
            const float *Wb = theta + offs[6 * l + 3], *Rb = theta + offs[6 * l + 4], *bb = theta + offs[6 * l + 5];
            TRY(pack_w(Wf, Wb, g.Drows[l], g.H, Hq, 2, g.Dn[l], g.rowmode[l], (__half *)(ws + w.w16[l]), st,
                       g.x2w ? g.Dn[l] : 0), "pack_w");
            TRY(pack_rt(Rf, Rb, g.H, Hq, 2, (__half *)(ws + w.rt16[l]), st), "pack_rt");
            TRY(pack_bias(bf, bb, g.H, Hq, 2, (float *)(ws + w.bq[l]), st), "pack_bias");
            TRY(init_hist((__half *)(ws + w.hist[l]), nullptr, g.T, g.B, g.H, Hq, 2, 1, st), "init_hist");
        }
    }
    // Overlap: layer l's recurrence is launched first and, once all its CTAs are resident, triggers
    // the Z GEMM as a programmatic dependent launch on the SMs its clusters leave free; the
    // recurrence waits per M-tile on the GEMM's completion counters.  Only when every GEMM CTA can
    // be co-resident with the clusters (one CTA per SM each): a GEMM CTA waiting for an SM would
    // deadlock the spinning recurrence.  Otherwise the GEMM simply runs first.
    // BLSTM_OVERLAP=0 disables it: profilers that serialize or replay kernels one at a time (ncu)
    // would otherwise leave the recurrence waiting for a GEMM that cannot run beside it.
    const int side_ctas = num_sms() - 2 * g.pl.G * g.pl.NC;
    // BLSTM_OVERLAP=0: never; =2: even in a serialized environment (tests of the arbitration)
    static const int overlap_mode = getenv("BLSTM_OVERLAP") ? atoi(getenv("BLSTM_OVERLAP")) : 1;
    static const bool overlap_env = overlap_mode == 2 || (overlap_mode != 0 && !serialized_env());
    const bool overlap = overlap_env && side_ctas >= 8 && !g.step;
    if (overlap && gemm_prepare()) return fail(BLSTM_ERR_CUDA, "gemm_prepare");
    for (int l = 0; l < g.L; ++l) {
        if (l == 1 && (split_pack || step_defer))  // layers 1..L-1's operand copies (side stream)
            TRY((int)cudaStreamWaitEvent(st, packed, 0), "cudaStreamWaitEvent");
        if (drop && l > 0)  // layer l's input = layer l-1's output, dropped in place (site l)
            TRY(dropout_f16((__half *)(ws + w.y16[l - 1]), g.TB, g.H, Hq, l, g.dr, st), "dropout");
        const __half *A = l == 0 ? x16 : (const __half *)(ws + w.y16[l - 1]);
        const long lda = l == 0 ? g.Dp0 : 2L * Hq;
        if (g.step) {  // row-major Z, then one launch pair per time step (rec_step.h)
            GemmParams gz{(int)g.TB, 8 * Hq, (g.x2w ? 2 : 1) * g.Dn[l], Z, 8L * Hq, 1.f, 0, (const float *)(ws + w.bq[l]), 0, 0};
            gz.tail_ws = (float *)(ws + w.tsk); gz.tail_elems = gemm_tail_elems();
            gz.a_kwrap = g.x2w ? g.Dn[l] / GEMM_BK_ELEMS : 0;
            TRY(gemm_f16({A, lda, 0}, {ws + w.w16[l], 8L * Hq, 1}, gz, 0, st), "gemm Z");
            if (l == 0 && step_defer) {  // the deferred operand packs, beside layer 0's recurrence
                TRY((int)cudaEventRecord(z0done, st), "cudaEventRecord");
                TRY((int)cudaStreamWaitEvent(side, z0done, 0), "cudaStreamWaitEvent");
                if (g.L > 1) {
                    PackLayers pk{};
                    pack_range(1, g.L, pk);
                    TRY(pack_layers(pk, side), "pack_layers (side)");
                }
                if (defer_r16)  // R of every layer in pack_w's K-major layout (the persistent BPTT's A)
                    for (int l2 = 0; l2 < g.L; ++l2)
                        TRY(pack_w(theta + offs[6 * l2 + 1], theta + offs[6 * l2 + 4], g.H, g.H, Hq, 2, Hq, 0,
                                   (__half *)(ws + w.r16[l2]), side), "pack_w R16");
                TRY((int)cudaEventRecord(packed, side), "cudaEventRecord");
            }
            __half *hist = (__half *)(ws + w.hist[l]);
            RecStepFwd q{};
            q.T = g.T; q.B = g.B; q.H = g.H; q.Hq = Hq; q.ndir = 2; q.dir0 = 1;
            q.Z = Z; q.mask = mask; q.RT16 = (const __half *)(ws + w.rt16[l]);
            q.P = (float *)(ws + w.stepF);
            if (Cout) { q.C = Cout + (size_t)l * 2 * g.TB * g.H; q.ldc = g.H; q.c_doff = g.TB * g.H; }
            else { q.C = (float *)(ws + w.C[l]); q.ldc = Hq; q.c_doff = g.TB * Hq; }
            if (Yout) { q.y = Yout + (size_t)l * g.TB * 2 * g.H; q.ldy = 2L * g.H; q.y_doff = g.H; }
            q.y16 = (__half *)(ws + w.y16[l]);
            q.gates = (__half *)(ws + w.gates[l]);
            q.hist = hist;
            TRY(rec_step_fwd(q, st), "rec_step_fwd");
            continue;
        }
        GemmParams gp{(int)g.TB, 8 * Hq, (g.x2w ? 2 : 1) * g.Dn[l], Z, 8L * Hq, 1.f, 0, (const float *)(ws + w.bq[l]), 0, 0};
        gp.a_kwrap = g.x2w ? g.Dn[l] / GEMM_BK_ELEMS : 0;
        set_native(gp, g.pl, g.B);  // Z in the recurrence kernels' CTA-native layout
        gp.flags = zflags + (size_t)l * 2 * num_m;
        gp.flag_desc = 2;  // direction 1 (backward) reads time steps in descending order
        gp.pdl = overlap;
        if (!overlap) TRY(gemm_f16({A, lda, 0}, {ws + w.w16[l], 8L * Hq, 1}, gp, 0, st), "gemm Z");
        __half *hist = (__half *)(ws + w.hist[l]);
        RecParams p = base_params(LayerGeo{g.T, g.B, g.D, g.H, Hq, 0, g.TB, g.pl}, 2, 1, mask);
        p.maskN = maskN;
        p.Z = Z; p.ldz = 8L * Hq;
        p.zflags = gp.flags; p.zflag_target = 4 * Hq / gemm_bn(8 * Hq); p.zflag_nm = num_m;
        if (Yout) { p.y = Yout + (size_t)l * g.TB * 2 * g.H; p.ldy = 2L * g.H; p.y_doff = g.H; }
        p.y16 = (__half *)(ws + w.y16[l]); p.ldy16 = 2L * Hq;
        if (Cout) { p.C = Cout + (size_t)l * 2 * g.TB * g.H; p.ldc = g.H; p.c_doff = g.TB * g.H; }
        else { p.C = (float *)(ws + w.C[l]); p.ldc = Hq; p.c_doff = g.TB * Hq; }
        p.gates = (__half *)(ws + w.gates[l]); p.ldg = 8L * Hq;
        p.hist = hist;
        p.counters = (uint32_t *)(ws + w.cnt);
        if (overlap) {  // the three launches are timed as one forward-recurrence scope (prof_suspend)
            // start arbitration (common.cuh): the recurrence goes ahead only once every GEMM CTA is
            // resident; otherwise it exits and the conditional re-launch after the GEMM runs it
            static const int arb_mode = getenv("BLSTM_ARB") ? atoi(getenv("BLSTM_ARB")) : 3;  // A/B: bit 0 arb, bit 1 rerun
            uint32_t *arb = zflags + zflag_words(g) - 2 * g.L + 2 * l;
            gp.arb = (arb_mode & 1) ? arb : nullptr;
            p.arb = (arb_mode & 1) ? arb : nullptr;
            p.arb_target = (uint32_t)gemm_grid((int)g.TB, 8 * Hq, 0, side_ctas);
            RecParams p2 = p;
            p2.arb = nullptr;
            p2.rerun = arb;
            ProfScope ps(PROF_REC_FWD, st);
            prof_suspend(1);
            const int rc1 = lstm_rec_fwd(p, (const __half *)(ws + w.rt16[l]), st);
            const int rc2 = rc1 ? 0 : gemm_f16({A, lda, 0}, {ws + w.w16[l], 8L * Hq, 1}, gp, side_ctas, st);
            const int rc3 = (rc1 || rc2 || !(arb_mode & 2)) ? 0 : lstm_rec_fwd(p2, (const __half *)(ws + w.rt16[l]), st);
            prof_suspend(0);
            TRY(rc1, "lstm_rec_fwd");
            TRY(rc2, "gemm Z");
            TRY(rc3, "lstm_rec_fwd (conditional re-launch)");
        } else {
            TRY(lstm_rec_fwd(p, (const __half *)(ws + w.rt16[l]), st), "lstm_rec_fwd");
        }
    }
    return 0;
}

static int check_stack_ptrs(const StackWS &w, const float *theta, const float *x, const uint8_t *mask, void *workspace,
                            size_t workspace_bytes) {
    if (!theta || !x || !mask || !workspace) return fail(BLSTM_ERR_ARG, "null required pointer");
    if (!al16(theta) || !al4(x) || !al16(workspace)) return fail(BLSTM_ERR_ALIGN, "theta/workspace must be 16-byte aligned");
    if (workspace_bytes < w.total) return fail(BLSTM_ERR_WORKSPACE, "workspace %zu < %zu bytes", workspace_bytes, w.total);
    return 0;
}

extern "C" int blstm_stack_fwd(const blstm_stack_desc *d, const float *theta, const float *x, const uint8_t *mask,
                               float *Y, float *C, void *workspace, size_t workspace_bytes, void *stream) {
    if (int rc = mask_pending()) return rc;
    StackGeo g;
    if (int rc = stack_geo(d, g)) return rc;
    const StackWS w = stack_ws(g);
    if (int rc = check_stack_ptrs(w, theta, x, mask, workspace, workspace_bytes)) return rc;
    return stack_forward(d, g, w, (uint8_t *)workspace, theta, x, mask, Y, C, (cudaStream_t)stream);
}

int dp_allreduce_grads_impl(dp_comm *c, float *grad, size_t n, cudaStream_t st);

static int opt_range(const blstm_opt_params *p, const blstm_stack_desc *layout, float *theta, float *grad,
                     float *state, size_t n, size_t lo, size_t hi, int zero_grad, double *partial, cudaStream_t st);
static int opt_check(const blstm_opt_params *p, float *theta, float *grad, float *state, size_t n);

// forward + BPTT (+ the update rule opt, when given: per bucket on the side stream as soon as the
// bucket is final -- after its scatters and its allreduce -- or, with the global norm constraint,
// once over everything at the end)
static int stack_step_impl(const blstm_stack_desc *d, const float *theta, float *grad, const float *x,
                           const uint8_t *mask, const int32_t *labels, const float *dy_top, double *loss_sum,
                           int32_t *frame_errors, dp_comm *comm, const blstm_opt_params *opt, float *opt_state,
                           void *workspace, size_t workspace_bytes, void *s_main, void *s_side) {
    if (int rc = mask_pending()) return rc;
    StackGeo g;
    if (int rc = stack_geo(d, g)) return rc;
    const StackWS w = stack_ws(g);
    if (int rc = check_stack_ptrs(w, theta, x, mask, workspace, workspace_bytes)) return rc;
    if (!grad || !loss_sum) return fail(BLSTM_ERR_ARG, "null grad / loss_sum");
    if (!al16(grad)) return fail(BLSTM_ERR_ALIGN, "grad must be 16-byte aligned");
    if (g.K > 0 && !labels) return fail(BLSTM_ERR_ARG, "K > 0 needs labels");
    if (g.K == 0 && !dy_top) return fail(BLSTM_ERR_ARG, "K == 0 needs dy_top");
    cudaStream_t st = (cudaStream_t)s_main;
    uint8_t *ws = (uint8_t *)workspace;
    std::vector<size_t> offs(6 * g.L + 2);
    const size_t nparam = param_layout(d, offs.data());
    // BLSTM_NO_SIDE=1: run the off-critical-path work on s_main too (experiments)
    static const bool no_side = getenv("BLSTM_NO_SIDE") && atoi(getenv("BLSTM_NO_SIDE")) != 0;
    cudaStream_t side = (s_side && s_side != s_main && !no_side) ? (cudaStream_t)s_side : st;
    const bool overlap = side != st;
    // events: [l] main -> side (dA of layer l ready), [L] side -> main (all done), [L+1] start,
    // [L+2+l] side -> main (layer l's gradient work done: its parity buffers may be reused),
    // [2L+2] side -> main (the side stream's latest GEMMs are done with the split-K scratch),
    // [2L+3] main -> side (layer 0's dW and direction-1 dR are accumulated: the forked tail, side_layer),
    // [2L+4] main -> side (start of the call), [2L+5] main -> side (step mode: layer 0's Z GEMM done),
    // [2L+6] main -> side (ce_head done: the loss reduction runs on the side stream),
    // [2L+7] side -> main (the operand packs of layers 1..L-1 done, stack_forward)
    // (per thread and per device: an event may only be recorded on a stream of its own device)
    static thread_local std::map<int, std::vector<cudaEvent_t>> evs_by_dev;
    int cur_dev = 0;
    if (cudaGetDevice(&cur_dev) != cudaSuccess) return fail(BLSTM_ERR_CUDA, "cudaGetDevice");
    std::vector<cudaEvent_t> &evs = evs_by_dev[cur_dev];
    const int GSK_FREE = 2 * g.L + 2;
    if (overlap && evs.size() < 2 * (size_t)g.L + 8) {
        while (evs.size() < 2 * (size_t)g.L + 8) {
            cudaEvent_t e;
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return fail(BLSTM_ERR_CUDA, "event");
            evs.push_back(e);
        }
    }
    if (overlap) {  // the side stream starts behind everything issued so far on s_main
        TRY((int)cudaEventRecord(evs[2 * g.L + 4], st), "cudaEventRecord");
        TRY((int)cudaStreamWaitEvent(side, evs[2 * g.L + 4], 0), "cudaStreamWaitEvent");
    }
    bool r16_on_side = false;
    if (int rc = stack_forward(d, g, w, ws, theta, x, mask, nullptr, nullptr, st, true, overlap ? side : nullptr,
                               overlap ? evs[2 * g.L + 7] : nullptr, true, overlap ? evs[2 * g.L + 5] : nullptr,
                               &r16_on_side))
        return rc;
    if (g.dr.on && g.K > 0)  // the head's input (site L)
        TRY(dropout_f16((__half *)(ws + w.y16[g.L - 1]), g.TB, g.H, g.Hq, g.L, g.dr, st), "dropout");

    const int Hq = g.Hq;
    const float a = 1.f / (float)(1 << DA_SHIFT);
    float *dY[2] = {(float *)(ws + w.dY0), (float *)(ws + w.dY1)};
    const __half *ytop = (const __half *)(ws + w.y16[g.L - 1]);
    // Weight gradients (dW, dR, db) of layer l are off the critical path (PAPER.md P:233-234 only
    // needs them after BPTT of layer l): with a side stream they run on the SMs the recurrence
    // clusters leave free, overlapping BPTT of layer l-1.  Their inputs (dA, dbpart) and scratch
    // are double-buffered by layer parity.
    const int rec_ctas = 2 * g.pl.G * g.pl.NC;
    const bool bucket_update = opt && !(opt->max_norm > 0.0);
    // exchange / update buckets (dp_buckets): index 0 = head (K > 0), then layers L-1 .. 0
    std::vector<size_t> blo(g.L + 1), bhi(g.L + 1);
    dp_buckets(d, blo.data(), bhi.data());
    const int bhead = g.K > 0 ? 1 : 0;
    // per-layer BPTT start counters (zeroed with the Z flags by stack_forward)
    uint32_t *bstarted = (uint32_t *)(ws + w.zflags) + (zflag_words(g) - 3 * g.L);
    // Side-stream work that overlaps BPTT(l) must not take SMs before BPTT(l)'s clusters are all
    // placed: GEMM CTAs dispatched first spread over every GPC, no GPC keeps 16 free SMs and the
    // BPTT waits for the whole GEMM (measured: 0.98 instead of 0.63 ms per layer).  Both become
    // ready when the same main-stream kernel completes, so the order is a race; a one-CTA kernel
    // on the side stream waits for BPTT(l)'s CTAs to check in first.
    static const bool no_guard = getenv("BLSTM_NO_GUARD") && atoi(getenv("BLSTM_NO_GUARD")) != 0;  // A/B
    // step mode: the persistent BPTT (rec_step.cu) when it applies, else the launched chain
    const int step_bwd_ctas = g.step ? rec_step_bwd_persist_ctas(g.B, g.Hq, 2) : 0;
    std::vector<char> bwd_persist(g.L, 0);
    std::vector<int> db_groups(g.L, g.step ? 1 : g.pl.G);
    auto side_guard = [&](int l) -> int {
        if (!overlap || no_guard || (g.step && !bwd_persist[l])) return 0;  // (chain: nothing resident to place)
        TRY(wait_count(bstarted + l, (uint32_t)(g.step ? step_bwd_ctas : rec_ctas), side), "wait_count");
        return 0;
    };
    // persistent recurrence: the side GEMMs get the SMs its clusters leave free.  Step-launched
    // recurrence (no resident clusters): a share of the GPU sized so that it and the per-step BPTT
    // GEMM (64 CTAs, rec_step.cu SB) run in one wave (C5 sweep: 64 best of 40..74)
    static const int step_side = getenv("BLSTM_STEP_SIDE_CTAS") ? atoi(getenv("BLSTM_STEP_SIDE_CTAS")) : 64;
    static const bool step_side_env = getenv("BLSTM_STEP_SIDE_CTAS") != nullptr;
    const int step_share = (step_bwd_ctas && !step_side_env) ? num_sms() - step_bwd_ctas : step_side;
    const int side_ctas = !overlap ? 0 : g.step ? step_share : (num_sms() - rec_ctas > 8 ? num_sms() - rec_ctas : 8);
    if (step_bwd_ctas && r16_on_side)  // packed on the side stream during the forward (stack_forward)
        TRY((int)cudaStreamWaitEvent(st, evs[2 * g.L + 7], 0), "cudaStreamWaitEvent");
    else if (step_bwd_ctas)  // R of every layer in pack_w's K-major layout: the persistent BPTT's A operand
        for (int l = 0; l < g.L; ++l)
            TRY(pack_w(theta + offs[6 * l + 1], theta + offs[6 * l + 4], g.H, g.H, Hq, 2, Hq, 0,
                       (__half *)(ws + w.r16[l]), st), "pack_w R16");
    if (overlap && g.K == 0) {  // the side stream may start only after everything issued so far on s_main
        TRY((int)cudaEventRecord(evs[g.L + 1], st), "cudaEventRecord");
        TRY((int)cudaStreamWaitEvent(side, evs[g.L + 1], 0), "cudaStreamWaitEvent");
    }
    if (g.K > 0) {
        __half *wo16 = (__half *)(ws + w.wo16), *dlog = (__half *)(ws + w.dlog16);
        float *boq = (float *)(ws + w.boq), *logits = (float *)(ws + w.Z);
        (void)wo16; (void)boq;  // packed by the preamble launch (stack_forward)
        GemmParams gl{(int)g.TB, g.K, 2 * Hq, logits, g.Kp, 1.f, 0, boq, 0, 0};
        gl.tail_ws = (float *)(ws + w.tsk); gl.tail_elems = gemm_tail_elems();
        TRY(gemm_f16({ytop, 2L * Hq, 0}, {wo16, g.Kp, 1}, gl, 0, st), "gemm logits");
        TRY(ce_head(logits, g.Kp, g.K, g.Kp, mask, labels, (float)(1 << DA_SHIFT), dlog, (double *)(ws + w.rowloss),
                    (int32_t *)(ws + w.rowerr), g.TB, st), "ce_head");
        // the loss and frame-error sums are read only after the call: side stream
        if (overlap) {
            TRY((int)cudaEventRecord(evs[2 * g.L + 6], st), "cudaEventRecord");
            TRY((int)cudaStreamWaitEvent(side, evs[2 * g.L + 6], 0), "cudaStreamWaitEvent");
        }
        TRY(reduce_loss((double *)(ws + w.rowloss), (int32_t *)(ws + w.rowerr), g.TB, loss_sum, frame_errors,
                        overlap ? side : st), "reduce_loss");
        GemmParams gd{(int)g.TB, 2 * Hq, g.Kp, dY[0], 2L * Hq, a, 0, nullptr, 0, 0};
        gd.tail_ws = (float *)(ws + w.tsk); gd.tail_elems = gemm_tail_elems();
        TRY(gemm_f16({dlog, g.Kp, 0}, {wo16, g.Kp, 0}, gd, 0, st), "gemm dY_top");
        if (g.dr.on) TRY(dropout_f32(dY[0], g.TB, g.H, Hq, g.L, g.dr, st), "dropout dY_top");
        // the head's parameter gradients are off the critical path too: side stream (side_head)
        if (overlap) TRY((int)cudaEventRecord(evs[g.L + 1], st), "cudaEventRecord");
    } else {
        TRY(pad_halves(dy_top, g.H, Hq, g.TB, dY[0], st), "pad dy_top");
        if (cudaMemsetAsync(loss_sum, 0, sizeof(double), st) != cudaSuccess) return fail(BLSTM_ERR_CUDA, "memset");
        if (frame_errors && cudaMemsetAsync(frame_errors, 0, sizeof(int32_t), st) != cudaSuccess)
            return fail(BLSTM_ERR_CUDA, "memset");
    }

    // Side-stream work is enqueued (host order) after the BPTT launch it overlaps: both become ready
    // when the same main-stream kernel completes, and side GEMM CTAs dispatched first would spread
    // over the GPCs and keep the recurrence clusters out until they finish.
    auto side_head = [&]() -> int {  // dW_out, db_out of the head
        if (g.K == 0) return 0;
        __half *dlog = (__half *)(ws + w.dlog16);
        float *dWoT = (float *)(ws + w.dWoT);
        if (overlap) TRY((int)cudaStreamWaitEvent(side, evs[g.L + 1], 0), "cudaStreamWaitEvent");
        if (int rc = side_guard(g.L - 1)) return rc;
        // dW_out [2H, K] += (dlogits^T Y)^T, scattered from the padded halves of Y by the GEMM
        GemmParams gw{g.K, 2 * Hq, (int)g.TB, dWoT, 2L * Hq, a, 0, nullptr, 0, 0};
        gw.splitk_ws = (float *)(ws + w.gsk); gw.splitk_elems = GSK_ELEMS;
        gw.scat.dst = grad + offs[6 * g.L]; gw.scat.rowmode = 0; gw.scat.nrows = g.K;
        gw.scat.colmode = 1; gw.scat.H = g.H; gw.scat.Hq = Hq; gw.scat.ld = g.K;
        TRY(gemm_f16({dlog, g.Kp, 1}, {ytop, 2L * Hq, 1}, gw, side_ctas, side), "gemm dW_out");
        if (overlap) TRY((int)cudaEventRecord(evs[GSK_FREE], side), "cudaEventRecord");
        TRY(colsum_f16_add(dlog, g.TB, g.K, g.Kp, a, grad + offs[6 * g.L + 1], (float *)(ws + w.cs), side), "db_out");
        if (comm) {  // sync-mode exchange of this bucket (the head), overlapping the BPTT below
            if (int rc = dp_allreduce_grads_impl(comm, grad + blo[0], bhi[0] - blo[0], side)) return rc;
        }
        if (bucket_update)  // the head's parameters are final: update them now (NEXT-3, fused)
            if (int rc = opt_range(opt, d, (float *)theta, grad, opt_state, nparam, blo[0], bhi[0], 1, nullptr, side))
                return rc;
        return 0;
    };
    // ss: the side stream, or (layer 0, which follows the last BPTT) s_main, which is idle then
    auto side_layer = [&](int l, cudaStream_t ss) -> int {  // dW, dR, db of layer l (its parity's dA / dbpart)
        const int par = l & 1;
        const __half *dA = (__half *)(ws + w.dA) + (size_t)par * g.TB * 8 * Hq;
        float *dWT = (float *)(ws + w.dWT) + (size_t)par * 8 * Hq * w.maxDn;
        float *dRT = (float *)(ws + w.dRT) + (size_t)par * 2 * 4 * Hq * Hq;
        const float *dbp = (float *)(ws + w.dbp) + (size_t)par * 2 * g.dbs * 4 * Hq;
        // layer 0 on s_main (after the last BPTT): fork -- dW and then direction 1's dR stay on s_main,
        // direction 0's dR and the rest go to the side stream once it finished layer 1's work, each
        // stream with its own half of the split-K scratch; the three small GEMMs then run side by side
        // instead of one after another
        const bool fork = l == 0 && overlap && ss != side && !comm;
        cudaStream_t sw = ss, sr = fork ? side : ss;
        float *gsk_w = (float *)(ws + w.gsk), *gsk_r = fork ? gsk_w + GSK_ELEMS / 2 : gsk_w;
        const long gsk_n = fork ? GSK_ELEMS / 2 : GSK_ELEMS;
        if (overlap && sr == side) TRY((int)cudaStreamWaitEvent(side, evs[l], 0), "cudaStreamWaitEvent");
        if (l > 0)  // overlaps BPTT(l-1)
            if (int rc = side_guard(l - 1)) return rc;
        // on s_main: the split-K scratch is shared with the side stream's GEMMs (the last layer's)
        if (overlap && sw != side) TRY((int)cudaStreamWaitEvent(sw, evs[GSK_FREE], 0), "cudaStreamWaitEvent");
        const __half *X = l == 0 ? (const __half *)(ws + w.x16) : (const __half *)(ws + w.y16[l - 1]);
        // the last layer's weight gradients run after all BPTT work: every SM is free then
        const int wctas = l == 0 ? 0 : side_ctas;
        // dW_d [Drows, 4H] of both directions += (dA^T X)^T, scattered into grad by the GEMM
        GemmParams gw{8 * Hq, g.Dn[l], (int)g.TB, dWT, g.Dn[l], a, 0, nullptr, 0, 0};
        gw.splitk_ws = gsk_w; gw.splitk_elems = gsk_n;
        gw.scat = scatter_gate_rows(grad + offs[6 * l], g.H, Hq, (long)(offs[6 * l + 3] - offs[6 * l]), g.rowmode[l],
                                    g.Drows[l], 4L * g.H);
        TRY(gemm_f16({dA, 8L * Hq, 1}, {X, (long)g.Dn[l], 1}, gw, wctas, sw), "gemm dW");
        const __half *hist = (const __half *)(ws + w.hist[l]);
        for (int dd = 0; dd < 2; ++dd) {
            // forked tail: direction 1's dR follows dW on s_main (its half of the scratch), beside
            // direction 0's on the side stream
            const bool on_w = fork && dd == 1;
            const __half *hprev = hist + ((long)dd * (g.T + 1) + dd) * g.B * Hq;
            GemmParams gr{4 * Hq, Hq, (int)g.TB, dRT + (size_t)dd * 4 * Hq * Hq, Hq, a, 0, nullptr, 0, 0};
            gr.splitk_ws = on_w ? gsk_w : gsk_r; gr.splitk_elems = gsk_n;
            gr.scat = scatter_gate_rows(grad + offs[6 * l + 3 * dd + 1], g.H, Hq, 0, 0, g.H, 4L * g.H);
            TRY(gemm_f16({dA + (size_t)dd * 4 * Hq, 8L * Hq, 1}, {hprev, Hq, 1}, gr, wctas, on_w ? sw : sr), "gemm dR");
        }
        if (fork) TRY((int)cudaEventRecord(evs[2 * g.L + 3], sw), "cudaEventRecord");
        if (overlap && ss == side) TRY((int)cudaEventRecord(evs[GSK_FREE], side), "cudaEventRecord");
        for (int dd = 0; dd < 2; ++dd)
            TRY(scatter_b(grad + offs[6 * l + 3 * dd + 2], g.H, Hq, dbp, db_groups[l], dd, sr), "scatter db");
        if (fork) {  // the rest of layer 0's work (update, completion event) follows on the side stream
            TRY((int)cudaStreamWaitEvent(sr, evs[2 * g.L + 3], 0), "cudaStreamWaitEvent");
            ss = sr;
        }
        const size_t b0 = blo[bhead + g.L - 1 - l], b1 = bhi[bhead + g.L - 1 - l];  // layer l's bucket
        if (comm) {  // sync-mode exchange of layer l's bucket (§4.1), overlapping BPTT
            if (int rc = dp_allreduce_grads_impl(comm, grad + b0, b1 - b0, ss)) return rc;
        }
        if (bucket_update)  // layer l's parameters are final: update them while BPTT continues below
            if (int rc = opt_range(opt, d, (float *)theta, grad, opt_state, nparam, b0, b1, 1, nullptr, ss))
                return rc;
        if (overlap) TRY((int)cudaEventRecord(evs[g.L + 2 + l], ss), "cudaEventRecord");
        return 0;
    };
    int cur = 0;
    for (int l = g.L - 1; l >= 0; --l) {
        const int par = l & 1;
        __half *dA = (__half *)(ws + w.dA) + (size_t)par * g.TB * 8 * Hq;
        float *dbp = (float *)(ws + w.dbp) + (size_t)par * 2 * g.dbs * 4 * Hq;
        // layer l+2 used the same parity buffers: its side-stream GEMMs must be done reading them
        if (overlap && l + 2 < g.L) TRY((int)cudaStreamWaitEvent(st, evs[g.L + 2 + l + 2], 0), "cudaStreamWaitEvent");
        RecParams p = base_params(LayerGeo{g.T, g.B, g.D, g.H, Hq, 0, g.TB, g.pl}, 2, 1, mask);
        p.maskN = (const uint8_t *)(ws + w.maskN);  // packed by stack_forward
        p.C = (float *)(ws + w.C[l]); p.ldc = Hq; p.c_doff = g.TB * Hq;
        p.gates = (__half *)(ws + w.gates[l]); p.ldg = 8L * Hq;
        p.dy = dY[cur]; p.lddy = 2L * Hq; p.dy_doff = Hq;
        p.dA = dA; p.ldda = 8L * Hq;
        p.dbpart = dbp;
        p.P = (float *)(ws + w.P);
        p.counters = (uint32_t *)(ws + w.cnt);
        p.started = overlap ? bstarted + l : nullptr;
        if (g.step) {  // one launch group per time step (rec_step.h); db = column sums of dA
            RecStepBwd q{};
            q.T = g.T; q.B = g.B; q.H = g.H; q.Hq = Hq; q.ndir = 2; q.dir0 = 1;
            q.mask = mask; q.RT16 = (const __half *)(ws + w.rt16[l]);
            q.C = p.C; q.ldc = p.ldc; q.c_doff = p.c_doff;
            q.gates = p.gates;
            q.dy = p.dy; q.lddy = p.lddy; q.dy_doff = p.dy_doff;
            q.dA = dA;
            float *sb = (float *)(ws + w.stepB);
            q.dhR = sb;
            q.dhc = sb + rec_step_bwd_partial_floats(g.B, Hq);
            q.dcc = q.dhc + 2L * g.B * Hq;
            q.splitk_ws = (float *)(ws + w.gsk); q.splitk_elems = GSK_ELEMS;
            q.R16 = (const __half *)(ws + w.r16[l]);
            q.dbpart = dbp;  // the persistent BPTT's db partials ([2][8][4Hq], dbs >= 8)
            q.started = p.started;
            const int rc = rec_step_bwd(q, st);
            if (rc < 0) TRY(rc, "rec_step_bwd");
            bwd_persist[l] = rc == 1;
            db_groups[l] = rc == 1 ? rec_step_bwd_db_groups() : 1;
            if (rc == 0) {  // the step chain: db = column sums of dA ([2][1][4Hq])
                if (cudaMemsetAsync(dbp, 0, (size_t)8 * Hq * 4, st) != cudaSuccess) return fail(BLSTM_ERR_CUDA, "memset");
                TRY(colsum_f16_add(dA, g.TB, 8 * Hq, 8L * Hq, 1.f / (float)(1 << DA_SHIFT), dbp, (float *)(ws + w.cs2), st),
                    "db colsum");
            }
        } else {
            TRY(lstm_rec_bwd(p, (const __half *)(ws + w.rt16[l]), st), "lstm_rec_bwd");
        }
        // the gradient work this BPTT overlaps, enqueued after it
        if (int rc = (l == g.L - 1) ? side_head() : side_layer(l + 1, side)) return rc;
        const __half *w16 = (const __half *)(ws + w.w16[l]);
        if (l > 0) {  // critical path: gradient of the layer below's output
            GemmParams gx{(int)g.TB, g.Dn[l], 8 * Hq, dY[1 - cur], 2L * Hq, a, 0, nullptr, 0, 0};
            gx.tail_ws = (float *)(ws + w.tsk); gx.tail_elems = gemm_tail_elems();
            TRY(gemm_f16({dA, 8L * Hq, 0}, {w16, 8L * Hq, 0}, gx, 0, st), "gemm dX");
            // gradient of the undropped output of layer l-1 (site l)
            if (g.dr.on) TRY(dropout_f32(dY[1 - cur], g.TB, g.H, Hq, l, g.dr, st), "dropout dX");
        }
        if (overlap) TRY((int)cudaEventRecord(evs[l], st), "cudaEventRecord");
        cur = 1 - cur;
    }
    // layer 0's gradient work follows the last BPTT: on s_main it starts while the side stream
    // finishes layer 1's scatters and update (with NCCL, on the side stream: one stream issues the
    // collectives, in bucket order)
    if (int rc = side_layer(0, (overlap && !comm) ? st : side)) return rc;
    if (overlap) {  // s_main's view: all gradient work of this call is complete
        TRY((int)cudaEventRecord(evs[g.L], side), "cudaEventRecord");
        TRY((int)cudaStreamWaitEvent(st, evs[g.L], 0), "cudaStreamWaitEvent");
    }
    if (opt && !bucket_update)  // the global norm constraint needs every gradient: one update at the end
        if (int rc = opt_range(opt, d, (float *)theta, grad, opt_state, nparam, 0, nparam, 1, (double *)(ws + w.optp), st))
            return rc;
    return 0;
}

extern "C" int blstm_stack_fwd_bwd(const blstm_stack_desc *d, const float *theta, float *grad, const float *x,
                                   const uint8_t *mask, const int32_t *labels, const float *dy_top, double *loss_sum,
                                   int32_t *frame_errors, dp_comm *comm, void *workspace, size_t workspace_bytes,
                                   void *s_main, void *s_side) {
    return stack_step_impl(d, theta, grad, x, mask, labels, dy_top, loss_sum, frame_errors, comm, nullptr, nullptr,
                           workspace, workspace_bytes, s_main, s_side);
}

extern "C" int blstm_stack_train_step(const blstm_stack_desc *d, float *theta, float *grad, const float *x,
                                      const uint8_t *mask, const int32_t *labels, const float *dy_top, double *loss_sum,
                                      int32_t *frame_errors, dp_comm *comm, const blstm_opt_params *opt,
                                      float *opt_state, void *workspace, size_t workspace_bytes, void *s_main,
                                      void *s_side) {
    const size_t n = blstm_param_count(d);
    if (n == 0) return fail(BLSTM_ERR_ARG, "blstm_stack_train_step: bad descriptor");
    if (int rc = opt_check(opt, theta, grad, opt_state, n)) return rc;
    if (d->L > 31) return fail(BLSTM_ERR_UNSUPPORTED, "update with L=%d > 31", d->L);
    return stack_step_impl(d, theta, grad, x, mask, labels, dy_top, loss_sum, frame_errors, comm, opt, opt_state,
                           workspace, workspace_bytes, s_main, s_side);
}

extern "C" int sgd_update(float *theta, float *grad, size_t n, float lr, int zero_grad, void *stream) {
    if (!theta || !grad) return fail(BLSTM_ERR_ARG, "null theta / grad");
    if (!al16(theta) || !al16(grad)) return fail(BLSTM_ERR_ALIGN, "theta/grad must be 16-byte aligned");
    TRY(sgd(theta, grad, (long)n, lr, zero_grad, (cudaStream_t)stream), "sgd");
    return 0;
}

// ---------------------------------------------------------------------------
// update rules (§4.3; optim.cu)
// ---------------------------------------------------------------------------
static inline size_t rup4(size_t n) { return (n + 3) & ~(size_t)3; }
extern "C" size_t blstm_opt_state_floats(int rule, size_t n) {
    switch (rule) {
    case BLSTM_OPT_SGD: return 0;
    case BLSTM_OPT_MOMENTUM: case BLSTM_OPT_NESTEROV: case BLSTM_OPT_ADAGRAD: return rup4(n);
    case BLSTM_OPT_ADADELTA: case BLSTM_OPT_ADAM: return 2 * rup4(n);
    default: return 0;
    }
}
extern "C" size_t blstm_opt_workspace_bytes(size_t) { return sizeof(double) * (size_t)opt_norm_partials(); }

// One update over [lo, hi) of an n-entry vector (state slot s0 at state + i, s1 at state + n4 + i);
// the layout's bias ranges are rebased to lo (a boundary before lo still counts: the pairing of
// [start, end) boundaries is what marks an index as a bias entry).  lo must be a multiple of 4.
static int opt_range(const blstm_opt_params *p, const blstm_stack_desc *layout, float *theta, float *grad,
                     float *state, size_t n, size_t lo, size_t hi, int zero_grad, double *partial, cudaStream_t st) {
    OptBiasTable tab;
    tab.nb = 0;
    for (int k = 0; k < OPT_MAX_BOUNDS; ++k) tab.bnd[k] = 0x7fffffffffffffffL;
    if (layout) {
        std::vector<size_t> offs(6 * layout->L + 2);
        param_layout(layout, offs.data());
        const long h4 = 4L * layout->H;
        for (int l = 0; l < layout->L; ++l)
            for (int dd = 0; dd < 2; ++dd) {
                const long b0 = (long)offs[6 * l + 3 * dd + 2] - (long)lo;
                tab.bnd[tab.nb++] = b0;
                tab.bnd[tab.nb++] = b0 + h4;
            }
        if (layout->K > 0) {
            tab.bnd[tab.nb++] = (long)offs[6 * layout->L + 1] - (long)lo;
            tab.bnd[tab.nb++] = (long)offs[6 * layout->L + 1] + layout->K - (long)lo;
        }
    }
    const size_t ns = blstm_opt_state_floats(p->rule, n), n4 = rup4(n);
    float *s0 = ns ? state + lo : nullptr;
    float *s1 = ns > n4 ? state + n4 + lo : nullptr;
    OptArgs a{(float)p->lr, (float)p->mu, (float)p->rho, (float)p->beta1, (float)p->beta2, (float)p->eps,
              (float)p->l2, (float)p->max_norm, (float)(1.0 - p->rho), (float)(1.0 - p->beta1),
              (float)(1.0 - p->beta2), 1.f, 1.f};
    if (p->rule == BLSTM_OPT_ADAM) {
        a.c1 = (float)(1.0 / (1.0 - pow(p->beta1, (double)p->step)));
        a.c2 = (float)(1.0 / (1.0 - pow(p->beta2, (double)p->step)));
    }
    if (hi <= lo) return 0;
    TRY(opt_update(p->rule, theta + lo, grad + lo, s0, s1, (long)(hi - lo), a, p->max_norm, tab, partial, zero_grad, st),
        "opt_update");
    return 0;
}

static int opt_check(const blstm_opt_params *p, float *theta, float *grad, float *state, size_t n) {
    if (!p || !theta || !grad) return fail(BLSTM_ERR_ARG, "update: null params / theta / grad");
    if (p->rule < BLSTM_OPT_SGD || p->rule > BLSTM_OPT_ADAM) return fail(BLSTM_ERR_ARG, "unknown rule %d", p->rule);
    if (p->rule == BLSTM_OPT_ADAM && p->step < 1) return fail(BLSTM_ERR_ARG, "ADAM needs step >= 1");
    const size_t ns = blstm_opt_state_floats(p->rule, n);
    if (ns && !state) return fail(BLSTM_ERR_ARG, "rule %d needs %zu floats of state", p->rule, ns);
    if (!al16(theta) || !al16(grad) || (ns && !al16(state)))
        return fail(BLSTM_ERR_ALIGN, "theta / grad / state must be 16-byte aligned");
    return 0;
}

extern "C" int blstm_opt_update(const blstm_opt_params *p, const blstm_stack_desc *layout, float *theta, float *grad,
                                float *state, size_t n, int zero_grad, void *workspace, size_t workspace_bytes,
                                void *stream) {
    if (int rc = opt_check(p, theta, grad, state, n)) return rc;
    if (p->max_norm > 0.0) {
        if (!workspace || !al16(workspace)) return fail(BLSTM_ERR_ALIGN, "norm constraint needs an aligned workspace");
        if (workspace_bytes < blstm_opt_workspace_bytes(n))
            return fail(BLSTM_ERR_WORKSPACE, "workspace %zu < %zu bytes", workspace_bytes, blstm_opt_workspace_bytes(n));
    }
    if (layout) {
        if (layout->L > 31) return fail(BLSTM_ERR_UNSUPPORTED, "layout with L=%d > 31", layout->L);
        const size_t np = blstm_param_count(layout);
        if (np == 0 || np != n) return fail(BLSTM_ERR_ARG, "n=%zu != blstm_param_count(layout)=%zu", n, np);
    }
    return opt_range(p, layout, theta, grad, state, n, 0, n, zero_grad, (double *)workspace, (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------
// MDLSTM (NEXT-2; mdlstm.cu)
// ---------------------------------------------------------------------------
static int md_check(const mdlstm_desc *d, MdGeo &g) {
    if (!d) return fail(BLSTM_ERR_ARG, "null mdlstm_desc");
    if (d->U < 1 || d->V < 1 || d->B < 1 || d->D < 1 || d->H < 1)
        return fail(BLSTM_ERR_SHAPE, "need U, V, B, D, H >= 1");
    if (d->H > 256) return fail(BLSTM_ERR_UNSUPPORTED, "mdlstm: H=%d > 256", d->H);
    g = md_geo(d->U, d->V, d->B, d->D, d->H, d->stable ? 1 : 0);
    if (g.cells * 20L * g.Hp > 0x7fffffffL) return fail(BLSTM_ERR_UNSUPPORTED, "mdlstm: grid too large");
    return 0;
}
extern "C" size_t mdlstm_param_count(const mdlstm_desc *d) {
    MdGeo g;
    return md_check(d, g) ? 0 : md_param_count(g);
}
extern "C" size_t mdlstm_workspace_bytes(const mdlstm_desc *d) {
    MdGeo g;
    return md_check(d, g) ? 0 : md_ws(g).total;
}
extern "C" size_t mdlstm_reserve_bytes(const mdlstm_desc *d) {
    MdGeo g;
    return md_check(d, g) ? 0 : md_ws(g).rtotal;
}
extern "C" int mdlstm_fwd(const mdlstm_desc *d, const float *theta, const float *x, const uint8_t *mask, float *y,
                          void *reserve, void *workspace, size_t workspace_bytes, void *stream) {
    MdGeo g;
    if (int rc = md_check(d, g)) return rc;
    if (!theta || !x || !mask || !y || !reserve || !workspace) return fail(BLSTM_ERR_ARG, "mdlstm_fwd: null pointer");
    if (!al16(reserve) || !al16(workspace) || !al4(theta) || !al4(x) || !al4(y))
        return fail(BLSTM_ERR_ALIGN, "mdlstm_fwd: misaligned buffer");
    if (workspace_bytes < md_ws(g).total) return fail(BLSTM_ERR_WORKSPACE, "workspace %zu < %zu", workspace_bytes, md_ws(g).total);
    TRY(md_forward(g, theta, x, mask, y, (uint8_t *)workspace, (uint8_t *)reserve, (cudaStream_t)stream), "mdlstm fwd");
    return 0;
}
extern "C" int mdlstm_bwd(const mdlstm_desc *d, const float *theta, const float *x, const uint8_t *mask,
                          const void *reserve, const float *dy, float *dx, float *grad, void *workspace,
                          size_t workspace_bytes, void *stream) {
    MdGeo g;
    if (int rc = md_check(d, g)) return rc;
    if (!theta || !x || !mask || !reserve || !dy || !grad || !workspace)
        return fail(BLSTM_ERR_ARG, "mdlstm_bwd: null pointer");
    if (!al16(reserve) || !al16(workspace)) return fail(BLSTM_ERR_ALIGN, "mdlstm_bwd: misaligned buffer");
    if (workspace_bytes < md_ws(g).total) return fail(BLSTM_ERR_WORKSPACE, "workspace %zu < %zu", workspace_bytes, md_ws(g).total);
    TRY(md_backward(g, theta, x, mask, dy, dx, grad, (uint8_t *)workspace, (uint8_t *)reserve, (cudaStream_t)stream),
        "mdlstm bwd");
    return 0;
}

extern "C" int blstm_gather_chunks(const float *frames, const int32_t *frame_labels, int D, const int64_t *cstart,
                                   const int32_t *clen, int B, int T, float *x, uint8_t *mask, int32_t *labels,
                                   void *stream) {
    if (!frames || !cstart || !clen || !x || !mask || D < 1 || B < 1 || T < 0)
        return fail(BLSTM_ERR_ARG, "blstm_gather_chunks: bad argument");
    if ((long)T * B * D == 0) return 0;
    TRY(gather_chunks(frames, frame_labels, D, cstart, clen, B, T, x, mask, labels, (cudaStream_t)stream),
        "gather_chunks");
    return 0;
}

extern "C" int blstm_reduce_replicas(float *const *ptrs, int n, size_t len, float scale, void *stream) {
    if (!ptrs || n < 1 || n > MAX_REPLICAS) return fail(BLSTM_ERR_ARG, "need 1 <= n <= %d replicas", MAX_REPLICAS);
    ReplicaPtrs rp{};
    for (int r = 0; r < n; ++r) {
        if (!ptrs[r]) return fail(BLSTM_ERR_ARG, "null replica pointer %d", r);
        if (!al16(ptrs[r])) return fail(BLSTM_ERR_ALIGN, "replica %d not 16-byte aligned", r);
        for (int q = 0; q < r; ++q)
            if (ptrs[q] == ptrs[r]) return fail(BLSTM_ERR_ARG, "replicas %d and %d alias", q, r);
        rp.p[r] = ptrs[r];
    }
    if (len == 0) return 0;
    TRY(reduce_replicas(rp, n, (long)len, scale, (cudaStream_t)stream), "reduce_replicas");
    return 0;
}

extern "C" int blstm_gemm_f16(int M, int N, int K, const void *A, long lda, int a_mn, const void *B, long ldb,
                              int b_mn, float *C, long ldc, float alpha, int beta, const float *bias, void *stream) {
    if (!A || !B || !C || M < 0 || N < 0 || K < 1) return fail(BLSTM_ERR_ARG, "blstm_gemm_f16: bad argument");
    if (!al16(A) || !al16(B) || (lda & 7) || (ldb & 7)) return fail(BLSTM_ERR_ALIGN, "A/B must be 16-byte aligned, ld % 8 == 0");
    GemmParams gp{M, N, K, C, ldc, alpha, beta, bias, 0, 0};
    // the same split-K and tail-wave scratch the stack gives its GEMMs (library-owned, per device,
    // allocated on first use), so the hook times and tests the kernels the stack runs
    static std::mutex mu;
    static std::map<int, std::pair<float *, float *>> scratch;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail(BLSTM_ERR_CUDA, "cudaGetDevice");
    std::pair<float *, float *> sc{nullptr, nullptr};
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = scratch.find(dev);
        if (it == scratch.end()) {
            float *a = nullptr, *b = nullptr;
            if (cudaMalloc(&a, (size_t)GSK_ELEMS * 4) != cudaSuccess ||
                cudaMalloc(&b, (size_t)gemm_tail_elems() * 4) != cudaSuccess) {
                cudaGetLastError();
                return fail(BLSTM_ERR_CUDA, "blstm_gemm_f16: scratch allocation");
            }
            it = scratch.emplace(dev, std::make_pair(a, b)).first;
        }
        sc = it->second;
    }
    gp.splitk_ws = sc.first; gp.splitk_elems = GSK_ELEMS;
    gp.tail_ws = sc.second; gp.tail_elems = gemm_tail_elems();
    TRY(gemm_f16({A, lda, a_mn}, {B, ldb, b_mn}, gp, 0, (cudaStream_t)stream), "gemm");
    return 0;
}

// debug hook: per-step phase timestamps of the next recurrence launches (8 u64 per step,
// CTA 0 thread 0), nullptr to disable
extern "C" int blstm_debug_set_trace(void *fwd, void *bwd) {
    rec_set_trace((unsigned long long *)fwd, (unsigned long long *)bwd);
    return 0;
}
