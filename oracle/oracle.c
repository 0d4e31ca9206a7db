/*
 * oracle.c -- plain fp64 CPU oracle for the BLSTM training step.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant with the CUDA path
 * (paper_1608_00895_b200/csrc), and the CUDA path never calls it.
 *
 * What it computes:
 *   - the LSTM layer of PAPER.md §4.2: "The non-recurrent part of
 *     the LSTM forward computations are performed in a single matrix
 *     multiplication for the whole mini-batch"; the recurrence with the gating
 *     mechanism; back propagation through time, then the gradients "with
 *     respect to the weights and the inputs".  Here everything is written as the
 *     plain sequential definition (no blocking, no fusion): the pre-activation
 *     of every frame is bias + x.W + h.R summed in ascending index order.
 *   - LSTM variant (paper silent; reading R1 = SPEC S:171/S:193/S:241):
 *     no peepholes, gate blocks [i | f | g | o] of W[D,4H], R[H,4H], b[4H].
 *   - index tensor / mask (§5; reading R2): at a masked
 *     frame the state (h, c) is carried unchanged and the output is 0; the
 *     backward pass gives dA = 0 there and lets dh, dc pass through (R4).
 *   - bidirectional stacking (reading A2/A3): Y_l = [fwd | bwd].
 *   - softmax cross-entropy head, summed over valid frames, no
 *     scaling of the gradient (§4.3, reading R7).
 *   - SGD theta' = theta - lr*g (§4.3), the other update rules of §4.3 (momentum,
 *     simplified Nesterov, Adagrad, Adadelta, Adam, L2 penalty, norm constraint:
 *     ref_opt_update) and parameter averaging theta = (1/N) sum_r theta_r
 *     (§4.1).
 *
 * Reductions run in ascending index order.  OpenMP (when compiled with
 * -fopenmp) only splits independent batch rows / output elements, so the
 * result is bitwise independent of the thread count.
 *
 * Pins: tests/test_oracle_pins.py (closed forms, worked examples W1/W2,
 * torch.nn.LSTM float64 on packed sequences, central finite differences,
 * direction duality, mask extension, sum semantics, DP algebra).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static double sigm(double z)
{
    /* numerically stable logistic */
    if (z >= 0.0) return 1.0 / (1.0 + exp(-z));
    double e = exp(z);
    return e / (1.0 + e);
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/*
 * One LSTM layer, one direction, forward.
 *   x [T,B,D], mask [T,B], W [D,4H], R [H,4H], bias [4H], h0/c0 [B,H] or NULL.
 * Outputs: y [T,B,H] (0 at masked frames), C [T,B,H] (cell state after frame t,
 * carried at masked frames), hT/cT [B,H] (state after the whole scan, may be NULL),
 * and the saved state the backward pass needs:
 *   G [T,B,4H] gate activations (i,f,g,o), Hprev/Cprev [T,B,H] the state before frame t.
 */
int ref_lstm_fwd(int T, int B, int D, int H, int dir,
                 const double *x, const uint8_t *mask,
                 const double *W, const double *R, const double *bias,
                 const double *h0, const double *c0,
                 double *y, double *C, double *hT, double *cT,
                 double *G, double *Hprev, double *Cprev)
{
    if (T < 0 || B < 1 || D < 0 || H < 1 || (dir != 1 && dir != -1)) return -1;
    const int G4 = 4 * H;
    double *h = (double *)calloc((size_t)B * H, sizeof(double));
    double *c = (double *)calloc((size_t)B * H, sizeof(double));
    if (!h || !c) { free(h); free(c); return -2; }
    if (h0) memcpy(h, h0, sizeof(double) * B * H);
    if (c0) memcpy(c, c0, sizeof(double) * B * H);

    for (int s = 0; s < T; ++s) {
        const int t = dir > 0 ? s : T - 1 - s;
#pragma omp parallel for schedule(static)
        for (int b = 0; b < B; ++b) {
            const size_t fr = (size_t)t * B + b;
            double *hb = h + (size_t)b * H, *cb = c + (size_t)b * H;
            memcpy(Hprev + fr * H, hb, sizeof(double) * H);
            memcpy(Cprev + fr * H, cb, sizeof(double) * H);
            if (!mask[fr]) {
                for (int j = 0; j < H; ++j) { y[fr * H + j] = 0.0; C[fr * H + j] = cb[j]; }
                for (int n = 0; n < G4; ++n) G[fr * G4 + n] = 0.0;
                continue;
            }
            /* a[n] = bias[n] + sum_d x[d] W[d][n] + sum_k h[k] R[k][n], each a[n] summed in
             * ascending d then k (rows of W and R traversed contiguously) */
            double *a = (double *)malloc(sizeof(double) * G4);
            for (int n = 0; n < G4; ++n) a[n] = bias[n];
            for (int d = 0; d < D; ++d) {
                const double xd = x[fr * D + d];
                const double *Wd = W + (size_t)d * G4;
                for (int n = 0; n < G4; ++n) a[n] += xd * Wd[n];
            }
            for (int k = 0; k < H; ++k) {
                const double hk = hb[k];
                const double *Rk = R + (size_t)k * G4;
                for (int n = 0; n < G4; ++n) a[n] += hk * Rk[n];
            }
            for (int j = 0; j < H; ++j) {
                const double i = sigm(a[j]);
                const double f = sigm(a[H + j]);
                const double g = tanh(a[2 * H + j]);
                const double o = sigm(a[3 * H + j]);
                const double cn = f * cb[j] + i * g;
                const double hn = o * tanh(cn);
                G[fr * G4 + j] = i;
                G[fr * G4 + H + j] = f;
                G[fr * G4 + 2 * H + j] = g;
                G[fr * G4 + 3 * H + j] = o;
                cb[j] = cn;
                hb[j] = hn;
                y[fr * H + j] = hn;
                C[fr * H + j] = cn;
            }
            free(a);
        }
    }
    if (hT) memcpy(hT, h, sizeof(double) * B * H);
    if (cT) memcpy(cT, c, sizeof(double) * B * H);
    free(h);
    free(c);
    return 0;
}

/*
 * Backward through time (the
 * recurrent part first, then the weight and input gradients).
 *   dy [T,B,H] (ignored at masked frames), dhT/dcT [B,H] or NULL.
 * Outputs: dx [T,B,D] overwritten (may be NULL), dW/dR/db accumulated (+=),
 * dh0/dc0 [B,H] (may be NULL).  dA [T,B,4H] is scratch supplied by the caller
 * (returned so tests can inspect it).
 */
int ref_lstm_bwd(int T, int B, int D, int H, int dir,
                 const double *x, const uint8_t *mask,
                 const double *W, const double *R,
                 const double *C, const double *G, const double *Hprev, const double *Cprev,
                 const double *dy, const double *dhT, const double *dcT,
                 double *dx, double *dW, double *dR, double *db,
                 double *dh0, double *dc0, double *dA)
{
    if (T < 0 || B < 1 || D < 0 || H < 1 || (dir != 1 && dir != -1)) return -1;
    const int G4 = 4 * H;
    double *dh = (double *)calloc((size_t)B * H, sizeof(double));
    double *dc = (double *)calloc((size_t)B * H, sizeof(double));
    if (!dh || !dc) { free(dh); free(dc); return -2; }
    if (dhT) memcpy(dh, dhT, sizeof(double) * B * H);
    if (dcT) memcpy(dc, dcT, sizeof(double) * B * H);

    for (int s = T - 1; s >= 0; --s) {
        const int t = dir > 0 ? s : T - 1 - s;
#pragma omp parallel for schedule(static)
        for (int b = 0; b < B; ++b) {
            const size_t fr = (size_t)t * B + b;
            double *dab = dA + fr * G4;
            if (!mask[fr]) {
                for (int n = 0; n < G4; ++n) dab[n] = 0.0;
                continue; /* dh, dc pass through unchanged */
            }
            double *dhb = dh + (size_t)b * H, *dcb = dc + (size_t)b * H;
            for (int j = 0; j < H; ++j) {
                const double i = G[fr * G4 + j];
                const double f = G[fr * G4 + H + j];
                const double g = G[fr * G4 + 2 * H + j];
                const double o = G[fr * G4 + 3 * H + j];
                const double th = tanh(C[fr * H + j]);
                const double dH = dhb[j] + dy[fr * H + j];
                const double dC = dcb[j] + dH * o * (1.0 - th * th);
                dab[j] = dC * g * i * (1.0 - i);
                dab[H + j] = dC * Cprev[fr * H + j] * f * (1.0 - f);
                dab[2 * H + j] = dC * i * (1.0 - g * g);
                dab[3 * H + j] = dH * th * o * (1.0 - o);
                dcb[j] = dC * f;
            }
            for (int k = 0; k < H; ++k) {
                double acc = 0.0;
                for (int n = 0; n < G4; ++n) acc += dab[n] * R[(size_t)k * G4 + n];
                dhb[k] = acc;
            }
        }
    }
    const size_t TB = (size_t)T * B;
    /* dW[d][n] += sum_{t,b} x[t,b,d] dA[t,b,n]  (each element summed over rows r = t*B+b in
     * ascending order into a zeroed accumulator, then added) */
#pragma omp parallel for schedule(static)
    for (int d = 0; d < D; ++d) {
        double *acc = (double *)calloc(G4, sizeof(double));
        for (size_t r = 0; r < TB; ++r) {
            const double xd = x[r * D + d];
            const double *dar = dA + r * G4;
            for (int n = 0; n < G4; ++n) acc[n] += xd * dar[n];
        }
        for (int n = 0; n < G4; ++n) dW[(size_t)d * G4 + n] += acc[n];
        free(acc);
    }
    /* dR[k][n] += sum_{t,b} Hprev[t,b,k] dA[t,b,n] */
#pragma omp parallel for schedule(static)
    for (int k = 0; k < H; ++k) {
        double *acc = (double *)calloc(G4, sizeof(double));
        for (size_t r = 0; r < TB; ++r) {
            const double hk = Hprev[r * H + k];
            const double *dar = dA + r * G4;
            for (int n = 0; n < G4; ++n) acc[n] += hk * dar[n];
        }
        for (int n = 0; n < G4; ++n) dR[(size_t)k * G4 + n] += acc[n];
        free(acc);
    }
    {
        double *acc = (double *)calloc(G4, sizeof(double));
        for (size_t r = 0; r < TB; ++r)
            for (int n = 0; n < G4; ++n) acc[n] += dA[r * G4 + n];
        for (int n = 0; n < G4; ++n) db[n] += acc[n];
        free(acc);
    }
    /* dx[t,b,d] = sum_n dA[t,b,n] W[d][n] */
    if (dx) {
#pragma omp parallel for schedule(static)
        for (long r = 0; r < (long)TB; ++r)
            for (int d = 0; d < D; ++d) {
                double acc = 0.0;
                for (int n = 0; n < G4; ++n) acc += dA[(size_t)r * G4 + n] * W[(size_t)d * G4 + n];
                dx[(size_t)r * D + d] = acc;
            }
    }
    if (dh0) memcpy(dh0, dh, sizeof(double) * B * H);
    if (dc0) memcpy(dc0, dc, sizeof(double) * B * H);
    free(dh);
    free(dc);
    return 0;
}

/*
 * Flat parameter layout (interface contract stated in include/blstm.h; the
 * oracle computes it on its own): for l = 0..L-1, for d in (fwd, bwd):
 * W [D_l,4H], R [H,4H], b [4H]; then W_out [2H,K], b_out [K] when K > 0.
 * D_0 = D, D_l = 2H for l >= 1.  Returns the count; fills offs (6L+2 entries).
 */
long ref_param_layout(int L, int D, int H, int K, long *offs)
{
    long o = 0;
    for (int l = 0; l < L; ++l) {
        const long Dl = l == 0 ? D : 2L * H;
        for (int d = 0; d < 2; ++d) {
            const int e = 6 * l + 3 * d;
            if (offs) { offs[e] = o; offs[e + 1] = o + Dl * 4 * H; offs[e + 2] = o + Dl * 4 * H + 4L * H * H; }
            o += Dl * 4 * H + 4L * H * H + 4L * H;
        }
    }
    if (offs) { offs[6 * L] = o; offs[6 * L + 1] = o + (K > 0 ? 2L * H * K : 0); }
    if (K > 0) o += 2L * H * K + K;
    return o;
}

/*
 * One BLSTM training step: forward through L
 * bidirectional layers, softmax-CE head summed over valid frames (or, when
 * K == 0, the caller's dy_top [T,B,2H] as the gradient of the top output),
 * backward through time, gradients written to grad (overwritten, flat layout).
 * Optional outputs: Ys [L,T,B,2H] per-layer outputs, Cs [L,2,T,B,H] cell
 * states, dX1 [T,B,D] gradient of the input, theta_new = theta - lr*grad.
 * loss / frame_errors may be NULL.
 */
/*
 * Input dropout (§4.3: "dropout on the layer inputs of any layer"; DESIGN.md
 * reading R20).  The input of layer l (l = 0: x; l >= 1: Y_{l-1} = [y_f | y_b]) and, with a head,
 * the head's input Y_{L-1} (site L) are replaced by X~ = X * keep / (1 - p); X~ feeds the layer
 * (so dW = X~^T dA) and the gradient reaching X is dX = dX~ * keep / (1 - p).  keep of element
 * (row r = t*B + b, feature j) of site s is the counter-based draw
 *     h = mix(seed + 0x9E3779B9 * (s + 1));  h = mix(h ^ lo32(i));  h = mix(h ^ hi32(i)),
 *     i = r * D_s + j,  keep  <=>  h >= floor(p * 2^32),
 * mix = the "lowbias32" integer finalizer.  Padded frames are dropped or kept alike: their
 * inputs are 0 and their gradients 0.
 */
static uint32_t mix32(uint32_t x)
{
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}
int ref_dropout_keep(uint32_t seed, int site, uint64_t i, double p)
{
    uint32_t h = mix32(seed + 0x9E3779B9u * (uint32_t)(site + 1));
    h = mix32(h ^ (uint32_t)i);
    h = mix32(h ^ (uint32_t)(i >> 32));
    const uint32_t thr = (uint32_t)floor(p * 4294967296.0);
    return h >= thr;
}
/* X~ = X * keep / (1-p) over rows x Dl (site s) */
static void ref_dropout_apply(double *X, size_t rows, int Dl, int site, double p, uint32_t seed)
{
    const double sc = 1.0 / (1.0 - p);
    for (size_t r = 0; r < rows; ++r)
        for (int j = 0; j < Dl; ++j) {
            const size_t i = r * (size_t)Dl + j;
            X[i] = ref_dropout_keep(seed, site, i, p) ? X[i] * sc : 0.0;
        }
}

int ref_blstm_step_ex(int L, int D, int H, int K, int T, int B,
                      const double *theta, const double *x, const uint8_t *mask,
                      const int32_t *labels, const double *dy_top,
                      double lr, double *loss, long *frame_errors,
                      double *grad, double *Ys, double *Cs, double *dX1,
                      double *theta_new, double p_drop, uint32_t seed)
{
    if (L < 1 || B < 1 || H < 1 || T < 0 || p_drop < 0.0 || p_drop >= 1.0) return -1;
    const int drop = p_drop > 0.0;
    const size_t TB = (size_t)T * B, W2 = 2 * (size_t)H;
    long *offs = (long *)malloc(sizeof(long) * (6 * L + 2));
    const long P = ref_param_layout(L, D, H, K, offs);
    memset(grad, 0, sizeof(double) * P);

    /* per-layer, per-direction saved state */
    double **Xin = (double **)calloc(L + 1, sizeof(double *));
    double **Xd = (double **)calloc(L + 1, sizeof(double *)); /* the inputs the layers see */
    double **sv = (double **)calloc(8 * L, sizeof(double *)); /* y,C,G,Hp,Cp per dir */
    Xin[0] = (double *)x;
    for (int l = 0; l < L; ++l) {
        const int Dl = l == 0 ? D : 2 * H;
        if (drop) {
            Xd[l] = (double *)malloc(sizeof(double) * TB * Dl);
            memcpy(Xd[l], Xin[l], sizeof(double) * TB * Dl);
            ref_dropout_apply(Xd[l], TB, Dl, l, p_drop, seed);
        } else {
            Xd[l] = Xin[l];
        }
        double *Y = (double *)malloc(sizeof(double) * TB * W2);
        for (int d = 0; d < 2; ++d) {
            const int e = 6 * l + 3 * d;
            double *y = (double *)malloc(sizeof(double) * TB * H);
            double *C = (double *)malloc(sizeof(double) * TB * H);
            double *Gs = (double *)malloc(sizeof(double) * TB * 4 * H);
            double *Hp = (double *)malloc(sizeof(double) * TB * H);
            double *Cp = (double *)malloc(sizeof(double) * TB * H);
            ref_lstm_fwd(T, B, Dl, H, d == 0 ? 1 : -1, Xd[l], mask,
                         theta + offs[e], theta + offs[e + 1], theta + offs[e + 2],
                         NULL, NULL, y, C, NULL, NULL, Gs, Hp, Cp);
            for (size_t r = 0; r < TB; ++r)
                for (int j = 0; j < H; ++j) Y[r * W2 + (size_t)d * H + j] = y[r * H + j];
            if (Cs) memcpy(Cs + ((size_t)(2 * l + d)) * TB * H, C, sizeof(double) * TB * H);
            double **p = sv + 8 * l + 4 * d;
            p[0] = C; p[1] = Gs; p[2] = Hp; p[3] = Cp;
            free(y);
        }
        if (Ys) memcpy(Ys + (size_t)l * TB * W2, Y, sizeof(double) * TB * W2);
        Xin[l + 1] = Y;
    }

    /* head (summed, unscaled P:253-254) */
    double *dY = (double *)calloc(TB * W2, sizeof(double));
    double lsum = 0.0;
    long ferr = 0;
    if (K > 0) {
        const double *Wo = theta + offs[6 * L], *bo = theta + offs[6 * L + 1];
        double *gWo = grad + offs[6 * L], *gbo = grad + offs[6 * L + 1];
        double *dlog = (double *)calloc(TB * (size_t)K, sizeof(double));
        double *rl = (double *)calloc(TB, sizeof(double));
        long *re = (long *)calloc(TB, sizeof(long));
        if (drop) {
            Xd[L] = (double *)malloc(sizeof(double) * TB * W2);
            memcpy(Xd[L], Xin[L], sizeof(double) * TB * W2);
            ref_dropout_apply(Xd[L], TB, (int)W2, L, p_drop, seed);
        } else {
            Xd[L] = Xin[L];
        }
        const double *YL = Xd[L];
#pragma omp parallel for schedule(static)
        for (long r = 0; r < (long)TB; ++r) {
            if (!mask[r]) continue;
            /* logits[k] = b_out[k] + sum_j Y[r][j] W_out[j][k], ascending j */
            double *lg = dlog + (size_t)r * K;
            for (int k = 0; k < K; ++k) lg[k] = bo[k];
            for (size_t j = 0; j < W2; ++j) {
                const double yj = YL[(size_t)r * W2 + j];
                const double *Woj = Wo + j * K;
                for (int k = 0; k < K; ++k) lg[k] += yj * Woj[k];
            }
            int am = 0;
            double m = lg[0];
            for (int k = 1; k < K; ++k) if (lg[k] > m) { m = lg[k]; am = k; } /* ties: lowest index */
            double se = 0.0;
            for (int k = 0; k < K; ++k) se += exp(lg[k] - m);
            const double lse = m + log(se);
            const int lab = labels[r];
            rl[r] = lse - lg[lab];
            re[r] = (am != lab);
            for (int k = 0; k < K; ++k) lg[k] = exp(lg[k] - lse);
            lg[lab] -= 1.0;
        }
        for (size_t r = 0; r < TB; ++r) { lsum += rl[r]; ferr += re[r]; }
        /* dW_out[j][k] = sum_r Y[r][j] dlog[r][k]; db_out[k] = sum_r dlog[r][k] */
#pragma omp parallel for schedule(static)
        for (long j = 0; j < (long)W2; ++j) {
            double *acc = (double *)calloc(K, sizeof(double));
            for (size_t r = 0; r < TB; ++r) {
                const double yrj = YL[r * W2 + j];
                const double *dl = dlog + r * K;
                for (int k = 0; k < K; ++k) acc[k] += yrj * dl[k];
            }
            for (int k = 0; k < K; ++k) gWo[(size_t)j * K + k] += acc[k];
            free(acc);
        }
        {
            double *acc = (double *)calloc(K, sizeof(double));
            for (size_t r = 0; r < TB; ++r)
                for (int k = 0; k < K; ++k) acc[k] += dlog[r * K + k];
            for (int k = 0; k < K; ++k) gbo[k] += acc[k];
            free(acc);
        }
        /* dY[r][j] = sum_k dlog[r][k] W_out[j][k] */
#pragma omp parallel for schedule(static)
        for (long r = 0; r < (long)TB; ++r)
            for (size_t j = 0; j < W2; ++j) {
                double acc = 0.0;
                for (int k = 0; k < K; ++k) acc += dlog[(size_t)r * K + k] * Wo[j * K + k];
                dY[(size_t)r * W2 + j] = acc;
            }
        free(dlog); free(rl); free(re);
        if (drop) ref_dropout_apply(dY, TB, (int)W2, L, p_drop, seed); /* dY_{L-1} = dY~ * keep/(1-p) */
    } else {
        memcpy(dY, dy_top, sizeof(double) * TB * W2);
    }

    /* backward through the stack, l = L-1 .. 0 */
    double *dyd = (double *)malloc(sizeof(double) * TB * H);
    for (int l = L - 1; l >= 0; --l) {
        const int Dl = l == 0 ? D : 2 * H;
        double *dXl = (double *)calloc(TB * (size_t)Dl, sizeof(double));
        double *dxd = (double *)malloc(sizeof(double) * TB * Dl);
        double *dA = (double *)malloc(sizeof(double) * TB * 4 * H);
        for (int d = 0; d < 2; ++d) {
            const int e = 6 * l + 3 * d;
            double **p = sv + 8 * l + 4 * d;
            for (size_t r = 0; r < TB; ++r)
                for (int j = 0; j < H; ++j) dyd[r * H + j] = dY[r * W2 + (size_t)d * H + j];
            ref_lstm_bwd(T, B, Dl, H, d == 0 ? 1 : -1, Xd[l], mask,
                         theta + offs[e], theta + offs[e + 1],
                         p[0], p[1], p[2], p[3], dyd, NULL, NULL,
                         dxd, grad + offs[e], grad + offs[e + 1], grad + offs[e + 2],
                         NULL, NULL, dA);
            for (size_t i = 0; i < TB * (size_t)Dl; ++i) dXl[i] += dxd[i];
        }
        free(dxd); free(dA);
        if (drop) ref_dropout_apply(dXl, TB, Dl, l, p_drop, seed); /* gradient of the undropped input */
        if (l == 0) {
            if (dX1) memcpy(dX1, dXl, sizeof(double) * TB * D);
            free(dXl);
        } else {
            free(dY);
            dY = dXl; /* [T,B,2H] = gradient of Y_{l-1} */
        }
    }
    free(dyd);
    free(dY);
    if (loss) *loss = lsum;
    if (frame_errors) *frame_errors = ferr;
    if (theta_new)
        for (long i = 0; i < P; ++i) theta_new[i] = theta[i] - lr * grad[i];

    for (int l = 0; l <= L; ++l)
        if (drop && Xd[l]) free(Xd[l]);
    for (int l = 0; l < L; ++l) {
        free(Xin[l + 1]);
        for (int d = 0; d < 2; ++d)
            for (int q = 0; q < 4; ++q) free(sv[8 * l + 4 * d + q]);
    }
    free(Xin); free(Xd); free(sv); free(offs);
    return 0;
}

int ref_blstm_step(int L, int D, int H, int K, int T, int B,
                   const double *theta, const double *x, const uint8_t *mask,
                   const int32_t *labels, const double *dy_top,
                   double lr, double *loss, long *frame_errors,
                   double *grad, double *Ys, double *Cs, double *dX1,
                   double *theta_new)
{
    return ref_blstm_step_ex(L, D, H, K, T, B, theta, x, mask, labels, dy_top, lr, loss, frame_errors, grad, Ys,
                             Cs, dX1, theta_new, 0.0, 0u);
}

/* SGD (§4.3): theta -= lr * grad, gradients unscaled. */
void ref_sgd(double *theta, const double *grad, long n, double lr)
{
    for (long i = 0; i < n; ++i) theta[i] -= lr * grad[i];
}

/* Update rules of PAPER.md §4.3: "Adagrad, Adadelta and Adam", "the classical momentum
 * term and also the simplified Nesterov accelerated gradient"; "penalizing large L2 norms of the
 * weight matrices" and the "norm constraints".  The paper gives no formulas; these
 * are the standard definitions of the cited works as SPEC S:391/S:398 restates them (DESIGN.md
 * reading R19), one update of n parameters:
 *   conditioning, in this order: g += 2*l2*theta on weight-matrix entries (is_bias == 0);
 *     then, if max_norm > 0 and ||g||_2 > max_norm, g *= max_norm / ||g||_2;
 *   rule 0 sgd      theta -= lr*g
 *   rule 1 momentum v = mu*v - lr*g; theta += v                               (s0 = v)
 *   rule 2 nesterov v = mu*v - lr*g; theta += mu*v - lr*g  (simplified form)  (s0 = v)
 *   rule 3 adagrad  a += g^2; theta -= lr*g / (sqrt(a) + eps)                  (s0 = a)
 *   rule 4 adadelta Eg = rho*Eg + (1-rho)*g^2; u = g*sqrt(Ed + eps)/sqrt(Eg + eps);
 *                   Ed = rho*Ed + (1-rho)*u^2; theta -= lr*u                   (s0 = Eg, s1 = Ed)
 *   rule 5 adam     m = b1*m + (1-b1)*g; v = b2*v + (1-b2)*g^2;
 *                   theta -= lr * (m/(1-b1^t)) / (sqrt(v/(1-b2^t)) + eps)      (s0 = m, s1 = v)
 *   zero_grad: g = 0 afterwards (the gradient buffer, not the conditioned copy).
 * is_bias may be NULL (every entry is a weight). */
void ref_opt_update(int rule, double lr, double mu, double rho, double b1, double b2, double eps, double l2,
                    double max_norm, long step, long n, double *theta, double *grad, double *s0, double *s1,
                    const uint8_t *is_bias, int zero_grad)
{
    double *g = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    for (long i = 0; i < n; ++i) {
        g[i] = grad[i];
        if (l2 > 0.0 && !(is_bias && is_bias[i])) g[i] += 2.0 * l2 * theta[i];
    }
    if (max_norm > 0.0) {
        double ss = 0.0;
        for (long i = 0; i < n; ++i) ss += g[i] * g[i];
        const double norm = sqrt(ss);
        if (norm > max_norm)
            for (long i = 0; i < n; ++i) g[i] *= max_norm / norm;
    }
    for (long i = 0; i < n; ++i) {
        const double gi = g[i];
        switch (rule) {
        case 0: theta[i] -= lr * gi; break;
        case 1: s0[i] = mu * s0[i] - lr * gi; theta[i] += s0[i]; break;
        case 2: s0[i] = mu * s0[i] - lr * gi; theta[i] += mu * s0[i] - lr * gi; break;
        case 3: s0[i] += gi * gi; theta[i] -= lr * gi / (sqrt(s0[i]) + eps); break;
        case 4: {
            s0[i] = rho * s0[i] + (1.0 - rho) * gi * gi;
            const double u = gi * sqrt(s1[i] + eps) / sqrt(s0[i] + eps);
            s1[i] = rho * s1[i] + (1.0 - rho) * u * u;
            theta[i] -= lr * u;
            break;
        }
        case 5: {
            s0[i] = b1 * s0[i] + (1.0 - b1) * gi;
            s1[i] = b2 * s1[i] + (1.0 - b2) * gi * gi;
            const double mh = s0[i] / (1.0 - pow(b1, (double)step)), vh = s1[i] / (1.0 - pow(b2, (double)step));
            theta[i] -= lr * mh / (sqrt(vh) + eps);
            break;
        }
        }
        if (zero_grad) grad[i] = 0.0;
    }
    free(g);
}

/* Parameter averaging (§4.1): out = (1/N) sum_r theta_r,
 * thetas laid out [N][n], summed in ascending rank order. */
void ref_dp_average(int nranks, long n, const double *thetas, double *out)
{
    for (long i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int r = 0; r < nranks; ++r) acc += thetas[(size_t)r * n + i];
        out[i] = acc / nranks;
    }
}

/*
 * MDLSTM, one direction (§4.2: 2-D LSTM whose cell at (u,v) depends on the
 * predecessor states (u-1,v) and (u,v-1); SPEC S:256-306 fixes the equations, R21).
 * Plain raster order (u outer, v inner) -- the CPU scheme P:241-242 describes; the GPU path uses
 * the anti-diagonal wavefront instead.
 *   x [U][V][B][D], mask [U][V][B] (1 = pixel of the image), W [D][5H], Ru, Rv [H][5H], b [5H].
 *   a = x W + h(u-1,v) Ru + h(u,v-1) Rv + b   (out-of-grid predecessors: h = c = 0)
 *   stable = 0, blocks [i, fu, fv, g, o]: c = s(fu) c(u-1,v) + s(fv) c(u,v-1) + s(i) tanh(g)
 *   stable = 1, blocks [i, f, g, o, l]:   c = s(f) (s(l) c(u-1,v) + (1-s(l)) c(u,v-1)) + s(i) tanh(g)
 *   h = s(o) tanh(c).  Masked cell: h = 0, c = c(u-1,v) if u > 0, else c(u,v-1) if v > 0, else 0.
 * Outputs h, c [U][V][B][H] and act [U][V][B][5H] (gate activations: sigmoid of each block,
 * tanh of the g block; 0 at masked cells).
 */
static double *mdl_at(double *a, int U, int V, int B, int n, int u, int v, int b)
{
    (void)U;
    return a + (((size_t)u * V + v) * B + b) * n;
}
int ref_mdlstm_fwd(int U, int V, int B, int D, int H, int stable, const double *x, const uint8_t *mask,
                   const double *W, const double *Ru, const double *Rv, const double *bias,
                   double *h, double *c, double *act)
{
    if (U < 1 || V < 1 || B < 1 || D < 1 || H < 1) return -1;
    const int G = 5 * H;
    const int gg = stable ? 2 : 3;  /* index of the tanh block */
    double *a = (double *)malloc(sizeof(double) * G);
    for (int u = 0; u < U; ++u)
        for (int v = 0; v < V; ++v)
            for (int b = 0; b < B; ++b) {
                double *hc = mdl_at(h, U, V, B, H, u, v, b), *cc = mdl_at(c, U, V, B, H, u, v, b);
                double *ac = mdl_at(act, U, V, B, G, u, v, b);
                const double *hu = u > 0 ? mdl_at(h, U, V, B, H, u - 1, v, b) : NULL;
                const double *hv = v > 0 ? mdl_at(h, U, V, B, H, u, v - 1, b) : NULL;
                const double *cu = u > 0 ? mdl_at(c, U, V, B, H, u - 1, v, b) : NULL;
                const double *cv = v > 0 ? mdl_at(c, U, V, B, H, u, v - 1, b) : NULL;
                if (!mask[((size_t)u * V + v) * B + b]) {
                    for (int j = 0; j < H; ++j) { hc[j] = 0.0; cc[j] = cu ? cu[j] : (cv ? cv[j] : 0.0); }
                    for (int n = 0; n < G; ++n) ac[n] = 0.0;
                    continue;
                }
                const double *xc = x + (((size_t)u * V + v) * B + b) * D;
                for (int n = 0; n < G; ++n) a[n] = bias[n];
                for (int k = 0; k < D; ++k) for (int n = 0; n < G; ++n) a[n] += xc[k] * W[(size_t)k * G + n];
                if (hu) for (int k = 0; k < H; ++k) for (int n = 0; n < G; ++n) a[n] += hu[k] * Ru[(size_t)k * G + n];
                if (hv) for (int k = 0; k < H; ++k) for (int n = 0; n < G; ++n) a[n] += hv[k] * Rv[(size_t)k * G + n];
                for (int n = 0; n < G; ++n) ac[n] = (n / H == gg) ? tanh(a[n]) : sigm(a[n]);
                for (int j = 0; j < H; ++j) {
                    const double cuj = cu ? cu[j] : 0.0, cvj = cv ? cv[j] : 0.0;
                    double cn;
                    if (!stable) {
                        cn = ac[H + j] * cuj + ac[2 * H + j] * cvj + ac[j] * ac[3 * H + j];
                    } else {
                        const double lam = ac[4 * H + j];
                        cn = ac[H + j] * (lam * cuj + (1.0 - lam) * cvj) + ac[j] * ac[2 * H + j];
                    }
                    cc[j] = cn;
                    hc[j] = ac[(stable ? 3 : 4) * H + j] * tanh(cn);
                }
            }
    free(a);
    return 0;
}

/*
 * Backward of ref_mdlstm_fwd (reverse raster order), from the saved h, c, act and the output
 * gradient dh_out [U][V][B][H]:  dx [U][V][B][D] (overwritten), dW, dRu, dRv, db (accumulated).
 * A masked cell passes its dc to the predecessor its c was carried from; its dh is dropped.
 */
int ref_mdlstm_bwd(int U, int V, int B, int D, int H, int stable, const double *x, const uint8_t *mask,
                   const double *W, const double *Ru, const double *Rv, const double *h, const double *c,
                   const double *act, const double *dh_out, double *dx, double *dW, double *dRu, double *dRv,
                   double *db)
{
    if (U < 1 || V < 1 || B < 1 || D < 1 || H < 1) return -1;
    const int G = 5 * H;
    const size_t NC = (size_t)U * V * B;
    double *dh = (double *)calloc(NC * H, sizeof(double)), *dc = (double *)calloc(NC * H, sizeof(double));
    double *da = (double *)malloc(sizeof(double) * G);
    memcpy(dh, dh_out, sizeof(double) * NC * H);
    for (int u = U - 1; u >= 0; --u)
        for (int v = V - 1; v >= 0; --v)
            for (int b = 0; b < B; ++b) {
                const size_t cell = ((size_t)u * V + v) * B + b;
                double *dhc = dh + cell * H, *dcc = dc + cell * H;
                double *dhu = u > 0 ? dh + (cell - (size_t)V * B) * H : NULL;
                double *dhv = v > 0 ? dh + (cell - B) * H : NULL;
                double *dcu = u > 0 ? dc + (cell - (size_t)V * B) * H : NULL;
                double *dcv = v > 0 ? dc + (cell - B) * H : NULL;
                double *dxc = dx + cell * D;
                for (int k = 0; k < D; ++k) dxc[k] = 0.0;
                if (!mask[cell]) {
                    for (int j = 0; j < H; ++j) {
                        if (dcu) dcu[j] += dcc[j];
                        else if (dcv) dcv[j] += dcc[j];
                    }
                    continue;
                }
                const double *ac = act + cell * G, *cc = c + cell * H;
                const double *cu = u > 0 ? c + (cell - (size_t)V * B) * H : NULL;
                const double *cv = v > 0 ? c + (cell - B) * H : NULL;
                for (int j = 0; j < H; ++j) {
                    const double cuj = cu ? cu[j] : 0.0, cvj = cv ? cv[j] : 0.0;
                    const double tc = tanh(cc[j]);
                    const int oi = (stable ? 3 : 4) * H + j;
                    const double o = ac[oi];
                    const double dct = dcc[j] + dhc[j] * o * (1.0 - tc * tc);
                    da[oi] = dhc[j] * tc * o * (1.0 - o);
                    const double ig = ac[j];
                    if (!stable) {
                        const double fu = ac[H + j], fv = ac[2 * H + j], g = ac[3 * H + j];
                        da[j] = dct * g * ig * (1.0 - ig);
                        da[H + j] = dct * cuj * fu * (1.0 - fu);
                        da[2 * H + j] = dct * cvj * fv * (1.0 - fv);
                        da[3 * H + j] = dct * ig * (1.0 - g * g);
                        if (dcu) dcu[j] += dct * fu;
                        if (dcv) dcv[j] += dct * fv;
                    } else {
                        const double f = ac[H + j], g = ac[2 * H + j], lam = ac[4 * H + j];
                        const double m = lam * cuj + (1.0 - lam) * cvj;
                        da[j] = dct * g * ig * (1.0 - ig);
                        da[H + j] = dct * m * f * (1.0 - f);
                        da[2 * H + j] = dct * ig * (1.0 - g * g);
                        da[4 * H + j] = dct * f * (cuj - cvj) * lam * (1.0 - lam);
                        if (dcu) dcu[j] += dct * f * lam;
                        if (dcv) dcv[j] += dct * f * (1.0 - lam);
                    }
                }
                const double *xc = x + cell * D;
                const double *hu = u > 0 ? h + (cell - (size_t)V * B) * H : NULL;
                const double *hv = v > 0 ? h + (cell - B) * H : NULL;
                for (int n = 0; n < G; ++n) db[n] += da[n];
                for (int k = 0; k < D; ++k) {
                    double acc = 0.0;
                    for (int n = 0; n < G; ++n) { dW[(size_t)k * G + n] += xc[k] * da[n]; acc += da[n] * W[(size_t)k * G + n]; }
                    dxc[k] = acc;
                }
                for (int k = 0; k < H; ++k) {
                    double au = 0.0, av = 0.0;
                    for (int n = 0; n < G; ++n) {
                        if (hu) dRu[(size_t)k * G + n] += hu[k] * da[n];
                        if (hv) dRv[(size_t)k * G + n] += hv[k] * da[n];
                        au += da[n] * Ru[(size_t)k * G + n];
                        av += da[n] * Rv[(size_t)k * G + n];
                    }
                    if (dhu) dhu[k] += au;
                    if (dhv) dhv[k] += av;
                }
            }
    free(dh); free(dc); free(da);
    return 0;
}
