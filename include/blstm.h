/*
 * blstm.h -- C-ABI of libblstm.so, the B200 (sm_100a) fused BLSTM training hot
 * path of RETURNN (arXiv:1608.00895).
 *
 * Citations: P:n = /root/reference/PAPER.md line n (section given), S:n =
 * SPEC.md line n.  The operation each entry point computes is defined by the
 * paper passage cited beside it and made exact by DESIGN.md §2 (the readings
 * R1..R18 of the paper's silent points).
 *
 * Conventions for every call:
 *   - Tensors are row-major and time-major: a sequence tensor is [T, B, F]
 *     (§5: "time ... as first, the batch index as second and
 *     the layer output size as third dimension").  Floating tensors are fp32.
 *   - The mask is the paper's index tensor: uint8 [T, B], 1 = real
 *     frame, 0 = padding.  Any 0/1 pattern is accepted.  An entry outside {0,1}
 *     is detected on device and reported lazily: the first call
 *     after the kernel that saw it has completed returns BLSTM_ERR_ARG (or
 *     blstm_check_errors() does); that launch read it as 1.  At
 *     a masked frame the LSTM state (h, c) is carried unchanged, the output is 0
 *     and the backward pass emits zero gate gradient (R2/R4).
 *   - LSTM variant (paper silent, R1): no peepholes, gate blocks
 *     [i | f | g | o]; W [D, 4H], R [H, 4H], b [4H];
 *       a = x W + h_{t-1} R + b,  i,f,o = sigmoid, g = tanh,
 *       c_t = f c_{t-1} + i g,  h_t = o tanh(c_t).
 *   - Pointers marked DEVICE are CUDA device pointers; streams are cudaStream_t
 *     passed as void*.  The caller owns every buffer.  The library never
 *     allocates device memory on the hot path and keeps no pointer after a call
 *     returns (the dp_comm handle excepted).  Calls are asynchronous on the
 *     given stream; an error detected by a kernel surfaces as BLSTM_ERR_CUDA on a
 *     later call.
 *   - Return 0 (BLSTM_OK) on success, < 0 on error; the text of the last error
 *     of the calling thread is returned by blstm_last_error().  No exception or
 *     abort crosses the ABI.  All argument checks happen before any launch.
 *   - Gradients are SUMS over valid frames (§4.3: "batches
 *     gradients are not scaled"); parameter gradients accumulate (+=).
 *   - Arithmetic: fp16 tensor-core operands with round-to-nearest, fp32
 *     accumulation, fp32 gate math and state (R9/R10).
 *   - Results are bitwise reproducible for fixed inputs, shapes and device
 *     (no floating-point atomics).
 */
#ifndef BLSTM_H
#define BLSTM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    BLSTM_OK = 0,
    BLSTM_ERR_ARG = -1,         /* null / out-of-range argument */
    BLSTM_ERR_SHAPE = -2,       /* inconsistent sizes or strides */
    BLSTM_ERR_ALIGN = -3,       /* pointer not 16-byte aligned */
    BLSTM_ERR_WORKSPACE = -4,   /* workspace / reserve too small */
    BLSTM_ERR_CUDA = -5,        /* CUDA runtime or launch error */
    BLSTM_ERR_UNSUPPORTED = -6, /* size beyond the kernels' on-chip capacity; never a silent fallback */
    BLSTM_ERR_NCCL = -7         /* NCCL error */
} blstm_status;

/* Text of the last error on this thread (valid until the next call on this thread). */
const char *blstm_last_error(void);
/* ABI version (major*100 + minor). */
int blstm_version(void);
/* Errors detected by kernels of completed earlier calls (a mask entry outside {0,1}): returns
   BLSTM_ERR_ARG once per detection and clears it, else BLSTM_OK.  Synchronize the stream first to
   see the calls issued on it. */
int blstm_check_errors(void);

/* ------------------------------------------------------------------------ */
/* One LSTM layer, one direction: PAPER.md §4.2 P:232-236.                   */
/* ------------------------------------------------------------------------ */
enum { BLSTM_NO_DX = 4, BLSTM_ACCUM_DX = 2 };
/* Precision of the tensor-core operands (R9; SURVEY §8(c) precision table):
 *   BLSTM_PREC_FP16    fp16 operands (round to nearest), fp32 accumulation and state (default);
 *   BLSTM_PREC_FP16X2W the input projection Z = x W + b (the a1 GEMM) with W split into
 *                      W_hi = fp16(W) and W_lo = fp16(W - W_hi), Z = x W_hi + x W_lo in one GEMM over
 *                      a doubled K: removes W's rounding, the dominant error term at small D
 *                      (measured in profiles/r02_parity_*.jsonl); everything else as FP16.
 * Other values (a 3-term split, TF32) return BLSTM_ERR_UNSUPPORTED: the remaining error is the
 * recurrent h R product, whose split would triple the MMAs on the serial chain. */
enum { BLSTM_PREC_FP16 = 0, BLSTM_PREC_FP16X2W = 1 };

typedef struct {
    int T, B, D, H;   /* frames, batch, input width, hidden units; T >= 0, B, D, H >= 1 */
    int direction;    /* +1: scan t = 0..T-1; -1: scan t = T-1..0 (each sequence then starts at its
                         own last valid frame) */
    int ldx, ldy;     /* row strides (elements) of x/dx and of y/dy; ldx >= D, ldy >= H.  A BLSTM
                         direction writes its half of [T,B,2H] with ldy = 2H. */
    int flags;        /* BLSTM_NO_DX / BLSTM_ACCUM_DX (lstm_bwd only) */
    int precision;    /* BLSTM_PREC_FP16 or BLSTM_PREC_FP16X2W */
} lstm_desc;

/* Scratch bytes for one lstm_fwd / lstm_bwd call. */
size_t lstm_workspace_bytes(const lstm_desc *d);
/* Bytes of saved forward state (gate activations, h history); the reserve must
 * live unchanged from lstm_fwd to the matching lstm_bwd ("reuse memory"). */
size_t lstm_reserve_bytes(const lstm_desc *d);

/*
 * Forward: "the non-recurrent part ... in a single matrix
 * multiplication for the whole mini-batch", then the recurrence with the gating
 * fused into the recurrent matmul's epilogue.
 *   x  [T,B,ldx] DEVICE, mask [T,B] DEVICE, W [D,4H], R [H,4H], b [4H] DEVICE
 *   h0, c0 [B,H] DEVICE or NULL (= 0)
 *   y  [T,B,ldy] DEVICE out (0 at masked frames), c [T,B,H] DEVICE out (cell state
 *   after frame t, carried at masked frames), hT, cT [B,H] DEVICE out or NULL
 *   (state after the whole scan).  reserve: lstm_reserve_bytes, workspace:
 *   lstm_workspace_bytes, both DEVICE, 256-byte aligned.
 */
int lstm_fwd(const lstm_desc *d, const float *x, const uint8_t *mask, const float *W, const float *R,
             const float *b, const float *h0, const float *c0, float *y, float *c, float *hT, float *cT,
             void *reserve, void *workspace, size_t workspace_bytes, void *stream);

/*
 * Backward through time (the recurrent part is back
 * propagated first, then the weight and input gradients are single matrix
 * multiplications).  Same x, mask, W, R, h0, c0 and the c / reserve written by
 * lstm_fwd.  dy [T,B,ldy] (ignored where mask = 0), dhT, dcT [B,H] or NULL.
 *   dx [T,B,ldx]: overwritten, or += with BLSTM_ACCUM_DX, untouched with BLSTM_NO_DX
 *   dW [D,4H], dR [H,4H], db [4H]: accumulated (+=)
 *   dh0, dc0 [B,H] or NULL: gradient w.r.t. h0, c0 (overwritten)
 */
int lstm_bwd(const lstm_desc *d, const float *x, const uint8_t *mask, const float *W, const float *R,
             const float *h0, const float *c0, const float *c, const void *reserve, const float *dy,
             const float *dhT, const float *dcT, float *dx, float *dW, float *dR, float *db, float *dh0,
             float *dc0, void *workspace, size_t workspace_bytes, void *stream);

/* ------------------------------------------------------------------------ */
/* Deep bidirectional stack + softmax-CE head: one training step's fwd+BPTT.  */
/* ------------------------------------------------------------------------ */
typedef struct {
    int L, D, H;  /* layers, input width, units per direction */
    int K;        /* classes of the softmax-CE head; 0 = no head, dy_top drives BPTT */
    int T, B;     /* frames, batch (chunks) */
    int flags;    /* reserved, 0 */
    int precision;/* BLSTM_PREC_FP16 or BLSTM_PREC_FP16X2W */
    /* Input dropout of blstm_stack_fwd_bwd ("dropout on the layer inputs of any
     * layer"; R20): 0 <= dropout < 1 is the drop probability of every element of every
     * layer's input and of the head's input; dropout_seed selects the masks (a counter-based draw
     * of (seed, site, element), reproducible; pass a new seed per step).  0 = off.
     * blstm_stack_fwd (inference) never drops. */
    float dropout;
    uint32_t dropout_seed;
} blstm_stack_desc;

/*
 * Flat parameter vector theta (fp32) and its gradient share one layout (the
 * paper's "image of the current network parameters"):
 *   for l = 0..L-1, for dir in (forward, backward):  W [D_l,4H], R [H,4H], b [4H]
 *   then, if K > 0:  W_out [2H,K], b_out [K]
 * with D_0 = D and D_l = 2H (input of layer l+1 = [y_fwd | y_bwd]).
 * blstm_param_offsets fills 6L+2 element offsets: offs[6l+3d+{0,1,2}] = W, R, b of
 * (l, d); offs[6L], offs[6L+1] = W_out, b_out.  Returns the element count.
 */
size_t blstm_param_count(const blstm_stack_desc *d);
size_t blstm_param_offsets(const blstm_stack_desc *d, size_t *offs);
size_t blstm_stack_workspace_bytes(const blstm_stack_desc *d);

typedef struct dp_comm dp_comm;

/*
 * One step's forward + BPTT of the stack:
 *   theta [P] DEVICE; grad [P] DEVICE, accumulated (+=) in theta's layout
 *   x [T,B,D], mask [T,B], labels [T,B] int32 (K > 0) DEVICE
 *   dy_top [T,B,2H] DEVICE (K == 0 only), gradient of the top layer's output
 *   loss_sum: DEVICE double, overwritten with sum over valid frames of
 *     -log softmax(logits)[label] (K > 0; 0 otherwise)
 *   frame_errors: DEVICE int32 or NULL, overwritten with #valid frames whose argmax
 *     (lowest index on ties) differs from the label
 *   comm: NULL, or a dp_comm: grad is then allreduce-SUMmed over ranks (sync data
 *     parallelism, R8), one bucket per layer (and one for the head) as soon as
 *     that bucket is accumulated, on s_side: the exchange overlaps the BPTT of the layers
 *     below.  Every rank must make the same calls in the same order.
 *   workspace: blstm_stack_workspace_bytes DEVICE bytes
 *   s_main: the stream of the call; s_side: a second stream for work off the
 *     critical path (may equal s_main or be NULL)
 */
int blstm_stack_fwd_bwd(const blstm_stack_desc *d, const float *theta, float *grad, const float *x,
                        const uint8_t *mask, const int32_t *labels, const float *dy_top, double *loss_sum,
                        int32_t *frame_errors, dp_comm *comm, void *workspace, size_t workspace_bytes,
                        void *s_main, void *s_side);

/* Forward-only view of the stack for parity checks: Y [L,T,B,2H] and C [L,2,T,B,H]
 * DEVICE outputs (either may be NULL); same workspace as blstm_stack_fwd_bwd. */
int blstm_stack_fwd(const blstm_stack_desc *d, const float *theta, const float *x, const uint8_t *mask,
                    float *Y, float *C, void *workspace, size_t workspace_bytes, void *stream);

/*
 * Chunked batches from a device-resident corpus (§4: sequences chunked
 * into "(possibly overlapping) segments of constant length").  Column b of the
 * batch is the chunk of clen[b] frames starting at corpus frame cstart[b]:
 *   frames [F, D] fp32, frame_labels [F] int32 or NULL: the corpus (sequences concatenated)
 *   cstart [B] int64, clen [B] int32 (0 <= clen <= T; 0 = empty column): DEVICE
 *   x [T, B, D] fp32, mask [T, B] uint8, labels [T, B] int32 or NULL: DEVICE outputs,
 *   x = 0 / mask = 0 / label = 0 at t >= clen[b].  Bit-exact copies (no arithmetic).
 * Errors: BLSTM_ERR_ARG.  Frame indices are not range-checked (the caller's table).
 */
int blstm_gather_chunks(const float *frames, const int32_t *frame_labels, int D, const int64_t *cstart,
                        const int32_t *clen, int B, int T, float *x, uint8_t *mask, int32_t *labels, void *stream);

/* SGD (§4.3): theta -= lr * grad over n elements (gradients unscaled,
 * P:253-254); zero_grad != 0 then sets grad = 0.  DEVICE pointers. */
int sgd_update(float *theta, float *grad, size_t n, float lr, int zero_grad, void *stream);

/*
 * Update rules (§4.3: "Adagrad, Adadelta and Adam ... the classical
 * momentum term and also the simplified Nesterov accelerated gradient ... norm constraints
 * ... penalizing large L2 norms of the weight matrices"; formulas as restated in DESIGN.md
 * R19).  One step over the flat vector theta[n] with gradient grad[n] (unscaled):
 *   g = grad + 2*l2*theta on weight entries (l2 > 0; bias entries are not penalised)
 *   g *= max_norm / ||g||_2 when max_norm > 0 and ||g||_2 exceeds it (global norm constraint)
 *   SGD       theta -= lr*g
 *   MOMENTUM  v = mu*v - lr*g;  theta += v
 *   NESTEROV  v = mu*v - lr*g;  theta += mu*v - lr*g
 *   ADAGRAD   a += g^2;  theta -= lr*g/(sqrt(a) + eps)
 *   ADADELTA  Eg = rho*Eg + (1-rho)g^2;  u = g*sqrt(Eu+eps)/sqrt(Eg+eps);  Eu = rho*Eu + (1-rho)u^2;
 *             theta -= lr*u
 *   ADAM      m = b1*m + (1-b1)g;  v = b2*v + (1-b2)g^2;
 *             theta -= lr*(m/(1-b1^step)) / (sqrt(v/(1-b2^step)) + eps)
 * then grad = 0 if zero_grad.  Arithmetic fp32 (norm sum fp64, reproducible bit for bit).
 */
enum { BLSTM_OPT_SGD = 0, BLSTM_OPT_MOMENTUM = 1, BLSTM_OPT_NESTEROV = 2, BLSTM_OPT_ADAGRAD = 3,
       BLSTM_OPT_ADADELTA = 4, BLSTM_OPT_ADAM = 5 };
typedef struct {
    int rule;       /* BLSTM_OPT_* */
    double lr, mu, rho, beta1, beta2, eps;
    double l2;       /* L2 penalty factor on weight entries, 0 = off */
    double max_norm; /* global gradient norm constraint, 0 = off */
    long step;       /* 1-based count of this update (Adam's bias correction) */
} blstm_opt_params;
/* Hyper-parameters are fp64 at the boundary: 1-beta2, 1-rho etc. are formed in fp64 on the
 * host (1 - 0.999f would carry a 1.3e-5 relative error into every second moment). */
/* Floats of optimizer state for n parameters: 0 (SGD), n4 (MOMENTUM, NESTEROV: v; ADAGRAD: a),
 * 2*n4 (ADADELTA: Eg then Eu; ADAM: m then v), n4 = n rounded up to a multiple of 4: the
 * second slot starts at state + n4.  The caller zero-fills it before the first step. */
size_t blstm_opt_state_floats(int rule, size_t n);
/* DEVICE workspace bytes blstm_opt_update needs (the norm pass's fp64 partials). */
size_t blstm_opt_workspace_bytes(size_t n);
/*
 * theta, grad [n], state [blstm_opt_state_floats] (NULL if 0), workspace: DEVICE, 16-byte
 * aligned, owned by the caller; updated in place on `stream` (asynchronous).
 * layout: NULL = every entry is a weight; else n must equal blstm_param_count(layout) and the
 * b / b_out ranges of its layout are the bias entries (L <= 31).
 * Errors (nothing launched): BLSTM_ERR_ARG (null pointer, unknown rule, step < 1 for ADAM,
 * n mismatch), BLSTM_ERR_ALIGN, BLSTM_ERR_WORKSPACE, BLSTM_ERR_UNSUPPORTED (L > 31).
 */
int blstm_opt_update(const blstm_opt_params *p, const blstm_stack_desc *layout, float *theta, float *grad,
                     float *state, size_t n, int zero_grad, void *workspace, size_t workspace_bytes,
                     void *stream);

/*
 * One whole training step: blstm_stack_fwd_bwd, then the update rule opt (blstm_opt_update
 * semantics with the stack's layout: L2 on weights only, optional global norm constraint) applied
 * to theta, grad set to 0 afterwards (the update "fused into the allreduce
 * epilogue").  Each gradient bucket (one per layer, one for the head) is updated on s_side as soon
 * as it is final -- after its scatters and, with comm, its allreduce -- overlapping the BPTT of the
 * layers below; with opt->max_norm > 0 (the norm needs every gradient) one update runs at the end.
 *   theta [P] DEVICE, updated in place; grad [P] DEVICE (+= then consumed: 0 on return)
 *   opt_state: blstm_opt_state_floats(opt->rule, P) DEVICE floats (NULL if 0)
 * Other arguments as blstm_stack_fwd_bwd.  The result equals blstm_stack_fwd_bwd followed by
 * blstm_opt_update(opt, d, ..., zero_grad = 1) bit for bit.
 */
int blstm_stack_train_step(const blstm_stack_desc *d, float *theta, float *grad, const float *x, const uint8_t *mask,
                           const int32_t *labels, const float *dy_top, double *loss_sum, int32_t *frame_errors,
                           dp_comm *comm, const blstm_opt_params *opt, float *opt_state, void *workspace,
                           size_t workspace_bytes, void *s_main, void *s_side);


/* ------------------------------------------------------------------------ */
/* Data parallelism over NCCL (§4.1).                      */
/* ------------------------------------------------------------------------ */
/* Rank 0 creates the 128-byte NCCL id; the caller broadcasts it (e.g. torch PG). */
int dp_get_unique_id(unsigned char id[128]);
/* Create a communicator for this rank on the current CUDA device. */
int dp_comm_init(int nranks, int rank, const unsigned char id[128], dp_comm **out);
/* grad <- sum over ranks (in place, fp32): sync mode, one big batch (P:254 unscaled). */
int dp_allreduce_grads(dp_comm *c, float *grad, size_t n, void *stream);
/* theta <- (1/N) sum over ranks (in place, fp32): the paper's parameter averaging
 * "combined into a single set of parameters by averaging". */
int dp_average_params(dp_comm *c, float *theta, size_t n, void *stream);
int dp_comm_destroy(dp_comm *c);
/*
 * The sync-mode exchange buckets of blstm_stack_fwd_bwd / blstm_stack_train_step (host-only,
 * no device work): [lo[i], hi[i]) of theta's layout, in the order the step issues the bucket
 * allreduces (and, in blstm_stack_train_step, the bucket updates): the head (K > 0) first,
 * then layer L-1 down to layer 0, each as soon as its gradients are final.
 * The buckets partition [0, blstm_param_count).  lo, hi: HOST arrays of max_buckets >= L + 1
 * entries.  Returns the bucket count, or BLSTM_ERR_ARG.
 */
int blstm_dp_buckets(const blstm_stack_desc *d, size_t *lo, size_t *hi, int max_buckets);
/*
 * N replicas resident on ONE device (a single-GPU simulation of N workers, SURVEY.md §8(f)
 * NEXT-1): x_r <- scale * sum_{q<n} x_q for every r < n, summed in replica order 0..n-1 in
 * fp32, so all replicas receive identical bits.  scale = 1/n is the paper's parameter
 * averaging; scale = 1 is the sync-mode gradient sum (R8).
 *   ptrs: HOST array of n DEVICE pointers (16-byte aligned, pairwise distinct), 1 <= n <= 16
 *   len: elements per replica.  Errors: BLSTM_ERR_ARG, BLSTM_ERR_ALIGN.
 */
int blstm_reduce_replicas(float *const *ptrs, int n, size_t len, float scale, void *stream);

/* ------------------------------------------------------------------------ */
/* Multi-directional 2-D LSTM layer (NEXT-2): PAPER.md §4.2 P:238-245.        */
/* ------------------------------------------------------------------------ */
/*
 * A grid x [U, V, B, D] (rows u, columns v, B images) is scanned by four 2-D LSTMs, one per
 * corner: direction k runs on the grid flipped by (k & 1: flip u, k & 2: flip v) and its output
 * is flipped back; y [U, V, B, 4H] = [y_0 | y_1 | y_2 | y_3].  In a direction's
 * frame (R21):
 *   a = x W + h(u-1,v) Ru + h(u,v-1) Rv + b        (missing predecessors: h = c = 0)
 *   stable = 0, gate blocks [i, fu, fv, g, o]:  c = s(fu) c(u-1,v) + s(fv) c(u,v-1) + s(i) tanh(g)
 *   stable = 1, gate blocks [i, f, g, o, l]:    c = s(f) (s(l) c(u-1,v) + (1-s(l)) c(u,v-1)) + s(i) tanh(g)
 *   h = s(o) tanh(c);  mask [U, V, B] = 0: h = 0, c carried from (u-1,v), else (u,v-1), else 0.
 * Cells on one anti-diagonal are independent ("activations for all positions on a common
 * diagonal can be computed at the same time"): one launch per diagonal for all four
 * directions and all images.
 * theta / grad: per direction k: W [D, 5H], Ru [H, 5H], Rv [H, 5H], b [5H] (fp32, DEVICE).
 */
typedef struct {
    int U, V, B, D, H;
    int stable;
} mdlstm_desc;
size_t mdlstm_param_count(const mdlstm_desc *d);
size_t mdlstm_workspace_bytes(const mdlstm_desc *d);
/* saved forward state (kept unchanged from mdlstm_fwd to the matching mdlstm_bwd) */
size_t mdlstm_reserve_bytes(const mdlstm_desc *d);
/* x [U,V,B,D], mask [U,V,B] uint8, y [U,V,B,4H] out; DEVICE, 16-byte aligned buffers. */
int mdlstm_fwd(const mdlstm_desc *d, const float *theta, const float *x, const uint8_t *mask, float *y,
               void *reserve, void *workspace, size_t workspace_bytes, void *stream);
/* Gradients of sum(y * dy): dx [U,V,B,D] overwritten (NULL: not computed), grad += (theta's layout). */
int mdlstm_bwd(const mdlstm_desc *d, const float *theta, const float *x, const uint8_t *mask, const void *reserve,
               const float *dy, float *dx, float *grad, void *workspace, size_t workspace_bytes, void *stream);

/* ------------------------------------------------------------------------ */
/* Test hook: the tcgen05 GEMM used by every dense contraction of the path.   */
/* ------------------------------------------------------------------------ */
/* C[m,n] = alpha * sum_k A(m,k) B(n,k) (+ C[m,n] if beta) (+ bias[n]), A and B fp16
 * DEVICE (16-byte aligned, ld a multiple of 8), each K-major (element (r,k) at
 * ptr[r*ld + k], *_mn = 0) or MN-major (at ptr[k*ld + r], *_mn = 1); C fp32.  The same kernels
 * the stack runs: split-K over a long K, CTA-pair tiles and tail-wave splits, with a
 * library-owned scratch per device (288 MB, allocated on the first call). */
int blstm_gemm_f16(int M, int N, int K, const void *A, long lda, int a_mn, const void *B, long ldb, int b_mn,
                   float *C, long ldc, float alpha, int beta, const float *bias, void *stream);

/* ------------------------------------------------------------------------ */
/* Measurement hooks (bench.py).                                              */
/* ------------------------------------------------------------------------ */
/* Number of kernels this library has launched since it was loaded. */
long blstm_launch_count(void);
/* on = 1: from now on bracket every launch of the categories below with CUDA events on the
 * launching stream (records are reset); on = 2: also the helper kernels (category 3, for
 * blstm_profile_timeline; adds two events per helper launch); on == 0: stop. */
int blstm_profile_enable(int on);
/* Restrict the recording to the categories whose bit is set in cat_mask (bit c: category c; the
 * default, and -1, is every category).  Each bracket is two event records between the stream's
 * kernels (~1.7 us per C3 launch): bench.py times only the dominant category inside its timed
 * region and the others in an untimed pass.  Returns 0. */
int blstm_profile_select(int cat_mask);
/* cat: 0 forward recurrence, 1 BPTT recurrence, 2 GEMM.  Synchronizes the
 * recorded events; returns the summed device time (ms) and launch count. */
int blstm_profile_read(int cat, double *total_ms, long *launches);
/* Timeline of the launches recorded since blstm_profile_enable(1) (synchronizes them):
 * 7 doubles per launch into host `rec` (at most max_recs launches): category (0-2 as above,
 * 3 = helper kernels), stream index (order of first appearance), start and end (ms, relative
 * to the first recorded start), and the launch shape (GEMM: M, N, K; else 0).  Returns the
 * number of launches written, < 0 on error. */
int blstm_profile_timeline(double *rec, int max_recs);
/* Debug: record per-step phase timestamps (SM clock64 cycles, 16 slots per step, CTA 0 /
 * thread 0) of the following forward / BPTT recurrence launches into DEVICE buffers of
 * 16*T uint64 each; NULL disables.  Only a library built with -DBLSTM_TRACE writes them. */
int blstm_debug_set_trace(void *fwd, void *bwd);

#ifdef __cplusplus
}
#endif
#endif /* BLSTM_H */
