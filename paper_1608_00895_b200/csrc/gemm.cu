// gemm.cu -- TMA-fed tcgen05 GEMM for the dense contractions of the path:
//   a1  Z  = X W + b            (§4.2, "a single matrix multiplication
//                                 for the whole mini-batch of sequences")
//   a4  logits = Y W_out + b_out, dY = dlogits W_out^T, dW_out = Y^T dlogits
//   a6  dX = dA W^T, dW = X^T dA, dR = Hprev^T dA  ("after the recurrent part is
//                                 back propagated through time")
//
//   C[m, n] = alpha * sum_k A(m, k) * B(n, k)  (+ C[m, n] if beta)  (+ bias[n])
//
// A and B are fp16, each either K-major (element (r, k) at ptr[r*ld + k]) or MN-major
// (element (r, k) at ptr[k*ld + r]); C is fp32 row-major.  fp32 accumulation in TMEM.
//
// Structure (persistent, one CTA per SM, 10 warps):
//   warp 0      TMA producer (one elected lane), STAGES-deep smem ring, 128B swizzle
//   warp 1      TMEM allocator + MMA issuer (one lane), tcgen05.mma M=128 N=BN K=16
//   warps 2..9  epilogue (two per TMEM lane quarter, each half of the columns):
//               tcgen05.ld -> alpha/bias (bias staged in smem)/beta -> fp32 global stores
//   Two TMEM accumulators (2 x BN columns) let the epilogue of tile i overlap the
//   MMAs of tile i+1.
#include "common.cuh"
#include "gemm.h"
#include "prof.h"

namespace blstm {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
constexpr int GEMM_EPI_WARPS = 8;  // two per TMEM lane quarter, each half of the tile's columns
constexpr int GEMM_THREADS = 64 + 32 * GEMM_EPI_WARPS;

template <int BN>
struct GemmCfg {
    static constexpr int STAGES = BN >= 256 ? 4 : 6;
    static constexpr int A_BYTES = GEMM_BM * GEMM_BK * 2;
    static constexpr int B_BYTES = BN * GEMM_BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ +
                                      GEMM_EPI_WARPS * 4096 /*store staging*/;
    static constexpr int TMEM_COLS = 2 * BN;
};

// tile index -> (M-tile, N-tile).  Default: N fastest, so the N-tiles of one M block run on
// neighbouring CTAs at about the same time and the (large) A operand streams from HBM once while
// the (small) B operand stays in L2; M-fastest re-read A once per N-tile (the dX GEMM read 4x its
// 166 MB A from DRAM).  With completion flags: round r visits, per direction d, all N-tiles of
// that direction at M-tile r (ascending) or num_m-1-r (descending), so Z becomes complete in the
// order the recurrence reads it.
template <int BN>
DEVI void tile_coords(int tile, int num_m, int num_n, const GemmParams &p, int &mt, int &nt) {
    if (!p.flags) {
        mt = tile / num_n;
        nt = tile - mt * num_n;
        return;
    }
    const int ntd = p.natHq4 / BN, per = p.natNdir * ntd;
    const int r = tile / per, w = tile - r * per, d = w / ntd;
    mt = ((p.flag_desc >> d) & 1) ? num_m - 1 - r : r;
    nt = w;
}

// work item -> (batch, split, tile, k-block range, tail partial slot or -1); identical in the
// producer, MMA and epilogue loops
struct GemmItem {
    int bt, split, tile, kb0, kb1, tslot;
};
DEVI GemmItem gemm_item(const GemmParams &p, int item, int num_tiles, int per_batch, int kbs, int num_kb) {
    GemmItem it;
    if (p.tail_split > 1 && item >= p.full_items) {  // a K-split of a tile of the partial last wave
        const int ti = item - p.full_items, kbt = (num_kb + p.tail_split - 1) / p.tail_split;
        it.bt = 0;
        it.tslot = ti;
        it.tile = p.full_items + ti / p.tail_split;
        it.split = ti % p.tail_split;
        it.kb0 = it.split * kbt;
        it.kb1 = min(num_kb, it.kb0 + kbt);
    } else {
        it.bt = item / per_batch;
        const int bi = item - it.bt * per_batch;
        it.split = bi / num_tiles;
        it.tile = bi - it.split * num_tiles;
        it.kb0 = it.split * kbs;
        it.kb1 = min(num_kb, (it.split + 1) * kbs);
        it.tslot = -1;
    }
    return it;
}

// scatter-mode addresses (gemm.h GemmScatter); -1: the element has no destination (padding)
DEVI long scat_row(const GemmScatter &s, int m) {
    if (s.rowmode == 0) return m < s.nrows ? (long)m : -1L;
    const int d = m / (4 * s.Hq), r = m - d * 4 * s.Hq, u = r >> 2, gam = r & 3;
    return u < s.H ? d * s.dstride + (long)gam * s.H + u : -1L;
}
DEVI long scat_col(const GemmScatter &s, int n) {
    if (s.colmode == 0) return n < s.ncols ? (long)n * s.ld : -1L;
    const int h = n / s.Hq, u = n - h * s.Hq;
    return u < s.H ? ((long)h * s.H + u) * s.ld : -1L;
}

template <int BN>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_f16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmA2, GemmParams p) {
    using Cfg = GemmCfg<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *full = (uint64_t *)(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
    uint64_t *empty = full + Cfg::STAGES;
    uint64_t *tfull = empty + Cfg::STAGES;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = (uint32_t *)(tempty + 2);

    const int warp = warp_id();
    const int num_m = (p.M + GEMM_BM - 1) / GEMM_BM;
    const int num_n = (p.N + BN - 1) / BN;
    const int num_tiles = num_m * num_n;
    const int num_kb = (p.K + GEMM_BK - 1) / GEMM_BK;
    // split-K: work item = (split, tile); split s covers k-blocks [s*kbs, min(num_kb, (s+1)*kbs))
    const int kbs = (num_kb + p.ksplit - 1) / p.ksplit;
    const int per_batch = num_tiles * p.ksplit;
    const int num_items = p.tail_split > 1 ? p.full_items + (num_tiles - p.full_items) * p.tail_split
                                           : per_batch * p.nbatch;

    if (warp == 0 && lane_id() == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        if (p.nbatch > 1) tma_prefetch_desc(&tmA2);
        for (int s = 0; s < Cfg::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], GEMM_EPI_WARPS);
        }
        fence_mbar_init();
    }
    if (p.arb) {  // resident (common.cuh); the conditional re-launch of the recurrence may launch
        if (threadIdx.x == 64) arb_checkin(p.arb);
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
    if (warp == 1) {
        tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (p.pdl_chain) {  // (gemm.h) the previous kernel of the chain completed and is visible from here
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int item = blockIdx.x; item < num_items; item += gridDim.x) {
                const GemmItem itm = gemm_item(p, item, num_tiles, per_batch, kbs, num_kb);
                const int bt = itm.bt;
                int mt, nt;
                tile_coords<BN>(itm.tile, num_m, num_n, p, mt, nt);
                const int m0 = mt * GEMM_BM, n0 = nt * BN;
                const CUtensorMap *mA = bt ? &tmA2 : &tmA;
                const int boff = bt * (int)p.b_boff;  // along B's outer dimension
                for (int kb = itm.kb0; kb < itm.kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t *sa = smem + stage * Cfg::STAGE_BYTES;
                    uint8_t *sb = sa + Cfg::A_BYTES;
                    mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
                    const int k0 = kb * GEMM_BK;
                    if (!p.a_mn) {
                        const int ka = p.a_kwrap ? (kb % p.a_kwrap) * GEMM_BK : k0;
                        tma_load_2d(sa, mA, &full[stage], ka, m0);
                    } else {
                        tma_load_2d(sa, mA, &full[stage], m0, k0);
                        tma_load_2d(sa + 8192, mA, &full[stage], m0 + 64, k0);
                    }
                    if (!p.b_mn) {
                        tma_load_2d(sb, &tmB, &full[stage], k0, n0 + boff);
                    } else {
#pragma unroll
                        for (int j = 0; j < BN / 64; ++j)
                            tma_load_2d(sb + j * 8192, &tmB, &full[stage], n0 + 64 * j, k0 + boff);
                    }
                    if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        const uint32_t idesc = idesc_f16(GEMM_BM, BN, p.a_mn, p.b_mn);
        const int a_mn = warp_uniform(p.a_mn), b_mn = warp_uniform(p.b_mn);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int item = blockIdx.x; item < num_items; item += gridDim.x) {
            const GemmItem itm = gemm_item(p, item, num_tiles, per_batch, kbs, num_kb);
            const int kb0 = itm.kb0, kb1 = itm.kb1;
            mbar_wait(&tempty[acc], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + acc * BN;
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                {  // warp-collective issue (one elected lane), operands warp-uniform
                    const uint32_t sa = smem_u32(smem + stage * Cfg::STAGE_BYTES);
                    const uint32_t sb = sa + Cfg::A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < GEMM_BK / 16; ++kk) {
                        const uint64_t ad = a_mn ? sdesc_sw128(sa + kk * 2048, 8192, 1024)
                                                 : sdesc_sw128(sa + kk * 32, 16, 1024);
                        const uint64_t bd = b_mn ? sdesc_sw128(sb + kk * 2048, 8192, 1024)
                                                 : sdesc_sw128(sb + kk * 32, 16, 1024);
                        mma_f16_ss_w(d_tmem, ad, bd, idesc, (kb != kb0) | (kk != 0));
                    }
                    mma_commit_w(&empty[stage]);
                    if (kb == kb1 - 1) mma_commit_w(&tfull[acc]);
                }
                __syncwarp();
                if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
            }
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    } else {
        // ---------------- epilogue (warps 2..9) ----------------
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        const int row_in_tile = q * 32 + lane_id();
        int acc = 0;
        uint32_t acc_phase = 0;
        const int et = threadIdx.x - 64;                           // 0..255 over the epilogue warps
        const int chalf = (warp - 2) / 4;                          // column half of this warp
        // row-major stores go through a per-warp [32 rows][32 cols] staging tile (float4 index
        // XOR-swizzled by row), so each store instruction writes 4 rows x 128 contiguous bytes (whole
        // lines); two TMEM loads are in flight per wait, and the bias comes from warp-uniform L1
        // loads issued before that wait (no per-tile barrier to stage it)
        float4 *stg4 = reinterpret_cast<float4 *>(tmem_slot + 4) + (warp - 2) * 256;
        const int lane = lane_id();
        (void)et;
        for (int item = blockIdx.x; item < num_items; item += gridDim.x) {
            const GemmItem itm = gemm_item(p, item, num_tiles, per_batch, kbs, num_kb);
            const int bt = itm.bt, split = itm.split, tslot = itm.tslot;
            int mt, nt;
            tile_coords<BN>(itm.tile, num_m, num_n, p, mt, nt);
            const int m0 = mt * GEMM_BM, n0 = nt * BN;
            float *Cbase = p.C + bt * p.c_bstride + split * p.split_stride;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int m = m0 + row_in_tile;
            float *crow = Cbase + (size_t)m * p.ldc;
#pragma unroll 1
            for (int c = chalf * (BN / 2); c < (chalf + 1) * (BN / 2); c += 32) {
                float v[32];
                const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c;
                tmem_ld16(ta, *reinterpret_cast<float(*)[16]>(&v[0]));
                tmem_ld16(ta + 16, *reinterpret_cast<float(*)[16]>(&v[16]));
                const int n = n0 + c;
                float bv[32];
                if (p.bias && n + 32 <= p.N && ((uintptr_t)(p.bias + n) & 15) == 0) {  // warp-uniform: broadcast
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        const float4 b4 = __ldg(reinterpret_cast<const float4 *>(p.bias + n + j));
                        bv[j] = b4.x; bv[j + 1] = b4.y; bv[j + 2] = b4.z; bv[j + 3] = b4.w;
                    }
                } else if (p.bias) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) bv[j] = n + j < p.N ? __ldg(p.bias + n + j) : 0.f;
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) bv[j] = 0.f;
                }
                tmem_ld_wait();
                if (tslot >= 0) {  // tail split: the raw partial tile [128][BN] (the reduction finishes it)
                    float4 *dst = reinterpret_cast<float4 *>(p.tail_ws + (size_t)tslot * GEMM_BM * BN +
                                                             (size_t)row_in_tile * BN + c);
#pragma unroll
                    for (int j = 0; j < 8; ++j) dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                    continue;
                }
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = v[j] * p.alpha + bv[j];
                if (p.scat.dst) {  // scatter-add into the parameter layout (split-K: the reduction does it)
                    if (m >= p.M) continue;
                    const long ro = scat_row(p.scat, m);
                    if (ro < 0) continue;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const long co = n + j < p.N ? scat_col(p.scat, n + j) : -1L;
                        if (co >= 0) p.scat.dst[ro + co] += v[j];
                    }
                } else if (p.natB) {
                    if (m >= p.M || n >= p.N) continue;
                    // CTA-native layout of the recurrence (see lstm_rec.h): the 32 columns stay in
                    // one 128-row block of one CTA, consecutive columns are NQ floats apart
                    const long t = m / p.natB, b = m - t * p.natB;
                    const int g = (int)(b / p.natBg), nn = (int)(b - (long)g * p.natBg);
                    const int cb = nn / p.natNQ, i = nn - cb * p.natNQ;
                    const long blk = 512L * p.natNQ;
                    const long rm = ((t * p.natNdir * p.natG + g) * p.natNC) * blk + (long)cb * 128 * p.natNQ + i;
                    const int d = n / p.natHq4, rr = n - d * p.natHq4;
                    const long cn = ((long)d * p.natG * p.natNC + (rr >> 7)) * blk + (long)(rr & 127) * p.natNQ;
                    float *base = p.C + rm + cn;
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (n + j < p.N) base[(long)j * p.natNQ] = v[j];
                } else if ((p.ldc & 3) == 0 && ((uintptr_t)Cbase & 15) == 0) {
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        stg4[lane * 8 + (k ^ (lane & 7))] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
                    __syncwarp();
#pragma unroll
                    for (int it = 0; it < 8; ++it) {
                        const int r = 4 * it + (lane >> 3), k = lane & 7;
                        float4 o = stg4[r * 8 + (k ^ (r & 7))];
                        const int mm = m0 + 32 * q + r, nn = n + 4 * k;
                        if (mm < p.M && nn < p.N) {
                            float *dst = Cbase + (size_t)mm * p.ldc + nn;
                            if (nn + 4 <= p.N) {
                                if (p.beta) {
                                    const float4 old = *reinterpret_cast<const float4 *>(dst);
                                    o.x += old.x; o.y += old.y; o.z += old.z; o.w += old.w;
                                }
                                *reinterpret_cast<float4 *>(dst) = o;
                            } else {
                                const float ov[4] = {o.x, o.y, o.z, o.w};
                                for (int e = 0; e < p.N - nn; ++e) dst[e] = p.beta ? dst[e] + ov[e] : ov[e];
                            }
                        }
                    }
                    __syncwarp();
                } else if (m < p.M && n < p.N) {
                    if (n + 32 <= p.N && (p.ldc & 3) == 0) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4) {
                            float4 o = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                            float4 *dst = reinterpret_cast<float4 *>(crow + n + j);
                            if (p.beta) {
                                const float4 old = *dst;
                                o.x += old.x; o.y += old.y; o.z += old.z; o.w += old.w;
                            }
                            *dst = o;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (n + j < p.N) crow[n + j] = p.beta ? crow[n + j] + v[j] : v[j];
                    }
                }
            }
            if (p.flags) {  // publish the tile to the concurrently running recurrence
                asm volatile("bar.sync 2, %0;" ::"n"(32 * GEMM_EPI_WARPS) : "memory");
                if (et == 0) {
                    __threadfence();
                    red_release_gpu_add(p.flags + (n0 / p.natHq4) * num_m + mt, 1);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane_id() == 0) mbar_arrive(&tempty[acc]);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
    }
    // programmatic dependent launch: complete only after the primary grid (the recurrence this GEMM
    // feeds) has, so later work in the stream keeps plain stream order.  All tiles are published
    // before this point, hence no cycle.
    if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2) for plain GEMMs with many tiles: a 2-CTA cluster computes a
// 256 x 256 tile; CTA r loads its 128 rows of A and its 128 columns of B (B split by N) per
// k-block, both completing on the even CTA's full barrier (TMA .cta_group::2); the even CTA
// issues M = 256, N = 256 MMAs that read both CTAs' shared memory and write each CTA's 128 rows
// of D into its own TMEM; commits are multicast to both CTAs.  Per SM a k-block is 32 KB of
// operands instead of 48 KB, and the pair MMA keeps the tensor pipe busier (ncu: the single-CTA
// kernel's TC pipe at 80 % on C5's Z GEMM).  Plain row-major output with alpha / beta / bias only.
// ---------------------------------------------------------------------------
constexpr int GP_STAGES = 6;
constexpr int GP_A_BYTES = GEMM_BM * GEMM_BK * 2;           // 16 KB: this CTA's 128 rows of A
constexpr int GP_B_BYTES = 128 * GEMM_BK * 2;               // 16 KB: this CTA's 128 columns of B
constexpr int GP_STAGE_BYTES = GP_A_BYTES + GP_B_BYTES;
// [stages][barriers, 1 KB][store staging: 8 warps x 4 KB, 1024-aligned for the SW128 TMA stores]
constexpr int GP_SMEM_BYTES = GP_STAGES * GP_STAGE_BYTES + 1024 + 1024 + GEMM_EPI_WARPS * 4096;

DEVI void tma_load_2d_pair(void *dst, const CUtensorMap *m, uint32_t bar_cluster, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(c0), "r"(c1)
        : "memory");
}
DEVI void mma_f16_ss2_w(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
        " @e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
DEVI void mbar_remote_arrive_release(uint32_t bar_cluster) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM_THREADS, 1)
    gemm_f16_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const __grid_constant__ CUtensorMap tmC, GemmParams p, int tma_store) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *full = (uint64_t *)(smem + GP_STAGES * GP_STAGE_BYTES);
    uint64_t *empty = full + GP_STAGES;
    uint64_t *tfull = empty + GP_STAGES;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = (uint32_t *)(tempty + 2);
    constexpr int BN = 256;

    const int warp = warp_id();
    const int r = (int)cluster_ctarank();
    const int num_mp = (p.M + 2 * GEMM_BM - 1) / (2 * GEMM_BM);
    const int num_n = (p.N + BN - 1) / BN;
    const int num_tiles = num_mp * num_n;
    const int ks = p.ksplit > 1 ? p.ksplit : 1;  // split-K: item = (split, tile); partials at split * split_stride
    const int num_items = num_tiles * ks;
    const int num_kb = (p.K + GEMM_BK - 1) / GEMM_BK;
    const int kbs = (num_kb + ks - 1) / ks;
    const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;

    if (warp == 0 && lane_id() == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int s = 0; s < GP_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 2 * GEMM_EPI_WARPS);  // (the even CTA's: both CTAs' epilogue warps)
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        tmem_alloc2(tmem_slot, 2 * BN);
        tmem_relinquish2();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // every barrier of the pair initialised before any remote arrive / complete_tx
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer (both CTAs) ----------------
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int item = cl; item < num_items; item += ncl) {
                const int split = item / num_tiles, tile = item - split * num_tiles;
                const int mp = tile / num_n, nt = tile - mp * num_n;
                const int m0 = mp * 2 * GEMM_BM + r * GEMM_BM, n0 = nt * BN + r * 128;
                const int kb1 = min(num_kb, (split + 1) * kbs);
                for (int kb = split * kbs; kb < kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t *sa = smem + stage * GP_STAGE_BYTES;
                    uint8_t *sb = sa + GP_A_BYTES;
                    const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);  // the even CTA's barrier
                    if (r == 0) mbar_arrive_expect_tx(&full[stage], 2 * GP_STAGE_BYTES);
                    const int k0 = kb * GEMM_BK;
                    if (!p.a_mn) {
                        tma_load_2d_pair(sa, &tmA, fb, k0, m0);
                    } else {
                        tma_load_2d_pair(sa, &tmA, fb, m0, k0);
                        tma_load_2d_pair(sa + 8192, &tmA, fb, m0 + 64, k0);
                    }
                    if (!p.b_mn) {
                        tma_load_2d_pair(sb, &tmB, fb, k0, n0);
                    } else {
                        tma_load_2d_pair(sb, &tmB, fb, n0, k0);
                        tma_load_2d_pair(sb + 8192, &tmB, fb, n0 + 64, k0);
                    }
                    if (++stage == GP_STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (the even CTA) ----------------
        if (r == 0) {
            const uint32_t idesc = idesc_f16(2 * GEMM_BM, BN, p.a_mn, p.b_mn);
            const int a_mn = warp_uniform(p.a_mn), b_mn = warp_uniform(p.b_mn);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int item = cl; item < num_items; item += ncl) {
                const int split = item / num_tiles;
                const int kb0 = split * kbs, kb1 = min(num_kb, (split + 1) * kbs);
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + stage * GP_STAGE_BYTES);
                    const uint32_t sb = sa + GP_A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < GEMM_BK / 16; ++kk) {
                        const uint64_t ad = a_mn ? sdesc_sw128(sa + kk * 2048, 8192, 1024) : sdesc_sw128(sa + kk * 32, 16, 1024);
                        const uint64_t bd = b_mn ? sdesc_sw128(sb + kk * 2048, 8192, 1024) : sdesc_sw128(sb + kk * 32, 16, 1024);
                        mma_f16_ss2_w(d_tmem, ad, bd, idesc, (kb != kb0) | (kk != 0));
                    }
                    mma_commit2_w(&empty[stage], (uint16_t)3);
                    if (kb == kb1 - 1) mma_commit2_w(&tfull[acc], (uint16_t)3);
                    __syncwarp();
                    if (++stage == GP_STAGES) { stage = 0; phase ^= 1; }
                }
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else {
        // ---------------- epilogue (both CTAs, warps 2..9): this CTA's 128 rows x 256 columns ----------------
        const int q = warp & 3;
        const int row_in_tile = q * 32 + lane_id();
        const int chalf = (warp - 2) / 4;
        // (1024-aligned: the SW128 layout of a [32 rows][32 fp32] box, chunk k of row r at k ^ (r & 7))
        float4 *stg4 = reinterpret_cast<float4 *>(smem + GP_STAGES * GP_STAGE_BYTES + 1024) + (warp - 2) * 256;
        const int lane = lane_id();
        const uint32_t tempty0 = mapa_shared(smem_u32(&tempty[0]), 0);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int item = cl; item < num_items; item += ncl) {
            const int split = item / num_tiles, tile = item - split * num_tiles;
            const int mp = tile / num_n, nt = tile - mp * num_n;
            const int m0 = mp * 2 * GEMM_BM + r * GEMM_BM, n0 = nt * BN;
            float *Cb = p.C + split * p.split_stride;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int m = m0 + row_in_tile;
            float *crow = Cb + (size_t)m * p.ldc;
#pragma unroll 1
            for (int c = chalf * (BN / 2); c < (chalf + 1) * (BN / 2); c += 32) {
                float v[32];
                const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c;
                tmem_ld16(ta, *reinterpret_cast<float(*)[16]>(&v[0]));
                tmem_ld16(ta + 16, *reinterpret_cast<float(*)[16]>(&v[16]));
                const int n = n0 + c;
                float bv[32];
                if (p.bias && n + 32 <= p.N && ((uintptr_t)(p.bias + n) & 15) == 0) {
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        const float4 b4 = __ldg(reinterpret_cast<const float4 *>(p.bias + n + j));
                        bv[j] = b4.x; bv[j + 1] = b4.y; bv[j + 2] = b4.z; bv[j + 3] = b4.w;
                    }
                } else if (p.bias) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) bv[j] = n + j < p.N ? __ldg(p.bias + n + j) : 0.f;
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) bv[j] = 0.f;
                }
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = v[j] * p.alpha + bv[j];
                if (tma_store) {  // the staged [32 x 32] box leaves by one TMA store (bounds clipped by TMA)
                    if (lane == 0) bulk_wait_read<0>();  // the previous box has been read out
                    __syncwarp();
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        stg4[lane * 8 + (k ^ (lane & 7))] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
                    fence_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        asm volatile(
                            "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                reinterpret_cast<uint64_t>(&tmC)),
                            "r"(n), "r"(m0 + 32 * q), "r"(smem_u32(stg4))
                            : "memory");
                        bulk_commit();
                    }
                    continue;
                }
                if ((p.ldc & 3) == 0 && ((uintptr_t)Cb & 15) == 0) {
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        stg4[lane * 8 + (k ^ (lane & 7))] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
                    __syncwarp();
#pragma unroll
                    for (int it = 0; it < 8; ++it) {
                        const int rr = 4 * it + (lane >> 3), k = lane & 7;
                        float4 o = stg4[rr * 8 + (k ^ (rr & 7))];
                        const int mm = m0 + 32 * q + rr, nn = n + 4 * k;
                        if (mm < p.M && nn < p.N) {
                            float *dst = Cb + (size_t)mm * p.ldc + nn;
                            if (nn + 4 <= p.N) {
                                if (p.beta) {
                                    const float4 old = *reinterpret_cast<const float4 *>(dst);
                                    o.x += old.x; o.y += old.y; o.z += old.z; o.w += old.w;
                                }
                                *reinterpret_cast<float4 *>(dst) = o;
                            } else {
                                const float ov[4] = {o.x, o.y, o.z, o.w};
                                for (int e = 0; e < p.N - nn; ++e) dst[e] = p.beta ? dst[e] + ov[e] : ov[e];
                            }
                        }
                    }
                    __syncwarp();
                } else if (m < p.M && n < p.N) {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (n + j < p.N) crow[n + j] = p.beta ? crow[n + j] + v[j] : v[j];
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane_id() == 0) mbar_remote_arrive_release(tempty0 + (uint32_t)acc * 8u);  // the even CTA's tempty[acc]
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    }
    if (tma_store && warp >= 2 && lane_id() == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // no remote arrive / complete_tx / MMA into this CTA is outstanding
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc2(tmem_base, 2 * BN);
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                    const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                    CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_encodeTiled)ptr;
    }
    return fn;
}

// 2-D fp16 tensor map over a row-major [outer, inner] array with row stride ld
// (elements), box {64 inner, box_outer}, 128B swizzle, OOB reads as zero.
int make_tmap_f16(CUtensorMap *map, const void *ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                  uint32_t box_outer) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return -1;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {ld * 2};
    cuuint32_t box[2] = {64, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -2;
}

// 2-D fp32 tensor map over a row-major [outer, inner] array with row stride ld (elements),
// box {32 inner (128 B), box_outer}, 128B swizzle, OOB reads as zero.  Needs ld*4 % 16 == 0 and
// a 16-byte aligned base.
int make_tmap_f32_rows(CUtensorMap *map, const void *ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                       uint32_t box_outer) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return -1;
    if (((uintptr_t)ptr & 15) || ((ld * 4) & 15)) return -3;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {ld * 4};
    cuuint32_t box[2] = {32, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -2;
}

static int g_num_sms = 0;
int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

template <int BN>
static cudaError_t gemm_setup() {
    static bool done[64] = {};  // per device: a function attribute is set per context
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!done[dev]) {
        cudaError_t e = cudaFuncSetAttribute(gemm_f16_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             GemmCfg<BN>::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        cudaFuncAttributes a;
        e = cudaFuncGetAttributes(&a, gemm_f16_kernel<BN>);  // forces the (lazy) module load
        if (e != cudaSuccess) return e;
        done[dev] = true;
    }
    return cudaSuccess;
}
__global__ void splitk_reduce_kernel(const float *__restrict__ part, int S, long stride, int M, int N, float *C,
                                     long ldc, float alpha, int beta, const float *__restrict__ bias, GemmScatter sc);
__global__ void splitk_scatter_kernel(const float *__restrict__ part, int S, long stride, int M, int N, float alpha,
                                      GemmScatter sc);
// the partial last wave's tiles: sum the tail_split (<= 4) partial tiles in split order, then
// alpha, bias and beta as the epilogue would.  TAIL_BLK blocks per tile, every load of a thread
// issued before its first use (a latency-bound loop over 44 blocks cost more than the split saved)
constexpr int TAIL_BLK = 8;
template <int BN>
__global__ void __launch_bounds__(256) gemm_tail_reduce_kernel(GemmParams p, int num_n) {
    const int tt = blockIdx.x / TAIL_BLK, part_i = blockIdx.x - tt * TAIL_BLK;
    const int tile = p.full_items + tt, mt = tile / num_n, nt = tile - mt * num_n;
    const float4 *part = reinterpret_cast<const float4 *>(p.tail_ws + (size_t)tt * p.tail_split * GEMM_BM * BN);
    constexpr int PER = GEMM_BM * BN / 4 / TAIL_BLK / 256;  // float4 per thread
    const long sstride = (long)GEMM_BM * BN / 4;
    float4 acc[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) acc[i] = part[(part_i * PER + i) * 256 + threadIdx.x];
#pragma unroll
    for (int sp = 1; sp < 4; ++sp) {
        if (sp >= p.tail_split) break;
        float4 b[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) b[i] = part[sp * sstride + (part_i * PER + i) * 256 + threadIdx.x];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            acc[i].x += b[i].x; acc[i].y += b[i].y; acc[i].z += b[i].z; acc[i].w += b[i].w;
        }
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e4 = (part_i * PER + i) * 256 + threadIdx.x;
        const int r = (4 * e4) / BN, c = 4 * e4 - r * BN;
        const int m = mt * GEMM_BM + r, n = nt * BN + c;
        if (m >= p.M || n >= p.N) continue;
        float v[4] = {acc[i].x, acc[i].y, acc[i].z, acc[i].w};
        float *dst = p.C + (size_t)m * p.ldc + n;
        if (n + 4 <= p.N && (p.ldc & 3) == 0 && ((uintptr_t)dst & 15) == 0) {
            float4 o;
            o.x = v[0] * p.alpha + (p.bias ? p.bias[n] : 0.f);
            o.y = v[1] * p.alpha + (p.bias ? p.bias[n + 1] : 0.f);
            o.z = v[2] * p.alpha + (p.bias ? p.bias[n + 2] : 0.f);
            o.w = v[3] * p.alpha + (p.bias ? p.bias[n + 3] : 0.f);
            if (p.beta) {
                const float4 old = *reinterpret_cast<const float4 *>(dst);
                o.x += old.x; o.y += old.y; o.z += old.z; o.w += old.w;
            }
            *reinterpret_cast<float4 *>(dst) = o;
        } else {
            for (int j = 0; j < 4 && n + j < p.N; ++j) {
                const float x = v[j] * p.alpha + (p.bias ? p.bias[n + j] : 0.f);
                dst[j] = p.beta ? dst[j] + x : x;
            }
        }
    }
}
long gemm_tail_elems() { return 148L * GEMM_BM * 256; }

int gemm_prepare() {
    cudaFuncAttributes a;
    if (cudaFuncGetAttributes(&a, splitk_reduce_kernel) != cudaSuccess) return -5;
    if (cudaFuncGetAttributes(&a, splitk_scatter_kernel) != cudaSuccess) return -5;
    if (cudaFuncGetAttributes(&a, gemm_f16_pair_kernel) != cudaSuccess) return -5;
    return (gemm_setup<128>() == cudaSuccess && gemm_setup<256>() == cudaSuccess) ? 0 : -5;
}

template <int BN>
static cudaError_t launch_gemm(const CUtensorMap &ta, const CUtensorMap &tb, const CUtensorMap &ta2,
                               const GemmParams &p, int max_ctas, cudaStream_t st) {
    using Cfg = GemmCfg<BN>;
    if (cudaError_t e = gemm_setup<BN>()) return e;
    const int tiles = ((p.M + GEMM_BM - 1) / GEMM_BM) * ((p.N + BN - 1) / BN) * p.ksplit * p.nbatch;
    int grid = tiles < max_ctas ? tiles : max_ctas;
    if (grid < 1) grid = 1;
    ProfScope ps(PROF_GEMM, st, p.M, p.N, p.K);
    note_launch();
    if (!p.pdl && !p.pdl_chain) {
        gemm_f16_kernel<BN><<<grid, GEMM_THREADS, Cfg::SMEM_BYTES, st>>>(ta, tb, ta2, p);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(GEMM_THREADS);
    cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, gemm_f16_kernel<BN>, ta, tb, ta2, p);
}

// split-K reduction: C = alpha * sum_s part[s] (+C) (+bias), in fixed order
// (scatter mode, sc.dst: dst[row_off(m) + col_off(c)] += alpha * sum_s part[s] instead)
__global__ void splitk_reduce_kernel(const float *__restrict__ part, int S, long stride, int M, int N, float *C,
                                     long ldc, float alpha, int beta, const float *__restrict__ bias, GemmScatter sc) {
    const long n = (long)M * N;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const long m = i / N;
        const int c = (int)(i - m * N);
        float acc = 0.f;
        for (int s = 0; s < S; ++s) acc += part[s * stride + i];
        if (sc.dst) {
            const long ro = scat_row(sc, (int)m), co = scat_col(sc, c);
            if (ro >= 0 && co >= 0) sc.dst[ro + co] += acc * alpha;
            continue;
        }
        float v = acc * alpha + (bias ? bias[c] : 0.f);
        float *dst = C + m * ldc + c;
        *dst = beta ? *dst + v : v;
    }
}

// split-K reduction in scatter mode: the destination runs along m (the gate columns of the
// parameter matrices), the partials along n, so the sum is transposed through a 32 x 32 shared tile:
// reads coalesced along n, scatter-adds along m (8 consecutive floats per (unit block, gate))
__global__ void __launch_bounds__(256) splitk_scatter_kernel(const float *__restrict__ part, int S, long stride, int M,
                                                             int N, float alpha, GemmScatter sc) {
    __shared__ float tile[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int tn = (N + 31) / 32, tm = (M + 31) / 32;
    for (int tb = blockIdx.x; tb < tm * tn; tb += gridDim.x) {
        const int m0 = (tb / tn) * 32, n0 = (tb % tn) * 32;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int m = m0 + ty + 8 * k, n = n0 + tx;
            float acc = 0.f;
            if (m < M && n < N)
                for (int s = 0; s < S; ++s) acc += part[s * stride + (long)m * N + n];
            tile[ty + 8 * k][tx] = acc;
        }
        __syncthreads();
        const int m = m0 + tx;
        const long ro = m < M ? scat_row(sc, m) : -1L;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int n = n0 + ty + 8 * k;
            if (ro >= 0 && n < N) {
                const long co = scat_col(sc, n);
                if (co >= 0) sc.dst[ro + co] += tile[tx][ty + 8 * k] * alpha;
            }
        }
        __syncthreads();
    }
}

int gemm_grid(int M, int N, int bn, int max_ctas) {
    const int BN = bn == 128 ? 128 : gemm_bn(N);
    if (max_ctas <= 0) max_ctas = num_sms();
    const int tiles = ((M + GEMM_BM - 1) / GEMM_BM) * ((N + BN - 1) / BN);
    return tiles < max_ctas ? (tiles < 1 ? 1 : tiles) : max_ctas;
}

// the fixed-order reduction of S split-K partials (splitk_ws) into C or the scatter destination
static int splitk_finish(const GemmParams &p, int S, cudaStream_t st) {
    const long n = (long)p.M * p.N;
    long g = (n + 255) / 256;
    if (g > 148 * 8) g = 148 * 8;
    if (p.scat.dst) {
        long tiles32 = (long)((p.M + 31) / 32) * ((p.N + 31) / 32);
        splitk_scatter_kernel<<<(int)(tiles32 < 148 * 8 ? tiles32 : 148 * 8), 256, 0, st>>>(
            p.splitk_ws, S, (long)p.M * p.N, p.M, p.N, p.alpha, p.scat);
    } else {
        splitk_reduce_kernel<<<(int)g, 256, 0, st>>>(p.splitk_ws, S, (long)p.M * p.N, p.M, p.N, p.C, p.ldc, p.alpha,
                                                    p.beta, p.bias, p.scat);
    }
    note_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

// C = alpha * op(A) op(B)^T (+C) (+bias).  Returns 0 / negative error.
int gemm_f16(const GemmOperand &A, const GemmOperand &B, const GemmParams &pin, int max_ctas, cudaStream_t st) {
    GemmParams p = pin;
    p.a_mn = A.mn_major;
    p.b_mn = B.mn_major;
    if (p.M <= 0 || p.N <= 0) return 0;
    if (p.K <= 0) return -3;  // callers never ask for an empty contraction
    const int BN = p.bn == 128 ? 128 : gemm_bn(p.N);
    // two products in one launch (gemm.h a2): partials mode only; batch 1's B lies b_boff rows
    // (K-major: along N, MN-major: along K) after batch 0's, which must be whole tiles / k-blocks so
    // no tile of batch 0 reads batch 1's data in place of the zero fill
    p.nbatch = p.a2 ? 2 : 1;
    if (p.a2 && (p.partials <= 0 || p.b_boff <= 0 || p.c_bstride < (long)p.partials * p.M * p.N ||
                 (B.mn_major ? p.K % GEMM_BK : p.N % BN) || p.b_boff < (B.mn_major ? p.K : p.N)))
        return -3;
    const long bext = p.a2 ? p.b_boff : 0;  // extra extent of B's outer dimension
    if (p.a_kwrap && (A.mn_major || p.a2 || p.K % (p.a_kwrap * GEMM_BK))) return -3;
    const long ka_ext = p.a_kwrap ? (long)p.a_kwrap * GEMM_BK : p.K;  // A's K extent (zero fill beyond ld)
    CUtensorMap ta, tb, ta2;
    int rc;
    if (!A.mn_major) rc = make_tmap_f16(&ta, A.ptr, ka_ext < A.ld ? ka_ext : A.ld, p.M, A.ld, GEMM_BM);
    else rc = make_tmap_f16(&ta, A.ptr, p.M, p.K, A.ld, GEMM_BK);
    if (rc) return rc;
    if (p.a2) {
        if (!A.mn_major) rc = make_tmap_f16(&ta2, p.a2, p.K, p.M, A.ld, GEMM_BM);
        else rc = make_tmap_f16(&ta2, p.a2, p.M, p.K, A.ld, GEMM_BK);
        if (rc) return rc;
    } else {
        ta2 = ta;
    }
    if (!B.mn_major) rc = make_tmap_f16(&tb, B.ptr, p.K, p.N + bext, B.ld, BN);
    else rc = make_tmap_f16(&tb, B.ptr, p.N, p.K + bext, B.ld, GEMM_BK);
    if (rc) return rc;
    if (max_ctas <= 0) max_ctas = num_sms();
    // split K when the output tiles leave at least half of the allowed CTAs idle
    const int tiles = ((p.M + GEMM_BM - 1) / GEMM_BM) * ((p.N + BN - 1) / BN);
    const int num_kb = (p.K + GEMM_BK - 1) / GEMM_BK;
    if (p.partials > 0) {  // fixed split, partials left for the consumer (no reduction launch)
        if (!p.splitk_ws || p.natB || p.flags || p.beta || p.bias || (long)p.partials * p.M * p.N > p.splitk_elems)
            return -3;
        GemmParams q = p;
        q.C = p.splitk_ws; q.ldc = p.N; q.ksplit = p.partials; q.split_stride = (long)p.M * p.N;
        cudaError_t e = BN == 256 ? launch_gemm<256>(ta, tb, ta2, q, max_ctas, st)
                                  : launch_gemm<128>(ta, tb, ta2, q, max_ctas, st);
        return e == cudaSuccess ? 0 : -5;
    }
    // split K when it shortens the launch: the estimate is the waves of (split, tile) work items over
    // the allowed CTAs, each 1/S of a full-K tile, plus the fixed-order reduction's HBM pass over
    // the S partial tiles (e.g. dR^T at C3: 32 tiles on the 52 SMs the recurrence leaves -> S = 3)
    int S = 1;
    if (p.splitk_ws && !p.natB && !p.flags && num_kb >= 32) {
        const double t_tile = 2.0 * GEMM_BM * BN * (double)p.K / 9.0e12;   // one full-K tile on one SM (s)
        const double mn_bytes = 8.0 * (double)p.M * p.N;                    // a partial written + read (fp32)
        double best = (double)((tiles + max_ctas - 1) / max_ctas) * t_tile;
        for (int s = 2; s <= 64; ++s) {  // (few-tile GEMMs over a very long K: the MDLSTM dR, 3 tiles x K = 132k)
            if (num_kb / s < 16 || (long)s * p.M * p.N > p.splitk_elems) break;  // >= 16 k-blocks per split
            const double est = (double)((tiles * s + max_ctas - 1) / max_ctas) * t_tile / s + s * mn_bytes / 5.0e12;
            if (est < 0.97 * best) { best = est; S = s; }
        }
        if (S > 1) S = (num_kb + (num_kb + S - 1) / S - 1) / ((num_kb + S - 1) / S);  // no empty split
    }
    GemmParams q = p;
    if (S > 1) {
        q.C = p.splitk_ws; q.ldc = p.N; q.alpha = 1.f; q.beta = 0; q.bias = nullptr;
        q.ksplit = S; q.split_stride = (long)p.M * p.N;
        q.scat = GemmScatter{};  // the partials are plain; the reduction scatters
    }
    // CTA pairs (gemm_f16_pair_kernel): plain GEMMs with at least a wave of 256 x 256 tiles;
    // BLSTM_GEMM_PAIR=0: off
    // (split-K GEMMs too: their partial tiles are plain rows of splitk_ws, reduced below)
    static const bool pair_env = !(getenv("BLSTM_GEMM_PAIR") && getenv("BLSTM_GEMM_PAIR")[0] == '0');
    if (pair_env && BN == 256 && !p.natB && !p.flags && !p.a2 && (S > 1 || !p.scat.dst) && !p.pdl && !p.pdl_chain &&
        !p.arb && p.partials == 0 && p.a_kwrap == 0 && p.nbatch == 1 && max_ctas >= 2) {
        const int pair_tiles = ((p.M + 2 * GEMM_BM - 1) / (2 * GEMM_BM)) * ((p.N + 255) / 256);
        const int clusters = max_ctas / 2;
        if ((long)pair_tiles * S >= clusters) {
            CUtensorMap tbp;
            int rc2;
            if (!B.mn_major) rc2 = make_tmap_f16(&tbp, B.ptr, p.K, p.N, B.ld, 128);
            else rc2 = make_tmap_f16(&tbp, B.ptr, p.N, p.K, B.ld, GEMM_BK);
            if (rc2) return rc2;
            static bool attr_done[64] = {};  // per device
            int dev = 0;
            cudaGetDevice(&dev);
            if (dev < 0 || dev >= 64) dev = 0;
            if (!attr_done[dev]) {
                if (cudaFuncSetAttribute(gemm_f16_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         GP_SMEM_BYTES) != cudaSuccess)
                    return -5;
                attr_done[dev] = true;
            }
            const int grid = 2 * (pair_tiles < clusters ? pair_tiles : clusters);
            // TMA stores of the output (plain overwrite of a 16-byte-aligned fp32 C; BLSTM_GEMM_TMA_STORE=0: off)
            static const bool tstore_env = !(getenv("BLSTM_GEMM_TMA_STORE") && getenv("BLSTM_GEMM_TMA_STORE")[0] == '0');
            CUtensorMap tmc;
            int tma_store = 0;
            // (not for split-K partials: rows past M of one split are the next split's rows)
            if (tstore_env && S == 1 && !q.beta && make_tmap_f32_rows(&tmc, q.C, q.N, q.M, q.ldc, 32) == 0) tma_store = 1;
            else tmc = tbp;  // (unused)
            const int gridp = 2 * ((long)pair_tiles * S < clusters ? pair_tiles * S : clusters);
            {
                ProfScope ps(PROF_GEMM, st, p.M, p.N, p.K);
                note_launch();
                gemm_f16_pair_kernel<<<gridp, GEMM_THREADS, GP_SMEM_BYTES, st>>>(ta, tbp, tmc, q, tma_store);
                if (cudaGetLastError() != cudaSuccess) return -5;
            }
            (void)grid;
            if (S == 1) return 0;
            return splitk_finish(p, S, st);
        }
    }
    // tail split (gemm.h tail_ws): the r tiles of a partial last wave, each split St ways over K,
    // so the wave's idle SMs take a share (BLSTM_GEMM_TAIL=0: off)
    static const bool tail_env = !(getenv("BLSTM_GEMM_TAIL") && getenv("BLSTM_GEMM_TAIL")[0] == '0');
    q.tail_split = 0;
    if (tail_env && S == 1 && p.tail_ws && !p.natB && !p.flags && !p.a2 && !p.scat.dst && !p.pdl && !p.pdl_chain &&
        !p.arb && p.ksplit <= 1 && tiles > max_ctas) {
        const int r = tiles % max_ctas;
        if (r > 0 && 2 * r <= max_ctas) {
            int St = max_ctas / r < 4 ? max_ctas / r : 4;
            while (St > 1 && num_kb / St < 8) --St;  // >= 8 k-blocks per split
            // worth it when the saved (1 - 1/St) of a tile's time beats the reduction launch (~10 us):
            // a tile of K >= 3072 (C3 dX, ~27 us) yes; the head's K = 1024 / 1536 GEMMs measured no
            if (St > 1 && num_kb >= 48 && (long)r * St * GEMM_BM * BN <= p.tail_elems) {
                q.tail_split = St;
                q.full_items = tiles - r;
            }
        }
    }
    cudaError_t e = BN == 256 ? launch_gemm<256>(ta, tb, ta2, q, max_ctas, st)
                              : launch_gemm<128>(ta, tb, ta2, q, max_ctas, st);
    if (e != cudaSuccess) return -5;
    if (q.tail_split > 1) {
        const int num_n = (p.N + BN - 1) / BN;
        ProfScope ps(PROF_GEMM, st, p.M, p.N, p.K);
        const unsigned nb = (unsigned)(tiles - q.full_items) * TAIL_BLK;
        if (BN == 256) gemm_tail_reduce_kernel<256><<<nb, 256, 0, st>>>(q, num_n);
        else gemm_tail_reduce_kernel<128><<<nb, 256, 0, st>>>(q, num_n);
        note_launch();
        if (cudaGetLastError() != cudaSuccess) return -5;
    }
    if (S > 1) return splitk_finish(p, S, st);
    return 0;
}

}  // namespace blstm
