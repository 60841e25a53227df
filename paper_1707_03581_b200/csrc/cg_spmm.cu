// cg_spmm.cu -- batched Jacobi-PCG with the shared volume operator applied as a TMA-staged
// SpMM: S independent scenarios (BASELINE.json configs[4]) advanced together,
// per-column alpha, beta and convergence masks.  Replaces the gather kernel of cg_batched.cu
// (kept as the fallback for meshes whose numbering fails the window test).
//
// Layout of every block vector (state, z, p, q'): column groups of CW scenarios,
// [G][N][CW] (CW = 16 for S > 16, else CW = SP and G = 1, i.e. the plain row-major N x SP
// block): a run of consecutive rows of one column group is one contiguous range, so a chunk's
// column window is a few bulk copies.  CTA b works on group b % G only.
//
// One persistent cooperative launch per implicit-Euler step, one CTA per SM:
//   * phase 0: r0 = b - K~ x0, z0 = D^{-1} r0, p0 = z0 (b = M_L T^n + dt (b_env + b_G));
//     sums b.b, r.r, r.z per column (+ |Gamma_R| of scenario 0)
//   * per iteration, z-primary as in the single-vector kernel (cg.cu):
//       S: q = K~ p (window of p in shared memory), q' = D^{-1} q stored, and per column the
//          seven sums p.q, sum d z^2, sum z q, sum q q', sum d^2 z^2, sum d z q, sum q^2 that
//          give alpha = r.z / p.q and, with r = D z,
//            r'.z' = sum d z^2 - 2 alpha sum z q + alpha^2 sum q q'
//            r'.r' = sum d^2 z^2 - 2 alpha sum d z q + alpha^2 sum q^2
//          so that beta is known after S's reduction;
//       U: x += alpha p, z -= alpha q', p = z + beta p (one streaming pass, no reduction).
// S streams, per chunk = (one 32-row slice, the CTA's column group): the slice's matrix values
// and 16-bit window-local columns (k_chunk_windows with W = 1), the window of p -- at most 32
// runs of rows -- and the slice's own rows of z, D^{-1} and interface indices through a
// cp.async.bulk + mbarrier ring filled by one producer warp; eight consumer warps take 4 rows
// each (a half-warp per row, lane & 15 = scenario column: every entry one broadcast value and
// one 128-byte window row), read everything a row needs from the stage, release it, and only
// then do the global work (q' stores, interface rows).  Interface rows (per scenario) add their entries with
// per-lane gathers.  The Jacobi diagonal: d = the row's entry 0 (the volume diagonal) with
// 1/d = Dinv, except interface rows, whose per-scenario d and 1/d the interface kernels write
// (k_rows: if_d, if_dinv).
//
// Reductions are deterministic: per-lane sums in row order, CTA partials summed over warps in a
// fixed order, then each (value, column) total summed over the CTAs by one warp of one CTA in a
// fixed order (distributed: 7 x 64 totals over 148 CTAs), a grid barrier, and every CTA reads the
// same totals.  Converged columns are frozen (alpha = 0).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ctx.h"

namespace cg = cooperative_groups;

namespace thermo {

#define CK(x)                                                                    \
    do {                                                                         \
        cudaError_t e_ = (x);                                                    \
        if (e_ != cudaSuccess) {                                                 \
            c.err = std::string("CUDA: ") + cudaGetErrorString(e_) + " at " #x; \
            return -3;                                                           \
        }                                                                        \
    } while (0)

#define SB_NCW 8                        // consumer warps
#define SB_RPW (32 / SB_NCW)            // rows of a slice per consumer warp (two per half-warp pass)
#ifndef SB_NPW
#define SB_NPW 1   // producer warps (chunks k = p mod SB_NPW; ring slots likewise).  2 producers measured no
                   // faster (the consumers bound the sweep) and runs were not bitwise reproducible
#endif
#define SB_NIW 2                        // interface warps (gather the interface rows during the sweep)
#define SB_THREADS ((SB_NCW + SB_NPW + SB_NIW) * 32)
#define SB_NV 7                         // reduction values per column (S phase)
#define SB_MAXS 64
#define SB_M (SB_NV * SB_MAXS)          // partial slots per CTA
#define SB_HDR 128
#define SB_MAXSTAGES 6
#define SB_GAP 8                        // column-window gaps up to 8 rows are bridged
#define SB_CW 16                        // scenario columns per group (S > 16)

struct SBParams {
    int64_t N, nslices;
    int S, SP, CW, G;
    int Gw;                        // CTAs working in the sweeps: (grid / G) * G; CTA b -> group b % G
    const int64_t *slice_ptr;
    const uint16_t *lcol;          // window-local columns, row-major per slice (sbcg_prepare)
    const double *val;             // K~_vol values, row-major per slice: [32 rows][w8] (w8 = width
                                   // rounded up to 8, padding: value 0, column = the row itself)
    const struct SBRec *recs;      // per CTA, in sweep order: the chunk metadata (host-packed)
    const int32_t *rec_ptr;        // [Gw + 1]
    const double *ML, *benv, *Dinv;
    const int32_t *if_of_row;      // [nslices * 32] interface index of a row, -1 if none
    const int32_t *if_rows;        // [n_if] row of each interface node
    const int32_t *if_cta_ptr, *if_cta_k;   // [Gw + 1] / list: interface rows in the slices of CTA b
    double *ai;                    // [list][SB_CW] interface sums of the current sweep
    int n_if, nA, cap;
    const int32_t *ell_cnt, *ell_col;
    const double *ell_val, *if_b, *if_phi, *if_d, *if_dinv;   // [k][c][s] / [k][s]
    const double *T_in, *X0;
    double *T_out, *z, *p, *q;
    double *partials;              // [grid][SB_M]
    double *totals;                // [2][SB_M]
    int *status;
    double *fail_relres;
    int32_t *iters_out;
    double *relres_out, *area_out;
    double dt, rtol2;
    int maxit, step;
    int nstages;
    uint32_t stage_bytes, col_off, win_off, own_off, aux_off;
    uint32_t meta_off;             // metadata batch buffers (after the ring and the reduction scratch)
    unsigned long long *trace;
    int trace_fine;   // THERMO_CG_TRACE=3: stamps after the sweep, the interface pass, the CTA
                      // partials and the first grid barrier of every reduction (CTA 0)
    int debug;   // THERMO_CGB_DEBUG bits (measurement only, results invalid): 1 consumers skip the
                 // row sums, 2 no window copies, 4 no epilogue (post), 8 no copies at all; (results
                 // valid:) 16 no interface gathers during the sweep; with -DSB_STAGE_CHECKS: 64
                 // consumers check the values they kept for their own rows against global memory
                 // (sb_check_light), 128 every value of every stage (sb_check), mismatches printed
    int *dbg;    // [4] mismatch counter of sb_check
};

__device__ __forceinline__ int64_t brow(const SBParams &P, int g, int64_t i) {   // first element of row i, group g
    return ((int64_t)g * P.N + i) * P.CW;
}

struct SBRing {
    uint64_t *full, *empty;
    unsigned char *stage;
    uint32_t n;
    uint64_t *mbar;     // [2] metadata batch buffers
    SBRec *meta;        // [2][SB_RB]
    uint32_t mph;       // phase bits of mbar[0..1]
    int *ictr;          // interface units claimed in this sweep (sb_iface_gather)
};

// Metadata of one chunk (one slice of the CTA's column group), packed on the host per CTA in
// sweep order and streamed into shared memory in batches of SB_RB by the producer (one bulk copy
// per batch): no global round trip per chunk on the producer's critical path.
#define SB_MAXR 16   // window runs per chunk in the packed record
#define SB_RB 32     // records per batch
struct SBRec {
    long long e0;     // first matrix entry of the slice
    int cnt, lown, nruns, s;
    int2 run[SB_MAXR];
    int pad[2];
};
static_assert(sizeof(SBRec) == 160, "SBRec layout");

// Per-row operands of the consumer epilogue, read from the stage before it is released.
struct SBRow {
    double acc, pw, own, dinv, diag;
    int ik;
    int64_t i;
};

// Interface rows of this CTA's slices (its own column group), in two parts:
//  * gather (the SB_NIW interface warps, during the sweep): ai = sum_e val_e w[col_e] of every
//    (interface row, column), two rows in flight per half-warp, every load of a round issued
//    before the next dependent round (count; entries; gathers) -> P.ai;
//  * finish (all warps, after the sweep): body(k, i, g, l, ai) adds the volume part the sweep
//    stored for the row and completes it.
__device__ __forceinline__ void sb_iface_gather(const SBParams &P, const double *w, int *ctr) {
    // units (interface rows of the CTA's list) are claimed four at a time per warp from a
    // shared counter: the interface warps start during the sweep, every warp helps after it.
    // Each unit's sum has a fixed order (the entries'), so the values are reproducible; only
    // which warp computes them varies.
    const int lane = threadIdx.x & 31, h = lane >> 4, l = lane & 15;
    const int g = blockIdx.x % P.G;
    const int j0 = P.if_cta_ptr[blockIdx.x], j1 = P.if_cta_ptr[blockIdx.x + 1];
    const int sc = g * P.CW + l;
    const bool col = l < P.CW && sc < P.S;
    while (true) {   // warp-uniform: the warp claims four units, two per half-warp
        int jb = 0;
        if (lane == 0) jb = j0 + atomicAdd(ctr, 4);
        jb = __shfl_sync(0xffffffffu, jb, 0);
        if (jb >= j1) break;
        const int j = jb + 2 * h;
        int k[2], cnt[2];
        double a[2] = {0.0, 0.0};
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            k[u] = j + u < j1 ? P.if_cta_k[j + u] : -1;
            cnt[u] = (k[u] >= 0 && col) ? P.ell_cnt[(int64_t)k[u] * P.S + sc] : 0;
        }
        const int cmax = max(cnt[0], cnt[1]);
        for (int c0 = 0; c0 < cmax; c0 += 8) {
            int jc[2][8];
            double v[2][8], y[2][8];
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int ce = min(c0 + e, max(cnt[u] - 1, 0));
                    const int64_t ix = ((int64_t)max(k[u], 0) * P.cap + ce) * P.S + (col ? sc : 0);
                    jc[u][e] = cnt[u] ? P.ell_col[ix] : 0;
                    v[u][e] = cnt[u] ? P.ell_val[ix] : 0.0;
                }
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int e = 0; e < 8; ++e) y[u][e] = cnt[u] ? ld_cg1(w + brow(P, g, jc[u][e]) + l) : 0.0;
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    if (c0 + e < cnt[u]) a[u] = fma(v[u][e], y[u][e], a[u]);
        }
        if (l < P.CW) {
#pragma unroll
            for (int u = 0; u < 2; ++u)
                if (k[u] >= 0) P.ai[(int64_t)(j + u) * SB_CW + l] = a[u];
        }
    }
}

#ifdef SB_STAGE_CHECKS   // compiled in for diagnosis only: the checks change the consumers' code
// Debug (THERMO_CGB_DEBUG bit 128): compare what a consumer warp reads from a stage with the
// global memory the producer copied it from -- matrix values and columns (constant), the window
// rows of w, the own rows of ownv, D^{-1} -- and print the first mismatches.
__device__ __noinline__ void sb_check(const SBParams &P, uint32_t k, const unsigned char *sb, const double *w,
                                      const double *ownv, int64_t s, int wd, int g) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, h = lane >> 4, l = lane & 15;
    const SBRec &rec = P.recs[P.rec_ptr[blockIdx.x] + k];
    const double *vals = reinterpret_cast<const double *>(sb + SB_HDR);
    const uint16_t *lc = reinterpret_cast<const uint16_t *>(sb + P.col_off);
    const double *win = reinterpret_cast<const double *>(sb + P.win_off);
    const double *own = reinterpret_cast<const double *>(sb + P.own_off);
    const double *dv = reinterpret_cast<const double *>(sb + P.aux_off);
    auto report = [&](int kind, int r, int e, int cidx, int64_t grow, double a, double b) {
        const int c = atomicAdd(P.dbg, 1);
        if (c < 16)
            printf("[sbchk] kind %d step %d cta %d chunk %u slice %lld (rec %d) row %d e %d cidx %d grow %lld l %d "
                   "stage %.17g global %.17g\n", kind, P.step, (int)blockIdx.x, k, (long long)s, rec.s, r, e, cidx,
                   (long long)grow, l, a, b);
    };
    if (rec.s != s) report(0, -1, -1, -1, -1, 0.0, 0.0);
    for (int pp = 0; pp < SB_RPW / 2; ++pp) {
        const int r = warp * SB_RPW + 2 * pp + h;
        const int64_t i = 32 * s + r;
        if (i >= P.N || l >= P.CW) continue;
        for (int kk = 0; kk < wd; ++kk) {
            const int e = r * wd + kk;
            const double gv = P.val[rec.e0 + e];
            if (__double_as_longlong(vals[e]) != __double_as_longlong(gv)) report(1, r, e, -1, -1, vals[e], gv);
            const int cidx = lc[e];
            if (cidx != P.lcol[rec.e0 + e]) report(2, r, e, cidx, -1, cidx, P.lcol[rec.e0 + e]);
            int off = 0;
            int64_t grow = -1;
            for (int q = 0; q < rec.nruns; ++q) {
                if (cidx < off + rec.run[q].y) { grow = rec.run[q].x + cidx - off; break; }
                off += rec.run[q].y;
            }
            if (grow < 0) { report(3, r, e, cidx, grow, 0.0, 0.0); continue; }
            const double a = win[cidx * P.CW + l], b = ld_cg1(w + brow(P, g, grow) + l);
            if (__double_as_longlong(a) != __double_as_longlong(b)) report(4, r, e, cidx, grow, a, b);
        }
        const double a = own[r * P.CW + l], b = ld_cg1(ownv + brow(P, g, i) + l);
        if (__double_as_longlong(a) != __double_as_longlong(b)) report(5, r, -1, -1, i, a, b);
        if (__double_as_longlong(dv[r]) != __double_as_longlong(P.Dinv[i])) report(6, r, -1, -1, i, dv[r], P.Dinv[i]);
    }
}

// Debug (bit 64, cheap, after the release): the values a consumer kept from the stage for its
// own rows (p of the row from the window, ownv, D^{-1}, the diagonal) against global memory.
__device__ __noinline__ void sb_check_light(const SBParams &P, uint32_t k, const double *w, const double *ownv,
                                            int64_t s, int wd, int g, int r, double pw, double ow, double dinv,
                                            double diag) {
    const int l = threadIdx.x & 15;
    const int64_t i = 32 * s + r;
    const SBRec &rec = P.recs[P.rec_ptr[blockIdx.x] + k];
    const double v[4] = {ld_cg1(w + brow(P, g, i) + l), ld_cg1(ownv + brow(P, g, i) + l), P.Dinv[i],
                         P.val[rec.e0 + r * wd]};
    const double u[4] = {pw, ow, dinv, diag};
    for (int q = 0; q < 4; ++q)
        if (__double_as_longlong(u[q]) != __double_as_longlong(v[q])) {
            const int c = atomicAdd(P.dbg, 1);
            if (c < 16)
                printf("[sbchk-light] kind %d step %d cta %d chunk %u slice %lld row %d l %d stage %.17g global %.17g\n",
                       q, P.step, (int)blockIdx.x, k, (long long)s, r, l, u[q], v[q]);
        }
}

#endif

// One sweep over the slices of this CTA's column group g = b % G (slices b / G + k Gw / G,
// a static order).  Stage = [hdr | values | 16-bit window columns | window of w (runs) | own
// rows of ownv | D^{-1} of the slice's rows | interface index of the slice's rows].  Consumers
// (half-warp per row, lane & 15 = column) form acc = (K~_vol w)_i from shared memory, read the
// rest of the row's operands, release the stage and then call post(row) (global stores and the
// interface rows' gathers run while the producer refills the ring).
template <class Post>
__device__ __forceinline__ void sb_sweep(const SBParams &P, SBRing &R, const double *w, const double *ownv,
                                         Post &&post) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t NS = (uint32_t)P.nstages;
    if ((int)blockIdx.x >= P.Gw) return;
    const int g = blockIdx.x % P.G;
    const uint32_t base = R.n;   // ring slot of this sweep's chunk 0 (the same in every warp)
    if (warp >= SB_NCW + SB_NPW) {   // ---------------- interface warps
        if (P.n_if && !(P.debug & 16)) sb_iface_gather(P, w, R.ictr);
        R.n = base + (uint32_t)(P.rec_ptr[SB_NPW * blockIdx.x + SB_NPW] - P.rec_ptr[SB_NPW * blockIdx.x]) + 1u;
        return;
    }
    if (warp >= SB_NCW) {   // ---------------- producers: warp SB_NCW + p takes chunks k = p (mod 2)
        const int pw = warp - SB_NCW;
        const int r0i = P.rec_ptr[SB_NPW * blockIdx.x + pw], r1i = P.rec_ptr[SB_NPW * blockIdx.x + pw + 1];
        const SBRec *recs = P.recs + r0i;
        const int nmine = r1i - r0i;
        const int nrec = P.rec_ptr[SB_NPW * blockIdx.x + SB_NPW] - P.rec_ptr[SB_NPW * blockIdx.x];   // chunks of the CTA
        SBRec *meta = R.meta + pw * 2 * SB_RB;
        uint64_t *mbar = R.mbar + 2 * pw;
        auto fetch = [&](int bt) {   // batch bt of this producer's records -> buffer bt & 1
            const int n = min(SB_RB, nmine - bt * SB_RB);
            if (n <= 0 || lane != 0) return;
            uint64_t *mb = &mbar[bt & 1];
            fence_proxy_async_smem();   // earlier generic reads of the buffer before the async write
            mbar_arrive_expect_tx(mb, (uint32_t)n * (uint32_t)sizeof(SBRec));
            bulk_g2s_nohint(meta + (bt & 1) * SB_RB, recs + bt * SB_RB, (uint32_t)n * (uint32_t)sizeof(SBRec), mb);
        };
        // issuer side of the cross-proxy ordering: the vectors this sweep streams by TMA were
        // written by plain stores before the last grid barrier
        fence_proxy_async_global();
        fetch(0);
        fetch(1);
        for (int j = 0;; ++j) {
            const int k = pw + SB_NPW * j;   // CTA-local chunk index
            if (k > nrec) break;
            const uint32_t n = base + (uint32_t)k;
            const uint32_t st = n % NS, ph = (n / NS) & 1u;
            unsigned char *sb = R.stage + (size_t)st * P.stage_bytes;
            int *hdr = reinterpret_cast<int *>(sb);
            if (k == nrec) {   // end marker
                if (lane == 0) {
                    mbar_wait(&R.empty[st], ph ^ 1u);
                    hdr[31] = -1;
                    mbar_arrive(&R.full[st]);
                }
                __syncwarp();
                break;
            }
            const int bt = j / SB_RB, bb = bt & 1;
            if (j % SB_RB == 0) {
                mbar_wait(&mbar[bb], (R.mph >> (2 * pw + bb)) & 1u);
                R.mph ^= 1u << (2 * pw + bb);
            }
            const SBRec &mm = meta[bb * SB_RB + j % SB_RB];
            const long long e0 = mm.e0;
            const int cntr = mm.cnt, lown = mm.lown, nruns = mm.nruns, s = mm.s;
            const int2 run = lane < SB_MAXR ? mm.run[lane] : make_int2(0, 0);
            if (j % SB_RB == SB_RB - 1) {   // batch done (read into registers): refill its buffer
                __syncwarp();
                fetch(bt + 2);
            }
            const int len = lane < nruns ? run.y : 0;
            int x = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            const int woff = x - len, wtot = (P.debug & 2) ? 0 : __shfl_sync(0xffffffffu, x, 31);
            const uint32_t cnt = (uint32_t)cntr;
            const int64_t r0 = 32 * (int64_t)s;
            const uint32_t rows = (uint32_t)(((min((int64_t)32, P.N - r0)) + 1) & ~(int64_t)1);   // even: 16-B copies
            const uint32_t ownb = rows * (uint32_t)P.CW * 8u;
            if (lane == 0 && (P.debug & 8)) {   // measurement: no copies at all
                mbar_wait(&R.empty[st], ph ^ 1u);
                hdr[0] = (int)(cnt >> 5);
                hdr[1] = lown;
                hdr[31] = s;
                mbar_arrive(&R.full[st]);
            } else if (lane == 0) {
                mbar_wait(&R.empty[st], ph ^ 1u);
#ifndef SB_EXPERIMENT_EARLY_RELEASE
                // generic-proxy reads of this stage by the consumers (released through the empty
                // barrier) before the async-proxy writes into it (PTX: a proxy fence between them)
                fence_proxy_async_smem();
#endif
                hdr[0] = (int)(cnt >> 5);
                hdr[1] = lown;
                hdr[31] = s;
                mbar_arrive_expect_tx(&R.full[st],
                                      cnt * 10u + (uint32_t)wtot * (uint32_t)P.CW * 8u + ownb + rows * 8u + 128u);
                bulk_g2s_nohint(sb + SB_HDR, P.val + e0, cnt * 8u, &R.full[st]);
                bulk_g2s_nohint(sb + P.col_off, P.lcol + e0, cnt * 2u, &R.full[st]);
                bulk_g2s_nohint(sb + P.own_off, ownv + brow(P, g, r0), ownb, &R.full[st]);
                bulk_g2s_nohint(sb + P.aux_off, P.Dinv + r0, rows * 8u, &R.full[st]);
                bulk_g2s_nohint(sb + P.aux_off + 256, P.if_of_row + r0, 128u, &R.full[st]);
            }
            __syncwarp();
#ifndef SB_EXPERIMENT_EARLY_RELEASE
            if (len) fence_proxy_async_smem();   // the same for the lanes copying the window
#endif
            if (len && !(P.debug & 10))
                bulk_g2s_nohint(sb + P.win_off + (size_t)woff * P.CW * 8, w + brow(P, g, run.x),
                                (uint32_t)len * (uint32_t)P.CW * 8u, &R.full[st]);
            __syncwarp();
        }
        R.n = base + (uint32_t)nrec + 1u;
        return;
    }
    // ---------------- consumers: rows warp * SB_RPW + [0, SB_RPW) of each slice, a half-warp
    // per row (lanes 0-15 the even, 16-31 the odd row of a pair), lane & 15 = column
    const int h = lane >> 4, l = lane & 15;
    const bool lok = l < P.CW;
    while (true) {
        const uint32_t st = R.n % NS, ph = (R.n / NS) & 1u;
        mbar_wait(&R.full[st], ph);
        const unsigned char *sb = R.stage + (size_t)st * P.stage_bytes;
        const int *hdr = reinterpret_cast<const int *>(sb);
        const int64_t s = hdr[31];
        if (s < 0) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&R.empty[st]);
            ++R.n;
            break;
        }
        const int wd = hdr[0], lown = hdr[1];
        const double *vals = reinterpret_cast<const double *>(sb + SB_HDR);
        const uint16_t *lc = reinterpret_cast<const uint16_t *>(sb + P.col_off);
        const double *win = reinterpret_cast<const double *>(sb + P.win_off);
        const double *own = reinterpret_cast<const double *>(sb + P.own_off);
        const double *dv = reinterpret_cast<const double *>(sb + P.aux_off);
        const int *ifr = reinterpret_cast<const int *>(sb + P.aux_off + 256);
        SBRow rw[SB_RPW / 2];
        // both rows of this half-warp (two independent accumulation chains), entries in blocks of
        // 8 with every shared-memory load of a block issued before its FMAs; entries past the
        // row width read the row's own window slot with weight 0 (no tail loop)
        int rr_[SB_RPW / 2];
        bool ok_[SB_RPW / 2];
#pragma unroll
        for (int pp = 0; pp < SB_RPW / 2; ++pp) {
            rr_[pp] = warp * SB_RPW + 2 * pp + h;
            SBRow &x = rw[pp];
            x.i = 32 * s + rr_[pp];
            x.acc = x.pw = x.own = x.diag = 0.0;
            x.dinv = 1.0;
            x.ik = -1;
            ok_[pp] = x.i < P.N && lok && !(P.debug & 1);
        }
        if (ok_[0] || ok_[1]) {
            // wd = row width rounded to 8 (row-major slice): per block of 8 entries one 16-byte
            // broadcast load of the columns and four of the values per row
            for (int k = 0; k < wd; k += 8) {
                uint4 cq[SB_RPW / 2];
                double2 vq[SB_RPW / 2][4];
                double yy[SB_RPW / 2][8];
#pragma unroll
                for (int pp = 0; pp < SB_RPW / 2; ++pp) {
                    const int e = rr_[pp] * wd + k;
                    cq[pp] = *reinterpret_cast<const uint4 *>(lc + e);
#pragma unroll
                    for (int u = 0; u < 4; ++u) vq[pp][u] = reinterpret_cast<const double2 *>(vals + e)[u];
                }
#pragma unroll
                for (int pp = 0; pp < SB_RPW / 2; ++pp) {
                    const uint32_t w4[4] = {cq[pp].x, cq[pp].y, cq[pp].z, cq[pp].w};
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int cidx = (int)((w4[u >> 1] >> (16 * (u & 1))) & 0xffffu);
                        yy[pp][u] = win[cidx * P.CW + l];
                    }
                }
#pragma unroll
                for (int pp = 0; pp < SB_RPW / 2; ++pp)
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        rw[pp].acc = fma(vq[pp][u].x, yy[pp][2 * u], rw[pp].acc);
                        rw[pp].acc = fma(vq[pp][u].y, yy[pp][2 * u + 1], rw[pp].acc);
                    }
            }
        }
#pragma unroll
        for (int pp = 0; pp < SB_RPW / 2; ++pp) {
            SBRow &x = rw[pp];
            const int r = rr_[pp];
            if (ok_[pp]) {
                x.pw = win[(lown + r) * P.CW + l];
                x.own = own[r * P.CW + l];
                x.dinv = dv[r];
                x.diag = vals[r * wd];   // entry 0 of the row: the diagonal
                x.ik = ifr[r];
            }
        }
#ifdef SB_STAGE_CHECKS
        if (P.debug & 128) sb_check(P, R.n - base, sb, w, ownv, s, wd, g);
        if (P.debug & 64)
#pragma unroll
            for (int pp = 0; pp < SB_RPW / 2; ++pp)
                if (ok_[pp])
                    sb_check_light(P, R.n - base, w, ownv, s, wd, g, rr_[pp], rw[pp].pw, rw[pp].own, rw[pp].dinv,
                                   rw[pp].diag);
#endif
#ifdef SB_EXPERIMENT_EARLY_RELEASE   // the round-2 order (measurement of the race only)
        __syncwarp();
        if (lane == 0) mbar_arrive(&R.empty[st]);
#endif
        // the epilogue (global stores) consumes every value read from the stage; only then is
        // the stage released.  Released right after the loads, the producer's next bulk copy into
        // the stage could overtake a still outstanding shared-memory load (the arrive does not
        // wait for them): about one cfg-4 run in three had one stale row somewhere
        // (tools/diag_spmm_race.py; located with the SB_STAGE_CHECKS build)
#pragma unroll
        for (int pp = 0; pp < SB_RPW / 2; ++pp)
            if (rw[pp].i < P.N && lok && !(P.debug & 5)) post(rw[pp], g, l);
#ifndef SB_EXPERIMENT_EARLY_RELEASE
        __syncwarp();
        if (lane == 0) mbar_arrive(&R.empty[st]);   // the stage is free again
#endif
        ++R.n;
    }
}

template <class Body>
__device__ __forceinline__ void sb_iface_finish(const SBParams &P, const double *w, int *ctr, Body &&body) {
    if ((int)blockIdx.x >= P.Gw || !P.n_if) return;
    sb_iface_gather(P, w, ctr);   // the units the interface warps have not claimed yet
    __syncthreads();   // the sweep's volume parts and the gathered interface sums are visible
    if (threadIdx.x == 0) *ctr = 0;   // for the next sweep (after the reduction's barriers)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int h = lane >> 4, l = lane & 15;
    if (l >= P.CW) return;
    const int g = blockIdx.x % P.G;
    const int j0 = P.if_cta_ptr[blockIdx.x], j1 = P.if_cta_ptr[blockIdx.x + 1];
    const int nhw = 2 * (blockDim.x >> 5), hw = 2 * warp + h;
    for (int j = j0 + hw; j < j1; j += nhw) {
        const int k = P.if_cta_k[j];
        body(k, (int64_t)P.if_rows[k], g, l, ld_cg1(P.ai + (int64_t)j * SB_CW + l));
    }
}

// CTA sums of NV values per column (lane (h, l) of every warp holds column g * CW + l of its
// CTA's group in acc[v]; both halves) -> partials[cta][v * 64 + column]; grid barrier; the total
// of every (v, column) by one warp, over the CTAs of the column's group in a fixed order
// (distributed over the grid); grid barrier; totals -> tot (every CTA the same bits).
// THERMO_CG_TRACE=3: extra %globaltimer stamps inside an iteration (CTA 0, thread 0)
__device__ __forceinline__ void sb_stamp(const SBParams &P, int &ntr) {
    if (P.trace_fine && blockIdx.x == 0 && threadIdx.x == 0 && ntr < 1000) P.trace[ntr++] = gtimer();
}

template <int NV>
__device__ __forceinline__ void sb_reduce(const SBParams &P, const double (&acc)[NV], double *red, double *tot,
                                          double *totals, cg::grid_group &grid, int &ntr) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int M = NV * SB_MAXS;
    __syncthreads();   // the ring is idle: red aliases its stages
    const int nwb = blockDim.x >> 5;   // every warp: the consumers' rows and the interface rows
#pragma unroll
    for (int v = 0; v < NV; ++v) red[(warp * NV + v) * 32 + lane] = acc[v];
    __syncthreads();
    if ((int)blockIdx.x < P.Gw) {
        const int g = blockIdx.x % P.G;
        for (int j = threadIdx.x; j < NV * P.CW; j += blockDim.x) {
            const int v = j / P.CW, l = j - v * P.CW;
            double x = 0.0;
            for (int w = 0; w < nwb; ++w) x += red[(w * NV + v) * 32 + l] + red[(w * NV + v) * 32 + 16 + l];
            P.partials[(int64_t)blockIdx.x * SB_M + v * SB_MAXS + g * P.CW + l] = x;
        }
    }
    sb_stamp(P, ntr);
    fence_proxy_async_global();   // plain stores before the next TMA reads
    grid.sync();
    sb_stamp(P, ntr);
    const int nw = blockDim.x >> 5, Gc = gridDim.x;
    for (int j = blockIdx.x + Gc * warp; j < M; j += Gc * nw) {
        const int v = j / SB_MAXS, col = j - v * SB_MAXS;
        double x = 0.0;
        if (col < P.SP) {
            const int gg = col / P.CW;
            for (int b = gg + P.G * lane; b < P.Gw; b += 32 * P.G) x += ld_cg1(P.partials + (int64_t)b * SB_M + v * SB_MAXS + col);   // L2: written by other CTAs this launch
        }
        x = warp_sum(x);
        if (lane == 0) totals[j] = x;
    }
    fence_proxy_async_global();   // plain stores before the next TMA reads
    grid.sync();
    for (int j = threadIdx.x; j < M; j += blockDim.x) tot[j] = ld_cg1(totals + j);
    fence_proxy_async_smem();   // red (generic proxy) before the next sweep's bulk copies into the ring
    __syncthreads();
}

// 12 warps: <= 168 registers (3 warps on each SM sub-partition)
__global__ void __launch_bounds__(SB_THREADS, 1) k_sbcg_step(SBParams P) {
    extern __shared__ __align__(128) unsigned char sb_smem[];
    __shared__ uint64_t bar_full[SB_MAXSTAGES], bar_empty[SB_MAXSTAGES], bar_meta[2 * SB_NPW];
    __shared__ double s_tot[SB_M];
    __shared__ double s_alpha[SB_MAXS], s_beta[SB_MAXS], s_rho[SB_MAXS], s_rr[SB_MAXS], s_tol2[SB_MAXS],
        s_bb[SB_MAXS];
    __shared__ int s_conv[SB_MAXS], s_itc[SB_MAXS], s_any, s_ictr;
    // an earlier step failed, or the interface of this or an earlier step overflowed
    if (P.status[0] || (P.status[1] && P.status[4] <= P.step)) {
        if (!P.status[0] && blockIdx.x == 0 && threadIdx.x == 0) {
            P.status[0] = 2;
            P.status[2] = P.step;
        }
        return;
    }
    cg::grid_group grid = cg::this_grid();
    if (threadIdx.x == 0) {
        for (int k = 0; k < P.nstages; ++k) {
            mbar_init(&bar_full[k], 1);
            mbar_init(&bar_empty[k], SB_NCW);
        }
        for (int k = 0; k < 2 * SB_NPW; ++k) mbar_init(&bar_meta[k], 1);
        s_ictr = 0;
        fence_mbar_init();
    }
    __syncthreads();
    SBRing R{bar_full, bar_empty, sb_smem, 0u, bar_meta,
             reinterpret_cast<SBRec *>(sb_smem + P.meta_off), 0u, &s_ictr};
    double *red = reinterpret_cast<double *>(sb_smem);   // aliases the ring between sweeps
    const bool tr_on = P.trace && blockIdx.x == 0 && threadIdx.x == 0;
    int ntr = 0;
    if (tr_on) P.trace[ntr++] = gtimer();
    const double *const x0 = P.X0 ? P.X0 : P.T_in;
    const int64_t NU = (int64_t)P.G * P.N;   // rows of all column groups (U phase units)

    // ---- phase 0: r0 = b - K~ x0, z0 = D^{-1} r0, p0 = z0 (own rows: T^n)
    {
        double acc[4] = {0, 0, 0, 0};   // b.b, r.r, r.z, |Gamma_R| (scenario 0)
        // b, r, z of a row from its full (K~ x0)_i
        auto fin0 = [&](int64_t i, int g, int l, double ax, double Ti, double bg, double dinv) {
            const int sc = g * P.CW + l;
            const double b = fma(P.ML[i], Ti, P.dt * (P.benv[i] + bg));
            const double r = b - ax;
            const double zz = sc < P.S ? dinv * r : 0.0;
            P.z[brow(P, g, i) + l] = zz;
            P.p[brow(P, g, i) + l] = zz;
            if (sc < P.S) {
                acc[0] = fma(b, b, acc[0]);
                acc[1] = fma(r, r, acc[1]);
                acc[2] = fma(r, zz, acc[2]);
            }
        };
        sb_sweep(P, R, x0, P.T_in, [&](const SBRow &x, int g, int l) {
            if (x.ik >= 0) P.z[brow(P, g, x.i) + l] = x.acc;   // volume part; finished by the interface pass
            else fin0(x.i, g, l, x.acc, x.own, 0.0, x.dinv);
        });
        sb_iface_finish(P, x0, &s_ictr, [&](int k, int64_t i, int g, int l, double ai) {
            const int sc = g * P.CW + l;
            const int64_t e = brow(P, g, i) + l;
            const double ax = ld_cg1(P.z + e) + ai, Ti = ld_cg1(P.T_in + e);
            double bg = 0.0, dinv = P.Dinv[i];
            if (sc < P.S) {
                bg = P.if_b[(int64_t)k * P.S + sc];
                dinv = P.if_dinv[(int64_t)k * P.S + sc];
            }
            if (sc == 0 && k < P.nA) acc[3] += P.if_phi[(int64_t)k * P.S];
            fin0(i, g, l, ax, Ti, bg, dinv);
        });
        sb_reduce<4>(P, acc, red, s_tot, P.totals, grid, ntr);
    }
    if (tr_on) P.trace[ntr++] = gtimer();
    const double area = s_tot[3 * SB_MAXS + 0];
    if (threadIdx.x < SB_MAXS) {
        const int c = threadIdx.x;
        const double bb = s_tot[0 * SB_MAXS + c], rr = s_tot[1 * SB_MAXS + c];
        s_bb[c] = bb;
        s_tol2[c] = P.rtol2 * bb;
        s_rho[c] = s_tot[2 * SB_MAXS + c];
        s_rr[c] = rr;
        s_conv[c] = c >= P.S || rr <= P.rtol2 * bb;
        s_itc[c] = 0;
    }
    __syncthreads();
    const double *xsrc = x0;
    int it = 0;
    while (it < P.maxit) {
        if (threadIdx.x == 0) {
            int any = 0;
            for (int c = 0; c < P.S; ++c) any |= !s_conv[c];
            s_any = any;
        }
        __syncthreads();
        if (!s_any) break;
        // ---- S: q = K~ p, q' = D^{-1} q, seven sums per column (own rows: z)
        {
            double acc[SB_NV] = {0, 0, 0, 0, 0, 0, 0};
            auto finS = [&](int64_t i, int g, int l, double qv, double pi, double zz, double d, double dinv) {
                const int sc = g * P.CW + l;
                const double qp = dinv * qv;
                P.q[brow(P, g, i) + l] = qp;
                if (sc < P.S) {
                    const double dz = d * zz;
                    acc[0] = fma(pi, qv, acc[0]);
                    acc[1] = fma(dz, zz, acc[1]);
                    acc[2] = fma(zz, qv, acc[2]);
                    acc[3] = fma(qv, qp, acc[3]);
                    acc[4] = fma(dz, dz, acc[4]);
                    acc[5] = fma(dz, qv, acc[5]);
                    acc[6] = fma(qv, qv, acc[6]);
                }
            };
            sb_sweep(P, R, P.p, P.z, [&](const SBRow &x, int g, int l) {
                if (x.ik >= 0) P.q[brow(P, g, x.i) + l] = x.acc;   // volume part; finished by the interface pass
                else finS(x.i, g, l, x.acc, x.pw, x.own, x.diag, x.dinv);
            });
            sb_stamp(P, ntr);
            sb_iface_finish(P, P.p, &s_ictr, [&](int k, int64_t i, int g, int l, double ai) {
                const int sc = g * P.CW + l;
                const int64_t e = brow(P, g, i) + l;
                const double qv = ld_cg1(P.q + e) + ai, pi = ld_cg1(P.p + e), zz = ld_cg1(P.z + e);
                double d = 1.0, dinv = 1.0;
                if (sc < P.S) {
                    d = P.if_d[(int64_t)k * P.S + sc];
                    dinv = P.if_dinv[(int64_t)k * P.S + sc];
                }
                finS(i, g, l, qv, pi, zz, d, dinv);
            });
            sb_stamp(P, ntr);
            sb_reduce<SB_NV>(P, acc, red, s_tot, P.totals + SB_M, grid, ntr);
        }
        if (tr_on && ntr < 1000) P.trace[ntr++] = gtimer();
        if (threadIdx.x < SB_MAXS) {
            const int c = threadIdx.x;
            if (s_conv[c]) {
                s_alpha[c] = 0.0;
                s_beta[c] = 0.0;
            } else {
                const double pq = s_tot[c], A1 = s_tot[SB_MAXS + c], A2 = s_tot[2 * SB_MAXS + c],
                             A3 = s_tot[3 * SB_MAXS + c], B1 = s_tot[4 * SB_MAXS + c],
                             B2 = s_tot[5 * SB_MAXS + c], B3 = s_tot[6 * SB_MAXS + c];
                const double al = s_rho[c] / pq;
                const double rz = fma(al * al, A3, fma(-2.0 * al, A2, A1));
                const double rr = fma(al * al, B3, fma(-2.0 * al, B2, B1));
                s_alpha[c] = al;
                s_beta[c] = rz / s_rho[c];
                s_rho[c] = rz;
                s_rr[c] = rr;
                s_itc[c] = it + 1;
                s_conv[c] = rr <= s_tol2[c];
            }
        }
        __syncthreads();
        // ---- U: x += alpha p, z -= alpha q', p = z + beta p: one flat stream over the four block
        // vectors (identical layouts), 16-byte elements (two columns of one row), 6 in flight
        {
            const int64_t n2 = NU * P.CW / 2;
            const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, TT = (int64_t)gridDim.x * blockDim.x;
            const int64_t NC = P.N * P.CW;   // elements per column group
            auto upd = [&](int64_t e2, double2 pv, double2 qv, double2 xv, double2 zv) {
                const int64_t e = 2 * e2;
                const int sc = (int)(e / NC) * P.CW + (int)(e % P.CW);
                const double a0 = s_alpha[sc], a1 = s_alpha[sc + 1], b0 = s_beta[sc], b1 = s_beta[sc + 1];
                const double z0 = fma(-a0, qv.x, zv.x), z1 = fma(-a1, qv.y, zv.y);
                reinterpret_cast<double2 *>(P.T_out)[e2] = make_double2(fma(a0, pv.x, xv.x), fma(a1, pv.y, xv.y));
                reinterpret_cast<double2 *>(P.z)[e2] = make_double2(z0, z1);
                reinterpret_cast<double2 *>(P.p)[e2] = make_double2(fma(b0, pv.x, z0), fma(b1, pv.y, z1));
            };
            const double2 *p2 = reinterpret_cast<const double2 *>(P.p), *q2 = reinterpret_cast<const double2 *>(P.q),
                          *x2 = reinterpret_cast<const double2 *>(xsrc), *z2 = reinterpret_cast<const double2 *>(P.z);
            int64_t e2 = gt;
            for (; e2 + 5 * TT < n2; e2 += 6 * TT) {
                double2 pv[6], qv[6], xv[6], zv[6];
#pragma unroll
                for (int k = 0; k < 6; ++k) {
                    pv[k] = ld_cg2(p2 + e2 + k * TT);
                    qv[k] = ld_cg2(q2 + e2 + k * TT);
                    xv[k] = ld_cg2(x2 + e2 + k * TT);
                    zv[k] = ld_cg2(z2 + e2 + k * TT);
                }
#pragma unroll
                for (int k = 0; k < 6; ++k) upd(e2 + k * TT, pv[k], qv[k], xv[k], zv[k]);
            }
            for (; e2 < n2; e2 += TT) upd(e2, ld_cg2(p2 + e2), ld_cg2(q2 + e2), ld_cg2(x2 + e2), ld_cg2(z2 + e2));
        }
        fence_proxy_async_global();   // plain stores before the next TMA reads
        grid.sync();
        if (tr_on && ntr < 1000) P.trace[ntr++] = gtimer();
        xsrc = P.T_out;
        ++it;
    }
    if (it == 0) {   // converged at the start: T^{n+1} = x0
        const int64_t n = NU * P.CW;
        for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
            P.T_out[e] = x0[e];
    }
    if (blockIdx.x == 0 && threadIdx.x < SB_MAXS) {
        const int c = threadIdx.x;
        if (c < P.S) {
            const double rel = s_bb[c] > 0.0 ? sqrt(s_rr[c] / s_bb[c]) : sqrt(s_rr[c]);
            P.iters_out[(int64_t)P.step * P.S + c] = s_itc[c];
            P.relres_out[(int64_t)P.step * P.S + c] = rel;
            if (!s_conv[c] && atomicCAS(&P.status[0], 0, 1) == 0) {
                P.status[2] = P.step;
                P.status[3] = c;
                *P.fail_relres = rel;
            }
        }
        if (c == 0) P.area_out[P.step] = area;
    }
}

// Row-major copy of each slice of the sliced-ELL operator (after every rebuild of K~_vol):
// entry k of row r at ptr8[s] + r w8 + k; padding entries: value 0, the row's own window slot.
__global__ void k_sb_rowmajor(const int64_t *__restrict__ sp, const int64_t *__restrict__ sp8,
                              const double *__restrict__ val, const uint16_t *__restrict__ lcol,
                              const int32_t *__restrict__ lown, int64_t nslices, double *__restrict__ val8,
                              uint16_t *__restrict__ lcol8) {
    const int64_t s = blockIdx.x;
    if (s >= nslices) return;
    const int w = (int)((sp[s + 1] - sp[s]) / 32), w8 = (int)((sp8[s + 1] - sp8[s]) / 32);
    for (int t = threadIdx.x; t < 32 * w8; t += blockDim.x) {
        const int r = t / w8, k = t - r * w8;
        const int64_t src = sp[s] + 32 * (int64_t)k + r;
        val8[sp8[s] + t] = k < w ? val[src] : 0.0;
        lcol8[sp8[s] + t] = k < w ? lcol[src] : (uint16_t)(lown[s] + r);
    }
}

int sbcg_prepare(Ctx &c) {
    k_sb_rowmajor<<<(unsigned)c.nslices, 128, 0, c.stream>>>(c.d_slice_ptr, c.d_sb_ptr8, c.d_val, c.d_lcol,
                                                              c.d_chunk_lown, c.nslices, c.d_sb_val8, c.d_sb_lcol8);
    CK(cudaGetLastError());
    return 0;
}

// ---------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------
static size_t a16(size_t x) { return (x + 15) & ~(size_t)15; }

// Select the windowed SpMM kernel for a batched context: chunk windows of single slices,
// stage layout, ring depth.  Returns 0 and sets c.sb_on, or 0 with c.sb_on = false when the
// numbering / sizes do not fit (the gather kernel of cg_batched.cu is used then).
int sbcg_setup(Ctx &c) {
    c.sb_on = false;
    // the default batched kernel; THERMO_CGB=1 selects the gather kernel (cg_batched.cu), which
    // is also the fallback when the numbering or the sizes do not fit (below)
    const char *ev = getenv("THERMO_CGB");
    if (ev && atoi(ev) == 1) return 0;
    if (c.S > SB_MAXS) return 0;
    const int CW = c.SP > SB_CW ? SB_CW : c.SP;
    const int G = c.SP / CW;
    if (G * CW != c.SP || G > 4 || c.num_sms < G) return 0;
    // window runs of every slice (W = 1 chunk), 16-bit window-local columns
    CK(cudaMalloc(&c.d_chunk_runs, sizeof(int2) * (size_t)c.nslices * 32));
    CK(cudaMalloc(&c.d_chunk_nruns, sizeof(int32_t) * (size_t)c.nslices));
    CK(cudaMalloc(&c.d_chunk_lown, sizeof(int32_t) * (size_t)c.nslices));
    CK(cudaMalloc(&c.d_lcol, sizeof(uint16_t) * (size_t)c.nnz_pad));
    int *d_stats = nullptr;
    CK(cudaMalloc(&d_stats, sizeof(int) * 4));
    CK(cudaMemsetAsync(d_stats, 0, sizeof(int) * 4, c.stream));
    chunk_windows_launch(c, 1, SB_GAP, c.d_chunk_runs, c.d_chunk_nruns, c.d_chunk_lown, c.d_lcol, d_stats);
    CK(cudaGetLastError());
    int stats[4];
    std::vector<int64_t> sp(c.nslices + 1);
    CK(cudaMemcpyAsync(stats, d_stats, sizeof stats, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaMemcpyAsync(sp.data(), c.d_slice_ptr, sizeof(int64_t) * sp.size(), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    cudaFree(d_stats);
    const bool verbose = getenv("THERMO_CG_VERBOSE") != nullptr;
    if (stats[2] || stats[1] > SB_MAXR) {
        if (verbose) fprintf(stderr, "[thermo cgb] windows do not fit (runs %d, flags %d): gather kernel\n", stats[1], stats[2]);
        return 0;
    }
    // row-major copy of the matrix per slice, widths rounded up to 8 (sbcg_prepare fills it)
    std::vector<int64_t> sp8(c.nslices + 1, 0);
    for (int64_t s = 0; s < c.nslices; ++s) sp8[s + 1] = sp8[s] + 32 * (((sp[s + 1] - sp[s]) / 32 + 7) & ~(int64_t)7);
    int64_t emax = 0;
    for (int64_t s = 0; s < c.nslices; ++s) emax = std::max(emax, sp8[s + 1] - sp8[s]);
    CK(cudaMalloc(&c.d_sb_ptr8, sizeof(int64_t) * (c.nslices + 1)));
    CK(cudaMemcpy(c.d_sb_ptr8, sp8.data(), sizeof(int64_t) * (c.nslices + 1), cudaMemcpyHostToDevice));
    CK(cudaMalloc(&c.d_sb_val8, sizeof(double) * (size_t)(sp8[c.nslices] + 1)));
    CK(cudaMalloc(&c.d_sb_lcol8, sizeof(uint16_t) * (size_t)(sp8[c.nslices] + 8)));
    const int wc = (stats[0] + 2) & ~1;
    const size_t col_off = a16(SB_HDR + (size_t)emax * 8);
    const size_t win_off = a16(col_off + (size_t)emax * 2);
    const size_t own_off = a16(win_off + (size_t)wc * CW * 8);
    const size_t aux_off = a16(own_off + (size_t)32 * CW * 8);   // D^{-1} (256 B) + interface index (128 B)
    const size_t stage = a16(aux_off + 256 + 128);
    const size_t budget = 210 * 1024;
    int ns = (int)std::min<size_t>(SB_MAXSTAGES, budget / stage);
    if (const char *e = getenv("THERMO_CGB_STAGES")) ns = std::min(ns, std::max(2, atoi(e)));
    ns -= ns % SB_NPW;   // every ring slot belongs to one producer
    // the reduction scratch aliases the ring: (all warps) x 7 x 32 doubles; the metadata batch
    // buffers follow the ring
    const size_t meta_off = a16(std::max((size_t)ns * stage, (size_t)(SB_THREADS / 32) * SB_NV * 32 * 8));
    const size_t smem = meta_off + 2 * SB_NPW * SB_RB * sizeof(SBRec);
    if (ns < 2) {
        if (verbose) fprintf(stderr, "[thermo cgb] stage %zu B too large: gather kernel\n", stage);
        return 0;
    }
    CK(cudaFuncSetAttribute((const void *)k_sbcg_step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sbcg_step, SB_THREADS, smem));
    if (per_sm < 1) {
        if (verbose) fprintf(stderr, "[thermo cgb] SpMM kernel not resident (smem %zu B): gather kernel\n", smem);
        return 0;
    }
    // interface rows of each CTA's slices (CTA b: column group b % G, slices s with
    // s mod (Gw / G) = b / G -- the static assignment of sb_sweep)
    const int grid = c.num_sms, Gw = (grid / G) * G, step_s = Gw / G;
    {
        std::vector<int32_t> rows(c.n_if);
        if (c.n_if) CK(cudaMemcpy(rows.data(), c.d_if_rows, sizeof(int32_t) * c.n_if, cudaMemcpyDeviceToHost));
        std::vector<std::vector<int32_t>> lists(Gw);
        for (int k = 0; k < c.n_if; ++k) {
            const int64_t sl = rows[k] / 32;
            for (int g = 0; g < G; ++g) lists[(sl % step_s) * G + g].push_back(k);
        }
        std::vector<int32_t> ptr(Gw + 1, 0), ks;
        for (int b = 0; b < Gw; ++b) {
            ptr[b + 1] = ptr[b] + (int32_t)lists[b].size();
            ks.insert(ks.end(), lists[b].begin(), lists[b].end());
        }
        CK(cudaMalloc(&c.d_sb_ai, sizeof(double) * SB_CW * (ks.size() + 1)));
        CK(cudaMalloc(&c.d_sb_if_ptr, sizeof(int32_t) * (Gw + 1)));
        CK(cudaMalloc(&c.d_sb_if_k, sizeof(int32_t) * (ks.size() + 1)));
        CK(cudaMemcpy(c.d_sb_if_ptr, ptr.data(), sizeof(int32_t) * (Gw + 1), cudaMemcpyHostToDevice));
        if (!ks.empty()) CK(cudaMemcpy(c.d_sb_if_k, ks.data(), sizeof(int32_t) * ks.size(), cudaMemcpyHostToDevice));
    }
    {   // per-CTA chunk metadata in sweep order (CTA b: slices b / G + k step_s of group b % G)
        std::vector<int2> runs((size_t)c.nslices * 32);
        std::vector<int32_t> nr(c.nslices), lo(c.nslices);
        CK(cudaMemcpy(runs.data(), c.d_chunk_runs, sizeof(int2) * runs.size(), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(nr.data(), c.d_chunk_nruns, sizeof(int32_t) * nr.size(), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(lo.data(), c.d_chunk_lown, sizeof(int32_t) * lo.size(), cudaMemcpyDeviceToHost));
        // records of CTA b, producer p: its chunks k = p, p + 2, ... (rec_ptr[2 b + p])
        std::vector<SBRec> recs;
        std::vector<int32_t> rptr(SB_NPW * Gw + 1, 0);
        for (int b = 0; b < Gw; ++b) {
            for (int pw = 0; pw < SB_NPW; ++pw) {
                int64_t k = 0;
                for (int64_t sl = b / G; sl < c.nslices; sl += step_s, ++k) {
                    if (k % SB_NPW != pw) continue;
                    SBRec r;
                    memset(&r, 0, sizeof r);
                    r.e0 = sp8[sl];
                    r.cnt = (int)(sp8[sl + 1] - sp8[sl]);
                    r.lown = lo[sl];
                    r.nruns = nr[sl];
                    r.s = (int)sl;
                    for (int q = 0; q < nr[sl]; ++q) r.run[q] = runs[(size_t)sl * 32 + q];
                    recs.push_back(r);
                }
                rptr[SB_NPW * b + pw + 1] = (int32_t)recs.size();
            }
        }
        CK(cudaMalloc(&c.d_sb_recs, sizeof(SBRec) * (recs.size() + 1)));
        CK(cudaMalloc(&c.d_sb_rec_ptr, sizeof(int32_t) * (SB_NPW * Gw + 1)));
        CK(cudaMemcpy(c.d_sb_recs, recs.data(), sizeof(SBRec) * recs.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c.d_sb_rec_ptr, rptr.data(), sizeof(int32_t) * (SB_NPW * Gw + 1), cudaMemcpyHostToDevice));
    }
    CK(cudaMalloc(&c.d_sb_partials, sizeof(double) * SB_M * (size_t)c.num_sms));
    CK(cudaMalloc(&c.d_sb_totals, sizeof(double) * 2 * SB_M));
    CK(cudaMalloc(&c.d_sb_dbg, sizeof(int) * 4));
    CK(cudaMemset(c.d_sb_dbg, 0, sizeof(int) * 4));
    if (!c.d_if_d && c.n_if) CK(cudaMalloc(&c.d_if_d, sizeof(double) * (size_t)c.S * c.n_if));
    c.sb_on = true;
    c.CW = CW;
    c.sb_G = G;
    c.sb_stage = (uint32_t)stage;
    c.sb_col_off = (uint32_t)col_off;
    c.sb_win_off = (uint32_t)win_off;
    c.sb_own_off = (uint32_t)own_off;
    c.sb_meta_off = (uint32_t)meta_off;
    c.sb_aux_off = (uint32_t)aux_off;
    c.sb_nstages = ns;
    c.sb_smem = smem;
    c.cg_grid = c.num_sms;
    c.cg_block = SB_THREADS;
    c.cg_win_cap = wc;
    c.cg_max_runs = stats[1];
    if (getenv("THERMO_CG_VERBOSE"))
        fprintf(stderr, "[thermo cgb] windowed SpMM: CW %d, G %d, window cap %d rows (max runs %d), stage %zu B, "
                        "%d stages, smem %zu B\n", CW, G, wc, stats[1], stage, ns, smem);
    return 0;
}

// [G][N][CW] column groups -> [N][SP] rows (the gather kernel's layout)
__global__ void k_sb_to_rows(const double *__restrict__ in, int64_t N, int CW, int SP, double *__restrict__ out) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= N * SP) return;
    const int64_t i = t / SP;
    const int s = (int)(t % SP);
    out[t] = in[((int64_t)(s / CW) * N + i) * CW + s % CW];
}

// Switch a batched context from this kernel to the gather kernel (the SDC methods run on the
// latter): the current state moves to the row layout; the extrapolation history is dropped.
int sbcg_disable(Ctx &c) {
    if (!c.sb_on) return 0;
    const int64_t n = c.N * c.SP;
    double *cur = c.d_T[c.cur];
    k_sb_to_rows<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(cur, c.N, c.CW, c.SP, c.d_q);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(cur, c.d_q, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
    c.sb_on = false;
    c.CW = c.SP;
    c.hist = 0;
    if (int rc = cgb_gather_setup(c)) return rc;
    return c.built_dt > 0.0 ? cgb_prepare(c) : 0;
}

int sbcg_launch_step(Ctx &c, int step, double dt, const double *x0) {
    SBParams P;
    memset(&P, 0, sizeof P);
    P.N = c.N;
    P.nslices = c.nslices;
    P.S = c.S;
    P.SP = c.SP;
    P.CW = c.CW;
    P.G = c.sb_G;
    P.Gw = (c.cg_grid / P.G) * P.G;
    P.slice_ptr = c.d_slice_ptr;
    P.lcol = c.d_sb_lcol8;
    P.val = c.d_sb_val8;
    P.recs = (const SBRec *)c.d_sb_recs;
    P.rec_ptr = c.d_sb_rec_ptr;
    P.ML = c.d_ML;
    P.benv = c.d_benv;
    P.Dinv = c.d_Dinv;
    P.if_of_row = c.d_if_of_row;
    P.if_rows = c.d_if_rows;
    P.if_cta_ptr = c.d_sb_if_ptr;
    P.if_cta_k = c.d_sb_if_k;
    P.ai = c.d_sb_ai;
    P.n_if = c.n_if;
    P.nA = c.nA;
    P.cap = c.cap;
    P.ell_cnt = c.d_ell_cnt;
    P.ell_col = c.d_ell_col;
    P.ell_val = c.d_ell_val;
    P.if_b = c.d_if_b;
    P.if_phi = c.d_if_phi;
    P.if_d = c.d_if_d;
    P.if_dinv = c.d_if_dinv;
    P.T_in = c.d_T[(c.cur + step) & 1];
    P.X0 = x0;
    P.T_out = c.d_T[(c.cur + step + 1) & 1];
    P.z = c.d_z;
    P.p = c.d_p[0];
    P.q = c.d_q;
    P.partials = c.d_sb_partials;
    P.totals = c.d_sb_totals;
    P.status = c.d_status;
    P.fail_relres = c.d_fail_relres;
    P.iters_out = c.d_iters;
    P.relres_out = c.d_relres;
    P.area_out = c.d_area;
    P.dt = dt;
    P.rtol2 = c.rtol * c.rtol;
    P.maxit = c.maxit > 0 ? c.maxit : (int)std::min<int64_t>(10 * c.N, 10000);
    P.step = step;
    P.nstages = c.sb_nstages;
    P.stage_bytes = c.sb_stage;
    P.col_off = c.sb_col_off;
    P.win_off = c.sb_win_off;
    P.own_off = c.sb_own_off;
    P.meta_off = c.sb_meta_off;
    P.debug = getenv("THERMO_CGB_DEBUG") ? atoi(getenv("THERMO_CGB_DEBUG")) : 0;
    P.aux_off = c.sb_aux_off;
    P.trace = c.d_trace;
    P.trace_fine = getenv("THERMO_CG_TRACE") && atoi(getenv("THERMO_CG_TRACE")) == 3;
    P.dbg = c.d_sb_dbg;
    void *args[] = {&P};
    CK(cudaLaunchCooperativeKernel((const void *)k_sbcg_step, dim3(c.cg_grid), dim3(SB_THREADS), args, c.sb_smem,
                                   c.stream));
    return 0;
}

}  // namespace thermo
