// cg_batched.cu -- S independent scenarios advanced together (BASELINE.json config 4,
// SURVEY 8(a) a5): the implicit-Euler solve of every scenario by Jacobi-PCG with per-column
// alpha, beta and convergence mask, the shared volume operator applied as an SpMM.
//
// Layout: every state / workspace vector is an N x SP row-major block (SP even, >= S); lane l
// of a warp owns the columns 2l, 2l+1 of every row it touches, so one row of a block vector is
// one coalesced 512-byte access for S = 64.  Per-scenario pieces: the interface rows (ELL,
// [k][c][s]), the friction source, and the Jacobi diagonal DinvS[N][SP] (volume diagonal,
// interface rows rewritten per step by the interface kernels).
//
// Per CG iteration (same z-primary schedule as cg.cu, column-wise):
//   S: p = z + beta p_old on the fly, q = K~ p (warp per slice, rows in turn: the row's entries
//      are broadcast by shuffles, every lane gathers its two columns), partial p.q per column
//   U: x += alpha p, z -= alpha D^{-1} q, partial r.z, r.r per column
// Converged columns are frozen (alpha = 0).  Reductions are deterministic: lanes own columns,
// warps combine in fixed order, CTAs in fixed order; every CTA computes identical scalars.
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cmath>
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

#define CGB_BLOCK 512
#define CGB_WARPS (CGB_BLOCK / 32)
#define CGB_MAXS 64
#define CGB_NV 4   // reduction values per column and phase (max)

// windowed variant (k_cgb_step<true>): 2 groups of 8 consumer warps + 1 producer warp
#define CGW_NCW 8
#define CGW_WARPS 17
#define CGW_BLOCK (32 * CGW_WARPS)
#define CGW_MAXR 16     // window runs per chunk (one per producer lane)
#define CGW_HDR 128     // stage header bytes: [0] window index of the chunk's first row, [1] slice width

struct CGBParams {
    int64_t N, nslices;
    int S, SP;
    const int64_t *slice_ptr;
    const int32_t *col;
    const double *val;
    const double *ML, *benv, *DinvS;
    int n_if, nA, cap;
    const int32_t *if_rows, *slice_if, *ell_cnt, *ell_col;
    const int32_t *if_of_row;   // [N] interface index of a row, -1 if none
    const double *ell_val, *if_b, *if_phi;
    const double *T_in;
    double *T_out, *z, *pa, *pb, *q;
    double *partials;   // [G][CGB_NV][64]
    int *status;
    double *fail_relres;
    int32_t *iters_out;
    double *relres_out, *area_out;
    double dt, rtol2;
    int maxit, step;
    unsigned long long *trace;   // optional: %globaltimer after every grid barrier (CTA 0)
    int contiguous;              // 1: CTA b sweeps one contiguous block of row pairs (L1 reuse of
                                 // the gathered neighbour rows), 0: row pairs dealt round-robin
    // windowed sweeps: chunk = CR consecutive rows of one slice; the producer bulk-copies the
    // chunk's slice (values, window-local columns, interface map) and its column window (<=
    // CGW_MAXR runs of whole block-vector rows) into one stage of an NS-stage ring
    int CR, NS, wcap;
    int64_t nchunks;
    uint32_t stage_bytes, off_col, off_if, off_w1, off_w2;
    const int2 *wruns;           // [nchunks][CGW_MAXR] (first row, rows)
    const int32_t *wnruns;       // [nchunks]
    const int32_t *wlown;        // [nchunks] window index of the chunk's first row
    const uint16_t *wcol;        // [nnz_pad] window-local column of every stored entry
};

__device__ __forceinline__ int64_t ellb(const CGBParams &P, int s, int c, int k) {
    return ((int64_t)k * P.cap + c) * P.S + s;
}

// CTA + grid reduction of NV values per column (lanes own columns 2l, 2l+1).
template <int NV, int NW = CGB_WARPS>
__device__ __forceinline__ void cgb_reduce(double (&v)[NV][2], double *sm, double *partials, cg::grid_group &grid,
                                           double (&out)[NV][2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        sm[(warp * NV + j) * 64 + 2 * lane] = v[j][0];
        sm[(warp * NV + j) * 64 + 2 * lane + 1] = v[j][1];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < NV * 64; t += blockDim.x) {
        double a = 0.0;
        for (int w = 0; w < NW; ++w) a += sm[w * NV * 64 + t];
        partials[(int64_t)blockIdx.x * CGB_NV * 64 + t] = a;
    }
    grid.sync();
    for (int t = threadIdx.x; t < NV * 64; t += blockDim.x) {
        double a = 0.0;
        const int G = gridDim.x;
        int g = 0;
        for (; g + 8 <= G; g += 8) {   // loads issued together, adds in the serial order
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = partials[(int64_t)(g + u) * CGB_NV * 64 + t];
#pragma unroll
            for (int u = 0; u < 8; ++u) a += v[u];
        }
        for (; g < G; ++g) a += partials[(int64_t)g * CGB_NV * 64 + t];
        sm[t] = a;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        out[j][0] = sm[j * 64 + 2 * lane];
        out[j][1] = sm[j * 64 + 2 * lane + 1];
    }
    __syncthreads();
}

// Two rows (rA, rA + 1) of one slice at once: lanes 0-15 hold the entries of row A, lanes
// 16-31 those of row B (16 per round); the warp broadcasts them and every lane gathers its two
// columns for both rows, so 16 loads per lane are in flight.  The entries of a round are
// loaded by load_cv (for the first round one unit ahead, see unit_loop).
__device__ __forceinline__ void load_cv(const CGBParams &P, int64_t base, int w, int rA, bool validB, int k0,
                                        int lane, int &cl, double &vl) {
    const int half = lane >> 4, kk = k0 + (lane & 15);
    cl = 0;
    vl = 0.0;
    if (kk < w && (half == 0 || validB)) {
        cl = P.col[base + 32 * (int64_t)kk + rA + half];
        vl = P.val[base + 32 * (int64_t)kk + rA + half];
    }
}

// U entries per row and round: 4 with two gathered vectors, 8 with one (same register budget).
template <bool kTwo, int U>
__device__ __forceinline__ void gather_round(const CGBParams &P, int cl, double vl, int m, const double *x1,
                                             const double *x2, double2 beta, int ln, double2 &accA, double2 &accB) {
    for (int k = 0; k < m; k += U) {
        double2 yA[U], yB[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {   // all gathers of the round first
            const int ku = min(k + u, m - 1);
            const int cA = __shfl_sync(0xffffffffu, cl, ku);
            const int cB = __shfl_sync(0xffffffffu, cl, 16 + ku);
            const double2 a = reinterpret_cast<const double2 *>(x1 + (int64_t)cA * P.SP)[ln];
            const double2 b = reinterpret_cast<const double2 *>(x1 + (int64_t)cB * P.SP)[ln];
            if (kTwo) {
                const double2 a2 = reinterpret_cast<const double2 *>(x2 + (int64_t)cA * P.SP)[ln];
                const double2 b2 = reinterpret_cast<const double2 *>(x2 + (int64_t)cB * P.SP)[ln];
                yA[u] = make_double2(fma(beta.x, a2.x, a.x), fma(beta.y, a2.y, a.y));
                yB[u] = make_double2(fma(beta.x, b2.x, b.x), fma(beta.y, b2.y, b.y));
            } else {
                yA[u] = a;
                yB[u] = b;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {   // then the values (broadcast) and the row sums
            const int ku = min(k + u, m - 1);
            const double vA = __shfl_sync(0xffffffffu, vl, ku), vB = __shfl_sync(0xffffffffu, vl, 16 + ku);
            if (k + u < m) {
                accA.x = fma(vA, yA[u].x, accA.x);
                accA.y = fma(vA, yA[u].y, accA.y);
                accB.x = fma(vB, yB[u].x, accB.x);
                accB.y = fma(vB, yB[u].y, accB.y);
            }
        }
    }
}

// Row sums of the shared volume operator for rows rA, rA + 1 of a slice applied to the lane's
// two columns of y = x1 + beta x2 (kTwo = false: y = x1).  (cl, vl): entries 0..15, preloaded.
template <bool kTwo>
__device__ __forceinline__ void row_spmm2(const CGBParams &P, int64_t base, int w, int rA, bool validB, int cl,
                                          double vl, const double *x1, const double *x2, double2 beta, int lane,
                                          double2 &accA, double2 &accB) {
    accA = make_double2(0.0, 0.0);
    accB = make_double2(0.0, 0.0);
    const int ln = 2 * lane < P.SP ? lane : 0;   // lanes past the row stride re-read columns 0..1
    constexpr int U = kTwo ? 4 : 8;
    gather_round<kTwo, U>(P, cl, vl, min(16, w), x1, x2, beta, ln, accA, accB);
    for (int k0 = 16; k0 < w; k0 += 16) {
        load_cv(P, base, w, rA, validB, k0, lane, cl, vl);
        gather_round<kTwo, U>(P, cl, vl, min(16, w - k0), x1, x2, beta, ln, accA, accB);
    }
}

// Walk this warp's units (slice s, row pair rA, rA + 1; unit u = gw + k TW).  Per 32 units,
// lane k loads unit k's slice offset, width and interface indices in one round trip; the
// first round of matrix entries of the next unit is loaded while the current one gathers.
// body(u, base, w, rA, validB, ikA, ikB, cl, vl) runs once per unit, warp-uniformly.
template <class Body>
__device__ __forceinline__ void unit_loop(const CGBParams &P, int64_t npairs, int64_t gw, int64_t TW, int lane,
                                          Body body) {
    const int64_t N = P.N;
    for (int64_t c0 = gw; c0 < npairs; c0 += 32 * (int64_t)TW) {
        const int64_t uk = c0 + (int64_t)lane * TW;
        long long m_base = 0;
        int m_w = -1, m_ikA = -1, m_ikB = -1;
        if (uk < npairs) {
            const int64_t s = uk >> 4, iA = 32 * s + 2 * (uk & 15);
            if (iA < N) {
                m_base = P.slice_ptr[s];
                m_w = (int)((P.slice_ptr[s + 1] - m_base) >> 5);
                m_ikA = P.if_of_row[iA];
                m_ikB = iA + 1 < N ? P.if_of_row[iA + 1] : -1;
            }
        }
        const int64_t rem = (npairs - c0 + TW - 1) / TW;
        const int nun = rem < 32 ? (int)rem : 32;
        int cl = 0, cln = 0;
        double vl = 0.0, vln = 0.0;
        {
            const int w0 = __shfl_sync(0xffffffffu, m_w, 0);
            if (w0 >= 0) {
                const int64_t iA = 32 * (c0 >> 4) + 2 * (c0 & 15);
                load_cv(P, __shfl_sync(0xffffffffu, m_base, 0), w0, 2 * (int)(c0 & 15), iA + 1 < N, 0, lane, cl, vl);
            }
        }
        for (int k = 0; k < nun; ++k) {
            const int64_t u = c0 + (int64_t)k * TW;
            const int64_t base = __shfl_sync(0xffffffffu, m_base, k);
            const int w = __shfl_sync(0xffffffffu, m_w, k);
            const int ikA = __shfl_sync(0xffffffffu, m_ikA, k), ikB = __shfl_sync(0xffffffffu, m_ikB, k);
            if (k + 1 < nun) {   // next unit's first round of entries
                const int64_t un = u + TW;
                const int wn = __shfl_sync(0xffffffffu, m_w, k + 1);
                const long long bn = __shfl_sync(0xffffffffu, m_base, k + 1);
                if (wn >= 0) {
                    const int64_t iAn = 32 * (un >> 4) + 2 * (un & 15);
                    load_cv(P, bn, wn, 2 * (int)(un & 15), iAn + 1 < N, 0, lane, cln, vln);
                }
            }
            if (w >= 0) {
                const int rA = 2 * (int)(u & 15);
                const bool validB = 32 * (u >> 4) + rA + 1 < N;
                body(u, base, w, rA, validB, ikA, ikB, cl, vl);
            }
            cl = cln;
            vl = vln;
        }
    }
}

// Interface rows (per scenario): lane's two columns of row ik.
template <bool kTwo>
__device__ __forceinline__ double2 row_iface(const CGBParams &P, int ik, const double *x1, const double *x2,
                                             double2 beta, int lane) {
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int s = 2 * lane + h;
        if (s >= P.S) break;
        const int cnt = P.ell_cnt[(int64_t)ik * P.S + s];
        const double b = h ? beta.y : beta.x;
        double a = 0.0;
        for (int c = 0; c < cnt; ++c) {
            const int64_t e = ellb(P, s, c, ik);
            const int j = P.ell_col[e];
            double y = x1[(int64_t)j * P.SP + s];
            if (kTwo) y = fma(b, x2[(int64_t)j * P.SP + s], y);
            a = fma(P.ell_val[e], y, a);
        }
        if (h) acc.y = a; else acc.x = a;
    }
    return acc;
}

// U phase of one CG iteration (warp per row, lanes over the columns, 4 rows in flight):
// x += alpha p, z -= alpha D^{-1} q, partial r.z and r.r per column (r = z / D^{-1}).
__device__ __forceinline__ void cgb_update(const CGBParams &P, const double (&alpha)[2], const double *pnew,
                                       const double *xsrc, const bool (&col_ok)[2], bool lane_ok, int lane,
                                       int gw, int TW, double (&vu)[2][2]) {
    const int64_t N = P.N;
    auto upd = [&](double2 pv, double2 qv, double2 dv, double2 xv, double2 zv, int64_t i) {
        double2 xo, zo;
        xo.x = fma(alpha[0], pv.x, xv.x);
        xo.y = fma(alpha[1], pv.y, xv.y);
        zo.x = fma(-alpha[0] * dv.x, qv.x, zv.x);
        zo.y = fma(-alpha[1] * dv.y, qv.y, zv.y);
        reinterpret_cast<double2 *>(P.T_out + i * P.SP)[lane] = xo;
        reinterpret_cast<double2 *>(P.z + i * P.SP)[lane] = zo;
        if (col_ok[0]) {
            const double r0 = zo.x / dv.x;
            vu[0][0] = fma(r0, zo.x, vu[0][0]);
            vu[1][0] = fma(r0, r0, vu[1][0]);
        }
        if (col_ok[1]) {
            const double r1 = zo.y / dv.y;
            vu[0][1] = fma(r1, zo.y, vu[0][1]);
            vu[1][1] = fma(r1, r1, vu[1][1]);
        }
    };
    if (lane_ok) {
        int64_t i = gw;
        for (; i + 3 * (int64_t)TW < N; i += 4 * (int64_t)TW) {   // 4 rows in flight
            double2 pv[4], qv[4], dv[4], xv[4], zv[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int64_t ir = i + r * (int64_t)TW;
                pv[r] = ld_cg2(reinterpret_cast<const double2 *>(pnew + ir * P.SP) + lane);
                qv[r] = ld_cg2(reinterpret_cast<const double2 *>(P.q + ir * P.SP) + lane);
                dv[r] = ld_cg2(reinterpret_cast<const double2 *>(P.DinvS + ir * P.SP) + lane);
                xv[r] = ld_cg2(reinterpret_cast<const double2 *>(xsrc + ir * P.SP) + lane);
                zv[r] = ld_cg2(reinterpret_cast<const double2 *>(P.z + ir * P.SP) + lane);
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) upd(pv[r], qv[r], dv[r], xv[r], zv[r], i + r * (int64_t)TW);
        }
        for (; i < N; i += TW)
            upd(ld_cg2(reinterpret_cast<const double2 *>(pnew + i * P.SP) + lane),
                ld_cg2(reinterpret_cast<const double2 *>(P.q + i * P.SP) + lane),
                ld_cg2(reinterpret_cast<const double2 *>(P.DinvS + i * P.SP) + lane),
                ld_cg2(reinterpret_cast<const double2 *>(xsrc + i * P.SP) + lane),
                ld_cg2(reinterpret_cast<const double2 *>(P.z + i * P.SP) + lane), i);
    }
}

// ---------------------------------------------------------------------------------
// windowed sweeps (TMA ring)
// ---------------------------------------------------------------------------------
struct WinRing {
    uint64_t *full, *empty;
    unsigned char *stage;
    uint32_t n;   // stages passed through the ring so far (same count in every warp)
};

struct WinMeta {
    int64_t base;
    int w, s, lown, nruns;
    int2 run;
};

__device__ __forceinline__ WinMeta win_meta(const CGBParams &P, int64_t ch, int lane) {
    WinMeta m;
    m.base = 0; m.w = 0; m.s = 0; m.lown = 0; m.nruns = 0;
    m.run = make_int2(0, 0);
    if (ch >= P.nchunks) return m;
    m.s = (int)((ch * P.CR) >> 5);
    m.base = P.slice_ptr[m.s];
    m.w = (int)((P.slice_ptr[m.s + 1] - m.base) >> 5);
    m.lown = P.wlown[ch];
    m.nruns = P.wnruns[ch];
    if (lane < CGW_MAXR) m.run = P.wruns[ch * CGW_MAXR + lane];
    return m;
}

// Producer warp: CTA b streams its chunks b, b + G, ... (static order) into the ring.
template <int NVEC>
__device__ __forceinline__ void win_produce(const CGBParams &P, WinRing &R, const double *v1, const double *v2,
                                            int lane) {
    const int G = gridDim.x;
    const uint32_t RB = (uint32_t)P.SP * 8u;
    // the vectors were written by generic stores of other CTAs before the last grid barrier,
    // and the ring's first stage served as reduction scratch: order both before the copies
    asm volatile("fence.proxy.async.global;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    int64_t ch = blockIdx.x;
    WinMeta cur = win_meta(P, ch, lane), nxt = win_meta(P, ch + G, lane);
    uint32_t n = R.n;
    for (; ch < P.nchunks; ch += G, ++n) {
        const WinMeta m2 = win_meta(P, ch + 2 * (int64_t)G, lane);   // in flight meanwhile
        const uint32_t st = n % (uint32_t)P.NS, ph = (n / (uint32_t)P.NS) & 1u;
        const int len = lane < cur.nruns ? cur.run.y : 0;
        int off = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, off, o);
            if (lane >= o) off += y;
        }
        const int tot = __shfl_sync(0xffffffffu, off, 31);
        off -= len;
        unsigned char *stg = R.stage + (size_t)st * P.stage_bytes;
        if (lane == 0) {
            mbar_wait(&R.empty[st], ph ^ 1u);
            int *hdr = reinterpret_cast<int *>(stg);
            hdr[0] = cur.lown;
            hdr[1] = cur.w;
            const uint32_t bytes = (uint32_t)cur.w * 32u * 10u + 128u + (uint32_t)NVEC * (uint32_t)tot * RB;
            mbar_arrive_expect_tx(&R.full[st], bytes);
        }
        __syncwarp();
        if (lane == 0) bulk_g2s_nohint(stg + CGW_HDR, P.val + cur.base, (uint32_t)cur.w * 256u, &R.full[st]);
        if (lane == 1) bulk_g2s_nohint(stg + P.off_col, P.wcol + cur.base, (uint32_t)cur.w * 64u, &R.full[st]);
        if (lane == 2) bulk_g2s_nohint(stg + P.off_if, P.if_of_row + 32 * (int64_t)cur.s, 128u, &R.full[st]);
        if (len > 0) {
            bulk_g2s_nohint(stg + P.off_w1 + (size_t)off * RB, v1 + (int64_t)cur.run.x * P.SP, (uint32_t)len * RB,
                            &R.full[st]);
            if (NVEC == 2)
                bulk_g2s_nohint(stg + P.off_w2 + (size_t)off * RB, v2 + (int64_t)cur.run.x * P.SP,
                                (uint32_t)len * RB, &R.full[st]);
        }
        cur = nxt;
        nxt = m2;
    }
}

// Consumer warp: 16 consumer warps form NG = 16 / NCW groups of NCW = min(CR, 8) warps; group
// g takes the chunks j = g, g + NG, ... of the CTA, warp r of a group the rows r, r + NCW, ...
// of a chunk: body(i, rr, w, vals, cols, ifmap, win1, win2, own, SPh) per row.
template <class Body>
__device__ __forceinline__ void win_consume(const CGBParams &P, WinRing &R, int warp, int lane, Body body) {
    const int NCW = P.CR < CGW_NCW ? P.CR : CGW_NCW, NG = 2 * CGW_NCW / NCW;
    const int G = gridDim.x, g = warp / NCW, r = warp % NCW;
    const int64_t b = blockIdx.x;
    const int64_t nloc = b < P.nchunks ? (P.nchunks - 1 - b) / G + 1 : 0;
    const int SPh = P.SP >> 1;
    for (int64_t j = g; j < nloc; j += NG) {
        const uint32_t n = R.n + (uint32_t)j;
        const uint32_t st = n % (uint32_t)P.NS, ph = (n / (uint32_t)P.NS) & 1u;
        mbar_wait(&R.full[st], ph);
        const unsigned char *stg = R.stage + (size_t)st * P.stage_bytes;
        const int *hdr = reinterpret_cast<const int *>(stg);
        const int lown = hdr[0], w = hdr[1];
        const double *vals = reinterpret_cast<const double *>(stg + CGW_HDR);
        const uint16_t *cols = reinterpret_cast<const uint16_t *>(stg + P.off_col);
        const int32_t *ifmap = reinterpret_cast<const int32_t *>(stg + P.off_if);
        const double2 *w1 = reinterpret_cast<const double2 *>(stg + P.off_w1);
        const double2 *w2 = reinterpret_cast<const double2 *>(stg + P.off_w2);
        const int64_t row0 = (b + j * G) * P.CR;
        for (int m = r; m < P.CR; m += NCW) {
            const int64_t i = row0 + m;
            if (i >= P.N) break;
            body(i, (int)(i & 31), w, vals, cols, ifmap, w1, w2, (lown + m) * SPh, SPh);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&R.empty[st]);
    }
}

// sum_k val_k (w1[col_k] + beta w2[col_k]) of one row from the stage (same fma order as row_spmm2)
template <bool kTwo>
__device__ __forceinline__ double2 win_row(const double *vals, const uint16_t *cols, int rr, int w, const double2 *w1,
                                           const double2 *w2, int SPh, int ln, double2 beta) {
    double2 acc = make_double2(0.0, 0.0);
    int k = 0;
    for (; k + 4 <= w; k += 4) {
        double2 y[4];
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = cols[(k + u) * 32 + rr];
            v[u] = vals[(k + u) * 32 + rr];
            const double2 a = w1[c * SPh + ln];
            if (kTwo) {
                const double2 bb = w2[c * SPh + ln];
                y[u] = make_double2(fma(beta.x, bb.x, a.x), fma(beta.y, bb.y, a.y));
            } else {
                y[u] = a;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            acc.x = fma(v[u], y[u].x, acc.x);
            acc.y = fma(v[u], y[u].y, acc.y);
        }
    }
    for (; k < w; ++k) {
        const int c = cols[k * 32 + rr];
        const double v = vals[k * 32 + rr];
        double2 y = w1[c * SPh + ln];
        if (kTwo) {
            const double2 bb = w2[c * SPh + ln];
            y = make_double2(fma(beta.x, bb.x, y.x), fma(beta.y, bb.y, y.y));
        }
        acc.x = fma(v, y.x, acc.x);
        acc.y = fma(v, y.y, acc.y);
    }
    return acc;
}

template <bool WIN>
__global__ void __launch_bounds__(WIN ? CGW_BLOCK : CGB_BLOCK, 1) k_cgb_step(CGBParams P) {
    constexpr int NW = WIN ? CGW_WARPS : CGB_WARPS;
    __shared__ double sm_static[WIN ? 1 : CGB_WARPS * CGB_NV * 64];
    extern __shared__ __align__(128) unsigned char dsm[];
    // WIN: [full[NS] | empty[NS] | pad to 128 | NS stages]; the reduction scratch aliases the
    // stages (the ring is drained at every reduction)
    WinRing R;
    R.full = reinterpret_cast<uint64_t *>(dsm);
    R.empty = R.full + 8;
    R.stage = dsm + 128;
    R.n = 0;
    double *sm = WIN ? reinterpret_cast<double *>(dsm + 128) : sm_static;
    if (P.status[0] || P.status[1]) {
        if (!P.status[0] && blockIdx.x == 0 && threadIdx.x == 0) {
            P.status[0] = 2;
            P.status[2] = P.step;
        }
        return;
    }
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool tr_on = P.trace && blockIdx.x == 0 && threadIdx.x == 0;
    int ntr = 0;
    if (tr_on) P.trace[ntr++] = gtimer();
    const int64_t N = P.N;
    const int gw = blockIdx.x * NW + warp, TW = gridDim.x * NW;
    const bool col_ok[2] = {2 * lane < P.S, 2 * lane + 1 < P.S};
    const bool lane_ok = 2 * lane < P.SP;   // lanes past the row stride touch no memory
    const int ln = lane_ok ? lane : 0;
    if (WIN) {
        if (threadIdx.x < P.NS) {
            mbar_init(&R.full[threadIdx.x], 1);
            mbar_init(&R.empty[threadIdx.x], P.CR < CGW_NCW ? P.CR : CGW_NCW);
        }
        fence_mbar_init();
        __syncthreads();
    }
    const int64_t nloc = WIN ? (blockIdx.x < P.nchunks ? (P.nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0) : 0;

    // ---- phase 0: r0 = b - K~ x0, z0 = D^{-1} r0 per column
    double v0[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};   // b.b, r.r, r.z, |Gamma_R| (scenario 0)
    const int64_t npairs = P.nslices * 16;   // units: (slice, row pair)
    // this warp's units: u0, u0 + ust, ... < uend
    int64_t u0 = gw, ust = TW, uend = npairs;
    if (P.contiguous) {
        const int64_t upc = (npairs + gridDim.x - 1) / gridDim.x;
        u0 = (int64_t)blockIdx.x * upc + warp;
        ust = NW;
        uend = min(npairs, (int64_t)(blockIdx.x + 1) * upc);
    }
    // epilogue of one row: ax = (K~ x0)_i without the interface part, Ti = x0_i
    auto fin0 = [&](int64_t i, int ik, double2 ax, double2 Ti, double2 di) {
        double2 bg = make_double2(0.0, 0.0);
        if (ik >= 0) {
            const double2 ai = row_iface<false>(P, ik, P.T_in, nullptr, make_double2(0, 0), lane);
            ax.x += ai.x;
            ax.y += ai.y;
            if (col_ok[0]) bg.x = P.if_b[(int64_t)ik * P.S + 2 * lane];
            if (col_ok[1]) bg.y = P.if_b[(int64_t)ik * P.S + 2 * lane + 1];
            if (lane == 0 && ik < P.nA) v0[3][0] += P.if_phi[(int64_t)ik * P.S];
        }
        if (!lane_ok) return;
        const double ml = P.ML[i], be = P.benv[i];
        double2 b, rr, zz;
        b.x = fma(ml, Ti.x, P.dt * (be + bg.x));
        b.y = fma(ml, Ti.y, P.dt * (be + bg.y));
        rr.x = b.x - ax.x;
        rr.y = b.y - ax.y;
        zz.x = col_ok[0] ? di.x * rr.x : 0.0;
        zz.y = col_ok[1] ? di.y * rr.y : 0.0;
        reinterpret_cast<double2 *>(P.z + i * P.SP)[lane] = zz;
        if (col_ok[0]) {
            v0[0][0] = fma(b.x, b.x, v0[0][0]);
            v0[1][0] = fma(rr.x, rr.x, v0[1][0]);
            v0[2][0] = fma(rr.x, zz.x, v0[2][0]);
        }
        if (col_ok[1]) {
            v0[0][1] = fma(b.y, b.y, v0[0][1]);
            v0[1][1] = fma(rr.y, rr.y, v0[1][1]);
            v0[2][1] = fma(rr.y, zz.y, v0[2][1]);
        }
    };
    if constexpr (WIN) {
        if (warp == CGW_WARPS - 1) {
            win_produce<1>(P, R, P.T_in, nullptr, lane);
        } else {
            win_consume(P, R, warp, lane, [&](int64_t i, int rr, int w, const double *vals, const uint16_t *cols,
                                              const int32_t *ifmap, const double2 *w1, const double2 *, int own,
                                              int SPh) {
                const double2 di = lane_ok ? reinterpret_cast<const double2 *>(P.DinvS + i * P.SP)[lane]
                                           : make_double2(0.0, 0.0);
                const double2 ax = win_row<false>(vals, cols, rr, w, w1, nullptr, SPh, ln, make_double2(0, 0));
                fin0(i, ifmap[rr], ax, w1[own + ln], di);
            });
        }
        R.n += (uint32_t)nloc;
        __syncthreads();   // ring drained before its memory serves as reduction scratch
    } else {
        unit_loop(P, uend, u0, ust, lane, [&](int64_t u, int64_t base, int w, int rA, bool validB, int ikA,
                                               int ikB, int cl, double vl) {
            const int64_t iA = 32 * (u >> 4) + rA;
            double2 Tr[2], dr[2];   // own rows, loaded ahead of the gathers
            if (lane_ok) {
                Tr[0] = reinterpret_cast<const double2 *>(P.T_in + iA * P.SP)[lane];
                dr[0] = reinterpret_cast<const double2 *>(P.DinvS + iA * P.SP)[lane];
                if (validB) {
                    Tr[1] = reinterpret_cast<const double2 *>(P.T_in + (iA + 1) * P.SP)[lane];
                    dr[1] = reinterpret_cast<const double2 *>(P.DinvS + (iA + 1) * P.SP)[lane];
                }
            }
            double2 axr[2];
            row_spmm2<false>(P, base, w, rA, validB, cl, vl, P.T_in, nullptr, make_double2(0, 0), lane, axr[0],
                             axr[1]);
            fin0(iA, ikA, axr[0], Tr[0], dr[0]);
            if (validB) fin0(iA + 1, ikB, axr[1], Tr[1], dr[1]);
        });
    }
    double t0[4][2];
    cgb_reduce<4, NW>(v0, sm, P.partials, grid, t0);
    if (tr_on) P.trace[ntr++] = gtimer();
    double rho[2] = {t0[2][0], t0[2][1]}, rr2[2] = {t0[1][0], t0[1][1]}, tol2[2], beta[2] = {0.0, 0.0};
    bool conv[2];
    int itc[2] = {0, 0};
    for (int h = 0; h < 2; ++h) {
        tol2[h] = P.rtol2 * t0[0][h];
        conv[h] = !col_ok[h] || rr2[h] <= tol2[h];
    }
    const double area = __shfl_sync(0xffffffffu, t0[3][0], 0);
    const double *xsrc = P.T_in;
    double *pold = P.pa, *pnew = P.pb;
    int it = 0;
    while (it < P.maxit) {
        const bool any = __syncthreads_or(!(conv[0] && conv[1])) != 0;   // same in every CTA
        if (!any) break;
        // ---- S
        const bool first = it == 0;
        const double2 b2 = make_double2(beta[0], beta[1]);
        double vs[1][2] = {{0.0, 0.0}};
        // epilogue of one row: acc = (K~ p)_i without the interface part, pi = p_i
        auto finS = [&](int64_t i, int ik, double2 acc, double2 pi) {
            if (ik >= 0) {
                const double2 ai = first ? row_iface<false>(P, ik, P.z, nullptr, b2, lane)
                                         : row_iface<true>(P, ik, P.z, pold, b2, lane);
                acc.x += ai.x;
                acc.y += ai.y;
            }
            if (!lane_ok) return;
            reinterpret_cast<double2 *>(pnew + i * P.SP)[lane] = pi;
            reinterpret_cast<double2 *>(P.q + i * P.SP)[lane] = acc;
            vs[0][0] = fma(pi.x, acc.x, vs[0][0]);
            vs[0][1] = fma(pi.y, acc.y, vs[0][1]);
        };
        if constexpr (WIN) {
            if (warp == CGW_WARPS - 1) {
                if (first) win_produce<1>(P, R, P.z, nullptr, lane);
                else win_produce<2>(P, R, P.z, pold, lane);
            } else {
                win_consume(P, R, warp, lane, [&](int64_t i, int rr, int w, const double *vals, const uint16_t *cols,
                                                  const int32_t *ifmap, const double2 *w1, const double2 *w2, int own,
                                                  int SPh) {
                    double2 acc, pi = w1[own + ln];
                    if (first) {
                        acc = win_row<false>(vals, cols, rr, w, w1, nullptr, SPh, ln, b2);
                    } else {
                        acc = win_row<true>(vals, cols, rr, w, w1, w2, SPh, ln, b2);
                        const double2 po = w2[own + ln];
                        pi = make_double2(fma(b2.x, po.x, pi.x), fma(b2.y, po.y, pi.y));
                    }
                    finS(i, ifmap[rr], acc, pi);
                });
            }
            R.n += (uint32_t)nloc;
            __syncthreads();
        } else {
            unit_loop(P, uend, u0, ust, lane, [&](int64_t u, int64_t base, int w, int rA, bool validB, int ikA,
                                                   int ikB, int cl, double vl) {
                const int64_t iA = 32 * (u >> 4) + rA;
                double2 zr[2], pr[2];   // own rows, loaded ahead of the gathers
                if (lane_ok) {
                    zr[0] = reinterpret_cast<const double2 *>(P.z + iA * P.SP)[lane];
                    if (!first) pr[0] = reinterpret_cast<const double2 *>(pold + iA * P.SP)[lane];
                    if (validB) {
                        zr[1] = reinterpret_cast<const double2 *>(P.z + (iA + 1) * P.SP)[lane];
                        if (!first) pr[1] = reinterpret_cast<const double2 *>(pold + (iA + 1) * P.SP)[lane];
                    }
                }
                double2 accr[2];
                if (first) row_spmm2<false>(P, base, w, rA, validB, cl, vl, P.z, nullptr, b2, lane, accr[0], accr[1]);
                else row_spmm2<true>(P, base, w, rA, validB, cl, vl, P.z, pold, b2, lane, accr[0], accr[1]);
                for (int h = 0; h < 2; ++h) {
                    if (h == 1 && !validB) break;
                    double2 pi = zr[h];
                    if (!first && lane_ok) pi = make_double2(fma(b2.x, pr[h].x, pi.x), fma(b2.y, pr[h].y, pi.y));
                    finS(iA + h, h ? ikB : ikA, accr[h], pi);
                }
            });
        }
        double tpq[1][2];
        cgb_reduce<1, NW>(vs, sm, P.partials, grid, tpq);
        if (tr_on && ntr < 1000) P.trace[ntr++] = gtimer();
        double alpha[2];
        for (int h = 0; h < 2; ++h) alpha[h] = conv[h] ? 0.0 : rho[h] / tpq[0][h];   // frozen columns
        // ---- U (warp per row, lanes over columns)
        double vu[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
        cgb_update(P, alpha, pnew, xsrc, col_ok, lane_ok, lane, gw, TW, vu);
        double tu[2][2];
        cgb_reduce<2, NW>(vu, sm, P.partials, grid, tu);
        if (tr_on && ntr < 1000) P.trace[ntr++] = gtimer();
        ++it;
        for (int h = 0; h < 2; ++h) {
            if (conv[h]) continue;
            beta[h] = tu[0][h] / rho[h];
            rho[h] = tu[0][h];
            rr2[h] = tu[1][h];
            itc[h] = it;
            conv[h] = rr2[h] <= tol2[h];
        }
        xsrc = P.T_out;
        double *t = pold; pold = pnew; pnew = t;
    }
    if (it == 0 && lane_ok) {
        for (int64_t i = gw; i < N; i += TW)
            reinterpret_cast<double2 *>(P.T_out + i * P.SP)[lane] = reinterpret_cast<const double2 *>(P.T_in + i * P.SP)[lane];
    }
    if (blockIdx.x == 0 && warp == 0) {
        for (int h = 0; h < 2; ++h) {
            const int s = 2 * lane + h;
            if (s >= P.S) continue;
            const double rel = t0[0][h] > 0.0 ? sqrt(rr2[h] / t0[0][h]) : sqrt(rr2[h]);
            P.iters_out[(int64_t)P.step * P.S + s] = itc[h];
            P.relres_out[(int64_t)P.step * P.S + s] = rel;
            if (!conv[h]) {
                if (atomicCAS(&P.status[0], 0, 1) == 0) {
                    P.status[2] = P.step;
                    P.status[3] = s;
                    *P.fail_relres = rel;
                }
            }
        }
        if (lane == 0) P.area_out[P.step] = area;
    }
}

__global__ void k_dinv_broadcast(const double *Dinv, int64_t N, int S, int SP, double *DinvS) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= N * SP) return;
    const int64_t i = t / SP;
    const int s = (int)(t % SP);
    DinvS[t] = s < S ? Dinv[i] : 1.0;
}

// Column windows of the windowed sweeps (host, once per context): chunk = CR consecutive rows
// of one slice (CR = 8 for 64 columns: a window then holds ~64 block-vector rows = 64 KB per
// vector); the sorted column set of the chunk is cut into runs of consecutive rows, the
// closest runs merged until at most CGW_MAXR remain.  Returns 1 if the windows fit the
// shared-memory budget (else the register-gather kernel is used), < 0 on error.
static int cgw_build(Ctx &c) {
    const int SP = c.SP;
    int CR = SP >= 48 ? 8 : (SP >= 24 ? 16 : 32);
    if (const char *e = getenv("THERMO_CGB_CR")) {   // tuning override: 4, 8, 16 or 32
        const int v = atoi(e);
        if (v == 4 || v == 8 || v == 16 || v == 32) CR = v;
    }
    const int64_t N = c.N, nsl = c.nslices;
    std::vector<int64_t> sp(nsl + 1);
    std::vector<int32_t> col((size_t)c.nnz_pad);
    CK(cudaMemcpyAsync(sp.data(), c.d_slice_ptr, sizeof(int64_t) * (nsl + 1), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaMemcpyAsync(col.data(), c.d_col, sizeof(int32_t) * col.size(), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    int wmax = 0;
    for (int64_t s = 0; s < nsl; ++s) wmax = std::max(wmax, (int)((sp[s + 1] - sp[s]) >> 5));
    const int64_t nch = (N + CR - 1) / CR;
    std::vector<int2> runs((size_t)nch * CGW_MAXR, make_int2(0, 0));
    std::vector<int32_t> nruns(nch), lown(nch);
    std::vector<uint16_t> wcol(col.size(), 0);
    std::vector<int32_t> cs;
    std::vector<int2> rv;
    int wcap = 0;
    for (int64_t ch = 0; ch < nch; ++ch) {
        const int64_t r0 = ch * CR, r1 = std::min(r0 + CR, N), s = r0 >> 5, base = sp[s];
        const int w = (int)((sp[s + 1] - base) >> 5);
        cs.clear();
        for (int64_t i = r0; i < r1; ++i)
            for (int k = 0; k < w; ++k) cs.push_back(col[base + 32 * k + (i & 31)]);
        std::sort(cs.begin(), cs.end());
        cs.erase(std::unique(cs.begin(), cs.end()), cs.end());
        rv.clear();
        for (int32_t x : cs) {
            if (!rv.empty() && rv.back().x + rv.back().y == x) rv.back().y++;
            else rv.push_back(make_int2(x, 1));
        }
        while ((int)rv.size() > CGW_MAXR) {   // bridge the smallest gap
            size_t best = 0;
            int64_t bg = INT64_MAX;
            for (size_t q = 0; q + 1 < rv.size(); ++q) {
                const int64_t g = (int64_t)rv[q + 1].x - (rv[q].x + rv[q].y);
                if (g < bg) { bg = g; best = q; }
            }
            rv[best].y = rv[best + 1].x + rv[best + 1].y - rv[best].x;
            rv.erase(rv.begin() + best + 1);
        }
        int tot = 0;
        std::vector<int> off(rv.size());
        for (size_t q = 0; q < rv.size(); ++q) { off[q] = tot; tot += rv[q].y; }
        if (tot > 65535) return 0;
        wcap = std::max(wcap, tot);
        auto local = [&](int32_t x) {
            size_t q = std::upper_bound(rv.begin(), rv.end(), x, [](int32_t v, const int2 &r) { return v < r.x; }) -
                       rv.begin() - 1;
            return off[q] + (x - rv[q].x);
        };
        nruns[ch] = (int)rv.size();
        for (size_t q = 0; q < rv.size(); ++q) runs[ch * CGW_MAXR + q] = rv[q];
        lown[ch] = local((int32_t)r0);
        for (int64_t i = r0; i < r1; ++i)
            for (int k = 0; k < w; ++k) {
                const int64_t e = base + 32 * k + (i & 31);
                wcol[e] = (uint16_t)local(col[e]);
            }
    }
    // stage layout: header | values [wmax][32] | columns [wmax][32] | interface map [32] | windows
    const size_t RB = (size_t)SP * 8;
    wcap = (wcap + 7) & ~7;
    const size_t off_col = CGW_HDR + (size_t)wmax * 32 * 8;
    const size_t off_if = off_col + (((size_t)wmax * 32 * 2 + 127) & ~(size_t)127);
    const size_t off_w1 = off_if + 128;
    const size_t off_w2 = off_w1 + (size_t)wcap * RB;
    const size_t stage = (off_w2 + (size_t)wcap * RB + 127) & ~(size_t)127;
    const size_t budget = 227 * 1024 - 128;
    const size_t red = (size_t)CGW_WARPS * CGB_NV * 64 * 8;
    int NS = (int)std::min<size_t>(8, budget / stage);
    if (const char *e = getenv("THERMO_CGB_NS")) NS = std::min(NS, std::max(2, atoi(e)));
    // a consumer group waits on parity (n / NS) & 1 of its stage: with more groups than
    // stages - 1 a group could see the phase of the chunk NS earlier, so NS >= groups + 1
    const int ngroups = 2 * CGW_NCW / (CR < CGW_NCW ? CR : CGW_NCW);
    if (NS < ngroups + 1) return 0;
    if (NS < 2 || std::max((size_t)NS * stage, red) > budget) return 0;
    c.cgw_CR = CR;
    c.cgw_NS = NS;
    c.cgw_wcap = wcap;
    c.cgw_nchunks = nch;
    c.cgw_stage = (uint32_t)stage;
    c.cgw_off[0] = (uint32_t)off_col;
    c.cgw_off[1] = (uint32_t)off_if;
    c.cgw_off[2] = (uint32_t)off_w1;
    c.cgw_off[3] = (uint32_t)off_w2;
    c.cgw_smem = 128 + std::max((size_t)NS * stage, red);
    CK(cudaMalloc(&c.d_chunk_runs, sizeof(int2) * runs.size()));
    CK(cudaMalloc(&c.d_chunk_nruns, sizeof(int32_t) * nch));
    CK(cudaMalloc(&c.d_chunk_lown, sizeof(int32_t) * nch));
    CK(cudaMalloc(&c.d_lcol, sizeof(uint16_t) * wcol.size() + 64));
    CK(cudaMemcpyAsync(c.d_chunk_runs, runs.data(), sizeof(int2) * runs.size(), cudaMemcpyHostToDevice, c.stream));
    CK(cudaMemcpyAsync(c.d_chunk_nruns, nruns.data(), sizeof(int32_t) * nch, cudaMemcpyHostToDevice, c.stream));
    CK(cudaMemcpyAsync(c.d_chunk_lown, lown.data(), sizeof(int32_t) * nch, cudaMemcpyHostToDevice, c.stream));
    CK(cudaMemcpyAsync(c.d_lcol, wcol.data(), sizeof(uint16_t) * wcol.size(), cudaMemcpyHostToDevice, c.stream));
    CK(cudaStreamSynchronize(c.stream));   // host vectors die here
    return 1;
}

int cgb_setup(Ctx &c) {
    if (c.S > CGB_MAXS) { c.err = "at most 64 scenarios per context"; return -1; }
    if (int rc = build_if_of_row(c)) return rc;
    // THERMO_CGB_KIND=1 selects the windowed sweeps; measured slower than the register gathers
    // on cfg 4, so the register kernel is the default
    const char *kind = getenv("THERMO_CGB_KIND");
    c.cgw_on = 0;
    if (kind && atoi(kind) == 1) {
        const int r = cgw_build(c);
        if (r < 0) return r;
        c.cgw_on = r;
    }
    int per_sm = 0;
    if (c.cgw_on) {
        CK(cudaFuncSetAttribute((const void *)k_cgb_step<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)c.cgw_smem));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cgb_step<true>, CGW_BLOCK, c.cgw_smem));
        c.cg_block = CGW_BLOCK;
    } else {
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cgb_step<false>, CGB_BLOCK, 0));
        c.cg_block = CGB_BLOCK;
    }
    if (per_sm < 1) { c.err = "batched CG kernel cannot be resident"; return -3; }
    c.cg_grid = (c.cgw_on ? 1 : per_sm) * c.num_sms;
    const char *ord = getenv("THERMO_CGB_ORDER");
    c.cgb_contiguous = ord ? atoi(ord) : 0;   // contiguous blocks measured 3.5x slower (L2 thrash)
    if (getenv("THERMO_CG_TRACE"))
        fprintf(stderr, "[thermo] batched CG: %s, rows/chunk %d, stages %d, window rows %d, stage %u B\n",
                c.cgw_on ? "windows" : "register gathers", c.cgw_CR, c.cgw_NS, c.cgw_wcap, c.cgw_stage);
    CK(cudaMalloc(&c.d_partials, sizeof(double) * (size_t)CGB_NV * 64 * c.cg_grid));
    CK(cudaMalloc(&c.d_DinvS, sizeof(double) * (size_t)c.N * c.SP + 16));
    return 0;
}

int cgb_prepare(Ctx &c) {
    const int64_t n = c.N * c.SP;
    k_dinv_broadcast<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(c.d_Dinv, c.N, c.S, c.SP, c.d_DinvS);
    CK(cudaGetLastError());
    return 0;
}

int cgb_launch_step(Ctx &c, int step, double dt) {
    CGBParams P;
    memset(&P, 0, sizeof P);
    P.N = c.N;
    P.nslices = c.nslices;
    P.S = c.S;
    P.SP = c.SP;
    P.slice_ptr = c.d_slice_ptr;
    P.col = c.d_col;
    P.val = c.d_val;
    P.ML = c.d_ML;
    P.benv = c.d_benv;
    P.DinvS = c.d_DinvS;
    P.n_if = c.n_if;
    P.nA = c.nA;
    P.cap = c.cap;
    P.if_rows = c.d_if_rows;
    P.slice_if = c.d_slice_if;
    P.if_of_row = c.d_if_of_row;
    P.ell_cnt = c.d_ell_cnt;
    P.ell_col = c.d_ell_col;
    P.ell_val = c.d_ell_val;
    P.if_b = c.d_if_b;
    P.if_phi = c.d_if_phi;
    P.T_in = c.d_T[(c.cur + step) & 1];
    P.T_out = c.d_T[(c.cur + step + 1) & 1];
    P.z = c.d_z;
    P.pa = c.d_p[0];
    P.pb = c.d_p[1];
    P.q = c.d_q;
    P.partials = c.d_partials;
    P.status = c.d_status;
    P.fail_relres = c.d_fail_relres;
    P.iters_out = c.d_iters;
    P.relres_out = c.d_relres;
    P.area_out = c.d_area;
    P.dt = dt;
    P.rtol2 = c.rtol * c.rtol;
    P.maxit = c.maxit > 0 ? c.maxit : (int)std::min<int64_t>(10 * c.N, 10000);
    P.step = step;
    P.trace = c.d_trace;
    P.contiguous = c.cgb_contiguous;
    void *args[] = {&P};
    if (c.cgw_on) {
        P.CR = c.cgw_CR;
        P.NS = c.cgw_NS;
        P.wcap = c.cgw_wcap;
        P.nchunks = c.cgw_nchunks;
        P.stage_bytes = c.cgw_stage;
        P.off_col = c.cgw_off[0];
        P.off_if = c.cgw_off[1];
        P.off_w1 = c.cgw_off[2];
        P.off_w2 = c.cgw_off[3];
        P.wruns = c.d_chunk_runs;
        P.wnruns = c.d_chunk_nruns;
        P.wlown = c.d_chunk_lown;
        P.wcol = c.d_lcol;
        CK(cudaLaunchCooperativeKernel((const void *)k_cgb_step<true>, dim3(c.cg_grid), dim3(c.cg_block), args,
                                       c.cgw_smem, c.stream));
    } else {
        CK(cudaLaunchCooperativeKernel((const void *)k_cgb_step<false>, dim3(c.cg_grid), dim3(c.cg_block), args, 0,
                                       c.stream));
    }
    return 0;
}

}  // namespace thermo
