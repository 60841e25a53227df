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
// Per CG iteration (z-primary, column-wise):
//   P: p = z + beta p_old (streaming pass; first iteration p = z), grid barrier
//   S: q = K~ p (warp per row pair: the rows' entries are broadcast by shuffles, every lane
//      gathers its two columns of p with L2-only loads), partial p.q per column
//   U: x += alpha p, z -= alpha D^{-1} q, partial r.z, r.r per column
// Forming p in its own pass (instead of z + beta p_old on the fly for every gathered column, as
// the single-vector kernel does from shared memory) halves the gathered bytes: the gathers are
// latency-bound with the rows held in registers, so one vector per entry allows twice the
// entries per round.
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
    const double *X0;          // optional initial guess (extrapolated states); nullptr: x0 = T_in
    const double *rhs;         // optional explicit right-hand side block (SDC / MRSDC solves)
    int use_iface;             // 0: no interface rows (the MRSDC implicit operator is volume only)
    double *T_out, *z, *pa, *pb, *q;
    double *partials;   // [G][CGB_NV][64]
    int *status;
    double *fail_relres;
    int32_t *iters_out;
    double *relres_out, *area_out;
    double dt, rtol2;
    int maxit, step;
    unsigned long long *trace;   // optional: %globaltimer after every grid barrier (CTA 0)
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
            for (int u = 0; u < 8; ++u) v[u] = ld_cg1(partials + (int64_t)(g + u) * CGB_NV * 64 + t);   // L2, not a stale L1 line
#pragma unroll
            for (int u = 0; u < 8; ++u) a += v[u];
        }
        for (; g < G; ++g) a += ld_cg1(partials + (int64_t)g * CGB_NV * 64 + t);
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
template <bool kTwo, int U, bool CGL = false>
__device__ __forceinline__ void gather_round(const CGBParams &P, int cl, double vl, int m, const double *x1,
                                             const double *x2, double2 beta, int ln, double2 &accA, double2 &accB) {
    for (int k = 0; k < m; k += U) {
        double2 yA[U], yB[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {   // all gathers of the round first
            const int ku = min(k + u, m - 1);
            const int cA = __shfl_sync(0xffffffffu, cl, ku);
            const int cB = __shfl_sync(0xffffffffu, cl, 16 + ku);
            const double2 *pa = reinterpret_cast<const double2 *>(x1 + (int64_t)cA * P.SP) + ln;
            const double2 *pb = reinterpret_cast<const double2 *>(x1 + (int64_t)cB * P.SP) + ln;
            const double2 a = CGL ? ld_cg2(pa) : *pa;
            const double2 b = CGL ? ld_cg2(pb) : *pb;
            if (kTwo) {
                const double2 *qa = reinterpret_cast<const double2 *>(x2 + (int64_t)cA * P.SP) + ln;
                const double2 *qb = reinterpret_cast<const double2 *>(x2 + (int64_t)cB * P.SP) + ln;
                const double2 a2 = CGL ? ld_cg2(qa) : *qa;
                const double2 b2 = CGL ? ld_cg2(qb) : *qb;
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
template <bool kTwo, bool CGL = false>
__device__ __forceinline__ void row_spmm2(const CGBParams &P, int64_t base, int w, int rA, bool validB, int cl,
                                          double vl, const double *x1, const double *x2, double2 beta, int lane,
                                          double2 &accA, double2 &accB) {
    accA = make_double2(0.0, 0.0);
    accB = make_double2(0.0, 0.0);
    const int ln = 2 * lane < P.SP ? lane : 0;   // lanes past the row stride re-read columns 0..1
    constexpr int U = kTwo ? 4 : 8;
    gather_round<kTwo, U, CGL>(P, cl, vl, min(16, w), x1, x2, beta, ln, accA, accB);
    for (int k0 = 16; k0 < w; k0 += 16) {
        load_cv(P, base, w, rA, validB, k0, lane, cl, vl);
        gather_round<kTwo, U, CGL>(P, cl, vl, min(16, w - k0), x1, x2, beta, ln, accA, accB);
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
                m_ikA = P.use_iface ? P.if_of_row[iA] : -1;
                m_ikB = P.use_iface && iA + 1 < N ? P.if_of_row[iA + 1] : -1;
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
        // rounds of 8 entries: all column / value loads, then all gathers, then the sums in
        // ascending entry order (same order as one at a time)
        for (int c0 = 0; c0 < cnt; c0 += 8) {
            int j[8];
            double v[8], y[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t e = ellb(P, s, min(c0 + u, cnt - 1), ik);
                j[u] = P.ell_col[e];
                v[u] = P.ell_val[e];
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                y[u] = x1[(int64_t)j[u] * P.SP + s];
                if (kTwo) y[u] = fma(b, x2[(int64_t)j[u] * P.SP + s], y[u]);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (c0 + u < cnt) a = fma(v[u], y[u], a);
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

__global__ void __launch_bounds__(CGB_BLOCK, 1) k_cgb_step(CGBParams P) {
    constexpr int NW = CGB_WARPS;
    __shared__ double sm[CGB_WARPS * CGB_NV * 64];
    // an earlier step failed, or the interface of this or an earlier step overflowed
    if (P.status[0] || (P.status[1] && P.status[4] <= P.step)) {
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
    // ---- phase 0: r0 = b - K~ x0, z0 = D^{-1} r0 per column (b = M_L T^n + dt (b_env + b_G);
    // x0 = T^n or the extrapolated guess X0)
    const double *const x0 = P.X0 ? P.X0 : P.T_in;
    double v0[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};   // b.b, r.r, r.z, |Gamma_R| (scenario 0)
    const int64_t npairs = P.nslices * 16;   // units: (slice, row pair)
    // epilogue of one row: ax = (K~ x0)_i without the interface part, Ti = x0_i
    auto fin0 = [&](int64_t i, int ik, double2 ax, double2 Ti, double2 di) {
        double2 bg = make_double2(0.0, 0.0);
        if (ik >= 0) {
            const double2 ai = row_iface<false>(P, ik, x0, nullptr, make_double2(0, 0), lane);
            ax.x += ai.x;
            ax.y += ai.y;
            if (col_ok[0]) bg.x = P.if_b[(int64_t)ik * P.S + 2 * lane];
            if (col_ok[1]) bg.y = P.if_b[(int64_t)ik * P.S + 2 * lane + 1];
            if (lane == 0 && ik < P.nA) v0[3][0] += P.if_phi[(int64_t)ik * P.S];
        }
        if (!lane_ok) return;
        double2 b, rr, zz;
        if (P.rhs) {
            b = reinterpret_cast<const double2 *>(P.rhs + i * P.SP)[lane];
        } else {
            const double ml = P.ML[i], be = P.benv[i];
            b.x = fma(ml, Ti.x, P.dt * (be + bg.x));
            b.y = fma(ml, Ti.y, P.dt * (be + bg.y));
        }
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
    unit_loop(P, npairs, gw, TW, lane, [&](int64_t u, int64_t base, int w, int rA, bool validB, int ikA,
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
        row_spmm2<false>(P, base, w, rA, validB, cl, vl, x0, nullptr, make_double2(0, 0), lane, axr[0],
                         axr[1]);
        fin0(iA, ikA, axr[0], Tr[0], dr[0]);
        if (validB) fin0(iA + 1, ikB, axr[1], Tr[1], dr[1]);
    });
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
    const double *xsrc = x0;
    double *pold = P.pa, *pnew = P.pb;
    int it = 0;
    while (it < P.maxit) {
        const bool any = __syncthreads_or(!(conv[0] && conv[1])) != 0;   // same in every CTA
        if (!any) break;
        // ---- S: p = z + beta p_old in its own streaming pass (first iteration: p = z), then
        // q = K~ p gathering p only -- one vector, 8 entries per round -- with L2-only loads
        // (p was written by other SMs moments ago; L1-allocating gathers of it ran 2.8x slower)
        const bool first = it == 0;
        const double2 b2 = make_double2(beta[0], beta[1]);
        const double *pv = first ? P.z : pnew;
        double vs[1][2] = {{0.0, 0.0}};
        if (!first) {
            if (lane_ok) {
                int64_t i = gw;
                for (; i + 3 * (int64_t)TW < N; i += 4 * (int64_t)TW) {   // 4 rows in flight
                    double2 zv[4], po[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        zv[r] = ld_cg2(reinterpret_cast<const double2 *>(P.z + (i + r * (int64_t)TW) * P.SP) + lane);
                        po[r] = ld_cg2(reinterpret_cast<const double2 *>(pold + (i + r * (int64_t)TW) * P.SP) + lane);
                    }
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        reinterpret_cast<double2 *>(pnew + (i + r * (int64_t)TW) * P.SP)[lane] =
                            make_double2(fma(b2.x, po[r].x, zv[r].x), fma(b2.y, po[r].y, zv[r].y));
                }
                for (; i < N; i += TW) {
                    const double2 zv = ld_cg2(reinterpret_cast<const double2 *>(P.z + i * P.SP) + lane);
                    const double2 po = ld_cg2(reinterpret_cast<const double2 *>(pold + i * P.SP) + lane);
                    reinterpret_cast<double2 *>(pnew + i * P.SP)[lane] =
                        make_double2(fma(b2.x, po.x, zv.x), fma(b2.y, po.y, zv.y));
                }
            }
            grid.sync();
        }
        unit_loop(P, npairs, gw, TW, lane, [&](int64_t u, int64_t base, int w, int rA, bool validB, int ikA,
                                               int ikB, int cl, double vl) {
            const int64_t iA = 32 * (u >> 4) + rA;
            double2 own[2];   // own rows of p, loaded ahead of the gathers
            if (lane_ok) {
                own[0] = ld_cg2(reinterpret_cast<const double2 *>(pv + iA * P.SP) + lane);
                if (validB) own[1] = ld_cg2(reinterpret_cast<const double2 *>(pv + (iA + 1) * P.SP) + lane);
            }
            double2 accr[2];
            row_spmm2<false, true>(P, base, w, rA, validB, cl, vl, pv, nullptr, b2, lane, accr[0], accr[1]);
            for (int h = 0; h < 2; ++h) {
                if (h == 1 && !validB) break;
                const int64_t i = iA + h;
                const int ik = h ? ikB : ikA;
                double2 acc = accr[h];
                if (ik >= 0) {
                    const double2 ai = row_iface<false>(P, ik, pv, nullptr, b2, lane);
                    acc.x += ai.x;
                    acc.y += ai.y;
                }
                if (!lane_ok) continue;
                const double2 pi = own[h];
                if (first) reinterpret_cast<double2 *>(pnew + i * P.SP)[lane] = pi;   // p_0 = z_0
                reinterpret_cast<double2 *>(P.q + i * P.SP)[lane] = acc;
                vs[0][0] = fma(pi.x, acc.x, vs[0][0]);
                vs[0][1] = fma(pi.y, acc.y, vs[0][1]);
            }
        });
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
            reinterpret_cast<double2 *>(P.T_out + i * P.SP)[lane] = reinterpret_cast<const double2 *>(x0 + i * P.SP)[lane];
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
        if (lane == 0 && P.area_out) P.area_out[P.step] = area;
    }
}

__global__ void k_dinv_broadcast(const double *Dinv, int64_t N, int S, int SP, double *DinvS) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= N * SP) return;
    const int64_t i = t / SP;
    const int s = (int)(t % SP);
    DinvS[t] = s < S ? Dinv[i] : 1.0;
}

int cgb_setup(Ctx &c) {
    if (c.S > CGB_MAXS) { c.err = "at most 64 scenarios per context"; return -1; }
    if (int rc = build_if_of_row(c)) return rc;
    if (int rc = sbcg_setup(c)) return rc;
    if (c.sb_on) return 0;   // windowed SpMM kernel (cg_spmm.cu)
    return cgb_gather_setup(c);
}

int cgb_gather_setup(Ctx &c) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cgb_step, CGB_BLOCK, 0));
    if (per_sm < 1) { c.err = "batched CG kernel cannot be resident"; return -3; }
    c.cg_block = CGB_BLOCK;
    c.cg_grid = per_sm * c.num_sms;
    CK(cudaMalloc(&c.d_partials, sizeof(double) * (size_t)CGB_NV * 64 * c.cg_grid));
    CK(cudaMalloc(&c.d_DinvS, sizeof(double) * (size_t)c.N * c.SP + 16));
    return 0;
}

int cgb_prepare(Ctx &c) {
    if (c.sb_on) return sbcg_prepare(c);   // row-major copy of the rebuilt operator (cg_spmm.cu)
    const int64_t n = c.N * c.SP;
    k_dinv_broadcast<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(c.d_Dinv, c.N, c.S, c.SP, c.d_DinvS);
    CK(cudaGetLastError());
    return 0;
}

static void cgb_params(Ctx &c, CGBParams &P) {
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
    P.z = c.d_z;
    P.pa = c.d_p[0];
    P.pb = c.d_p[1];
    P.q = c.d_q;
    P.partials = c.d_partials;
    P.status = c.d_status;
    P.fail_relres = c.d_fail_relres;
    P.rtol2 = c.rtol * c.rtol;
    P.maxit = c.maxit > 0 ? c.maxit : (int)std::min<int64_t>(10 * c.N, 10000);
    P.trace = c.d_trace;
}

// Solve with an explicit right-hand side block (SDC / MRSDC implicit stages, every scenario)
int cgb_launch_solve(Ctx &c, const double *x0, double *x, const double *rhs, bool iface, int32_t *iters_out,
                     double *relres_out, int slot) {
    if (c.sb_on) { c.err = "internal: explicit-rhs solve on the windowed SpMM kernel (sbcg_disable first)"; return -1; }
    CGBParams P;
    cgb_params(c, P);
    P.T_in = x0;
    P.X0 = nullptr;
    P.T_out = x;
    P.rhs = rhs;
    P.use_iface = iface ? 1 : 0;
    P.iters_out = iters_out;
    P.relres_out = relres_out;
    P.area_out = nullptr;
    P.dt = 0.0;
    P.step = slot;
    void *args[] = {&P};
    CK(cudaLaunchCooperativeKernel((const void *)k_cgb_step, dim3(c.cg_grid), dim3(c.cg_block), args, 0, c.stream));
    return 0;
}

int cgb_launch_step(Ctx &c, int step, double dt, const double *x0) {
    if (c.sb_on) return sbcg_launch_step(c, step, dt, x0);
    CGBParams P;
    cgb_params(c, P);
    P.T_in = c.d_T[(c.cur + step) & 1];
    P.X0 = x0;
    P.T_out = c.d_T[(c.cur + step + 1) & 1];
    P.iters_out = c.d_iters;
    P.relres_out = c.d_relres;
    P.area_out = c.d_area;
    P.dt = dt;
    P.step = step;
    P.use_iface = 1;
    void *args[] = {&P};
    CK(cudaLaunchCooperativeKernel((const void *)k_cgb_step, dim3(c.cg_grid), dim3(c.cg_block), args, 0, c.stream));
    return 0;
}

}  // namespace thermo
