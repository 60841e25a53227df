// cg.cu -- the implicit-Euler solve (M_L - dt K(t')) T^{n+1} = M_L T^n + dt (b_env + b_G)
// by Jacobi-preconditioned CG, one persistent cooperative kernel per
// time step.
//
// Schedule per CG iteration, z-primary Jacobi-PCG:
//   S: p = z + beta p_old (recomputed on the fly for every gathered column),
//      q = K~ p (sliced-ELL volume part + per-step interface rows), partial p.q
//   -- grid barrier; alpha = rho / p.q
//   U: x += alpha p ; z -= alpha D^{-1} q ; r = z / D^{-1} ; partials r.z, r.r
//   -- grid barrier; beta = r.z / rho, convergence test ||r||^2 <= rtol^2 ||b||^2
// Every value of every reduction is combined in a fixed order (deterministic, identical in
// all CTAs), so all CTAs take the same control-flow decisions.
#include <cooperative_groups.h>

#include <cmath>

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

struct CGParams {
    int64_t N, nslices;
    const int64_t *slice_ptr;
    const int32_t *col;
    const double *val;
    const double *ML, *benv, *Dinv;
    int n_if, nA;
    const int32_t *if_rows, *slice_if, *ell_cnt, *ell_col;
    const double *ell_val, *if_b, *if_phi;
    const double *T_in;
    double *T_out, *z, *pa, *pb, *q;
    double *partials;
    int *status;
    double *fail_relres;
    int32_t *iters_out;
    double *relres_out, *area_out;
    double dt, rtol2;
    int maxit, step;
};

// Interface index of the row owned by this lane (-1 if none).  Warp-uniform call.
__device__ __forceinline__ int iface_index(const CGParams &P, int64_t s, int64_t i, int lane) {
    const int b = P.slice_if[s], e = P.slice_if[s + 1];
    if (b == e) return -1;
    const int m = e - b;
    const int mine = lane < m ? P.if_rows[b + lane] : -1;
    int ik = -1;
    for (int j = 0; j < m; ++j) {
        int rj = __shfl_sync(0xffffffffu, mine, j);
        if (rj == (int)i) ik = b + j;
    }
    return ik;
}

// y_i = sum_k val * (x1[col] + beta * x2[col]) over the sliced-ELL row of this lane.
template <bool kTwo>
__device__ __forceinline__ double sell_row(const CGParams &P, int64_t s, int lane, const double *x1,
                                           const double *x2, double beta) {
    const int64_t b0 = P.slice_ptr[s], b1 = P.slice_ptr[s + 1];
    const int w = (int)((b1 - b0) >> 5);
    const int32_t *cp = P.col + b0 + lane;
    const double *vp = P.val + b0 + lane;
    const uint64_t pol = policy_evict_first();
    double acc = 0.0;
    int k = 0;
    for (; k + 4 <= w; k += 4) {
        int c0 = ld_stream(cp + 32 * (k + 0), pol);
        int c1 = ld_stream(cp + 32 * (k + 1), pol);
        int c2 = ld_stream(cp + 32 * (k + 2), pol);
        int c3 = ld_stream(cp + 32 * (k + 3), pol);
        double v0 = ld_stream(vp + 32 * (k + 0), pol);
        double v1 = ld_stream(vp + 32 * (k + 1), pol);
        double v2 = ld_stream(vp + 32 * (k + 2), pol);
        double v3 = ld_stream(vp + 32 * (k + 3), pol);
        double y0 = x1[c0], y1 = x1[c1], y2 = x1[c2], y3 = x1[c3];
        if (kTwo) {
            y0 = fma(beta, x2[c0], y0);
            y1 = fma(beta, x2[c1], y1);
            y2 = fma(beta, x2[c2], y2);
            y3 = fma(beta, x2[c3], y3);
        }
        acc = fma(v0, y0, acc);
        acc = fma(v1, y1, acc);
        acc = fma(v2, y2, acc);
        acc = fma(v3, y3, acc);
    }
    for (; k < w; ++k) {
        int c0 = ld_stream(cp + 32 * k, pol);
        double v0 = ld_stream(vp + 32 * k, pol);
        double y0 = x1[c0];
        if (kTwo) y0 = fma(beta, x2[c0], y0);
        acc = fma(v0, y0, acc);
    }
    return acc;
}

template <bool kTwo>
__device__ __forceinline__ double ell_row(const CGParams &P, int ik, const double *x1, const double *x2,
                                          double beta) {
    const int cnt = P.ell_cnt[ik];
    double acc = 0.0;
    for (int c = 0; c < cnt; ++c) {
        const int64_t e = (int64_t)c * P.n_if + ik;
        const int j = P.ell_col[e];
        double y = x1[j];
        if (kTwo) y = fma(beta, x2[j], y);
        acc = fma(P.ell_val[e], y, acc);
    }
    return acc;
}

__global__ void __launch_bounds__(THERMO_BLOCK) k_cg_step(CGParams P) {
    __shared__ double smem[128];
    if (P.status[0] || P.status[1]) {   // an earlier step failed or the interface overflowed
        if (!P.status[0] && blockIdx.x == 0 && threadIdx.x == 0) {
            P.status[0] = 2;
            P.status[2] = P.step;
        }
        return;
    }
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * THERMO_WARPS + (threadIdx.x >> 5);
    const int TW = gridDim.x * THERMO_WARPS;
    const int G = gridDim.x;
    const int64_t N = P.N;

    // ---- r0 = b - K~ x0 with x0 = T^n, b = M_L T^n + dt (b_env + b_G); z0 = D^{-1} r0
    double red0[4] = {0.0, 0.0, 0.0, 0.0};   // b.b, r.r, r.z, |Gamma_R|
    for (int64_t s = gw; s < P.nslices; s += TW) {
        const int64_t i = 32 * s + lane;
        const int ik = iface_index(P, s, i, lane);
        double ax = sell_row<false>(P, s, lane, P.T_in, nullptr, 0.0);
        if (ik >= 0) ax += ell_row<false>(P, ik, P.T_in, nullptr, 0.0);
        if (i < N) {
            const double Ti = P.T_in[i];
            double bi = P.benv[i];
            if (ik >= 0) bi += P.if_b[ik];
            bi = fma(P.ML[i], Ti, P.dt * bi);
            const double r = bi - ax;
            const double zi = P.Dinv[i] * r;
            P.z[i] = zi;
            red0[0] = fma(bi, bi, red0[0]);
            red0[1] = fma(r, r, red0[1]);
            red0[2] = fma(r, zi, red0[2]);
            if (ik >= 0 && ik < P.nA) red0[3] += P.if_phi[ik];
        }
    }
    cta_reduce_store<4>(red0, smem, P.partials, 0);
    grid.sync();
    double tot0[4];
    grid_total<4>(P.partials, G, 0, smem, tot0);
    const double tol2 = P.rtol2 * tot0[0];
    double rho = tot0[2], rr = tot0[1];
    bool conv = rr <= tol2;
    double beta = 0.0;
    const double *xsrc = P.T_in;
    double *pold = P.pa, *pnew = P.pb;
    int it = 0;
    while (!conv && it < P.maxit) {
        // ---- S: p = z + beta p_old, q = K~ p, partial p.q
        double pq[1] = {0.0};
        const bool first = it == 0;
        for (int64_t s = gw; s < P.nslices; s += TW) {
            const int64_t i = 32 * s + lane;
            const int ik = iface_index(P, s, i, lane);
            double acc;
            if (first) {
                acc = sell_row<false>(P, s, lane, P.z, nullptr, 0.0);
                if (ik >= 0) acc += ell_row<false>(P, ik, P.z, nullptr, 0.0);
            } else {
                acc = sell_row<true>(P, s, lane, P.z, pold, beta);
                if (ik >= 0) acc += ell_row<true>(P, ik, P.z, pold, beta);
            }
            if (i < N) {
                const double pi = first ? P.z[i] : fma(beta, pold[i], P.z[i]);
                pnew[i] = pi;
                P.q[i] = acc;
                pq[0] = fma(pi, acc, pq[0]);
            }
        }
        cta_reduce_store<1>(pq, smem, P.partials, 4);
        grid.sync();
        double tpq[1];
        grid_total<1>(P.partials, G, 4, smem, tpq);
        const double alpha = rho / tpq[0];
        // ---- U: x += alpha p, z -= alpha D^{-1} q, partials r.z and r.r (r = z / D^{-1})
        double red[2] = {0.0, 0.0};
        for (int64_t s = gw; s < P.nslices; s += TW) {
            const int64_t i = 32 * s + lane;
            if (i < N) {
                const double di = P.Dinv[i];
                P.T_out[i] = fma(alpha, pnew[i], xsrc[i]);
                const double zi = fma(-alpha * di, P.q[i], P.z[i]);
                P.z[i] = zi;
                const double r = zi / di;
                red[0] = fma(r, zi, red[0]);
                red[1] = fma(r, r, red[1]);
            }
        }
        cta_reduce_store<2>(red, smem, P.partials, 5);
        grid.sync();
        double tr[2];
        grid_total<2>(P.partials, G, 5, smem, tr);
        beta = tr[0] / rho;
        rho = tr[0];
        rr = tr[1];
        conv = rr <= tol2;
        xsrc = P.T_out;
        double *t = pold; pold = pnew; pnew = t;
        ++it;
    }
    if (it == 0) {   // already converged: T^{n+1} = T^n
        for (int64_t s = gw; s < P.nslices; s += TW) {
            const int64_t i = 32 * s + lane;
            if (i < N) P.T_out[i] = P.T_in[i];
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const double rel = tot0[0] > 0.0 ? sqrt(rr / tot0[0]) : sqrt(rr);
        P.iters_out[P.step] = it;
        P.relres_out[P.step] = rel;
        P.area_out[P.step] = tot0[3];
        if (!conv) {
            P.status[0] = 1;
            P.status[2] = P.step;
            P.status[3] = 0;
            *P.fail_relres = rel;
        }
    }
}

int cg_setup(Ctx &c) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cg_step, THERMO_BLOCK, 0));
    if (per_sm < 1) { c.err = "CG kernel cannot be resident"; return -3; }
    c.cg_grid = per_sm * c.num_sms;
    CK(cudaMalloc(&c.d_partials, sizeof(double) * THERMO_NRED * c.cg_grid));
    return 0;
}

int cg_launch_step(Ctx &c, int step, double dt) {
    CGParams P;
    P.N = c.N;
    P.nslices = c.nslices;
    P.slice_ptr = c.d_slice_ptr;
    P.col = c.d_col;
    P.val = c.d_val;
    P.ML = c.d_ML;
    P.benv = c.d_benv;
    P.Dinv = c.d_Dinv;
    P.n_if = c.n_if;
    P.nA = c.nA;
    P.if_rows = c.d_if_rows;
    P.slice_if = c.d_slice_if;
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
    void *args[] = {&P};
    CK(cudaLaunchCooperativeKernel((const void *)k_cg_step, dim3(c.cg_grid), dim3(THERMO_BLOCK), args, 0,
                                   c.stream));
    return 0;
}

}  // namespace thermo
