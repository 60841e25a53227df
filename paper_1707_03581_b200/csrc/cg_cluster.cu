// cg_cluster.cu -- latency path of the single-scenario Jacobi-PCG solve for paper-scale
// problems (the paper's model has 16,626 DoF; its metric is the look-ahead factor,
// P:189-194).  At that size a solve is bound by synchronisation latency, not bandwidth: the
// persistent grid kernel (cg.cu) spends ~12 us per CG iteration in TMA round trips and grid-wide
// barriers over 148 CTAs.  Here one thread-block cluster of CL_CTAS CTAs (16, the non-portable
// Blackwell maximum) does the whole solve:
//   * every CTA owns a contiguous block of slices; its rows' x, z, p and q' live in shared
//     memory for the whole solve, only p is also stored to global memory (L2) for the other
//     CTAs' gathers;
//   * thread per row, sliced-ELL entries read through the read-only path (the matrix of a CTA
//     stays in its L1 across iterations), p gathered from L2 (ld.global.cg: written by other
//     CTAs of the cluster in the previous phase);
//   * reductions: per-thread sums in row order, warp xor-butterflies, warps in fixed order, then
//     the CTA partials of the cluster read through distributed shared memory in rank order
//     (double-buffered slots) -- deterministic, every CTA computes identical scalars;
//   * barrier.cluster (hardware, release/acquire at cluster scope) instead of grid.sync.
// Same z-primary iteration and the same safeguards as the grid kernel: S forms q = K~ p, q' =
// q / d and the seven sums that give alpha and beta; U forms x, z and the next p.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ctx.h"
#include "cg_params.h"

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

#define CL_CTAS 16
#define CL_THREADS 512
#define CL_RPT 8   // rows per thread (max): N <= CL_CTAS * CL_THREADS * CL_RPT

// sum of NV per-thread values over the cluster (deterministic): warp butterflies, warps in
// order, then the CTA partials of every rank in rank order via DSMEM; slot alternates so that a
// CTA can start the next reduction while a slower one still reads this one's partials
template <int NV>
__device__ __forceinline__ void cl_reduce(double (&v)[NV], double *wred, double *part, int slot,
                                          cg::cluster_group &cl, double (&out)[NV]) {
    __shared__ double tot_s[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = warp_sum(v[j]);
    if (lane == 0)
#pragma unroll
        for (int j = 0; j < NV; ++j) wred[warp * NV + j] = v[j];
    __syncthreads();
    if (warp < NV) {   // warp j: the CTA total of value j (lane w holds warp w's partial)
        const double a = warp_sum(lane < nw ? wred[lane * NV + warp] : 0.0);
        if (lane == 0) part[slot * 8 + warp] = a;
    }
    cl.sync();   // every rank's partials written (release / acquire at cluster scope)
    if (warp < NV) {   // warp j: lane r reads rank r's partial through DSMEM, all at once
        const int nr = (int)cl.num_blocks();
        const double a = warp_sum(lane < nr ? cl.map_shared_rank(part, lane)[slot * 8 + warp] : 0.0);
        if (lane == 0) tot_s[warp] = a;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NV; ++j) out[j] = tot_s[j];
}

// row sums sum_k val_k x[col_k] of up to two sliced-ELL rows (entries at stride 32) at once,
// every load of a round issued before its FMAs; x from L2.  d[] = entry 0 (the diagonal).
__device__ __forceinline__ void cl_rows2(const CGParams &P, const int64_t (&i)[2], int nr, const double *x,
                                         double (&acc)[2], double (&d)[2]) {
    const int32_t *cp[2];
    const double *vp[2];
    int w[2] = {0, 0};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        acc[h] = 0.0;
        d[h] = 1.0;
        cp[h] = P.col;
        vp[h] = P.val;
        if (h < nr) {
            const int64_t sl = i[h] >> 5, b0 = __ldg(P.slice_ptr + sl);
            w[h] = (int)((__ldg(P.slice_ptr + sl + 1) - b0) >> 5);
            cp[h] = P.col + b0 + (i[h] & 31);
            vp[h] = P.val + b0 + (i[h] & 31);
        }
    }
    const int wm = max(w[0], w[1]);
    for (int k = 0; k < wm; k += 4) {   // rounds of 4 entries of both rows
        int c[2][4];
        double v[2][4], y[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool on = k + u < w[h];
                c[h][u] = on ? __ldg(cp[h] + 32 * (k + u)) : 0;
                v[h][u] = on ? __ldg(vp[h] + 32 * (k + u)) : 0.0;
            }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int u = 0; u < 4; ++u) y[h][u] = k + u < w[h] ? ld_cg1(x + c[h][u]) : 0.0;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (k + u < w[h]) acc[h] = fma(v[h][u], y[h][u], acc[h]);
        if (k == 0)
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if (w[h] > 0) d[h] = v[h][0];   // entry 0 = the volume diagonal (assembly order)
    }
}

// Interface rows, spread over the whole cluster (the rail-top rows of lattice order sit in one
// or two CTAs' slices): a group of 8 threads per interface row k takes the entries c = g, g + 8,
// ... (columns / values through the read-only path: constant during the solve), gathers x from
// L2, sums in a fixed order (xor butterfly over the group) and stores ai[k] = sum val x[col] and
// aself[k] = the entry on the row's own column; the owner adds them after a cluster barrier.
__device__ __forceinline__ void cl_iface_pass(const CGParams &P, int rank, int nct, const double *x, double *ai,
                                              double *aself) {
    const int nif = P.n_if;
    if (!nif) return;
    const int k0 = (int)((int64_t)nif * rank / nct), k1 = (int)((int64_t)nif * (rank + 1) / nct);
    const int g = threadIdx.x & 7, grp = threadIdx.x >> 3, ngrp = blockDim.x >> 3;
    for (int kb = k0; kb < k1; kb += ngrp) {   // warp-uniform trip count
        const int k = kb + grp;
        const bool on = k < k1;
        const int cnt = on ? __ldg(P.ell_cnt + k) : 0;
        const int64_t row = on ? (int64_t)__ldg(P.if_rows + k) : -1;
        double a = 0.0, self = 0.0;
        for (int c0 = 0; c0 < cnt; c0 += 32) {   // 4 entries per thread per round
            int j[4];
            double v[4], y[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int c = c0 + g + 8 * u;
                const int64_t e = (int64_t)min(c, cnt - 1) * nif + k;
                j[u] = __ldg(P.ell_col + e);
                v[u] = c < cnt ? __ldg(P.ell_val + e) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) y[u] = ld_cg1(x + j[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                a = fma(v[u], y[u], a);
                if (j[u] == row) self += v[u];
            }
        }
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            self += __shfl_xor_sync(0xffffffffu, self, o);
        }
        if (on && g == 0) {
            ai[k] = a;
            aself[k] = self;
        }
    }
}

__global__ void __launch_bounds__(CL_THREADS, 1) k_cg_cluster(CGParams P) {
    extern __shared__ __align__(16) double cl_smem[];
    __shared__ double wred[(CL_THREADS / 32) * 8];
    __shared__ double part[2 * 8];
    cg::cluster_group cl = cg::this_cluster();
    // an earlier step failed, or the interface of this or an earlier step overflowed (read by
    // every CTA before any of them writes the status: the decision is uniform over the cluster)
    const bool skip = P.status[0] || (P.status[1] && P.status[4] <= P.step);
    cl.sync();
    if (skip) {
        if (!P.status[0] && cl.block_rank() == 0 && threadIdx.x == 0) {
            P.status[0] = 2;
            P.status[2] = P.step;
        }
        return;
    }
    const int rank = (int)cl.block_rank(), nct = (int)cl.num_blocks();
    const int64_t N = P.N;
    const int64_t s0 = P.nslices * rank / nct, s1 = P.nslices * (rank + 1) / nct;
    const int64_t r0 = 32 * s0, r1 = min(N, 32 * s1);
    const int64_t nloc = r1 - r0;                    // rows of this CTA
    const int64_t cap = P.cl_rows;                   // shared-memory rows per vector (host: max nloc)
    // own rows in shared memory: x, z, p, q' (q: the volume part of interface rows until their
    // interface sums arrive), the volume diagonal, the interface index
    double *xs = cl_smem, *zs = xs + cap, *ps = zs + cap, *qs = ps + cap, *dvs = qs + cap;
    int *iks = reinterpret_cast<int *>(dvs + cap);
    const int t = threadIdx.x;
    const bool tr_on = P.trace && rank == 0 && t == 0;
    int ntr = 0;
    if (tr_on) P.trace[ntr++] = gtimer();
    const double *const x0 = P.X0 ? P.X0 : P.T_in;
    double *const pg = P.pa;   // global p (gathered by every CTA)
    double *const ai = P.z2, *const aself = P.q2;   // interface sums (cluster scratch, n_if each)
    const bool iface = P.n_if > 0;
    // ---- phase 0: r0 = b - K~ x0, z0 = D^{-1} r0, p0 = z0; b = M_L T^n + dt (b_env + b_G) or rhs
    double red0[4] = {0.0, 0.0, 0.0, 0.0};   // b.b, r.r, r.z, |Gamma_R|
    auto fin0 = [&](int64_t i, int64_t l, double ax, int ik) {
        double bi = P.benv[i];
        if (ik >= 0) {
            bi += P.if_b[ik];
            if (ik < P.nA) red0[3] += P.if_phi[ik];
        }
        bi = P.rhs ? P.rhs[i] : fma(P.ML[i], P.T_in[i], P.dt * bi);
        const double r = bi - ax;
        const double zi = (ik >= 0 && P.if_dinv_s ? P.if_dinv_s[ik] : P.Dinv[i]) * r;   // (ahead mode: per-slot diagonal)
        zs[l] = zi;
        ps[l] = zi;
        pg[i] = zi;
        red0[0] = fma(bi, bi, red0[0]);
        red0[1] = fma(r, r, red0[1]);
        red0[2] = fma(r, zi, red0[2]);
    };
    for (int u = 0; u < CL_RPT; u += 2) {   // two rows of this thread at a time
        const int64_t l0 = t + (int64_t)u * CL_THREADS;
        if (l0 >= nloc) break;
        const int64_t ii[2] = {r0 + l0, r0 + l0 + CL_THREADS};
        const int nr = l0 + CL_THREADS < nloc ? 2 : 1;
        double ax2[2], dd[2];
        cl_rows2(P, ii, nr, x0, ax2, dd);
        for (int h = 0; h < nr; ++h) {
            const int64_t i = ii[h], l = i - r0;
            const int ik = iface ? P.if_of_row[i] : -1;
            xs[l] = x0[i];
            dvs[l] = dd[h];
            iks[l] = ik;
            if (ik >= 0) qs[l] = ax2[h];   // finished after the interface pass
            else fin0(i, l, ax2[h], -1);
        }
    }
    if (iface) {
        cl_iface_pass(P, rank, nct, x0, ai, aself);
        cl.sync();   // interface sums of every row visible to its owner
        for (int64_t l = t; l < nloc; l += CL_THREADS) {
            const int ik = iks[l];
            if (ik >= 0) fin0(r0 + l, l, qs[l] + ld_cg1(ai + ik), ik);
        }
    }
    double tot0[4];
    cl_reduce<4>(red0, wred, part, 0, cl, tot0);   // (its cluster barrier also publishes pg)
    if (tr_on) P.trace[ntr++] = gtimer();
    const double tol2 = P.rtol2 * tot0[0];
    double rho = tot0[2], rr = tot0[1];
    bool conv = rr <= tol2;
    int it = 0, slot = 1;
    while (!conv && it < P.maxit) {
        // ---- S: q = K~ p (own rows), q' = q / d (d = volume diagonal + interface self term),
        // the seven sums of p.q and of the expansions of the next r.z and r.r (cg.cu)
        double red[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        auto finS = [&](int64_t l, double acc, double dg) {
            const double qv = acc / dg, zo = zs[l], pi = ps[l], zd = zo * dg;
            qs[l] = qv;
            red[0] = fma(pi, acc, red[0]);
            red[1] = fma(zo, zd, red[1]);
            red[2] = fma(zo, acc, red[2]);
            red[3] = fma(acc, qv, red[3]);
            red[4] = fma(zd, zd, red[4]);
            red[5] = fma(zd, acc, red[5]);
            red[6] = fma(acc, acc, red[6]);
        };
        for (int u = 0; u < CL_RPT; u += 2) {
            const int64_t l0 = t + (int64_t)u * CL_THREADS;
            if (l0 >= nloc) break;
            const int64_t ii[2] = {r0 + l0, r0 + l0 + CL_THREADS};
            const int nr = l0 + CL_THREADS < nloc ? 2 : 1;
            double a2[2], dd[2];
            cl_rows2(P, ii, nr, pg, a2, dd);
            for (int h = 0; h < nr; ++h) {
                const int64_t l = ii[h] - r0;
                if (iks[l] >= 0) qs[l] = a2[h];   // finished after the interface pass
                else finS(l, a2[h], dd[h]);
            }
        }
        if (iface) {
            cl_iface_pass(P, rank, nct, pg, ai, aself);
            cl.sync();
            for (int64_t l = t; l < nloc; l += CL_THREADS) {
                const int ik = iks[l];
                if (ik >= 0) finS(l, qs[l] + ld_cg1(ai + ik), dvs[l] + ld_cg1(aself + ik));
            }
        }
        double t7[7];
        cl_reduce<7>(red, wred, part, slot, cl, t7);
        slot ^= 1;
        if (tr_on && ntr < 1000) P.trace[ntr++] = gtimer();
        if (it > 0) {   // t7[4] = sum (z d)^2: the current r.r directly (safeguard of cg.cu)
            rr = t7[4];
            if (rr <= tol2) { conv = true; break; }
        }
        const double alpha = rho / t7[0];
        const double rz_new = fma(alpha, fma(alpha, t7[3], -2.0 * t7[2]), t7[1]);
        const double rr_new = fma(alpha, fma(alpha, t7[6], -2.0 * t7[5]), t7[4]);
        const double rr_noise = 1e-13 * (t7[4] + fabs(2.0 * alpha * t7[5]) + alpha * alpha * t7[6]);
        const double beta = rz_new / rho;
        // ---- U: x += alpha p, z -= alpha q', p = z + beta p (own rows in shared memory; p also
        // to global for the next gathers)
        for (int64_t l = t; l < nloc; l += CL_THREADS) {
            const double pv = ps[l];
            xs[l] = fma(alpha, pv, xs[l]);
            const double zn = fma(-alpha, qs[l], zs[l]);
            zs[l] = zn;
            const double pn = fma(beta, pv, zn);
            ps[l] = pn;
            pg[r0 + l] = pn;
        }
        cl.sync();   // the new p of every rank visible to the next gathers
        if (tr_on && ntr < 1000) P.trace[ntr++] = gtimer();
        rho = rz_new;
        rr = rr_new;
        conv = rr <= tol2 && rr > rr_noise;
        ++it;
    }
    for (int64_t l = t; l < nloc; l += CL_THREADS) P.T_out[r0 + l] = xs[l];
    if (rank == 0 && t == 0) {
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
    cl.sync();   // no CTA leaves while another may still read its shared memory (DSMEM)
}

// Use the cluster kernel for this context?  N small enough for its shared-memory rows, a
// 16-CTA cluster schedulable (THERMO_CG_CLUSTER=0 disables, =1 forces where possible).
int cl_setup(Ctx &c) {
    c.cl_on = false;
    const char *e = getenv("THERMO_CG_CLUSTER");
    const int mode = e ? atoi(e) : -1;
    if (mode == 0 || c.S != 1) return 0;
    int64_t rmax = 0;
    for (int r = 0; r < CL_CTAS; ++r) {
        const int64_t s0 = c.nslices * r / CL_CTAS, s1 = c.nslices * (r + 1) / CL_CTAS;
        rmax = std::max(rmax, std::min(c.N, 32 * s1) - 32 * s0);
    }
    // default: one row per thread (N <= 8,192), where it measured faster than the grid kernel
    // (cfg 0: 11.5 vs 12.8 us per CG iteration; 1,793 DoF: 11.2 vs 12.9); at two rows per thread
    // (11,856 DoF) it is slower (13.4 vs 11.9) -- THERMO_CG_CLUSTER=1 allows up to 8 rows/thread
    const int64_t limit = mode == 1 ? (int64_t)8 * CL_THREADS : (int64_t)CL_THREADS;
    if (rmax > limit) return 0;
    const size_t smem = (sizeof(double) * 5 + sizeof(int)) * (size_t)rmax + 16;
    if (smem > 200 * 1024) return 0;
    if (cudaFuncSetAttribute((const void *)k_cg_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
            cudaSuccess ||
        cudaFuncSetAttribute((const void *)k_cg_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof cfg);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL_CTAS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(CL_CTAS);
    cfg.blockDim = dim3(CL_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, (const void *)k_cg_cluster, &cfg) != cudaSuccess || ncl < 1) {
        cudaGetLastError();
        return 0;
    }
    if (int rc = build_if_of_row(c)) return rc;
    if (!c.d_cl_ai) CK(cudaMalloc(&c.d_cl_ai, sizeof(double) * (2 * (size_t)std::max(c.n_if, 1) + 16)));
    c.cl_on = true;
    c.cl_rows = rmax;
    c.cl_smem = smem;
    if (getenv("THERMO_CG_VERBOSE"))
        fprintf(stderr, "[thermo cg] cluster solve: %d CTAs x %d threads, %lld rows per CTA, smem %zu B\n", CL_CTAS,
                CL_THREADS, (long long)rmax, smem);
    return 0;
}

// Launch the cluster kernel with the parameters a grid launch would use (ovl: record the
// launch-completion event of the overlap mode).
int cl_launch(Ctx &c, CGParams &P, bool ovl, int buf) {
    P.cl_rows = c.cl_rows;
    P.if_of_row = c.d_if_of_row;
    P.z2 = c.d_cl_ai;                                   // interface sums ai[n_if] ...
    P.q2 = c.d_cl_ai + std::max(c.n_if, 1) + 8;         // ... and their own-column terms
    void *args[] = {&P};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL_CTAS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    int na = 1;
    if (ovl) {
        at[1].id = cudaLaunchAttributeLaunchCompletionEvent;
        at[1].val.launchCompletionEvent.event = c.ev_cg[buf];
        at[1].val.launchCompletionEvent.flags = 0;
        na = 2;
    }
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = dim3(CL_CTAS);
    cfg.blockDim = dim3(CL_THREADS);
    cfg.dynamicSmemBytes = c.cl_smem;
    cfg.stream = c.stream;
    cfg.attrs = at;
    cfg.numAttrs = na;
    CK(cudaLaunchKernelExC(&cfg, (const void *)k_cg_cluster, args));
    return 0;
}

}  // namespace thermo
