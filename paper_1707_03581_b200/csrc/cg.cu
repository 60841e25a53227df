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
//
// Two variants of the sliced-ELL sweeps (phase 0 and S):
//  kTMA = true  (default): one CTA per SM, CG_W consumer warps + 1 producer warp.  The
//    producer streams chunks of CG_W consecutive slices (values + columns, contiguous in HBM)
//    into a CG_NS-stage shared-memory ring with cp.async.bulk on the TMA engine
//    (mbarrier complete_tx); consumers read the matrix from shared memory and only gather
//    the vector entries from L1/L2.  HBM streaming is thereby decoupled from gather latency.
//  kTMA = false: every warp streams its slices with L1-bypassing, L2-evict-first loads
//    (fallback when a chunk does not fit the shared-memory ring).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
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

// TMA-ring geometry variants: CG_W slices per chunk = consumer warps per group, CG_G consumer
// groups (group g consumes chunks n with n % CG_G == g), CG_NS pipeline stages.
#define CG_HDR 128  // stage header bytes: chunk-relative slice offsets + interface ranges
#define CG_NVARIANT 3
__host__ __device__ constexpr int cg_w(int v) { return v == 2 ? 4 : 8; }
__host__ __device__ constexpr int cg_g(int v) { return v == 2 ? 4 : 2; }
__host__ __device__ constexpr int cg_ns(int v) { return v == 0 ? 4 : (v == 1 ? 3 : 6); }
__host__ __device__ constexpr int cg_threads(int v) { return (cg_w(v) * cg_g(v) + 1) * 32; }

struct CGParams {
    int64_t N, nslices, nchunks;
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
    int stage_entries;   // TMA: entries per stage buffer
    const int32_t *chunk_hi;   // TMA: largest column index referenced by each chunk
    int *chunk_ctr;            // TMA: two chunk-claim counters (zero between launches)
    const double *pf[4];       // TMA: vectors whose leading edge is prefetched into L2
    int npf;
};

// Prefetch into L2 the leading edge of the column window of a chunk: rows
// [hi - len + 1, hi] of each vector in pf (len = rows of the chunk, clamped, 16-B aligned).
template <int CG_W>
__device__ __forceinline__ void prefetch_edge(const CGParams &P, int64_t ch) {
    if (ch >= P.nchunks) return;
    const int64_t rows = (int64_t)CG_W * 32;
    int64_t hi = (int64_t)P.chunk_hi[ch] + 1;
    int64_t lo = hi - rows;
    if (lo < 0) lo = 0;
    lo &= ~(int64_t)1;
    hi = (hi + 1) & ~(int64_t)1;
    if (hi > P.N) hi = P.N & ~(int64_t)1;
    if (hi <= lo) return;
    for (int v = 0; v < P.npf; ++v) bulk_prefetch_l2(P.pf[v] + lo, (uint32_t)((hi - lo) * 8));
}

// sum_k val * (x1[col] + beta * x2[col]) over one sliced-ELL row (entries at stride 32).
// kSmem: the slice lives in shared memory (TMA ring); else in global memory (streamed).
template <bool kSmem, bool kTwo>
__device__ __forceinline__ double row_dot(const int32_t *cp, const double *vp, int w, const double *x1,
                                          const double *x2, double beta, uint64_t pol) {
    constexpr int B = kSmem ? 16 : 8;   // gathers issued together
    double acc = 0.0;
    int k = 0;
    for (; k + B <= w; k += B) {
        int c[B];
        double v[B], y[B];
#pragma unroll
        for (int u = 0; u < B; ++u) c[u] = kSmem ? cp[32 * (k + u)] : ld_stream(cp + 32 * (k + u), pol);
#pragma unroll
        for (int u = 0; u < B; ++u) y[u] = x1[c[u]];
        if (kTwo) {
#pragma unroll
            for (int u = 0; u < B; ++u) y[u] = fma(beta, x2[c[u]], y[u]);
        }
#pragma unroll
        for (int u = 0; u < B; ++u) v[u] = kSmem ? vp[32 * (k + u)] : ld_stream(vp + 32 * (k + u), pol);
#pragma unroll
        for (int u = 0; u < B; ++u) acc = fma(v[u], y[u], acc);
    }
    if (kSmem && k < w) {   // remainder: all loads first, then the ordered FMA chain
        int c[B];
        double y[B];
#pragma unroll
        for (int u = 0; u < B; ++u) c[u] = (k + u < w) ? cp[32 * (k + u)] : -1;
#pragma unroll
        for (int u = 0; u < B; ++u) {
            y[u] = c[u] >= 0 ? x1[c[u]] : 0.0;
            if (kTwo && c[u] >= 0) y[u] = fma(beta, x2[c[u]], y[u]);
        }
#pragma unroll
        for (int u = 0; u < B; ++u)
            if (k + u < w) acc = fma(vp[32 * (k + u)], y[u], acc);
        return acc;
    }
    for (; k < w; ++k) {
        const int c0 = kSmem ? cp[32 * k] : ld_stream(cp + 32 * k, pol);
        double y0 = x1[c0];
        if (kTwo) y0 = fma(beta, x2[c0], y0);
        const double v0 = kSmem ? vp[32 * k] : ld_stream(vp + 32 * k, pol);
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

// ---------------------------------------------------------------------------------
// slice sweep: calls body(s, cp, vp, w) for every slice owned by this warp, with the slice's
// columns / values (already offset by the lane) either in the shared-memory ring (kTMA) or
// in global memory.
// ---------------------------------------------------------------------------------
struct Ring {
    uint64_t *full, *empty;
    unsigned char *stage;   // CG_NS stages of [header | values | columns]
    size_t stage_bytes;
    uint32_t n;             // chunks passed through the ring so far (same count in every warp)
};

// Interface index of the row owned by this lane (-1 if none), given the slice's range
// [b, e) in if_rows.  Warp-uniform call.
__device__ __forceinline__ int iface_index_r(const CGParams &P, int b, int e, int64_t i, int lane) {
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

// Chunk order (TMA variant): CTA b takes chunks b, b + G, b + 2G, ... (static, so that every
// CTA's dot-product partial -- and hence every result bit -- is reproducible; dynamic claiming
// from a global counter was measured slower and breaks determinism).  The chunk id travels in
// the stage header; an id < 0 is the end marker (one per consumer group).
template <bool kTMA, int V, class Body>
__device__ __forceinline__ void sweep(const CGParams &P, Ring &R, int *ctr, Body &&body) {
    constexpr int CG_W = cg_w(V), CG_G = cg_g(V), CG_NS = cg_ns(V);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (kTMA) {
        const int G = gridDim.x;
        const int E = P.stage_entries;
        if (warp == CG_W * CG_G) {   // producer warp
            const uint64_t pol = policy_evict_first();
            int64_t next = blockIdx.x;   // static grid-stride order: deterministic partials
            while (true) {
                const uint32_t st = R.n % CG_NS, ph = (R.n / CG_NS) & 1u;
                const int64_t ch = next;
                next += G;
                if (ch >= P.nchunks) {   // end markers for every consumer group
                    const uint32_t m0 = R.n;
                    for (int q = 0; q < CG_G; ++q) {
                        const uint32_t sq = R.n % CG_NS, pq = (R.n / CG_NS) & 1u;
                        if (lane == 0) {
                            mbar_wait(&R.empty[sq], pq ^ 1u);
                            int *hdr = reinterpret_cast<int *>(R.stage + (size_t)sq * R.stage_bytes);
                            hdr[31] = -1;
                            hdr[30] = (int)m0;
                            mbar_arrive(&R.full[sq]);
                        }
                        __syncwarp();
                        ++R.n;
                    }
                    break;
                }
                const int64_t s0 = ch * CG_W, s1 = min(s0 + (int64_t)CG_W, P.nslices);
                const int64_t sl = min(s0 + lane, s1);
                const int64_t ptr = lane <= CG_W ? P.slice_ptr[sl] : 0;
                const int sif = lane <= CG_W ? P.slice_if[sl] : 0;
                const int64_t e0 = __shfl_sync(0xffffffffu, ptr, 0);
                const int64_t e1 = __shfl_sync(0xffffffffu, ptr, CG_W);
                if (lane == 0) mbar_wait(&R.empty[st], ph ^ 1u);
                __syncwarp();
                unsigned char *sb = R.stage + (size_t)st * R.stage_bytes;
                int *hdr = reinterpret_cast<int *>(sb);
                if (lane <= CG_W) {
                    hdr[lane] = (int)(ptr - e0);
                    hdr[16 + lane] = sif;
                }
                if (lane == 0) hdr[31] = (int)ch;
                __syncwarp();
                if (lane == 0) {
                    // leading edge of the column window two claim rounds ahead (and the
                    // current chunk during the first rounds)
                    if (ch < 2 * G) prefetch_edge<CG_W>(P, ch);
                    prefetch_edge<CG_W>(P, ch + 2 * G);
                    const uint32_t cnt = (uint32_t)(e1 - e0);
                    double *vals = reinterpret_cast<double *>(sb + CG_HDR);
                    int32_t *cols = reinterpret_cast<int32_t *>(vals + E);
                    mbar_arrive_expect_tx(&R.full[st], cnt * 12u);
                    bulk_g2s(vals, P.val + e0, cnt * 8u, &R.full[st], pol);
                    bulk_g2s(cols, P.col + e0, cnt * 4u, &R.full[st], pol);
                }
                __syncwarp();
                ++R.n;
            }
        } else {                     // consumer warps: group g takes every CG_G-th stage
            const int g = warp / CG_W, wg = warp % CG_W;
            while (true) {
                const uint32_t st = R.n % CG_NS, ph = (R.n / CG_NS) & 1u;
                if ((int)(R.n % CG_G) == g) {
                    mbar_wait(&R.full[st], ph);
                    const unsigned char *sb = R.stage + (size_t)st * R.stage_bytes;
                    const int *hdr = reinterpret_cast<const int *>(sb);
                    const int ch = hdr[31];
                    if (ch < 0) {
                        const uint32_t m0 = (uint32_t)hdr[30];
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&R.empty[st]);
                        R.n = m0 + CG_G;
                        break;
                    }
                    const int64_t s = (int64_t)ch * CG_W + wg;
                    if (s < P.nslices) {
                        const double *vals = reinterpret_cast<const double *>(sb + CG_HDR);
                        const int32_t *cols = reinterpret_cast<const int32_t *>(vals + E);
                        const int o0 = hdr[wg], o1 = hdr[wg + 1];
                        body(s, cols + o0 + lane, vals + o0 + lane, (o1 - o0) >> 5, hdr[16 + wg], hdr[17 + wg]);
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&R.empty[st]);
                }
                ++R.n;
            }
        }
    } else {
        const int nw = blockDim.x >> 5;
        const int gw = blockIdx.x * nw + warp;
        const int TW = gridDim.x * nw;
        for (int64_t s = gw; s < P.nslices; s += TW) {
            const int64_t b0 = P.slice_ptr[s], b1 = P.slice_ptr[s + 1];
            body(s, P.col + b0 + lane, P.val + b0 + lane, (int)((b1 - b0) >> 5), P.slice_if[s], P.slice_if[s + 1]);
        }
    }
}

template <bool kTMA, int V>
__global__ void __launch_bounds__(kTMA ? cg_threads(V) : THERMO_BLOCK, kTMA ? 1 : 2) k_cg_step(CGParams P) {
    constexpr int CG_W = cg_w(V), CG_NS = cg_ns(V);
    __shared__ double red_smem[THERMO_RED_SMEM];
    extern __shared__ __align__(128) unsigned char ring_raw[];
    if (P.status[0] || P.status[1]) {   // an earlier step failed or the interface overflowed
        if (!P.status[0] && blockIdx.x == 0 && threadIdx.x == 0) {
            P.status[0] = 2;
            P.status[2] = P.step;
        }
        return;
    }
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const int G = gridDim.x;
    const int64_t N = P.N;
    constexpr bool kSmem = kTMA;

    Ring R;
    R.n = 0;
    if (kTMA) {
        R.full = reinterpret_cast<uint64_t *>(ring_raw);
        R.empty = R.full + CG_NS;
        R.stage = ring_raw + 128;
        R.stage_bytes = CG_HDR + (size_t)P.stage_entries * 12;
        if (threadIdx.x == 0) {
            for (int s = 0; s < CG_NS; ++s) {
                mbar_init(&R.full[s], 1);
                mbar_init(&R.empty[s], CG_W);
            }
            fence_mbar_init();
        }
        __syncthreads();
    }
    const uint64_t pol = kTMA ? 0ull : policy_evict_first();

    // ---- r0 = b - K~ x0 with x0 = T^n, b = M_L T^n + dt (b_env + b_G); z0 = D^{-1} r0
    double red0[4] = {0.0, 0.0, 0.0, 0.0};   // b.b, r.r, r.z, |Gamma_R|
    P.pf[0] = P.T_in; P.pf[1] = P.ML; P.pf[2] = P.benv; P.pf[3] = P.Dinv;
    P.npf = 4;
    int sw = 0;   // sweep counter: sweep sw claims chunks from P.chunk_ctr[sw & 1]
    sweep<kTMA, V>(P, R, P.chunk_ctr + (sw & 1), [&](int64_t s, const int32_t *cp, const double *vp, int w, int ib, int ie) {
        const int64_t i = 32 * s + lane;
        const int ik = iface_index_r(P, ib, ie, i, lane);
        double ax = row_dot<kSmem, false>(cp, vp, w, P.T_in, nullptr, 0.0, pol);
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
    });
    cta_reduce_store<4>(red0, red_smem, P.partials, 0);
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) P.chunk_ctr[sw & 1] = 0;   // next used after >= 1 more barrier
    ++sw;
    double tot0[4];
    grid_total<4>(P.partials, G, 0, red_smem, tot0);
    const double tol2 = P.rtol2 * tot0[0];
    double rho = tot0[2], rr = tot0[1];
    bool conv = rr <= tol2;
    double beta = 0.0;
    const double *xsrc = P.T_in;
    double *pold = P.pa, *pnew = P.pb;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)G * blockDim.x;
    int it = 0;
    while (!conv && it < P.maxit) {
        // ---- S: p = z + beta p_old, q = K~ p, partial p.q
        double pq[1] = {0.0};
        const bool first = it == 0;
        P.pf[0] = P.z; P.pf[1] = pold;
        P.npf = first ? 1 : 2;
        sweep<kTMA, V>(P, R, P.chunk_ctr + (sw & 1), [&](int64_t s, const int32_t *cp, const double *vp, int w, int ib, int ie) {
            const int64_t i = 32 * s + lane;
            const int ik = iface_index_r(P, ib, ie, i, lane);
            double acc;
            if (first) {
                acc = row_dot<kSmem, false>(cp, vp, w, P.z, nullptr, 0.0, pol);
                if (ik >= 0) acc += ell_row<false>(P, ik, P.z, nullptr, 0.0);
            } else {
                acc = row_dot<kSmem, true>(cp, vp, w, P.z, pold, beta, pol);
                if (ik >= 0) acc += ell_row<true>(P, ik, P.z, pold, beta);
            }
            if (i < N) {
                const double pi = first ? P.z[i] : fma(beta, pold[i], P.z[i]);
                pnew[i] = pi;
                P.q[i] = acc;
                pq[0] = fma(pi, acc, pq[0]);
            }
        });
        cta_reduce_store<1>(pq, red_smem, P.partials, 4);
        grid.sync();
        if (blockIdx.x == 0 && threadIdx.x == 0) P.chunk_ctr[sw & 1] = 0;
        ++sw;
        double tpq[1];
        grid_total<1>(P.partials, G, 4, red_smem, tpq);
        const double alpha = rho / tpq[0];
        // ---- U: x += alpha p, z -= alpha D^{-1} q, partials r.z and r.r (r = z / D^{-1});
        // element pairs with 16-byte loads, two pairs in flight per thread and trip
        double red[2] = {0.0, 0.0};
        {
            const int64_t npair = N >> 1;
            const double2 *p2 = reinterpret_cast<const double2 *>(pnew);
            const double2 *q2 = reinterpret_cast<const double2 *>(P.q);
            const double2 *d2 = reinterpret_cast<const double2 *>(P.Dinv);
            const double2 *x2 = reinterpret_cast<const double2 *>(xsrc);
            double2 *z2 = reinterpret_cast<double2 *>(P.z);
            double2 *o2 = reinterpret_cast<double2 *>(P.T_out);
            auto upd = [&](double2 pv, double2 qv, double2 dv, double2 xv, double2 zv, int64_t j) {
                double2 xo, zo;
                xo.x = fma(alpha, pv.x, xv.x);
                xo.y = fma(alpha, pv.y, xv.y);
                zo.x = fma(-alpha * dv.x, qv.x, zv.x);
                zo.y = fma(-alpha * dv.y, qv.y, zv.y);
                o2[j] = xo;
                z2[j] = zo;
                const double r0 = zo.x / dv.x, r1 = zo.y / dv.y;
                red[0] = fma(r0, zo.x, red[0]);
                red[1] = fma(r0, r0, red[1]);
                red[0] = fma(r1, zo.y, red[0]);
                red[1] = fma(r1, r1, red[1]);
            };
            int64_t j = tid;
            for (; j + nthr < npair; j += 2 * nthr) {
                const int64_t j2 = j + nthr;
                const double2 pa = p2[j], pb = p2[j2], qa = q2[j], qb = q2[j2], da = d2[j], db = d2[j2];
                const double2 xa = x2[j], xb = x2[j2], za = z2[j], zb = z2[j2];
                upd(pa, qa, da, xa, za, j);
                upd(pb, qb, db, xb, zb, j2);
            }
            if (j < npair) upd(p2[j], q2[j], d2[j], x2[j], z2[j], j);
            if ((N & 1) && tid == nthr - 1) {
                const int64_t i = N - 1;
                const double di = P.Dinv[i];
                P.T_out[i] = fma(alpha, pnew[i], xsrc[i]);
                const double zi = fma(-alpha * di, P.q[i], P.z[i]);
                P.z[i] = zi;
                const double r = zi / di;
                red[0] = fma(r, zi, red[0]);
                red[1] = fma(r, r, red[1]);
            }
        }
        cta_reduce_store<2>(red, red_smem, P.partials, 5);
        grid.sync();
        double tr[2];
        grid_total<2>(P.partials, G, 5, red_smem, tr);
        beta = tr[0] / rho;
        rho = tr[0];
        rr = tr[1];
        conv = rr <= tol2;
        xsrc = P.T_out;
        double *t = pold; pold = pnew; pnew = t;
        ++it;
    }
    if (it == 0) {   // already converged: T^{n+1} = T^n
        for (int64_t i = tid; i < N; i += nthr) P.T_out[i] = P.T_in[i];
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

// largest column index of every chunk of CG_W slices (warp per chunk)
__global__ void k_chunk_hi(const int64_t *slice_ptr, const int32_t *col, int64_t nslices, int64_t nchunks,
                           int CG_W, int32_t *hi) {
    const int64_t ch = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (ch >= nchunks) return;
    const int64_t s0 = ch * CG_W, s1 = min(s0 + (int64_t)CG_W, nslices);
    int m = 0;
    for (int64_t e = slice_ptr[s0] + lane; e < slice_ptr[s1]; e += 32) m = max(m, col[e]);
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) hi[ch] = m;
}

template <int V>
static int setup_variant(Ctx &c, int *per_sm) {
    CK(cudaFuncSetAttribute(k_cg_step<true, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.cg_smem));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, k_cg_step<true, V>, cg_threads(V), c.cg_smem));
    return 0;
}

int cg_setup(Ctx &c) {
    const char *env = getenv("THERMO_CG_PATH");   // testing hook: 0 = register path, 1 = TMA
    const int force = env ? atoi(env) : -1;
    const char *envv = getenv("THERMO_CG_VARIANT");
    c.cg_variant = envv ? std::max(0, std::min(CG_NVARIANT - 1, atoi(envv))) : 0;
    const int W = cg_w(c.cg_variant);
    c.cg_chunk = W;
    // largest chunk of W consecutive slices -> stage size of the TMA ring
    std::vector<int64_t> sp(c.nslices + 1);
    CK(cudaMemcpy(sp.data(), c.d_slice_ptr, sizeof(int64_t) * (c.nslices + 1), cudaMemcpyDeviceToHost));
    int64_t emax = 0;
    for (int64_t s0 = 0; s0 < c.nslices; s0 += W) {
        const int64_t s1 = std::min<int64_t>(s0 + W, c.nslices);
        emax = std::max(emax, sp[s1] - sp[s0]);
    }
    c.cg_stage_entries = (int)((emax + 31) / 32 * 32);
    c.cg_smem = 128 + (size_t)cg_ns(c.cg_variant) * (CG_HDR + (size_t)c.cg_stage_entries * 12);
    c.cg_tma = c.cg_smem <= 220 * 1024 && force != 0;
    int per_sm = 0;
    if (c.cg_tma) {
        int rc = c.cg_variant == 0 ? setup_variant<0>(c, &per_sm)
                 : c.cg_variant == 1 ? setup_variant<1>(c, &per_sm) : setup_variant<2>(c, &per_sm);
        if (rc) return rc;
        c.cg_block = cg_threads(c.cg_variant);
    } else {
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cg_step<false, 0>, THERMO_BLOCK, 0));
        c.cg_block = THERMO_BLOCK;
        c.cg_smem = 0;
    }
    if (per_sm < 1) { c.err = "CG kernel cannot be resident"; return -3; }
    const int64_t nchunks = (c.nslices + W - 1) / W;
    CK(cudaMalloc(&c.d_chunk_hi, sizeof(int32_t) * (nchunks + 1)));
    CK(cudaMalloc(&c.d_chunk_ctr, sizeof(int) * 2));
    CK(cudaMemsetAsync(c.d_chunk_ctr, 0, sizeof(int) * 2, c.stream));
    k_chunk_hi<<<(unsigned)((nchunks * 32 + 255) / 256), 256, 0, c.stream>>>(c.d_slice_ptr, c.d_col, c.nslices,
                                                                           nchunks, W, c.d_chunk_hi);
    CK(cudaGetLastError());
    c.cg_grid = per_sm * c.num_sms;
    CK(cudaMalloc(&c.d_partials, sizeof(double) * THERMO_NRED * c.cg_grid));
    return 0;
}

int cg_launch_step(Ctx &c, int step, double dt) {
    CGParams P;
    P.N = c.N;
    P.nslices = c.nslices;
    P.nchunks = (c.nslices + c.cg_chunk - 1) / c.cg_chunk;
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
    P.stage_entries = c.cg_stage_entries;
    P.chunk_hi = c.d_chunk_hi;
    P.chunk_ctr = c.d_chunk_ctr;
    P.npf = 0;
    void *args[] = {&P};
    const void *fn = !c.cg_tma ? (const void *)k_cg_step<false, 0>
                     : c.cg_variant == 0 ? (const void *)k_cg_step<true, 0>
                     : c.cg_variant == 1 ? (const void *)k_cg_step<true, 1>
                                         : (const void *)k_cg_step<true, 2>;
    CK(cudaLaunchCooperativeKernel(fn, dim3(c.cg_grid), dim3(c.cg_block), args, c.cg_tma ? c.cg_smem : 0, c.stream));
    return 0;
}

}  // namespace thermo
