// cg_resident.cu -- resident-operator latency path of the single-scenario Jacobi-PCG solve for
// problems whose operator fits in the shared memory of the whole chip (N up to ~1.5e5: the paper's
// 16,626-DoF model, and BASELINE configs 0-1).  At that size a solve is bound by the chain of
// dependent latencies per iteration, not by bandwidth (the paper's metric is the look-ahead factor,
// P:189-194): the streaming grid kernel (cg.cu) pays a TMA ring pass plus a cooperative-groups
// grid barrier per iteration (~12-14 us), the single-cluster kernel (cg_cluster.cu) three cluster
// barriers with their GPU-scope fences (~11 us).  Here:
//   * one CTA per SM (cooperative launch), every CTA owns a contiguous block of slices and keeps
//     its rows of K~_vol (values + 32-bit columns, sliced ELL as stored) and of x, z, p, q' in
//     shared memory for the whole solve -- the matrix is read from L2 once per step;
//   * ONE grid barrier per iteration (as the one-barrier kernel of cg.cu): iteration k publishes
//     its rows of z_k, q'_k and p_k (double-buffered by iteration parity) before the barrier that
//     also carries the reduction, and iteration k + 1 forms every gathered column's
//       p_{k+1,j} = beta_k p_{k,j} + (z_{k,j} - alpha_k q'_{k,j})
//     with the owner's own expression (bitwise the same value);
//   * the barrier is an arrive counter in global memory (red.release / ld.acquire at GPU scope,
//     zeroed by the host before the launch) instead of cooperative-groups grid.sync; the CTA
//     partials of the seven sums are read by every CTA in one L2 round trip and summed in a fixed
//     order (every CTA computes identical scalars: deterministic, bitwise reproducible);
//   * a row's gathers are all in flight at once (4 threads per volume row, 8 per interface row,
//     whose per-step ELL entries are also loaded into shared memory at the start of the launch),
//     so a sweep costs one L2 round trip; the blocks of slices are balanced by entries, which
//     spreads the interface rows (3x the entries of a volume row) over more CTAs.
// Same z-primary iteration and the same safeguards as the other solve kernels.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "cg_params.h"
#include "ctx.h"

namespace thermo {

#define CK(x)                                                                    \
    do {                                                                         \
        cudaError_t e_ = (x);                                                    \
        if (e_ != cudaSuccess) {                                                 \
            c.err = std::string("CUDA: ") + cudaGetErrorString(e_) + " at " #x; \
            return -3;                                                           \
        }                                                                        \
    } while (0)

#define RS_THREADS 512
#define RS_MAXSL 64   // slices per CTA (<= 2048 rows)

// grid barrier: every CTA arrives once (release: its earlier global writes are visible to whoever
// acquires the count), thread 0 spins until all have
__device__ __forceinline__ void rs_barrier(unsigned *ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

__global__ void __launch_bounds__(RS_THREADS, 1) k_cg_resident(CGParams P) {
    extern __shared__ __align__(16) unsigned char rs_smem[];
    __shared__ double red_s[THERMO_RED_SMEM];
    __shared__ int sbase[RS_MAXSL + 1];
    __shared__ int s_nifl;
    // two arrive counters alternate between launches: this launch counts on gbar and zeroes
    // gbar_next for the next one (nobody touches it during this launch) -- no memset per step
    if (blockIdx.x == 0 && threadIdx.x == 0) *P.gbar_next = 0u;
    // an earlier step failed, or the interface of this or an earlier step overflowed (the
    // condition only depends on values written before the launch: uniform over the grid)
    if (P.status[0] || (P.status[1] && P.status[4] <= P.step)) {
        if (!P.status[0] && blockIdx.x == 0 && threadIdx.x == 0) {
            P.status[0] = 2;
            P.status[2] = P.step;
        }
        return;
    }
    const int rank = blockIdx.x, nct = gridDim.x;
    const int t = threadIdx.x;

    const int64_t N = P.N;
    const int64_t s0 = P.rs_part[rank], s1 = P.rs_part[rank + 1];   // this CTA's slices (host: balanced by entries)
    const int nsl = (int)(s1 - s0);
    const int64_t r0 = 32 * s0, r1 = min(N, 32 * s1);
    const int nloc = (int)max((int64_t)0, r1 - r0);   // rows of this CTA
    const int ell = P.rs_ell;
    const int64_t e0 = P.slice_ptr[s0];
    const int nent = (int)(P.slice_ptr[s1] - e0);
    // shared memory, packed by this CTA's own sizes (the host sized the allocation for the largest
    // block): volume values | x z p q' d | volume columns | interface index of a row | own
    // interface rows | their entry counts | interface values | interface columns
    const int ecap = (nent + 1) & ~1, cap = (32 * nsl + 1) & ~1;
    double *vs = reinterpret_cast<double *>(rs_smem);
    double *xs = vs + ecap, *zs = xs + cap, *ps = zs + cap, *qs = ps + cap, *ds = qs + cap;
    int *cs = reinterpret_cast<int *>(ds + cap);
    int *iks = cs + ecap, *ifl = iks + cap, *icn = ifl + cap;
    double *ivs = reinterpret_cast<double *>(icn + cap);   // (all counts above are even: 8-byte aligned)
    if (t == 0) s_nifl = 0;
    for (int s = t; s <= nsl; s += RS_THREADS) sbase[s] = (int)(P.slice_ptr[s0 + s] - e0);
    for (int e = t; e < nent; e += RS_THREADS) {
        vs[e] = __ldg(P.val + e0 + e);
        cs[e] = __ldg(P.col + e0 + e);
    }
    __syncthreads();
    const bool iface = P.n_if > 0;
    for (int l = t; l < nloc; l += RS_THREADS) {
        const int ik = iface ? P.if_of_row[r0 + l] : -1;
        iks[l] = ik;
        // the list order only decides where a row's entries sit in shared memory
        if (ik >= 0) ifl[atomicAdd(&s_nifl, 1)] = l;
    }
    __syncthreads();
    const int nifl = s_nifl;
    int *ics = reinterpret_cast<int *>(ivs + (((size_t)nifl * ell + 1) & ~(size_t)1));
    const bool tr_on = P.trace && rank == 0 && t == 0;
    unsigned nbar = 0;
    // ---- the steps of this launch (ahead mode: consecutive steps whose interfaces sit in
    // consecutive slots; otherwise one).  Step sti reads the state buffer the previous step wrote.
    for (int sti = 0; sti < P.nst; ++sti) {
    const int step = P.step + sti;
    if (sti > 0 && P.status[1] && P.status[4] <= step) {   // interface overflow at this step (known before the launch)
        if (rank == 0 && t == 0) {
            P.status[0] = 2;
            P.status[2] = step;
        }
        break;
    }
    const double *const Tin = (sti & 1) ? P.T_out : P.T_in;
    double *const Tout = (sti & 1) ? P.Tin_w : P.T_out;
    const int64_t so_if = (int64_t)sti * P.n_if;               // this step's slot behind the first one
    const int32_t *const ell_cnt = P.ell_cnt + so_if;
    const int32_t *const ell_col = P.ell_col + so_if * ell;
    const double *const ell_val = P.ell_val + so_if * ell;
    const double *const if_b = P.if_b + so_if, *const if_phi = P.if_phi + so_if;
    const double *const if_dinv_s = P.if_dinv_s ? P.if_dinv_s + so_if : nullptr;
    const int xorder = min(P.xhist + sti, P.xguess);   // states behind T^n available / wanted for the start
    const int xsave = P.xsave;
    for (int l = t; l < nloc; l += RS_THREADS) {
        const int sl = l >> 5;
        ds[l] = vs[sbase[sl] + (l & 31)];   // entry 0 of the row: the volume diagonal (assembly order)
    }
    __syncthreads();
    // this step's interface entries of the own interface rows -> shared memory (slot-major ELL
    // [c][k] in global memory; [j][c] here), and the interface self term on the diagonal
    for (int jb = 0; jb < nifl; jb += RS_THREADS >> 3) {   // warp-uniform trip count (shuffles inside)
        const int j = jb + (t >> 3);
        const bool on = j < nifl;
        const int l = on ? ifl[j] : 0, k = on ? iks[l] : 0;
        const int cnt = on ? min(__ldg(ell_cnt + k), ell) : 0;
        double self = 0.0;
        for (int c = t & 7; c < cnt; c += 8) {
            const int64_t e = (int64_t)c * P.n_if + k;
            const int jc = __ldg(ell_col + e);
            const double v = __ldg(ell_val + e);
            ics[j * ell + c] = jc;
            ivs[j * ell + c] = v;
            if (jc == r0 + l) self += v;
        }
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) self += __shfl_xor_sync(0xffffffffu, self, o);
        if (on && (t & 7) == 0) {
            icn[j] = cnt;
            ds[l] += self;
        }
    }
    __syncthreads();
    int ntr = 0;   // (the trace of the launch's last step survives)
    if (tr_on) P.trace[ntr++] = gtimer();
    const double *const x0 = P.X0 ? P.X0 : Tin;

    // One pass over the CTA's rows: (K~ w)_l for every own row l with w_j = gv(j), then fin(l, sum)
    // by one thread per row.  A volume row is summed by 4 threads (entries q, q + 4, ...), an
    // interface row by 8 (its volume entries, then its interface entries); every gather of a row is
    // in flight at once (rows of <= 16 volume and <= 48 interface entries: one round trip); the
    // partial sums are combined by xor butterflies -- a fixed order.
    auto sweep = [&](auto &&gv, auto &&fin) {
        for (int lb = 0; lb < nloc; lb += RS_THREADS >> 2) {   // volume rows: warp-uniform trip count
            const int l = lb + (t >> 2), q = t & 3;
            const bool on = l < nloc && iks[min(l, nloc - 1)] < 0;
            double acc = 0.0;
            if (on) {
                const int sl = l >> 5, b0 = sbase[sl] + (l & 31), w = (sbase[sl + 1] - sbase[sl]) >> 5;
                for (int k0 = 0; k0 < w; k0 += 16) {
                    double v[4], y[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int k = k0 + q + 4 * u;
                        v[u] = 0.0;
                        y[u] = 0.0;
                        if (k < w) {
                            v[u] = vs[b0 + 32 * k];
                            y[u] = gv(cs[b0 + 32 * k]);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) acc = fma(v[u], y[u], acc);
                }
            }
            acc += __shfl_xor_sync(0xffffffffu, acc, 1);
            acc += __shfl_xor_sync(0xffffffffu, acc, 2);
            if (on && q == 0) fin(l, acc);
        }
        for (int jb = 0; jb < nifl; jb += RS_THREADS >> 3) {   // interface rows
            const int j = jb + (t >> 3), o = t & 7;
            const bool on = j < nifl;
            const int l = on ? ifl[j] : 0;
            double acc = 0.0;
            if (on) {
                const int sl = l >> 5, b0 = sbase[sl] + (l & 31), w = (sbase[sl + 1] - sbase[sl]) >> 5;
                const int cnt = icn[j];
                for (int k0 = 0; k0 < w; k0 += 16) {
                    double v[2], y[2];
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int k = k0 + o + 8 * u;
                        v[u] = 0.0;
                        y[u] = 0.0;
                        if (k < w) {
                            v[u] = vs[b0 + 32 * k];
                            y[u] = gv(cs[b0 + 32 * k]);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 2; ++u) acc = fma(v[u], y[u], acc);
                }
                for (int c0 = 0; c0 < cnt; c0 += 48) {
                    double v[6], y[6];
#pragma unroll
                    for (int u = 0; u < 6; ++u) {
                        const int c = c0 + o + 8 * u;
                        v[u] = 0.0;
                        y[u] = 0.0;
                        if (c < cnt) {
                            v[u] = ivs[j * ell + c];
                            y[u] = gv(ics[j * ell + c]);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 6; ++u) acc = fma(v[u], y[u], acc);
                }
            }
#pragma unroll
            for (int x = 1; x < 8; x <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, x);
            if (on && o == 0) fin(l, acc);
        }
    };

    // ---- phase 0: r0 = b - K~ x0, z0 = D^{-1} r0, p0 = z0; b = M_L T^n + dt (b_env + b_G) or rhs
    double red0[4] = {0.0, 0.0, 0.0, 0.0};   // b.b, r.r, r.z, |Gamma_R|
    // x0 at column j: T^n (or the given X0), or the extrapolation of the last committed states
    // formed here with the expressions of k_extrap (thermo.cu) -- T^{n-1} still sits in T_out, which
    // is only written at the end of the launch, after every CTA has passed phase 0
    auto gx = [&](int64_t j) -> double {
        if (xorder == 0) return ld_cg1(x0 + j);
        const double a = ld_cg1(Tin + j), d = a - ld_cg1(Tout + j);
        return xorder >= 2 ? fma(3.0, d, ld_cg1(P.Th + j)) : a + d;
    };
    sweep([&](int j) { return gx(j); },
          [&](int l, double ax) {
              const int64_t i = r0 + l;
              const int ik = iks[l];
              double bi = P.benv[i];
              if (ik >= 0) {
                  bi += if_b[ik];
                  if (ik < P.nA) red0[3] += if_phi[ik];
              }
              bi = P.rhs ? P.rhs[i] : fma(P.ML[i], ld_cg1(Tin + i), P.dt * bi);
              const double r = bi - ax;
              const double zi = (ik >= 0 && if_dinv_s ? if_dinv_s[ik] : P.Dinv[i]) * r;
              xs[l] = gx(i);
              zs[l] = zi;
              ps[l] = zi;
              qs[l] = 0.0;
              // set 1 = the "previous iteration" of iteration 0 (alpha = beta = 0: p_0 = z_0)
              P.z2[i] = zi;
              P.q2[i] = 0.0;
              P.pb[i] = 0.0;
              red0[0] = fma(bi, bi, red0[0]);
              red0[1] = fma(r, r, red0[1]);
              red0[2] = fma(r, zi, red0[2]);
          });
    cta_reduce_store<4>(red0, red_s, P.partials, 0);
    rs_barrier(P.gbar, ++nbar * (unsigned)nct);
    double tot0[4];
    grid_total<4>(P.partials, nct, 0, red_s, tot0);
    if (tr_on) P.trace[ntr++] = gtimer();
    const double tol2 = P.rtol2 * tot0[0];
    double rho = tot0[2], rr = tot0[1];
    bool conv = rr <= tol2;
    int it = 0;
    double alpha = 0.0, beta = 0.0;   // coefficients of the update that is still to be applied
    while (!conv && it < P.maxit) {
        const int si = (it + 1) & 1, so = it & 1;   // published sets: read (previous iteration) / write
        const double *zi_ = si ? P.z2 : P.z, *qi_ = si ? P.q2 : P.q, *pi_ = si ? P.pb : P.pa;
        double *const zo_ = so ? P.z2 : P.z, *const qo_ = so ? P.q2 : P.q, *const po_ = so ? P.pb : P.pa;
        // S: q = K~ p with the direction of this iteration at column j formed from the previous
        // iteration's published rows (ld.global.cg: written by other CTAs during this launch);
        // the row's owner applies the previous iteration's update x += alpha p, z -= alpha q',
        // p = z + beta p to its own values (the same expression), then q' = q / d and the seven
        // sums (cg.cu), and publishes its z, q', p
        double red[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        sweep([&](int j) { return fma(beta, ld_cg1(pi_ + j), fma(-alpha, ld_cg1(qi_ + j), ld_cg1(zi_ + j))); },
              [&](int l, double acc) {
                  const double pv = ps[l];
                  xs[l] = fma(alpha, pv, xs[l]);
                  const double zo = fma(-alpha, qs[l], zs[l]);
                  const double pi = fma(beta, pv, zo);
                  const double dg = ds[l];
                  const double qv = acc / dg, zd = zo * dg;
                  zs[l] = zo;
                  ps[l] = pi;
                  qs[l] = qv;
                  const int64_t i = r0 + l;
                  zo_[i] = zo;
                  qo_[i] = qv;
                  po_[i] = pi;
                  red[0] = fma(pi, acc, red[0]);
                  red[1] = fma(zo, zd, red[1]);
                  red[2] = fma(zo, acc, red[2]);
                  red[3] = fma(acc, qv, red[3]);
                  red[4] = fma(zd, zd, red[4]);
                  red[5] = fma(zd, acc, red[5]);
                  red[6] = fma(acc, acc, red[6]);
              });
        const int slot = 4 + 7 * so;
        cta_reduce_store<7>(red, red_s, P.partials, slot);
        if (tr_on && ntr < 1000) P.trace[ntr++] = gtimer();
        rs_barrier(P.gbar, ++nbar * (unsigned)nct);   // also publishes this iteration's z, q', p
        double t7[7];
        grid_total<7>(P.partials, nct, slot, red_s, t7);
        if (tr_on && ntr < 1000) P.trace[ntr++] = gtimer();
        alpha = beta = 0.0;
        if (it > 0) {   // t7[4] = sum (z d)^2: the current r.r directly (safeguard of cg.cu)
            rr = t7[4];
            if (rr <= tol2) { conv = true; break; }
        }
        alpha = rho / t7[0];
        const double rz_new = fma(alpha, fma(alpha, t7[3], -2.0 * t7[2]), t7[1]);
        const double rr_new = fma(alpha, fma(alpha, t7[6], -2.0 * t7[5]), t7[4]);
        const double rr_noise = 1e-13 * (t7[4] + fabs(2.0 * alpha * t7[5]) + alpha * alpha * t7[6]);
        beta = rz_new / rho;
        rho = rz_new;
        rr = rr_new;
        conv = rr <= tol2 && rr > rr_noise;
        ++it;
    }
    __syncthreads();
    // the last update of x is still to be applied (alpha = 0 after an exit on the direct r.r test)
    for (int l = t; l < nloc; l += RS_THREADS) {
        if (xsave && xorder > 0) P.Th[r0 + l] = Tout[r0 + l];   // history shift: T^{n-1} before it is overwritten
        Tout[r0 + l] = fma(alpha, ps[l], xs[l]);
    }
    if (rank == 0 && t == 0) {
        const double rel = tot0[0] > 0.0 ? sqrt(rr / tot0[0]) : sqrt(rr);
        P.iters_out[step] = it;
        P.relres_out[step] = rel;
        P.area_out[step] = tot0[3];
        if (!conv) {
            P.status[0] = 1;
            P.status[2] = step;
            P.status[3] = 0;
            *P.fail_relres = rel;
        }
    }
    if (!conv) break;   // (the same decision in every CTA: identical totals)
    // the next step gathers this step's state (and the shifted history) from every CTA
    if (sti + 1 < P.nst) rs_barrier(P.gbar, ++nbar * (unsigned)nct);
    }   // steps of the launch
}

// CTAs of a launch: one per SM (the overlap mode leaves some SMs to the interface kernels), but
// never more than slices -- fewer arrivals make the barrier of a tiny problem cheaper
static int rs_grid(const Ctx &c, bool ovl) {
    int g = ovl && c.cg_grid_ovl > 0 ? c.cg_grid_ovl : c.num_sms;
    if (const char *e = getenv("THERMO_RS_CTAS")) g = std::max(1, std::min(g, atoi(e)));   // tuning hook
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, c.nslices));
}

// Contiguous blocks of slices for G CTAs, balanced by shared-memory bytes (= entries = work:
// volume entries, vector rows, interface rows with their ELL capacity): the smallest block size M
// for which a greedy cut needs <= G blocks.  Returns the bytes of the largest block (the kernel
// packs its arrays by its own sizes); part has G + 1 entries (trailing CTAs may be empty).
static size_t rs_block_bytes(int64_t nslices, int64_t entries, int64_t if_rows, int ell) {
    const size_t ent = (size_t)((entries + 1) & ~(int64_t)1), rows = (size_t)(32 * nslices),
                 ife = (size_t)((if_rows * ell + 1) & ~(int64_t)1);
    return (ent + ife) * 12 + rows * (5 * 8 + 3 * 4) + 16;
}

static bool rs_partition(const std::vector<int64_t> &sp, const std::vector<int> &nif_of_slice, int ell, int G,
                         std::vector<int64_t> &part, size_t &max_bytes) {
    const int64_t ns = (int64_t)sp.size() - 1;
    auto bytes_of = [&](int64_t s) { return rs_block_bytes(1, sp[s + 1] - sp[s], nif_of_slice[s], ell); };
    size_t lo = 0, hi = 0;
    for (int64_t s = 0; s < ns; ++s) {
        lo = std::max(lo, bytes_of(s));
        hi += bytes_of(s);
    }
    auto cut = [&](size_t M, std::vector<int64_t> *out) {
        int blocks = 0;
        int64_t s = 0;
        if (out) out->assign(1, 0);
        while (s < ns) {
            size_t acc = 0;
            int64_t b = s;
            while (s < ns && s - b < RS_MAXSL && acc + bytes_of(s) <= M) acc += bytes_of(s++);
            if (s == b) return 1 << 30;   // a single slice exceeds M
            ++blocks;
            if (out) out->push_back(s);
        }
        return blocks;
    };
    if (cut(hi, nullptr) > G) return false;   // RS_MAXSL slices per CTA are not enough
    while (lo < hi) {
        const size_t mid = lo + (hi - lo) / 2;
        if (cut(mid, nullptr) <= G) hi = mid; else lo = mid + 1;
    }
    cut(lo, &part);
    while ((int)part.size() < G + 1) part.push_back(ns);
    max_bytes = 0;
    for (int r = 0; r < G; ++r) {
        int64_t nifr = 0;
        for (int64_t s = part[r]; s < part[r + 1]; ++s) nifr += nif_of_slice[s];
        max_bytes = std::max(max_bytes, rs_block_bytes(part[r + 1] - part[r], sp[part[r + 1]] - sp[part[r]], nifr, ell));
    }
    return true;
}

// Use the resident kernel for this context?  Single scenario, every CTA's block of the operator,
// of the interface rows and of the vectors fits in shared memory for both grid sizes (all SMs /
// the overlap mode's smaller grid).
int rs_setup(Ctx &c) {
    c.rs_on = false;
    // THERMO_CG_RESIDENT=0 disables it, =1 forces it where it fits; a request for a specific grid
    // variant or for the cluster kernel (testing hooks) also switches it off
    const char *e = getenv("THERMO_CG_RESIDENT");
    const int mode = e ? atoi(e) : -1;
    if (mode == 0 || c.S != 1) return 0;
    if (mode != 1 && (getenv("THERMO_CG_VARIANT") || getenv("THERMO_CG_CLUSTER") || getenv("THERMO_CG_CTAS"))) return 0;
    if ((double)c.nnz_pad * 12 > 40e6) return 0;   // far beyond the chip's shared memory
    // default: up to ~256 rows per CTA (two passes of 128 rows per sweep), where it is faster than the
    // streaming kernel (11,856 DoF: 7.8 vs 12.4 us per iteration; 85,694 DoF, 580 rows per CTA: no gain)
    if (mode != 1 && c.N > (int64_t)256 * c.num_sms) return 0;
    std::vector<int64_t> sp(c.nslices + 1);
    CK(cudaMemcpy(sp.data(), c.d_slice_ptr, sizeof(int64_t) * (c.nslices + 1), cudaMemcpyDeviceToHost));
    std::vector<int32_t> ifr(std::max(c.n_if, 1));
    if (c.n_if) CK(cudaMemcpy(ifr.data(), c.d_if_rows, sizeof(int32_t) * c.n_if, cudaMemcpyDeviceToHost));
    std::vector<int> nif_of_slice(c.nslices, 0);
    for (int k = 0; k < c.n_if; ++k) ++nif_of_slice[ifr[k] / 32];
    const int ell = std::max(c.cap, 1);
    size_t smem = 0;
    std::vector<int64_t> parts[2];
    for (int gi = 0; gi < 2; ++gi) {
        size_t mb = 0;
        if (!rs_partition(sp, nif_of_slice, ell, rs_grid(c, gi == 1), parts[gi], mb)) return 0;
        smem = std::max(smem, mb);
    }
    if (smem > 216 * 1024) return 0;
    if (cudaFuncSetAttribute((const void *)k_cg_resident, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cg_resident, RS_THREADS, smem) != cudaSuccess ||
        per_sm < 1) {
        cudaGetLastError();
        return 0;
    }
    if (int rc = build_if_of_row(c)) return rc;
    if (!c.d_z2) {   // second published set of z, q' (p uses d_p[0] / d_p[1])
        CK(cudaMalloc(&c.d_z2, sizeof(double) * (c.N + 16)));
        CK(cudaMalloc(&c.d_q2, sizeof(double) * (c.N + 16)));
        CK(cudaMemsetAsync(c.d_z2, 0, sizeof(double) * (c.N + 16), c.stream));
        CK(cudaMemsetAsync(c.d_q2, 0, sizeof(double) * (c.N + 16), c.stream));
    }
    if (!c.d_gbar) {
        CK(cudaMalloc(&c.d_gbar, sizeof(unsigned) * 4));
        CK(cudaMemsetAsync(c.d_gbar, 0, sizeof(unsigned) * 4, c.stream));
        c.rs_parity = 0;
    }
    for (int gi = 0; gi < 2; ++gi) {
        if (!c.d_rs_part[gi]) CK(cudaMalloc(&c.d_rs_part[gi], sizeof(int64_t) * (c.num_sms + 1)));
        CK(cudaMemcpy(c.d_rs_part[gi], parts[gi].data(), sizeof(int64_t) * parts[gi].size(), cudaMemcpyHostToDevice));
    }
    c.rs_on = true;
    c.rs_smem = smem;
    if (getenv("THERMO_CG_VERBOSE"))
        fprintf(stderr, "[thermo cg] resident solve: %d CTAs x %d threads (overlap grid %d), interface ELL %d, smem %zu B"
                        "\n", rs_grid(c, false), RS_THREADS, rs_grid(c, true), ell, smem);
    return 0;
}

// Ahead mode (ctx.h, DESIGN 7.2): slot-major buffers for the interfaces of the next ah_slots step
// times.  On with the resident solve, and for the sizes that do not overlap the interface assembly
// with the previous solve (the overlap mode hides it completely where it is on); the slot count
// is limited by memory (<= 2 GB of pair records and rows).  THERMO_AHEAD: 0 off, n >= 2 slots.
int ahead_setup(Ctx &c) {
    c.ah_on = false;
    if (c.S != 1 || c.n_if == 0 || !(c.rs_on || !c.overlap)) return 0;
    const char *ea = getenv("THERMO_AHEAD");
    int slots = ea ? atoi(ea) : 16;
    const size_t nif = (size_t)c.n_if;
    const size_t per_slot = sizeof(PairRec) * (size_t)c.nTB * c.pcap + sizeof(int32_t) * (size_t)c.nTA * c.pcap +
                            sizeof(int32_t) * (size_t)(c.nTA + c.nTB) + nif * ((size_t)c.cap * 12 + 36);
    slots = (int)std::min<size_t>((size_t)std::min(slots, 64), ((size_t)2 << 30) / std::max<size_t>(per_slot, 1));
    if (slots < 2 || c.d_ah_sc) return 0;
    const size_t M = (size_t)slots;
    CK(cudaMalloc(&c.d_ah_pairs, sizeof(PairRec) * M * c.nTB * c.pcap));
    CK(cudaMalloc(&c.d_ah_refs, sizeof(int32_t) * M * c.nTA * c.pcap));
    CK(cudaMalloc(&c.d_ah_pcnt, sizeof(int32_t) * M * (c.nTA + c.nTB)));
    CK(cudaMalloc(&c.d_ah_ell_cnt, sizeof(int32_t) * M * nif));
    CK(cudaMalloc(&c.d_ah_ell_col, sizeof(int32_t) * M * c.cap * nif));
    CK(cudaMalloc(&c.d_ah_ell_val, sizeof(double) * M * c.cap * nif));
    CK(cudaMalloc(&c.d_ah_if_b, sizeof(double) * M * nif));
    CK(cudaMalloc(&c.d_ah_if_phi, sizeof(double) * M * nif));
    CK(cudaMalloc(&c.d_ah_dinv, sizeof(double) * M * nif));
    CK(cudaMalloc(&c.d_ah_d, sizeof(double) * M * nif));
    CK(cudaMalloc(&c.d_ah_sc, sizeof(double) * 4 * M));
    c.ah_slots = slots;
    c.ah_on = true;
    c.ah_valid = false;
    if (getenv("THERMO_CG_VERBOSE"))
        fprintf(stderr, "[thermo] ahead mode: %d slots of %.1f MB\n", slots, per_slot / 1048576.0);
    return 0;
}

// Launch the resident kernel with the parameters a grid launch would use (ovl: the overlap mode's
// smaller grid, and record its launch-completion event).
int rs_launch(Ctx &c, CGParams &P, bool ovl, int buf) {
    P.rs_ell = std::max(c.cap, 1);
    if (P.nst < 1) P.nst = 1;
    P.rs_part = c.d_rs_part[ovl ? 1 : 0];
    P.if_of_row = c.d_if_of_row;
    P.z2 = c.d_z2;
    P.q2 = c.d_q2;
    P.gbar = c.d_gbar + c.rs_parity;          // this launch's arrive counter (zeroed by the previous launch)
    P.gbar_next = c.d_gbar + (c.rs_parity ^ 1);
    c.rs_parity ^= 1;
    void *args[] = {&P};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    int na = 1;
    if (ovl) {
        at[1].id = cudaLaunchAttributeLaunchCompletionEvent;
        at[1].val.launchCompletionEvent.event = c.ev_cg[buf];
        at[1].val.launchCompletionEvent.flags = 0;
        na = 2;
    }
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = dim3(rs_grid(c, ovl));
    cfg.blockDim = dim3(RS_THREADS);
    cfg.dynamicSmemBytes = c.rs_smem;
    cfg.stream = c.stream;
    cfg.attrs = at;
    cfg.numAttrs = na;
    CK(cudaLaunchKernelExC(&cfg, (const void *)k_cg_resident, args));
    return 0;
}

}  // namespace thermo
