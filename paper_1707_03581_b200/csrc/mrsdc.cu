// mrsdc.cu -- multi-rate spectral deferred corrections, the paper's method, on the
// B200 kernels of the implicit-Euler path.
//
// Splitting: f^I(T) = (A + B_env) T (slow, implicit), g = b_env, f^E(T, t) =
// K_G(t) T + b_G(t) (interface coupling and friction, fast, explicit).  One step of size dt:
// M equidistant no-left standard nodes, P embedded nodes per standard interval.
//   Algorithm 1 (predictor): per standard interval one implicit solve
//       (M_L - dt/M (A + B_env)) T* = M_L T_{m-1} + dt/M g,   f* = f^I(T*) + g
//     then P explicit Euler sub-steps in f^E:  M_L T_{m,p} = M_L T_{m,p-1} + dt/(MP) (f* + f^E(T_{m,p-1}))
//   Algorithm 2 (sweep k -> k+1): the same structure with the quadrature terms I_{m-1}^m,
//     I_{m,p-1}^p of Table 1 built from the previous iterate.
// The implicit operator M_L - dt/M (A + B_env) never changes within a run, so the persistent CG
// kernel of cg.cu is reused with an explicit right-hand side and no interface rows; the
// interface operators K_G(t) at the M P + 1 node times of a step are integrated once per
// step by the interface kernels (unscaled, dt = -1) and applied explicitly.
#include <cmath>
#include <cstring>
#include <vector>

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

#define MR_MAX 8

struct MrW {            // one row of a weight family (by value)
    double a[MR_MAX];
    double b[MR_MAX];
};

static inline unsigned nbk(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

// Every kernel below works on S scenario columns: a block vector holds element (row i, scenario
// s) at i * SP + s (SP >= S; S = SP = 1 for a single run), node vectors follow each other at a
// stride of ldf elements, compact interface vectors (f^E on the interface rows) hold (k, s) at
// k * SP + s, and the node-time interface operators of scenario s and slot q are batch entry
// b = s * ns + q of the slot-major interface arrays ([b][c][k], [b][k]).  One thread per (row,
// scenario); padding columns s >= S are left alone.

// y = (A + B_env) x + sgn * addv   (sliced ELL)
__global__ void k_vol_apply(const int64_t *slice_ptr, const int32_t *col, const double *KV, int64_t N, int S,
                            int SP, const double *x, const double *addv, double sgn, double *y) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= N * S) return;
    const int64_t i = t / S;
    const int sc = (int)(t - i * S);
    const int64_t sl = i >> 5;
    const int lane = (int)(i & 31);
    const int64_t b0 = slice_ptr[sl], w = (slice_ptr[sl + 1] - b0) >> 5;
    double acc = 0.0;
    for (int64_t k = 0; k < w; ++k)
        acc = fma(KV[b0 + 32 * k + lane], x[(int64_t)col[b0 + 32 * k + lane] * SP + sc], acc);
    if (addv) acc = fma(sgn, addv[i * SP + sc], acc);
    y[i * SP + sc] = acc;
}

// The same for a single scenario (S = SP = 1): 4 threads per row (entries q, q + 4, ...), every
// gather of a row in flight at once, partial sums combined by an xor butterfly (a fixed order).  A
// thread per row walks its ~15 entries through dependent round trips: at paper scale (16,870 DoF)
// 11.5 us per launch, 12 launches per MRSDC(3,2) step.
__global__ void k_vol_apply4(const int64_t *slice_ptr, const int32_t *col, const double *KV, int64_t N,
                             const double *x, const double *addv, double sgn, double *y) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t i = t >> 2;
    const int q = (int)(t & 3);
    const bool on = i < N;
    double acc = 0.0;
    if (on) {
        const int64_t sl = i >> 5;
        const int64_t b0 = slice_ptr[sl] + (i & 31), w = (slice_ptr[sl + 1] - slice_ptr[sl]) >> 5;
        for (int64_t k0 = 0; k0 < w; k0 += 16) {
            double v[4], z[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t k = k0 + q + 4 * u;
                v[u] = 0.0;
                z[u] = 0.0;
                if (k < w) {
                    v[u] = KV[b0 + 32 * k];
                    z[u] = x[col[b0 + 32 * k]];
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) acc = fma(v[u], z[u], acc);
        }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (on && q == 0) y[i] = addv ? fma(sgn, addv[i], acc) : acc;
}

// f^E on the interface rows, single scenario: 8 threads per row (entries g, g + 8, ...)
__global__ void k_fe_apply8(int n_if, int q, int cap, const int32_t *cnt, const int32_t *ecol, const double *evals,
                            const double *bG, const double *x, double *y) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int k = (int)(t >> 3), g = (int)(t & 7);
    const bool on = k < n_if;
    double acc = 0.0;
    if (on) {
        const int64_t bt = q;   // batch entry of slot q (S = 1: ns slots of one scenario)
        const int m = cnt[bt * n_if + k];
        for (int c0 = 0; c0 < m; c0 += 48) {
            double v[6], z[6];
#pragma unroll
            for (int u = 0; u < 6; ++u) {
                const int c = c0 + g + 8 * u;
                v[u] = 0.0;
                z[u] = 0.0;
                if (c < m) {
                    const int64_t e = (bt * cap + c) * n_if + k;
                    v[u] = evals[e];
                    z[u] = x[ecol[e]];
                }
            }
#pragma unroll
            for (int u = 0; u < 6; ++u) acc = fma(v[u], z[u], acc);
        }
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (on && g == 0) y[k] = bG[(int64_t)q * n_if + k] + acc;
}

// compact f^E on the interface rows at node-time slot q of every scenario:
// y[k][s] = b_G[k] + sum_c K_G[k][c] x[col][s]   (operators of batch entry s * ns + q)
__global__ void k_fe_apply(int n_if, int q, int ns, int S, int SP, int cap, const int32_t *cnt, const int32_t *ecol,
                           const double *evals, const double *bG, const double *x, double *y) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)n_if * S) return;
    const int k = (int)(t / S), sc = (int)(t - (int64_t)k * S);
    const int64_t bt = (int64_t)sc * ns + q;
    double acc = bG[bt * n_if + k];
    const int m = cnt[bt * n_if + k];
    for (int c = 0; c < m; ++c) {
        const int64_t e = (bt * cap + c) * n_if + k;
        acc = fma(evals[e], x[(int64_t)ecol[e] * SP + sc], acc);
    }
    y[(int64_t)k * SP + sc] = acc;
}

// right-hand side of an implicit solve.
//  predictor:  rhs = M_L Tprev + a g
//  sweep:      rhs = M_L Tprev - a f^I(T^k_m) + I_{m-1}^m,
//              I_{m-1}^m = sum_j s_mj (f^I(T_j) + g) + sum_p shat_mp f^E(T_mp)
__global__ void k_mr_rhs(int64_t N, int S, int SP, int64_t ldf, const double *ML, const double *Tprev,
                         const double *benv, const double *KvTk, double a, const double *FI, const double *FE,
                         const int32_t *if_of_row, int n_if, int M, int P, MrW w, double *rhs) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= N * S) return;
    const int64_t i = t / S;
    const int sc = (int)(t - i * S);
    const int64_t e = i * SP + sc;
    double r = ML[i] * Tprev[e];
    if (!KvTk) {
        r = fma(a, benv[i], r);
    } else {
        double I = 0.0;
        for (int j = 0; j < M; ++j) I = fma(w.a[j], FI[(int64_t)j * ldf + e], I);
        const int k = if_of_row[i];
        if (k >= 0)
            for (int p = 0; p < P; ++p) I = fma(w.b[p], FE[((int64_t)p * n_if + k) * SP + sc], I);
        r = fma(-a, KvTk[e], r) + I;
    }
    rhs[e] = r;
}

// one embedded explicit-Euler sub-step (Algorithm 1 / 2 inner loop)
//  predictor: T = Tprev + dtp (fs + fe_new) / M_L
//  sweep:     T = Tprev + (dtp fs + dtp (fe_new - fe_old) + I_{m,p-1}^p) / M_L,
//             I_{m,p-1}^p = sum_j st_j (f^I(T_j) + g) + sum_q se_q f^E(T_mq)
__global__ void k_mr_emb(int64_t N, int S, int SP, int64_t ldf, const double *ML, const double *Tprev,
                         const double *fs, const double *fe_new, const double *fe_old, double dtp, const double *FI,
                         const double *FE, const int32_t *if_of_row, int n_if, int M, int P, MrW w, double *Tout) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= N * S) return;
    const int64_t i = t / S;
    const int sc = (int)(t - i * S);
    const int64_t e = i * SP + sc;
    const int k = if_of_row[i];
    const int64_t ek = (int64_t)k * SP + sc;
    double num;
    if (!fe_old) {
        num = dtp * (fs[e] + (k >= 0 ? fe_new[ek] : 0.0));
    } else {
        double I = 0.0;
        for (int j = 0; j < M; ++j) I = fma(w.a[j], FI[(int64_t)j * ldf + e], I);
        double fe = 0.0;
        if (k >= 0) {
            for (int q = 0; q < P; ++q) I = fma(w.b[q], FE[((int64_t)q * n_if + k) * SP + sc], I);
            fe = fe_new[ek] - fe_old[ek];
        }
        num = dtp * fs[e] + dtp * fe + I;
    }
    Tout[e] = Tprev[e] + num / ML[i];
}

// right-hand side of a single-rate SDC solve (every term implicit, reading R29):
//  predictor (KvTk == nullptr): rhs = M_L Tprev + a (b_env + b_G(tau_m))
//  sweep:  rhs = M_L Tprev - a K(tau_m) T^k_m + sum_j s_mj F(T^k_j, tau_j)
//          K(tau_m) T^k_m = KvTk + (FE_m - b_G(tau_m)) on the interface rows,
//          F(T^k_j, tau_j) = FI_j + FE_j (FI_j = (A + B_env) T^k_j + b_env, FE_j = K_G T^k_j + b_G)
__global__ void k_sdc_rhs(int64_t N, int S, int SP, int64_t ldf, const double *ML, const double *Tprev,
                          const double *benv, const double *KvTk, double a, const double *FI, const double *FE,
                          int nif, const double *bG, int ns, const int32_t *if_of_row, int M, int mcur, MrW w,
                          double *rhs) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= N * S) return;
    const int64_t i = t / S;
    const int sc = (int)(t - i * S);
    const int64_t e = i * SP + sc;
    const int k = nif ? if_of_row[i] : -1;
    const double bGm = k >= 0 ? bG[((int64_t)sc * ns + mcur) * nif + k] : 0.0;   // b_G(tau_m), slot m
    double r = ML[i] * Tprev[e];
    if (!KvTk) {
        r = fma(a, k >= 0 ? benv[i] + bGm : benv[i], r);
    } else {
        double KT = KvTk[e];
        if (k >= 0) KT += FE[((int64_t)(mcur - 1) * nif + k) * SP + sc] - bGm;
        double I = 0.0;
        for (int j = 0; j < M; ++j) {
            double Fj = FI[(int64_t)j * ldf + e];
            if (k >= 0) Fj += FE[((int64_t)j * nif + k) * SP + sc];
            I = fma(w.a[j], Fj, I);
        }
        r = fma(-a, KT, r) + I;
    }
    rhs[e] = r;
}

// g = b_env as a block (every scenario column the same), for the "+ g" forms of k_vol_apply
__global__ void k_bcast_rows(const double *v, int64_t N, int SP, double *vS) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < N * SP) vS[t] = v[t / SP];
}

__global__ void k_if_of_row(const int32_t *if_rows, int n_if, int32_t *map) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n_if) map[if_rows[k]] = k;
}

// row -> interface index map (-1 for volume-only rows), built once per context
int build_if_of_row(Ctx &c) {   // padded to whole slices (nslices * 32 entries)
    if (c.d_if_of_row) return 0;
    CK(cudaMalloc(&c.d_if_of_row, sizeof(int32_t) * (size_t)c.nslices * 32));
    CK(cudaMemsetAsync(c.d_if_of_row, 0xff, sizeof(int32_t) * (size_t)c.nslices * 32, c.stream));
    if (c.n_if) k_if_of_row<<<nbk(c.n_if), 256, 0, c.stream>>>(c.d_if_rows, c.n_if, c.d_if_of_row);
    CK(cudaGetLastError());
    return 0;
}

// ---------------------------------------------------------------------------------
// Table 1 weights on the host: exact integrals of Lagrange polynomials.
// ---------------------------------------------------------------------------------
static double lag_int(const double *x, int n, int j, double a, double b) {
    // l_j(s) = prod_{k != j} (s - x_k) / (x_j - x_k), integrated by Gauss-Legendre with n
    // points (exact for degree n - 1 <= 2n - 1)
    static const double gx[8][8] = {
        {0},
        {-0.5773502691896257, 0.5773502691896257},
        {-0.7745966692414834, 0.0, 0.7745966692414834},
        {-0.8611363115940526, -0.3399810435848563, 0.3399810435848563, 0.8611363115940526},
        {-0.9061798459386640, -0.5384693101056831, 0.0, 0.5384693101056831, 0.9061798459386640},
        {-0.9324695142031521, -0.6612093864662645, -0.2386191860831969, 0.2386191860831969, 0.6612093864662645,
         0.9324695142031521},
        {-0.9491079123427585, -0.7415311855993945, -0.4058451513773972, 0.0, 0.4058451513773972,
         0.7415311855993945, 0.9491079123427585},
        {-0.9602898564975363, -0.7966664774136267, -0.5255324099163290, -0.1834346424956498,
         0.1834346424956498, 0.5255324099163290, 0.7966664774136267, 0.9602898564975363}};
    static const double gw[8][8] = {
        {2.0},
        {1.0, 1.0},
        {0.5555555555555556, 0.8888888888888888, 0.5555555555555556},
        {0.3478548451374538, 0.6521451548625461, 0.6521451548625461, 0.3478548451374538},
        {0.2369268850561891, 0.4786286704993665, 0.5688888888888889, 0.4786286704993665, 0.2369268850561891},
        {0.1713244923791704, 0.3607615730481386, 0.4679139345726910, 0.4679139345726910, 0.3607615730481386,
         0.1713244923791704},
        {0.1294849661688697, 0.2797053914892766, 0.3818300505051189, 0.4179591836734694, 0.3818300505051189,
         0.2797053914892766, 0.1294849661688697},
        {0.1012285362903763, 0.2223810344533745, 0.3137066458778873, 0.3626837833783620, 0.3626837833783620,
         0.3137066458778873, 0.2223810344533745, 0.1012285362903763}};
    const int ng = n;   // n points integrate the degree n-1 polynomial exactly
    double acc = 0.0;
    const double hm = 0.5 * (b - a), cm = 0.5 * (a + b);
    for (int g = 0; g < ng; ++g) {
        const double sx = cm + hm * gx[ng - 1][g];
        double l = 1.0;
        for (int k = 0; k < n; ++k)
            if (k != j) l *= (sx - x[k]) / (x[j] - x[k]);
        acc += gw[ng - 1][g] * l;
    }
    return acc * hm;
}

struct MrTables {
    double tau[MR_MAX + 1];                 // tau[0] = t_n, tau[m] = standard node m
    double s[MR_MAX][MR_MAX];               // s[m-1][j]
    double shat[MR_MAX][MR_MAX];            // shat[m-1][p]
    double st[MR_MAX][MR_MAX][MR_MAX];      // stilde[m-1][p-1][j]
    double se[MR_MAX][MR_MAX][MR_MAX];      // s_{m,p,q}[m-1][p-1][q]
};

static void mr_tables(int M, int P, double tn, double dt, MrTables &T) {
    // work on the unit step (weights scale with dt)
    double x[MR_MAX];
    T.tau[0] = 0.0;
    for (int m = 1; m <= M; ++m) T.tau[m] = (double)m / M;
    for (int m = 0; m < M; ++m) x[m] = T.tau[m + 1];
    for (int m = 1; m <= M; ++m) {
        double e[MR_MAX];
        for (int p = 1; p <= P; ++p) e[p - 1] = T.tau[m - 1] + (T.tau[m] - T.tau[m - 1]) * p / P;
        for (int j = 0; j < M; ++j) T.s[m - 1][j] = dt * lag_int(x, M, j, T.tau[m - 1], T.tau[m]);
        for (int p = 0; p < P; ++p) T.shat[m - 1][p] = dt * lag_int(e, P, p, T.tau[m - 1], T.tau[m]);
        for (int p = 1; p <= P; ++p) {
            const double lo = p == 1 ? T.tau[m - 1] : e[p - 2], hi = e[p - 1];
            for (int j = 0; j < M; ++j) T.st[m - 1][p - 1][j] = dt * lag_int(x, M, j, lo, hi);
            for (int q = 0; q < P; ++q) T.se[m - 1][p - 1][q] = dt * lag_int(e, P, q, lo, hi);
        }
    }
    for (int m = 0; m <= M; ++m) T.tau[m] = tn + dt * T.tau[m];
}

// ---------------------------------------------------------------------------------
// setup and one step
// ---------------------------------------------------------------------------------
struct MrPtr {
    double *TSo[MR_MAX + 1], *TSn[MR_MAX + 1];
    double *TEo[MR_MAX][MR_MAX + 1], *TEn[MR_MAX][MR_MAX + 1];   // [m-1][p], p = 0..P
    double *FI, *FE, *fe_new, *fe_old, *fs, *rhs, *Tstar, *KvTk;
};

int mrsdc_setup(Ctx &c) {
    const int M = c.mr_M, P = c.mr_P, S = c.S, SP = c.SP;
    const int64_t N = c.N, nif = std::max(c.n_if, 1);
    const int64_t Np = (N + 31) & ~(int64_t)31;   // 256-byte aligned vectors (TMA windows, 16-B loads)
    const size_t nfull = 2 * (size_t)M + 2 * (size_t)M * (P - 1) + M + 4;   // TS (1..M) x2, interior TE x2, FI, 4 temps
    const size_t ncomp = (size_t)M * P + 2;
    if (c.d_mr) cudaFree(c.d_mr);
    const size_t bytes = sizeof(double) * ((nfull * Np + ncomp * nif) * SP + 64);
    CK(cudaMalloc(&c.d_mr, bytes));
    CK(cudaMemsetAsync(c.d_mr, 0, bytes, c.stream));
    c.mr_vectors = nfull;
    if (int rc = build_if_of_row(c)) return rc;
    // interface operators at the M P + 1 node times of a step, every scenario (batch entry
    // scenario * nslot + slot)
    const int nslot = M * P + 1;
    const int64_t nb = (int64_t)nslot * S;
    if (c.mr_nslots < nb && c.n_if) {
        for (void *p : {(void *)c.d_ell_cnt_s, (void *)c.d_ell_col_s, (void *)c.d_ell_val_s, (void *)c.d_if_b_s,
                        (void *)c.d_if_phi_s, (void *)c.d_pairs_s, (void *)c.d_pcnt_s, (void *)c.d_refs_s})
            if (p) cudaFree(p);
        // pair records of all node times at once (one launch set per step, batch = blockIdx.y)
        CK(cudaMalloc(&c.d_pairs_s, sizeof(PairRec) * (size_t)nb * c.nTB * c.pcap));
        CK(cudaMalloc(&c.d_refs_s, sizeof(int32_t) * (size_t)nb * c.nTA * c.pcap));
        CK(cudaMalloc(&c.d_pcnt_s, sizeof(int32_t) * (size_t)nb * (c.nTA + c.nTB)));
        CK(cudaMalloc(&c.d_ell_cnt_s, sizeof(int32_t) * nb * nif));
        CK(cudaMalloc(&c.d_ell_col_s, sizeof(int32_t) * (size_t)nb * c.cap * nif));
        CK(cudaMalloc(&c.d_ell_val_s, sizeof(double) * (size_t)nb * c.cap * nif));
        CK(cudaMalloc(&c.d_if_b_s, sizeof(double) * nb * nif));
        CK(cudaMalloc(&c.d_if_phi_s, sizeof(double) * nb * nif));
        c.mr_nslots = (int)nb;
    }
    // iterations / residual of every implicit solve of a step (solve-major, S per solve)
    const size_t nsol = (size_t)M * (c.mr_K + 1) + 8;
    if (c.d_mr_iters) cudaFree(c.d_mr_iters);
    if (c.d_mr_relres) cudaFree(c.d_mr_relres);
    CK(cudaMalloc(&c.d_mr_iters, sizeof(int32_t) * nsol * S));
    CK(cudaMalloc(&c.d_mr_relres, sizeof(double) * nsol * S));
    if (S > 1 && cgb_prepare(c)) return -3;
    return 0;
}

static MrPtr mr_pointers(Ctx &c, double *T0) {
    const int M = c.mr_M, P = c.mr_P;
    const int64_t SP = c.SP;
    const int64_t N = ((c.N + 31) & ~(int64_t)31) * SP, nif = std::max(c.n_if, 1) * SP;   // padded block strides
    MrPtr q;
    double *p = c.d_mr;
    q.TSo[0] = q.TSn[0] = T0;
    for (int m = 1; m <= M; ++m) { q.TSo[m] = p; p += N; }
    for (int m = 1; m <= M; ++m) { q.TSn[m] = p; p += N; }
    for (int m = 1; m <= M; ++m) {
        q.TEo[m - 1][0] = q.TSo[m - 1];
        q.TEn[m - 1][0] = q.TSn[m - 1];
        for (int e = 1; e < P; ++e) { q.TEo[m - 1][e] = p; p += N; }
        for (int e = 1; e < P; ++e) { q.TEn[m - 1][e] = p; p += N; }
        q.TEo[m - 1][P] = q.TSo[m];
        q.TEn[m - 1][P] = q.TSn[m];
    }
    q.FI = p; p += (size_t)M * N;
    q.fs = p; p += N;
    q.rhs = p; p += N;
    q.Tstar = p; p += N;
    q.KvTk = p; p += N;
    q.FE = p; p += (size_t)M * P * nif;
    q.fe_new = p; p += nif;
    q.fe_old = p; p += nif;
    return q;
}

// time scalars (offset, eta, s) of every scenario at the node times t_n + q dt / nq, q = 0..nq:
// sc[(s * (nq + 1) + q) * 4 ..] (batch entry s * (nq + 1) + q of assemble_slots) followed by the
// node-major copy sc[off + (q * S + s) * 4 ..] (one launch per node for the SDC reassembly)
static void node_scalars(const Ctx &c, double tn, double dt, int nq, std::vector<double> &sc) {
    const int S = c.S, ns = nq + 1;
    sc.assign(8 * (size_t)S * ns, 0.0);
    const size_t off = 4 * (size_t)S * ns;
    for (int s = 0; s < S; ++s) {
        const Scen &sn = c.scen[s];
        for (int q = 0; q < ns; ++q) {
            const double tq = tn + dt * (double)q / (double)nq;
            const double sv = sn.s0 + sn.amp * std::sin(2.0 * M_PI * tq / sn.period);
            const double v[4] = {sv * sn.d2[0], sv * sn.d2[1],
                                 sn.eta0 * (1.0 + sn.eta_amp * std::sin(2.0 * M_PI * tq / sn.eta_period)), sv};
            for (int j = 0; j < 4; ++j) {
                sc[4 * ((size_t)s * ns + q) + j] = v[j];
                sc[off + 4 * ((size_t)q * S + s) + j] = v[j];
            }
        }
    }
}

static int ensure_step_scalars(Ctx &c, size_t n) {   // d_step_sc with room for n doubles
    if ((int64_t)(n / 4) <= c.step_cap) return 0;
    for (void *p : {(void *)c.d_step_sc, (void *)c.d_iters, (void *)c.d_relres, (void *)c.d_area})
        if (p) cudaFree(p);
    c.step_cap = (int64_t)(n / 4);
    CK(cudaMalloc(&c.d_step_sc, sizeof(double) * n));
    CK(cudaMalloc(&c.d_iters, sizeof(int32_t) * (size_t)c.step_cap * c.S));
    CK(cudaMalloc(&c.d_relres, sizeof(double) * (size_t)c.step_cap * c.S));
    CK(cudaMalloc(&c.d_area, sizeof(double) * (size_t)c.step_cap));
    return 0;
}

// implicit solve number `slot` of a step: (M_L - a K_vol [- a K_G]) x = rhs from x0, every scenario
static int mr_solve(Ctx &c, const double *x0, double *x, const double *rhs, const double *Dinv, bool iface, int slot) {
    if (c.S == 1) return cg_launch_solve(c, x0, x, rhs, Dinv, iface, c.d_mr_iters, c.d_mr_relres, slot);
    return cgb_launch_solve(c, x0, x, rhs, iface, c.d_mr_iters, c.d_mr_relres, slot);
}

// K_G, b_G unscaled (dt = -1, Jacobi rows untouched) at the node times of d_step_sc[0..ns), all
// in one launch set with the slot as the batch index (layout [k][c][slot]).
static int assemble_slots(Ctx &c, int ns) {
    if (!c.n_if) return 0;
    IfaceParams Pf;
    memset(&Pf, 0, sizeof Pf);
    iface_params(c, Pf, c.d_step_sc, -1.0);
    Pf.S = ns * c.S;   // batch entry scenario * ns + slot
    Pf.pairs = c.d_pairs_s;
    Pf.pcnt = c.d_pcnt_s;
    Pf.refs = c.d_refs_s;
    Pf.ell_cnt = c.d_ell_cnt_s;
    Pf.ell_col = c.d_ell_col_s;
    Pf.ell_val = c.d_ell_val_s;
    Pf.if_b = c.d_if_b_s;
    Pf.if_phi = c.d_if_phi_s;
    Pf.no_dinv = 1;
    Pf.slot_major = 1;
    return iface_launch(c, Pf);
}

int mrsdc_step(Ctx &c, double tn, double dt, int step_index) {
    const int M = c.mr_M, P = c.mr_P, K = c.mr_K, S = c.S, SP = c.SP;
    const int64_t N = c.N;
    const int nif = c.n_if;
    const double a = dt / M, dtp = dt / (M * P);
    const int64_t ldf = ((N + 31) & ~(int64_t)31) * SP, nifs = (int64_t)std::max(nif, 1) * SP;
    cudaStream_t st = c.stream;
    if (c.built_dt != a) {
        if (build_operator(c, a)) return -3;
    }
    if (S > 1 && cgb_prepare(c)) return -3;   // Jacobi block = volume diagonal (implicit part only)
    const double *gS = c.d_benv;   // g per (row, scenario)
    if (S > 1) {
        if (!c.d_benvS) CK(cudaMalloc(&c.d_benvS, sizeof(double) * (size_t)N * SP));
        k_bcast_rows<<<nbk(N * SP), 256, 0, st>>>(c.d_benv, N, SP, c.d_benvS);
        CK(cudaGetLastError());
        gS = c.d_benvS;
    }
    MrTables W;
    mr_tables(M, P, tn, dt, W);
    // ---- interface operators K_G, b_G at the node times t_n + q dt/(MP), q = 0..MP, every scenario
    const int nslot = M * P + 1;
    std::vector<double> sc;
    node_scalars(c, tn, dt, M * P, sc);
    if (ensure_step_scalars(c, sc.size())) return -3;
    CK(cudaMemcpyAsync(c.d_step_sc, sc.data(), sizeof(double) * sc.size(), cudaMemcpyHostToDevice, st));
    if (assemble_slots(c, nslot)) return -3;
    double *T0 = c.d_T[c.cur];
    MrPtr q = mr_pointers(c, T0);
    auto fe_apply = [&](int slot, const double *x, double *y) -> int {
        if (!nif) return 0;
        if (S == 1)
            k_fe_apply8<<<nbk((int64_t)nif * 8), 256, 0, st>>>(nif, slot, c.cap, c.d_ell_cnt_s, c.d_ell_col_s, c.d_ell_val_s, c.d_if_b_s, x, y);
        else
            k_fe_apply<<<nbk((int64_t)nif * S), 256, 0, st>>>(nif, slot, nslot, S, SP, c.cap, c.d_ell_cnt_s,
                                                              c.d_ell_col_s, c.d_ell_val_s, c.d_if_b_s, x, y);
        CK(cudaGetLastError());
        return 0;
    };
    auto vol_apply = [&](const double *x, const double *addv, double sgn, double *y) -> int {
        if (S == 1) k_vol_apply4<<<nbk(N * 4), 256, 0, st>>>(c.d_slice_ptr, c.d_col, c.d_KV, N, x, addv, sgn, y);
        else k_vol_apply<<<nbk(N * S), 256, 0, st>>>(c.d_slice_ptr, c.d_col, c.d_KV, N, S, SP, x, addv, sgn, y);
        CK(cudaGetLastError());
        return 0;
    };
    int solve_no = 0;
    auto solve = [&](const double *x0, double *x, const double *rhs) -> int {
        return mr_solve(c, x0, x, rhs, c.d_Dinv_vol, false, solve_no++);
    };
    // g = b_env enters f^I + g per row (one value for every scenario): a block copy for the
    // vol_apply "+ addv" forms
    MrW w0;
    memset(&w0, 0, sizeof w0);
    // ---- Algorithm 1: predictor
    for (int m = 1; m <= M; ++m) {
        k_mr_rhs<<<nbk(N * S), 256, 0, st>>>(N, S, SP, ldf, c.d_ML, q.TSo[m - 1], c.d_benv, nullptr, a, nullptr,
                                             nullptr, c.d_if_of_row, nif, M, P, w0, q.rhs);
        CK(cudaGetLastError());
        if (solve(q.TSo[m - 1], q.Tstar, q.rhs)) return -3;
        if (vol_apply(q.Tstar, gS, 1.0, q.fs)) return -3;   // f* = f^I(T*) + g
        for (int p = 1; p <= P; ++p) {
            if (fe_apply((m - 1) * P + p - 1, q.TEo[m - 1][p - 1], q.fe_new)) return -3;
            k_mr_emb<<<nbk(N * S), 256, 0, st>>>(N, S, SP, ldf, c.d_ML, q.TEo[m - 1][p - 1], q.fs, q.fe_new, nullptr,
                                                 dtp, nullptr, nullptr, c.d_if_of_row, nif, M, P, w0,
                                                 q.TEo[m - 1][p]);
            CK(cudaGetLastError());
        }
    }
    // ---- Algorithm 2: K correction sweeps
    for (int k = 0; k < K; ++k) {
        for (int j = 1; j <= M; ++j)
            if (vol_apply(q.TSo[j], gS, 1.0, q.FI + (size_t)(j - 1) * ldf)) return -3;   // f^I(T^k_j) + g
        for (int m = 1; m <= M; ++m)
            for (int p = 1; p <= P; ++p)
                if (fe_apply((m - 1) * P + p, q.TEo[m - 1][p], q.FE + (size_t)((m - 1) * P + p - 1) * nifs))
                    return -3;
        for (int m = 1; m <= M; ++m) {
            MrW wr;
            memset(&wr, 0, sizeof wr);
            for (int j = 0; j < M; ++j) wr.a[j] = W.s[m - 1][j];
            for (int p = 0; p < P; ++p) wr.b[p] = W.shat[m - 1][p];
            if (vol_apply(q.TSo[m], nullptr, 0.0, q.KvTk)) return -3;                 // f^I(T^k_m)
            const double *FEm = q.FE + (size_t)(m - 1) * P * nifs;
            k_mr_rhs<<<nbk(N * S), 256, 0, st>>>(N, S, SP, ldf, c.d_ML, q.TSn[m - 1], c.d_benv, q.KvTk, a, q.FI,
                                                 FEm, c.d_if_of_row, nif, M, P, wr, q.rhs);
            CK(cudaGetLastError());
            if (solve(q.TSo[m], q.Tstar, q.rhs)) return -3;
            if (vol_apply(q.Tstar, q.KvTk, -1.0, q.fs)) return -3;                    // f^I(T*) - f^I(T^k_m)
            for (int p = 1; p <= P; ++p) {
                MrW we;
                memset(&we, 0, sizeof we);
                for (int j = 0; j < M; ++j) we.a[j] = W.st[m - 1][p - 1][j];
                for (int qq = 0; qq < P; ++qq) we.b[qq] = W.se[m - 1][p - 1][qq];
                const int slot = (m - 1) * P + p - 1;
                if (fe_apply(slot, q.TEn[m - 1][p - 1], q.fe_new)) return -3;
                if (fe_apply(slot, q.TEo[m - 1][p - 1], q.fe_old)) return -3;
                k_mr_emb<<<nbk(N * S), 256, 0, st>>>(N, S, SP, ldf, c.d_ML, q.TEn[m - 1][p - 1], q.fs, q.fe_new,
                                                     q.fe_old, dtp, q.FI, FEm, c.d_if_of_row, nif, M, P, we,
                                                     q.TEn[m - 1][p]);
                CK(cudaGetLastError());
            }
        }
        // T^{k+1} becomes T^k
        for (int m = 1; m <= M; ++m) std::swap(q.TSo[m], q.TSn[m]);
        for (int m = 1; m <= M; ++m) {
            for (int e = 1; e < P; ++e) std::swap(q.TEo[m - 1][e], q.TEn[m - 1][e]);
            q.TEo[m - 1][0] = q.TSo[m - 1];
            q.TEn[m - 1][0] = q.TSn[m - 1];
            q.TEo[m - 1][P] = q.TSo[m];
            q.TEn[m - 1][P] = q.TSn[m];
        }
    }
    // ---- commit T(t_{n+1}) = T_M
    CK(cudaMemcpyAsync(c.d_T[c.cur ^ 1], q.TSo[M], sizeof(double) * N * SP, cudaMemcpyDeviceToDevice, st));
    c.mr_solves = solve_no;
    (void)step_index;
    return 0;
}

// One single-rate SDC step (method 2; P:354-413 with every term implicit, reading R29):
// predictor = implicit Euler through the M nodes, then K sweeps; before every solve the
// interface Jacobian is reassembled at that node (the overhead the paper attributes to
// single-rate SDC).  Uses the MRSDC storage with P = 1 (slots = node times).
int sdc_step(Ctx &c, double tn, double dt, int step_index) {
    const int M = c.mr_M, K = c.mr_K, S = c.S, SP = c.SP;
    const int64_t N = c.N;
    const int nif = c.n_if;
    const int64_t nifs = (int64_t)std::max(nif, 1) * SP;
    const double a = dt / M;
    const int64_t ldf = ((N + 31) & ~(int64_t)31) * SP;
    cudaStream_t st = c.stream;
    if (c.built_dt != a) {
        if (build_operator(c, a)) return -3;
    }
    if (S > 1 && cgb_prepare(c)) return -3;   // Jacobi block: volume diagonal, interface rows per node below
    const double *gS = c.d_benv;   // g per (row, scenario)
    if (S > 1) {
        if (!c.d_benvS) CK(cudaMalloc(&c.d_benvS, sizeof(double) * (size_t)N * SP));
        k_bcast_rows<<<nbk(N * SP), 256, 0, st>>>(c.d_benv, N, SP, c.d_benvS);
        CK(cudaGetLastError());
        gS = c.d_benvS;
    }
    MrTables W;
    mr_tables(M, 1, tn, dt, W);
    const int nslot = M + 1;   // slot m = node tau_m (slot 0 = t_n, unused)
    std::vector<double> sc;
    node_scalars(c, tn, dt, M, sc);
    if (ensure_step_scalars(c, sc.size())) return -3;
    CK(cudaMemcpyAsync(c.d_step_sc, sc.data(), sizeof(double) * sc.size(), cudaMemcpyHostToDevice, st));
    // unscaled K_G, b_G at the node times (for F(T^k_j, tau_j) in the quadrature), one launch set
    if (assemble_slots(c, nslot)) return -3;
    // implicit Jacobian M_L - a K(tau_m): interface rows of every scenario reassembled into the
    // solve arrays (node-major scalars after the slot-major ones)
    auto reassemble = [&](int m) -> int {
        if (!nif) return 0;
        IfaceParams Pf;
        memset(&Pf, 0, sizeof Pf);
        iface_params(c, Pf, c.d_step_sc + 4 * (size_t)S * nslot + 4 * (size_t)m * S, a);
        return iface_launch(c, Pf);
    };
    double *T0 = c.d_T[c.cur];
    MrPtr q = mr_pointers(c, T0);
    auto fe_apply = [&](int slot, const double *x, double *y) -> int {
        if (!nif) return 0;
        if (S == 1)
            k_fe_apply8<<<nbk((int64_t)nif * 8), 256, 0, st>>>(nif, slot, c.cap, c.d_ell_cnt_s, c.d_ell_col_s, c.d_ell_val_s, c.d_if_b_s, x, y);
        else
            k_fe_apply<<<nbk((int64_t)nif * S), 256, 0, st>>>(nif, slot, nslot, S, SP, c.cap, c.d_ell_cnt_s,
                                                              c.d_ell_col_s, c.d_ell_val_s, c.d_if_b_s, x, y);
        CK(cudaGetLastError());
        return 0;
    };
    auto vol_apply = [&](const double *x, const double *addv, double sgn, double *y) -> int {
        if (S == 1) k_vol_apply4<<<nbk(N * 4), 256, 0, st>>>(c.d_slice_ptr, c.d_col, c.d_KV, N, x, addv, sgn, y);
        else k_vol_apply<<<nbk(N * S), 256, 0, st>>>(c.d_slice_ptr, c.d_col, c.d_KV, N, S, SP, x, addv, sgn, y);
        CK(cudaGetLastError());
        return 0;
    };
    int solve_no = 0;
    auto solve = [&](const double *x0, double *x, const double *rhs) -> int {
        return mr_solve(c, x0, x, rhs, c.d_Dinv, nif > 0, solve_no++);
    };
    MrW w0;
    memset(&w0, 0, sizeof w0);
    // ---- predictor: implicit Euler from node to node
    for (int m = 1; m <= M; ++m) {
        if (reassemble(m)) return -3;
        k_sdc_rhs<<<nbk(N * S), 256, 0, st>>>(N, S, SP, ldf, c.d_ML, q.TSo[m - 1], c.d_benv, nullptr, a, nullptr,
                                              nullptr, nif, c.d_if_b_s, nslot, c.d_if_of_row, M, m, w0, q.rhs);
        CK(cudaGetLastError());
        if (solve(q.TSo[m - 1], q.TSo[m], q.rhs)) return -3;
    }
    // ---- K sweeps
    for (int k = 0; k < K; ++k) {
        for (int j = 1; j <= M; ++j) {
            if (vol_apply(q.TSo[j], gS, 1.0, q.FI + (size_t)(j - 1) * ldf)) return -3;   // (A + B) T + b_env
            if (fe_apply(j, q.TSo[j], q.FE + (size_t)(j - 1) * nifs)) return -3;               // K_G T + b_G
        }
        for (int m = 1; m <= M; ++m) {
            MrW wr;
            memset(&wr, 0, sizeof wr);
            for (int j = 0; j < M; ++j) wr.a[j] = W.s[m - 1][j];
            if (vol_apply(q.TSo[m], nullptr, 0.0, q.KvTk)) return -3;   // (A + B_env) T^k_m
            if (reassemble(m)) return -3;
            k_sdc_rhs<<<nbk(N * S), 256, 0, st>>>(N, S, SP, ldf, c.d_ML, q.TSn[m - 1], c.d_benv, q.KvTk, a, q.FI,
                                                  q.FE, nif, c.d_if_b_s, nslot, c.d_if_of_row, M, m, wr, q.rhs);
            CK(cudaGetLastError());
            if (solve(q.TSo[m], q.TSn[m], q.rhs)) return -3;
        }
        for (int m = 1; m <= M; ++m) std::swap(q.TSo[m], q.TSn[m]);
    }
    CK(cudaMemcpyAsync(c.d_T[c.cur ^ 1], q.TSo[M], sizeof(double) * N * SP, cudaMemcpyDeviceToDevice, st));
    c.mr_solves = solve_no;
    (void)step_index;
    return 0;
}

}  // namespace thermo
