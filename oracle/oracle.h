/*
 * oracle.h -- plain, slow, obviously-correct CPU oracle for the implicit-Euler hot path of
 * arXiv 1707.03581 (Naumann, Ruprecht, Wensch).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code with the CUDA library
 * (paper_1707_03581_b200/csrc, include/thermo.h) and neither includes the other.
 *
 * Citations: P:n = /root/reference/PAPER.md line n.
 *
 * What it computes, per implicit-Euler step (readings R1-R8):
 *   (M_L - dt K(t')) T^{n+1} = M_L T^n + dt (b_env + b_G(t')),   t' = t + (n+1) dt
 *   K(t) = blockdiag(A_X + B_X,env) + [[M_B,fix(t), C_B(t)], [C_B(t)^T, M_B,mov(t)]]
 * with
 *   M_L   = row-sum lumped rho*Cp * int phi phi                  (reading R1)
 *   A_X   = -nu int grad phi . grad phi
 *   B_env = -int_{Gamma_env} alpha_i phi phi dS
 *   b_env =  int_{Gamma_env} alpha_i T_i phi dS
 *   b_X(t)= int_{Gamma_R(t)} eta(t)/2 phi dS
 *   M_B,X = -int_{Gamma_R(t)} alpha phi_X phi_X dS
 *   C_B   =  int_{Gamma_R(t)} alpha phi_Y phi_X dS
 * Gamma_R(t) integrals are evaluated on the exact intersection polygons of the two
 * non-matching surface triangulations (reading R6).
 *
 * Parity pins: see oracle/README.md and tests/test_oracle_*.py.
 */
#ifndef THERMO_ORACLE_H
#define THERMO_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct or_sys or_sys;

/* Build the oracle system: copies the two meshes, assembles M_L and A (element by element).
 * Node numbering of the coupled system: fixed nodes 0..nf-1, moving nodes nf..nf+nm-1.
 * Returns NULL on invalid input (non-positive tet, non-planar interface); or_last_error(). */
or_sys *or_create(int64_t nf, const double *xyz_f, int64_t ntf, const int32_t *tets_f,
                  int64_t nbf, const int32_t *faces_f, const int32_t *tags_f,
                  int64_t nm, const double *xyz_m, int64_t ntm, const int32_t *tets_m,
                  int64_t nbm, const int32_t *faces_m, const int32_t *tags_m,
                  int32_t iface_tag, double nu, double rho_cp, double alpha_iface);
const char *or_last_error(void);
/* host threads the CG loops use (OMP_NUM_THREADS; 1 without OpenMP) */
int or_threads(void);
void or_destroy(or_sys *s);

/* Robin data for (part, tag): alpha_i and T_i(x) = T_ref + g . x.  Re-assembles
 * B_env and b_env from scratch over all faces. */
int or_set_robin(or_sys *s, int32_t part, int32_t tag, double alpha, double T_ref,
                 double gx, double gy, double gz);

int64_t or_n(const or_sys *s);
int64_t or_n_fixed(const or_sys *s);
int64_t or_vol_nnz(const or_sys *s);
/* Volume operator on the fixed pattern: rowptr[N+1], col[nnz], A[nnz] (stiffness),
 * B[nnz] (Robin matrix), ML[N] (lumped mass incl. rho*Cp), benv[N]. Any pointer may be NULL. */
void or_get_volume(const or_sys *s, int64_t *rowptr, int32_t *col, double *A, double *B,
                   double *ML, double *benv);

/* Interface assembly at in-plane offset o of the moving mesh and friction eta.
 * Result kept inside s: K_G = M_B + C_B as CSR over all N rows, b_G[N], |Gamma_R|. */
int or_assemble_interface(or_sys *s, double ox, double oy, double oz, double eta);
int64_t or_iface_nnz(const or_sys *s);
void or_get_interface(const or_sys *s, int64_t *rowptr, int32_t *col, double *val,
                      double *bG, double *area);

/* Implicit-Euler time stepping (reading R3: everything at t' = t + (n+1) dt).
 * Scenario: s(t) = s0 + amp sin(2 pi t/period) along dir; eta(t) = eta0 (1 + eta_amp
 * sin(2 pi t/eta_period)).  T[N] in/out.  solver: 0 = Jacobi-PCG from x0 = T^n until
 * ||b - K x||_2 <= rtol ||b||_2 (reading R17); 1 = dense Cholesky.
 * stats (may be NULL): per step 4 doubles {iterations, recursive rel. residual,
 * true rel. residual, |Gamma_R|}.  Returns 0, or -4 if CG failed (stats of the failing
 * step written, T holds the last committed step). */
int or_step(or_sys *s, double t, double dt, int32_t nsteps,
            double s0, double amp, double period, double dx, double dy, double dz,
            double eta0, double eta_amp, double eta_period,
            double *T, int32_t solver, double rtol, int32_t maxit, double *stats);

/* CG start of or_step (default 0): 0 = x0 = T^n; 1 = T^n + (T^n - T^{n-1}); 2 = T^{n-2} +
 * 3 (T^n - T^{n-1}), the polynomial extrapolation of the last committed states (DESIGN.md
 * reading R17: the start is not part of the method; the CUDA path defaults to order 2).  The
 * history continues across or_step calls only when T is bitwise the state the previous call
 * returned and dt is unchanged; it restarts otherwise (lower orders until it has filled).
 * Returns 0, or -1 for another order. */
int or_set_guess(or_sys *s, int32_t order);

/* Residual rows of the IE system for given T^n, T^{n+1}: res[k] = (K~ T1 - b)[rows[k]],
 * with the system assembled at offset o, eta (both given).  Also returns ||b||_2 in bnorm. */
/* Stationary state at rest (reading R19): -(A + B_env [+ K_G(t)]) T = b_env
 * [+ b_G(t)]; with_interface selects the coupled variant (reading R28).  T: in = x0, out =
 * solution.  solver 1 = dense Cholesky, else Jacobi-PCG to rtol.  stats[3] = {iterations,
 * rel. residual, true rel. residual}.  Returns 0, -4 (no convergence), -5 (interface). */
int or_stationary(or_sys *s, double t, int32_t with_interface, double s0, double amp, double period,
                  double dx, double dy, double dz, double eta0, double eta_amp, double eta_period,
                  double *T, int32_t solver, double rtol, int32_t maxit, double *stats);

int or_ie_residual_rows(or_sys *s, double dt, double ox, double oy, double oz, double eta,
                        const double *T0, const double *T1, int64_t nrows,
                        const int64_t *rows, double *res, double *bnorm);

/* Apply y = K~ x with K~ = M_L - dt (A + B_env + K_G) (current interface). */
void or_apply_system(const or_sys *s, double dt, const double *x, double *y);

/* MRSDC: equidistant no-left standard nodes tau[M] of [t0, t0+dt], embedded
 * nodes taue[M*P] and the weights of Table 1: s[M*M], shat[M*P], stilde[M*P*M], semb[M*P*P]
 * (row-major in the index order of P:474-479), by exact integration of Lagrange polynomials. */
int or_mrsdc_weights(int M, int P, double t0, double dt, double *tau, double *taue,
                     double *s, double *shat, double *stilde, double *semb);

/* MRSDC(M, P) with K sweeps: Algorithm 1 (predictor) then K x Algorithm 2, with
 * f^I = (A + B_env) T, g = b_env, f^E = K_G(t) T + b_G(t).  Implicit solves
 * (M_L - dt/M (A + B_env)) x = rhs by Jacobi-PCG to rtol.  stats: per step {solves,
 * CG iterations, SDC residual r^K}.  T[N] in/out. */
int or_step_mrsdc(or_sys *s, double t, double dt, int32_t nsteps, int32_t M, int32_t P, int32_t K,
                  double s0, double amp, double period, double dx, double dy, double dz,
                  double eta0, double eta_amp, double eta_period, double *T, double rtol, double *stats);

/* Single-rate SDC with M equidistant no-left nodes and K sweeps, every term
 * implicit -- the interface operator reassembled at each node of each sweep (the "single-rate
 * SDC" of the work-precision study P:730-736, reading R29).  M = 1, K = 0 is implicit Euler.
 * stats (may be NULL): per step {solves, CG iterations, SDC residual}. */
int or_step_sdc(or_sys *s, double t, double dt, int32_t nsteps, int32_t M, int32_t K,
                double s0, double amp, double period, double dx, double dy, double dz,
                double eta0, double eta_amp, double eta_period, double *T, double rtol, double *stats);

#ifdef __cplusplus
}
#endif
#endif
