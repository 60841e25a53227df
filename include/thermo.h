/*
 * thermo.h -- C ABI of the B200 implicit-Euler hot path of arXiv 1707.03581
 * (Naumann, Ruprecht, Wensch, "Toward transient finite element simulation of thermal
 * deformation of machine tools in real-time").  P:n = /root/reference/PAPER.md line n.
 *
 * The library advances the semi-discrete, two-mesh P1 finite-element heat system
 *
 *   M dT/dt = (A + B_env + M_B(t)) T + C_B(t) T_other + b_env + b(t)
 *
 * of a fixed stand/rail (part 0) and a stock (part 1) sliding along it with implicit Euler
 * (P:211-213): per step n, with t' = t + (n+1) dt,
 *
 *   (M_L - dt K(t')) T^{n+1} = M_L T^n + dt (b_env + b_G(t'))
 *
 * where M_L is the row-sum lumped mass scaled by rho*Cp, K(t') = blockdiag(A + B_env)
 * + [[M_B,fix, C_B],[C_B^T, M_B,mov]](t') and b_G(t') the friction source eta(t')/2.
 * The interface terms are re-integrated every step on the exact intersection of the two
 * non-matching surface triangulations at the stock's current offset, and the
 * coupled system is solved monolithically by Jacobi-preconditioned CG in fp64 until
 * ||b - K~ x||_2 <= rtol ||b||_2 (default 1e-12).  CG starts from the quadratic extrapolation
 * of the last committed states by default (thermo_set_guess; order 0 = x0 = T^n): the start
 * changes the iterations, not the system or the stopping rule.
 *
 * Node numbering: the caller's numbering (per part, as passed to thermo_create_mesh) is what
 * every entry point reads and writes.  Internally the library may renumber each part
 * (reverse Cuthill-McKee) when the caller's numbering does not suit the windowed solve kernel
 * (thermo_get_stats: reordered); this is invisible at the ABI.
 *
 * Everything runs in hand-written sm_100a CUDA kernels on the caller's stream; there is no
 * CPU fallback.  Several independent scenarios (different motion / friction laws) may be
 * advanced together (batched mode, BASELINE.json config 4).
 *
 * Conventions for every entry point:
 *  - Return value: THERMO_OK (0) or a negative THERMO_E* code; functions never abort and
 *    never throw.  thermo_last_error(ctx) (or thermo_last_error(NULL) for a failed create)
 *    returns a human-readable message of the last failure on that context / thread.
 *  - Arrays are plain host pointers unless stated; all input arrays are copied during the
 *    call, so the caller may free them on return.  Indices are 0-based int32.
 *  - A context owns all device memory it allocates until thermo_destroy.  One context must
 *    not be used from two host threads at the same time.
 */
#ifndef THERMO_H
#define THERMO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Opaque context handle: owns all device memory of one coupled problem (thermo_create_mesh ..
 * thermo_destroy).  One context per host thread. */
typedef struct thermo_ctx thermo_ctx;

enum {
    THERMO_OK = 0,
    THERMO_EINVAL = -1,   /* bad argument: sizes, indices, inverted tet, non-planar interface */
    THERMO_ENOMEM = -2,   /* device or host allocation failed */
    THERMO_ECUDA = -3,    /* CUDA runtime error (message has the CUDA error string) */
    THERMO_ENOCONV = -4,  /* CG did not reach rtol within maxit; see thermo_get_stats */
    THERMO_EGEOM = -5     /* interface storage capacity exceeded.  No check of |Gamma_R| against the
                             stock-bottom area: a stock overhanging the rail is valid partial
                             contact (reading R30); |Gamma_R| of every step is
                             reported (thermo_get_stats: iface_area) */
};

/* One part's tetrahedral P1 mesh.
 *  xyz[n_nodes][3]   node coordinates (m), fp64, row-major
 *  tets[n_tets][4]   vertex indices; every tet must have positive det J (else EINVAL)
 *  bfaces[n_bfaces][3], bface_tag[n_bfaces]: boundary triangles and their tags.  Tags select
 *  Robin data (thermo_set_bc); tag 0 (or any tag without Robin data) is insulated.
 *  The moving part's coordinates are its reference position (offset s = 0). */
typedef struct {
    int64_t n_nodes;
    const double *xyz;
    int64_t n_tets;
    const int32_t *tets;
    int64_t n_bfaces;
    const int32_t *bfaces;
    const int32_t *bface_tag;
} thermo_mesh;

/* Motion and friction law of one scenario:
 *   offset s(t) = s0 + amp * sin(2 pi t / period)  along the unit vector dir (in the plane)
 *   eta(t)      = eta0 * (1 + eta_amp * sin(2 pi t / eta_period))   [W/m^2]            */
typedef struct {
    double s0, amp, period;
    double dir[3];
    double eta0, eta_amp, eta_period;
} thermo_scenario;

/* Create a context: copies both meshes to the device, assembles M_L and A
 * element by element on the device, extracts the interface triangulations (faces tagged
 * iface_tag_fixed on part 0 and iface_tag_moving on part 1; they must be coplanar), sizes
 * the per-step interface storage by sweeping each scenario's motion range, and sets the
 * state of every scenario to the uniform temperature T_init.
 *  nu [W/mK], rho_cp [J/m^3K], alpha_iface [W/m^2K]
 *  n_scen >= 1 scenarios, scen[n_scen]
 *  cuda_stream: a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream) or NULL for
 *  the legacy default stream; every later call enqueues its work on this stream.
 * On failure *out is NULL; message via thermo_last_error(NULL). */
int thermo_create_mesh(thermo_ctx **out, const thermo_mesh *fixed, const thermo_mesh *moving,
                       int32_t iface_tag_fixed, int32_t iface_tag_moving,
                       double nu, double rho_cp, double alpha_iface,
                       int32_t n_scen, const thermo_scenario *scen, double T_init,
                       void *cuda_stream);

/* Robin boundary data for faces of `part` (0 fixed, 1 moving) carrying `tag`:
 *   nu grad T . n = alpha (T_a(x) - T),   T_a(x) = T_ref + grad_T . x
 * Assembles B_env = -int alpha phi phi dS and b_env = int alpha T_a phi dS on the
 * device.  alpha = 0 removes the condition.  For part 1 grad_T must be orthogonal to every
 * scenario's motion direction (b_env of the stock is then time-independent), else EINVAL.
 * Interface tags cannot carry Robin data (EINVAL). */
int thermo_set_bc(thermo_ctx *ctx, int32_t part, int32_t tag, double alpha, double T_ref,
                  const double grad_T[3]);

/* Advance every scenario by nsteps implicit-Euler steps of size dt from time t:
 * step n uses t' = t + (n+1) dt for s, eta, M_B, C_B and b_G (fully implicit).
 * Work is enqueued on the context stream; the call synchronises that stream once at the
 * end to report status.  Returns THERMO_ENOCONV if some scenario's CG did not converge
 * within maxit (steps before the failing one are committed; the failing step and its
 * residual are in thermo_get_stats), THERMO_EGEOM if the interface storage overflowed.
 * Scheduling (no effect on the result beyond rounding of the reductions): the interface
 * operator of a step depends only on its time, so the library may assemble it early -- on a
 * side stream during the previous solve (overlap mode), or for the next 16 step times in one
 * launch set (ahead mode, with the resident-operator solve of small single-scenario problems);
 * operators assembled for times the caller then does not step to are discarded.  A call that
 * continues the previous call's time line with the same dt (t = the previous t + nsteps dt,
 * bitwise) reuses what was assembled for it. */
int thermo_step(thermo_ctx *ctx, double t, double dt, int32_t nsteps);

/* Copy the temperature of one scenario and part (0 fixed, 1 moving, -1 both: fixed nodes
 * first) into out[n]; n must equal the node count of the selection (EINVAL otherwise).
 * out_on_device != 0: out is a device pointer (e.g. a torch tensor's data_ptr()), the copy
 * is asynchronous on the context stream.  Otherwise out is host memory and the call
 * synchronises the stream. */
int thermo_get_T(thermo_ctx *ctx, int32_t scen, int32_t part, double *out, int64_t n,
                 int32_t out_on_device);

/* Asynchronous variant of thermo_get_T for host memory: enqueues the copy of the current state
 * (as of the work queued so far) on the context's copy stream and returns at once, so the
 * transfer overlaps the next thermo_step (the state is double-buffered; a later call that would
 * overwrite the buffer being copied waits for the copy on the device).  host_out should be
 * pinned (e.g. cudaHostAlloc / a pinned torch tensor) for a real overlap; its contents are valid
 * after thermo_sync().  Same selection rules and errors as thermo_get_T. */
int thermo_get_T_async(thermo_ctx *ctx, int32_t scen, int32_t part, double *host_out, int64_t n);

/* Asynchronous copy of every scenario's whole field (both parts, the caller's numbering) into
 * host_out[n_scen][n_nodes_fixed + n_nodes_moving], scenario-major, as one transfer: the
 * batched state block (N x SP, row-major on the device) is transposed by one kernel on the copy
 * stream into a staging buffer first.  n must equal n_scen * N.  Valid after thermo_sync().
 * EINVAL on a NULL pointer or a wrong n. */
int thermo_get_T_all_async(thermo_ctx *ctx, double *host_out, int64_t n);

/* Wait for all work of the context: its stream and every pending asynchronous copy. */
int thermo_sync(thermo_ctx *ctx);

/* Overwrite the temperature of one scenario and part (same selection rules as get_T). */
int thermo_set_T(thermo_ctx *ctx, int32_t scen, int32_t part, const double *in, int64_t n,
                 int32_t in_on_device);

/* Time-stepping method for thermo_step:
 *   method 0 (default): implicit Euler on the fully coupled system (above);
 *   method 1: multi-rate SDC, MRSDC(M, P) with K correction sweeps:
 *     f^I(T) = (A + B_env) T implicit with one solve of (M_L - dt/M (A + B_env)) per standard
 *     interval, f^E(T, t) = K_G(t) T + b_G(t) explicit on P embedded sub-steps (Algorithms 1-2),
 *     equidistant no-left nodes, Table-1 quadrature.  The paper's 3-D runs use M = 3, P = 2,
 *     K = 0..2.
 *   method 2: single-rate SDC(M) with K sweeps with every term implicit -- the
 *     comparison method of the work-precision study, whose interface Jacobian is reassembled
 *     at every node of every sweep (reading R29).  Implicit-Euler predictor through
 *     M equidistant no-left nodes; P is ignored.  M = 1 is implicit Euler.
 * Methods 1-2 run on batched contexts too: every scenario advances with its own motion and
 * friction law (node-time interface operators of every scenario in one launch set, the implicit
 * stages as batched solves with per-column convergence).
 * (A batched context whose implicit-Euler solves run on the windowed-SpMM kernel, the default,
 * moves its state to the gather kernel's row layout at this call: the SDC stages run there.)
 * EINVAL for other methods, M or P outside [1, 8] or K < 0. */
int thermo_set_method(thermo_ctx *ctx, int32_t method, int32_t M, int32_t P, int32_t K);

/* Replace the temperature by the stationary state of the machine at rest (the
 * initial data of the paper's 3-D runs; readings R19, R28):
 *   with_interface == 0:  0 = f^I(T) + g,  i.e. -(A + B_env) T = b_env for both parts
 *                         (uncoupled, as printed: f^E is not part of f^I);
 *   with_interface != 0:  -(A + B_env + K_G(t)) T = b_env + b_G(t), the coupling and friction
 *                         of the scenario's stock position s(t) and eta(t) included.
 * Solved by the same Jacobi-PCG kernel (x0 = current temperature, rtol / maxit of
 * thermo_set_solver; the unshifted operator needs O(1/h) iterations).  Requires a single
 * scenario (EINVAL otherwise: solve on a one-scenario context, copy with thermo_set_T).
 * ENOCONV if the solve did not converge (the temperature is then unchanged), EGEOM on
 * interface overflow.  Iterations / residual / |Gamma_R| are reported by thermo_get_stats
 * as a one-step run. */
int thermo_stationary(thermo_ctx *ctx, double t, int32_t with_interface);

/* CG stopping rule ||r||_2 <= rtol ||b||_2 (default 1e-12) and iteration cap
 * (default 0 = min(10 N, 10000)).  EINVAL if rtol <= 0 or maxit < 0. */
int thermo_set_solver(thermo_ctx *ctx, double rtol, int32_t maxit);

/* Initial guess x0 of the implicit-Euler CG solves (every scenario of a batched context alike):
 *   order 0:  x0 = T^n (reading R17; what the oracle does);
 *   order 1:  x0 = T^n + (T^n - T^{n-1});
 *   order 2:  x0 = T^{n-2} + 3 (T^n - T^{n-1})   (default),
 * the polynomial extrapolation of the last committed implicit-Euler states of equal dt (lower
 * order while fewer states exist: after create, thermo_set_T, thermo_stationary, an MRSDC/SDC
 * step, a dt change or a failed step the history restarts).  Only where CG starts changes: every
 * solve still stops at ||b - K~ x||_2 <= rtol ||b||_2, so results agree with x0 = T^n to the
 * solver tolerance, and the extrapolation saves iterations.
 * EINVAL for other orders. */
int thermo_set_guess(thermo_ctx *ctx, int32_t order);

/* Inspection / test aid (not needed for stepping): runs the interface kernels of every
 * scenario at time t (stock offset s(t), friction eta(t)) for step size dt, exactly
 * as thermo_step assembles a step, and copies scenario `scen`'s rows out.  n_if = the
 * interface row count and cap = the row capacity (thermo_get_stats: n_iface_rows,
 * iface_capacity); caller-owned host arrays:
 *   rows[n_if]      coupled row index of interface row k (rail-top nodes, then stock-bottom nodes)
 *   cnt[n_if]       entries of row k;  col[n_if][cap], val[n_if][cap]: column (coupled index) and
 *                   value of entry q < cnt[k] (col = -1, val = 0 beyond): val = -dt K_G(t) with
 *                   K_G = [[M_B,fix, C_B], [C_B^T, M_B,mov]], the term the operator
 *                   M_L - dt K(t) adds on those rows;
 *   b[n_if]         the friction source eta(t)/2 int phi_k of row k.
 * Order of the entries within a row is unspecified.  EINVAL for a bad scenario, dt <= 0,
 * non-finite t or NULL outputs; EGEOM on interface capacity overflow.  The solve data of the
 * next thermo_step are unaffected (it reassembles its own interface). */
int thermo_get_interface(thermo_ctx *ctx, int32_t scen, double t, double dt, int32_t *rows, int32_t *cnt,
                         int32_t *col, double *val, double *b);

typedef struct {
    int64_t n_fixed, n_moving;       /* node counts */
    int64_t nnz_volume;              /* stored nonzeros of the volume operator (unpadded) */
    int64_t nnz_volume_padded;       /* stored sliced-ELL entries incl. padding */
    int32_t n_scen;
    int32_t n_iface_rows;            /* rail-top + stock-bottom nodes */
    int32_t iface_capacity;          /* interface entries per row per scenario */
    int32_t last_nsteps;             /* nsteps of the last thermo_step */
    int64_t total_iters;             /* CG iterations of the last thermo_step, all scenarios */
    int32_t max_iters;               /* max over steps/scenarios of the last thermo_step */
    int32_t failed_step;             /* -1, or the first step (0-based, last call) that failed */
    int32_t failed_scen;
    double failed_relres;            /* achieved relative residual of the failing solve */
    double last_relres;              /* max over scenarios, last step */
    int64_t steps_done;              /* committed steps since create */
    double iface_area;               /* |Gamma_R| of scenario 0 at the last step (m^2) */
    double ms_iface;                 /* device time of the interface kernels and the initial-guess
                                        extrapolation, last call (ms); for small single-scenario
                                        runs the interface kernels of step n+1 run on a side stream
                                        during the solve of step n, and their time is included */
    double ms_solve;                 /* device time of the CG solve kernels, last call (ms) */
    int32_t solve_grid;              /* CTAs of the persistent CG kernel */
    int32_t solve_block;             /* threads per CTA */
    int32_t launches_per_step;       /* kernels per implicit-Euler step of the last call (interface,
                                        guess extrapolation, solve) */
    int32_t reordered;               /* 1: nodes renumbered internally at create (reverse
                                        Cuthill-McKee per part, because the caller's numbering
                                        failed the solve kernel's window test); the ABI keeps
                                        the caller's numbering either way */
    int32_t order_max_runs;          /* window test of the caller's numbering at create: max
                                        contiguous column runs of a 256-row chunk (0: not probed) */
    int32_t order_max_window;        /*   ... and max window entries of a chunk */
    int32_t solve_variant;           /* CG kernel variant chosen at create (S = 1): kind 2 =
                                        windowed TMA sweep */
    int32_t solve_kind;              /* sweep kind of the streaming grid kernel (S = 1: 0-2), 3: the
                                        batched windowed-SpMM kernel, -1: the batched gather kernel */
    int32_t solve_max_runs;          /* kind 2: max column-window runs of a chunk (internal order) */
    int32_t solve_window;            /* kind 2: max column-window entries of a chunk */
    int32_t latency_path;            /* S = 1, small problems: 0 = the streaming grid kernel solves,
                                        1 = the single-cluster kernel, 2 = the resident-operator
                                        kernel (operator and vectors in shared memory, one grid
                                        barrier per CG iteration) */
} thermo_stats;

int thermo_get_stats(const thermo_ctx *ctx, thermo_stats *out);

/* enable != 0: record CUDA events on the context stream around every interface and solve
 * kernel of thermo_step, so that thermo_get_stats reports ms_iface / ms_solve of the last
 * call (small overhead per step).  Default off. */
int thermo_set_timing(thermo_ctx *ctx, int32_t enable);

/* Per-step CG iteration counts of the last thermo_step: out[nsteps * n_scen], step-major. */
int thermo_get_step_iters(const thermo_ctx *ctx, int32_t *out, int64_t n);

const char *thermo_last_error(const thermo_ctx *ctx);
void thermo_destroy(thermo_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* THERMO_H */
