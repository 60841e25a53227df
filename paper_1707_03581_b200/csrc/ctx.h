// ctx.h -- host-side context of the thermo library (see include/thermo.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "common.cuh"

namespace thermo {

#define THERMO_MAX_ROW 96   // max distinct neighbours of one node in the volume pattern

struct Robin {
    int part, tag;
    double alpha, T_ref, g[3];
};

struct Scen {
    double s0, amp, period, dir[3], eta0, eta_amp, eta_period;
    double d2[2];  // in-plane motion direction
};

struct Ctx {
    cudaStream_t stream = nullptr;
    int dev = 0, num_sms = 0;
    std::string err;

    int64_t nf = 0, nm = 0, N = 0;
    int S = 1;
    int SP = 1;                      // scenario columns of the state / workspace block vectors (>= S)
    int CW = 1;                      // block layout [SP / CW][N][CW]: CW = SP (row-major N x SP) or 32
                                     // (column groups of the windowed SpMM kernel, cg_spmm.cu)
    double *d_DinvS = nullptr;       // S > 1: per-scenario Jacobi inverse diagonal [N][SP]
    double nu = 0, rho_cp = 0, alpha = 0;
    int iface_tag_f = 0, iface_tag_m = 0;
    std::vector<Scen> scen;
    std::vector<Robin> robin;

    // mesh on the device (coupled numbering: fixed nodes first)
    int64_t ntets = 0, nfaces = 0;
    double *d_xyz = nullptr;         // [N][3]
    int32_t *d_tets = nullptr;       // [ntets][4]
    int32_t *d_faces = nullptr;      // [nfaces][3]
    int32_t *d_fkey = nullptr;       // [nfaces] part * 65536 + tag
    int64_t *d_tinc_ptr = nullptr;   // node -> tet incidence
    int32_t *d_tinc = nullptr;
    int64_t *d_finc_ptr = nullptr;   // node -> boundary face incidence
    int32_t *d_finc = nullptr;

    // volume operator in sliced ELL (slice height 32)
    int64_t nslices = 0, nnz = 0, nnz_pad = 0;
    int64_t *d_slice_ptr = nullptr;  // [nslices + 1] entry offsets
    int32_t *d_col = nullptr;        // [nnz_pad]
    double *d_A = nullptr;           // stiffness  -nu int grad phi grad phi
    double *d_R = nullptr;           // Robin      -int alpha phi phi
    double *d_val = nullptr;         // K~ = M_L - dt (A + R) (volume part)
    int64_t *d_diagpos = nullptr;    // [N]
    double *d_ML = nullptr, *d_benv = nullptr, *d_Dvol = nullptr, *d_Dinv = nullptr;
    double *d_robin_tab = nullptr;   // [nrobin][8]
    double built_dt = -1.0;
    bool robin_dirty = true;

    // interface
    int n_if = 0, nA = 0, nTA = 0, nTB = 0, cap = 0, pcap = 0, cmax = 0;
    PairRec *d_pairs = nullptr;
    int32_t *d_pcnt = nullptr;
    int32_t *d_refs = nullptr;           // rail-side record references (k_pairs / k_refsort)
    int32_t *d_if_rows = nullptr;
    double2 *d_uv = nullptr;
    int32_t *d_star_ptr = nullptr, *d_star_tri = nullptr;
    int32_t *d_star_own = nullptr, *d_own_ptr = nullptr, *d_own_idx = nullptr;   // k_rows own-column slots
    int4 *d_triA = nullptr, *d_triB = nullptr;
    double4 *d_boxA = nullptr, *d_boxB = nullptr;
    BinGrid binA{}, binB{};
    int32_t *d_binA_ptr = nullptr, *d_binA_ids = nullptr, *d_binB_ptr = nullptr, *d_binB_ids = nullptr;
    int32_t *d_slice_if = nullptr;   // [nslices + 1]
    int32_t *d_ell_cnt = nullptr, *d_ell_col = nullptr;
    double *d_ell_val = nullptr, *d_if_b = nullptr, *d_if_phi = nullptr, *d_if_dinv = nullptr;
    double *d_if_d = nullptr;        // S > 1 (windowed SpMM): per-scenario diagonal of the interface rows
    double plane_n[3] = {0, 0, 1}, e1[3] = {1, 0, 0}, e2[3] = {0, 1, 0};
    double min_edge = 0.0;

    // state and CG workspace (N x S, row-major)
    double *d_T[2] = {nullptr, nullptr};
    int cur = 0;                     // index of the buffer holding the committed state
    double *d_z = nullptr, *d_p[2] = {nullptr, nullptr}, *d_q = nullptr;
    double *d_partials = nullptr;    // [grid][THERMO_NRED]
    int *d_status = nullptr;         // [0] failure, [1] overflow, [2] failed step, [3] failed scen
    double *d_fail_relres = nullptr;
    double *d_step_sc = nullptr;     // [steps][S][4]
    int32_t *d_iters = nullptr;      // [steps][S]
    double *d_relres = nullptr;      // [steps][S]
    double *d_area = nullptr;        // [steps]
    int64_t step_cap = 0;
    double *d_rhs = nullptr;           // [N] right-hand side of the stationary solve
    int cg_grid = 0, cg_block = 0, cg_stage_entries = 0;
    size_t cg_smem = 0;
    bool cg_tma = false;
    int cg_variant = 0, cg_kind = -1, cg_chunk = 8, cg_debug = 0, cg_prefetch = 0;
    bool cg_fused = false;           // one-barrier-per-iteration kernel (second z / q' set below)
    double *d_z2 = nullptr, *d_q2 = nullptr;
    int32_t *d_chunk_hi = nullptr;
    uint16_t *d_lcol = nullptr;      // chunk-local 16-bit columns (window kernels)
    int2 *d_chunk_runs = nullptr;    // window runs per chunk
    int32_t *d_chunk_nruns = nullptr;
    int32_t *d_chunk_lown = nullptr;
    unsigned long long *d_trace = nullptr;   // THERMO_CG_TRACE=1: barrier timestamps of the last solve
    int cg_win_cap = 0, cg_nstages = 1, cg_max_runs = 0;
    bool cl_on = false;              // single-cluster latency solve (cg_cluster.cu) for small N
    double *d_cl_ai = nullptr;       // its interface sums (2 n_if)
    int64_t cl_rows = 0;
    size_t cl_smem = 0;
    bool rs_on = false;              // resident-operator latency solve (cg_resident.cu)
    int64_t *d_rs_part[2] = {nullptr, nullptr};        // slice blocks of its CTAs (full grid, overlap grid)
    size_t rs_smem = 0;
    unsigned *d_gbar = nullptr;      // its two grid-barrier arrive counters (alternating between launches)
    int rs_parity = 0;
    // Ahead mode (single scenario, implicit Euler; with the resident solve, and for the sizes without
    // the overlap mode): the interface of a step depends only on
    // its time, so the interfaces of the next ah_slots step times are assembled in ONE launch set
    // (batch entry = step, slot-major buffers) and the solves run back to back; slots left over
    // at the end of a call belong to the presumed next call (same dt, t = the end of this one)
    bool ah_on = false, ah_valid = false;
    int ah_slots = 0, ah_next = 0, ah_count = 0;
    double ah_dt = 0.0;
    uint64_t ah_opver = 0, op_ver = 0;    // op_ver: rebuilds of the volume operator / Jacobi diagonal
    std::vector<double> ah_tp;            // step time of every assembled slot
    void *d_ah_pairs = nullptr;
    int32_t *d_ah_refs = nullptr, *d_ah_pcnt = nullptr, *d_ah_ell_cnt = nullptr, *d_ah_ell_col = nullptr;
    double *d_ah_ell_val = nullptr, *d_ah_if_b = nullptr, *d_ah_if_phi = nullptr, *d_ah_dinv = nullptr,
           *d_ah_d = nullptr, *d_ah_sc = nullptr;
    int64_t cg_u_rows = 0;
    int *d_chunk_ctr = nullptr;

    // Overlap (single scenario, implicit Euler, L2-resident sizes): the interface kernels of
    // step n+1 run on if_stream into the second interface buffer set (suffix _b) while the solve
    // of step n runs on the remaining SMs (the persistent CG grid leaves overlap_sms free).
    bool overlap = false;
    int overlap_sms = 0, cg_grid_ovl = 0;
    int32_t *d_ell_cnt_b = nullptr, *d_ell_col_b = nullptr;
    double *d_ell_val_b = nullptr, *d_if_b_b = nullptr, *d_if_phi_b = nullptr, *d_Dinv_b = nullptr;
    cudaStream_t if_stream = nullptr;
    // ev_if: interface(n) done; ev_cg: launch completion of solve(n) (all CTAs begun)
    cudaEvent_t ev_if[2] = {nullptr, nullptr}, ev_cg[2] = {nullptr, nullptr}, ev_main = nullptr;
    cudaEvent_t ev_done[2] = {nullptr, nullptr};   // solve(n) complete
    // buffer set of a call's step n: (if_phase + n) & 1 (if_phase advances by nsteps per call).
    // Speculation: after the last solve of a call, the interface of the presumed next step
    // (t + nsteps dt, same dt) is assembled on the side stream into the next buffer set, so a
    // caller stepping one step per call (a digital twin reading every field) still overlaps;
    // a mismatching next call (or any rebuild / SDC step / stationary solve) discards it.
    int if_phase = 0;
    bool spec_valid = false;
    double spec_t = 0.0, spec_dt = 0.0;
    double *d_step_sc_spec = nullptr;   // [4] scalars of the speculated step
    int *d_spec_status = nullptr;       // [8] overflow flag / step of the speculated assembly
    bool side_pending = false;          // side-stream work not yet ordered before the main stream
    cudaEvent_t ev_side_end = nullptr;  // recorded after the speculated assembly
    std::vector<cudaEvent_t> events_if;   // timing of the side-stream interface kernels

    double rtol = 1e-12;
    int maxit = 0;
    // initial guess of the implicit-Euler solves: 0 = T^n (reading R17), 1 = linear, 2 = quadratic
    // extrapolation of the last states (thermo_set_guess); hist = consecutive committed
    // implicit-Euler states with step hist_dt behind the current one (0..2)
    int guess = 2, hist = 0;
    double hist_dt = 0.0;
    double *d_x0 = nullptr, *d_Thist = nullptr;   // [N x SP] guess and T^{n-2}
    // time-stepping method: 0 implicit Euler, 1 MRSDC(M, P) with K sweeps
    int method = 0, mr_M = 3, mr_P = 2, mr_K = 1;
    int32_t *d_slice_if_zero = nullptr;   // all-empty interface ranges (volume-only solves)
    double *d_KV = nullptr;               // A + B_env values (sliced ELL), f^I operator
    double *d_Dinv_vol = nullptr;         // 1 / diag(M_L - a (A + B_env)), untouched by the interface
    int32_t *d_if_of_row = nullptr;       // [N] interface index of a row or -1
    double *d_mr = nullptr;               // MRSDC node states and caches (see mrsdc.cu)
    double *d_benvS = nullptr;            // S > 1: b_env broadcast over the scenario columns
    size_t mr_vectors = 0;
    int32_t *d_mr_iters = nullptr;        // per implicit solve of the last step
    double *d_mr_relres = nullptr;
    int32_t *d_ell_cnt_s = nullptr, *d_ell_col_s = nullptr;   // MRSDC: interface operators at the
    double *d_ell_val_s = nullptr, *d_if_b_s = nullptr;       // M P + 1 node times of a step
    double *d_if_phi_s = nullptr;
    int mr_nslots = 0, mr_solves = 0;
    bool timing = false;
    std::vector<cudaEvent_t> events;   // 2 * nsteps + 1 when timing
    // asynchronous host copies of the state (thermo_get_T_async): a copy stream, and per state
    // buffer the event after which a pending copy has read it
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_copy[2] = {nullptr, nullptr};
    int copy_pending[2] = {0, 0};
    PairRec *d_pairs_s = nullptr;        // pair records of the SDC node-time slots
    int32_t *d_pcnt_s = nullptr;
    int32_t *d_refs_s = nullptr;
    double ms_iface = 0.0, ms_solve = 0.0;

    // windowed SpMM batched kernel (cg_spmm.cu)
    bool sb_on = false;
    int sb_G = 1, sb_nstages = 0;
    uint32_t sb_stage = 0, sb_col_off = 0, sb_win_off = 0, sb_own_off = 0, sb_aux_off = 0, sb_meta_off = 0;
    size_t sb_smem = 0;
    double *d_sb_partials = nullptr, *d_sb_totals = nullptr;
    int32_t *d_sb_if_ptr = nullptr, *d_sb_if_k = nullptr;   // interface rows per CTA
    void *d_sb_recs = nullptr;                              // packed chunk metadata per CTA
    int32_t *d_sb_rec_ptr = nullptr;
    int *d_sb_dbg = nullptr;                                // sb_check mismatch counter (debug)
    double *d_sb_ai = nullptr;                              // interface sums of a sweep
    int64_t *d_sb_ptr8 = nullptr;                           // row-major operator copy per slice
    double *d_sb_val8 = nullptr;
    uint16_t *d_sb_lcol8 = nullptr;

    // internal numbering (reorder.cu): nullptr / empty = the caller's numbering
    int32_t *d_int_of_ext = nullptr;      // [N] internal index of the caller's node e
    std::vector<int32_t> h_ext_of_int;    // [N] the caller's index of internal node i
    int reorder = 0;                      // 0 caller's numbering kept, 1 RCM
    int probe_runs = 0, probe_window = 0; // window test of the caller's numbering (create)
    // staging of the host transfers: one contiguous field per scenario for state buffer b,
    // valid while stage_ver[b] == ver[b] (ver[b] counts the writes of d_T[b], see guard_write)
    double *d_stage[2] = {nullptr, nullptr};
    int64_t ver[2] = {0, 0}, stage_ver[2] = {-1, -1};

    // pinned host staging of a call's time scalars and status readback (thermo.cu: pin_reserve)
    void *h_pin = nullptr;
    size_t h_pin_bytes = 0;

    // stats of the last thermo_step
    int last_nsteps = 0;
    int64_t last_launches = 0;       // kernels launched by the last implicit-Euler thermo_step
    bool status_clean = false;   // d_status is in its initial state (see thermo_step)
    bool rep_pending = false;    // h_iters / h_relres / h_area of the last implicit-Euler call not fetched yet
    int rep_nsteps = 0;
    std::vector<int32_t> h_iters;
    std::vector<double> h_relres, h_area;
    int64_t steps_done = 0;
    int failed_step = -1, failed_scen = -1;
    double failed_relres = 0.0;
};

// assemble.cu
int assemble_create(Ctx &c, const double *xyz, const int32_t *tets, const int32_t *faces,
                    const int32_t *fkey);
int assemble_robin(Ctx &c);
int build_operator(Ctx &c, double dt, double mu = 1.0);   // K~ = mu M_L - dt (A + B_env)

// iface.cu
int iface_setup(Ctx &c, const double *h_xyz, const std::vector<int32_t> &facesA,
                const std::vector<int32_t> &facesB);
void iface_params(Ctx &c, IfaceParams &p, const double *step_sc, double dt, int buf = 0);
int iface_launch(Ctx &c, const IfaceParams &p, cudaStream_t stream = nullptr);

// cg.cu
int cg_setup(Ctx &c);
// cg_cluster.cu (single-cluster latency solve; cl_setup decides, cl_launch replaces the grid launch)
struct CGParams;
int cl_setup(Ctx &c);
int cl_launch(Ctx &c, CGParams &P, bool ovl, int buf);
// cg_resident.cu (resident-operator latency solve; rs_setup decides after overlap_setup, rs_launch
// replaces the grid / cluster launch)
int rs_setup(Ctx &c);
int rs_launch(Ctx &c, CGParams &P, bool ovl, int buf);
int ahead_setup(Ctx &c);   // after rs_setup: buffers of the ahead mode
// chunk windows of the current pattern (W slices per chunk, runs merged below `gap`);
// stats: [0] max window entries, [1] max runs, [2] flags (too many entries / window too wide)
void chunk_windows_launch(Ctx &c, int W, int gap, int2 *runs, int32_t *nruns, int32_t *lown, uint16_t *lcol,
                          int *d_stats);
// x0: initial guess (extrapolated state, see thermo.cu), nullptr = the committed state T^n
int cg_launch_step(Ctx &c, int step, double dt, const double *x0 = nullptr, int buf = 0, bool ovl = false,
                   int ah_slot = -1, int xhist = 0, int xguess = 0, int nst = 1);
// ah_slot >= 0: the interface rows of that slot of the ahead buffers; resident kernel: xhist / xguess = states
// behind T^n available / wanted for the extrapolated start formed inside the kernel, nst = steps of the launch
int overlap_setup(Ctx &c);   // second interface buffer set, side stream, reduced CG grid
// Solve (M_L - a K_vol [- a K_G]) x = rhs from x0 with the operator currently in d_val (a =
// built_dt); iface = false: no interface rows.  Iterations / residual to iters_out[slot].
int cg_launch_solve(Ctx &c, const double *x0, double *x, const double *rhs, const double *Dinv, bool iface,
                    int32_t *iters_out, double *relres_out, int slot);

// mrsdc.cu (multi-rate SDC)
int mrsdc_setup(Ctx &c);
int build_if_of_row(Ctx &c);
int mrsdc_step(Ctx &c, double tn, double dt, int step_index);
int sdc_step(Ctx &c, double tn, double dt, int step_index);   // single-rate SDC (method 2)

// cg_batched.cu (S > 1 scenarios advanced together)
int cgb_setup(Ctx &c);
int cgb_prepare(Ctx &c);   // broadcast the volume D^{-1} into DinvS (after build_operator)
int cgb_launch_step(Ctx &c, int step, double dt, const double *x0 = nullptr);
// Solve (M_L - a K_vol [- a K_G]) X = RHS for every scenario from X0 (explicit right-hand side
// block, operator in d_val, Jacobi block d_DinvS); iterations / residuals to [slot][S].
int cgb_launch_solve(Ctx &c, const double *x0, double *x, const double *rhs, bool iface, int32_t *iters_out,
                     double *relres_out, int slot);

// cg_spmm.cu (S > 1: windowed SpMM kernel, selected by cgb_setup when the windows fit)
int cgb_gather_setup(Ctx &c);   // grid and buffers of the gather kernel
int sbcg_setup(Ctx &c);
int sbcg_disable(Ctx &c);   // switch a batched context to the gather kernel (state re-laid out)
int sbcg_launch_step(Ctx &c, int step, double dt, const double *x0);
int sbcg_prepare(Ctx &c);   // after every rebuild of K~_vol

// reorder.cu (internal numbering, state transfers in the caller's numbering)
int order_probe(Ctx &c, bool *good, int *max_runs, int *max_window);
int rcm_order(Ctx &c, const std::vector<char> &is_iface, bool rooted, std::vector<int32_t> &new_to_old);
int gather_T(Ctx &c, int scen, int64_t off, int64_t cnt, const double *T, double *out, cudaStream_t st);
int scatter_T(Ctx &c, int scen, int64_t off, int64_t cnt, double *T, const double *in, cudaStream_t st);
int gather_all(Ctx &c, const double *T, double *out, cudaStream_t st);

}  // namespace thermo
