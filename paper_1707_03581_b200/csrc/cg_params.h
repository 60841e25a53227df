// cg_params.h -- parameter block of the single-scenario Jacobi-PCG solve kernels (cg.cu: the
// persistent grid kernels; cg_cluster.cu: the one-cluster latency kernel).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace thermo {

struct CGParams {
    int64_t N, nslices, nchunks;
    const int64_t *slice_ptr;
    const int32_t *col;
    const uint16_t *lcol;      // KIND 2: chunk-local 16-bit columns (same layout as col)
    const double *val;
    const double *ML, *benv, *Dinv;
    int n_if, nA;
    const int32_t *if_rows, *slice_if, *ell_cnt, *ell_col;
    const double *ell_val, *if_b, *if_phi;
    const double *T_in;
    const double *X0;          // optional initial guess (extrapolated state); nullptr: x0 = T_in
    const double *rhs;         // optional explicit right-hand side (MRSDC implicit solves)
    double *T_out, *z, *pa, *pb, *q;
    double *z2, *q2;           // FUSED: second buffer set of z and q' (p uses pa / pb)
    double *partials;
    int *status;
    double *fail_relres;
    int32_t *iters_out;
    double *relres_out, *area_out;
    double dt, rtol2;
    int maxit, step;
    int stage_entries;         // TMA: matrix entries per stage
    int nstages;               // TMA: ring stages (<= 8)
    int64_t u_rows;            // TMA: rows per update-phase chunk (4 streams per stage)
    int win_cap;               // KIND 2: window entries per vector per stage
    const int32_t *chunk_hi;   // TMA: largest column index referenced by each chunk
    const int2 *chunk_runs;    // KIND 2: [nchunks][CG_MAXR] (start, length) of the window runs
    const int32_t *chunk_nruns;
    const int32_t *chunk_lown;  // KIND 2: window-local index of the chunk's first row
    const double *pf[4];       // vectors whose leading edge is prefetched into L2
    int npf;
    const double *wv[3];       // KIND 2: vectors staged through the window (nwv <= nwin)
    int nwv;
    int nwin;                  // KIND 2: window slots of the stage layout (1, FUSED: 3)
    const double *ownv;        // KIND 2: vector of which only the chunk's own rows are staged
                               // (after the window, W * 32 rows)
    unsigned long long *trace; // optional: %globaltimer after every grid barrier (CTA 0)
    int trace_fine;            // fused kernel: also at the iteration start, sweep end, CTA reduction
    int prefetch;              // L2 leading-edge prefetch (THERMO_CG_PREFETCH=1; measured slower on cfg3)
    const int32_t *if_of_row;  // cluster kernel: interface index of a row (-1: none)
    int64_t cl_rows;           // cluster kernel: shared-memory rows per vector
    int rs_ell;                // resident kernel: ELL capacity of an interface row
    const int64_t *rs_part;    // resident kernel: [grid + 1] first slice of every CTA
    int xhist, xguess, xsave;  // resident kernel: the extrapolated start formed in phase 0 -- order min(xhist + step
                               // in launch, xguess) (0: x0 = X0 or T^n) from T^n, T_out's old content T^{n-1} and
                               // Th = T^{n-2}; xsave: shift the history (Th <- T^{n-1}) at the end of a step
    double *Th;
    int nst;                   // resident kernel: steps of this launch (ahead mode: their interfaces in
                               // consecutive slots from ell_cnt / ell_col / ... on; the state buffers alternate)
    double *Tin_w;             // = T_in, writable: the output buffer of the odd steps of a launch
    const double *if_dinv_s;   // resident kernel, ahead mode: Jacobi inverse diagonal of the interface rows of
                               // this step's slot ([n_if]; Dinv then holds the volume-only diagonal)
    unsigned *gbar, *gbar_next;   // resident kernel: grid-barrier arrive counter of this launch (zero at its
                                  // start) and the one it zeroes for the next launch
    int debug;                 // THERMO_CG_DEBUG bits (measurement only, results invalid):
                               // 1 consumers skip the row work, 2 no window copies, 4 no prefetch,
                               // 8 no q' store
};

}  // namespace thermo
