/*
 * oracle_sanitize.c -- every entry point of the CPU oracle (oracle/oracle.h) on a small two-slab
 * pair, built with -fsanitize=address,undefined by tests/test_oracle_sanitize.py (SURVEY 4.2:
 * "the oracle is also built with -fsanitize=address,undefined").  Test infrastructure only.
 *
 * Rail 0.3 x 0.2 x 0.1 m (6x4x2 cells, floor Robin 50 W/m^2K at 24 C) under a non-matching
 * stock (5x3x4 cells, cooled top 200 W/m^2K at 18 C), contact alpha = 1000, friction 500:
 *   1. coupled stationary state (or_stationary) vs the analytic two-slab profile;
 *   2. implicit Euler with dt = 1e7 s by CG with the quadratic-extrapolation start
 *      (or_set_guess) and by dense Cholesky -> the same profile;
 *   3. MRSDC(3,2) and SDC(3) steps from the uniform state stay finite and bounded;
 *   4. the MRSDC weight tables, interface / volume getters, residual rows.
 * Exit code 0 and "oracle_sanitize ok" on success.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "box_mesh.h"
#include "oracle.h"

static int check_profile(const double *T, const mesh_t *f, const mesh_t *s, const char *what) {
    const double Tbot = 22.5, T1 = 22.35, T2 = 22.025, Ttop = 20.875;   /* analytic, H1 = H2 = 0.1 */
    double err = 0.0;
    for (int i = 0; i < f->nn; i++) err = fmax(err, fabs(T[i] - (Tbot + (T1 - Tbot) * f->xyz[3 * i + 2] / 0.1)));
    for (int i = 0; i < s->nn; i++)
        err = fmax(err, fabs(T[f->nn + i] - (T2 + (Ttop - T2) * (s->xyz[3 * i + 2] - 0.1) / 0.1)));
    printf("%s: max |T - analytic| = %.3e\n", what, err);
    return err < 1e-8 ? 0 : 1;
}

int main(void) {
    mesh_t f, s;
    make_box(&f, 6, 4, 2, 0.3, 0.2, 0.1, 0.0, 3, 4);
    make_box(&s, 5, 3, 4, 0.3, 0.2, 0.1, 0.1, 4, 2);
    or_sys *o = or_create(f.nn, f.xyz, f.nt, f.tets, f.nf, f.faces, f.tags, s.nn, s.xyz, s.nt, s.tets, s.nf,
                          s.faces, s.tags, 4, 50.0, 3.6e6, 1000.0);
    if (!o) { fprintf(stderr, "or_create: %s\n", or_last_error()); return 1; }
    if (or_set_robin(o, 0, 3, 50.0, 24.0, 0, 0, 0) || or_set_robin(o, 1, 2, 200.0, 18.0, 0, 0, 0)) return 1;
    const int64_t n = or_n(o);
    double *T = malloc(sizeof(double) * n), stats[4 * 8];
    int bad = 0;
    /* 1. stationary, coupled */
    for (int64_t i = 0; i < n; i++) T[i] = 24.0;
    if (or_stationary(o, 0.0, 1, 0.0, 0.0, 1.0, 1, 0, 0, 500.0, 0.0, 1.0, T, 0, 1e-12, 0, stats)) return 1;
    bad |= check_profile(T, &f, &s, "stationary (CG)");
    /* 2. implicit Euler, dt -> infinity: CG with the extrapolated start, then dense Cholesky */
    if (or_set_guess(o, 2) || or_set_guess(o, 3) != -1) return 1;
    for (int64_t i = 0; i < n; i++) T[i] = 24.0;
    if (or_step(o, 0.0, 1e7, 5, 0.0, 0.0, 1.0, 1, 0, 0, 500.0, 0.0, 1.0, T, 0, 1e-12, 0, stats)) return 1;
    bad |= check_profile(T, &f, &s, "implicit Euler CG, extrapolated start");
    for (int64_t i = 0; i < n; i++) T[i] = 24.0;
    if (or_step(o, 0.0, 1e7, 5, 0.0, 0.0, 1.0, 1, 0, 0, 500.0, 0.0, 1.0, T, 1, 1e-12, 0, stats)) return 1;
    bad |= check_profile(T, &f, &s, "implicit Euler Cholesky");
    /* 3. the SDC methods from the uniform state (moving stock, time-varying friction) */
    for (int64_t i = 0; i < n; i++) T[i] = 24.0;
    if (or_step_mrsdc(o, 0.0, 1.0, 2, 3, 2, 1, 0.0, 0.02, 10.0, 1, 0, 0, 500.0, 0.5, 5.0, T, 1e-12, stats)) return 1;
    for (int64_t i = 0; i < n; i++) if (!(T[i] > 17.0 && T[i] < 26.0)) bad = 1;
    if (or_step_sdc(o, 2.0, 1.0, 2, 3, 1, 0.0, 0.02, 10.0, 1, 0, 0, 500.0, 0.5, 5.0, T, 1e-12, stats)) return 1;
    for (int64_t i = 0; i < n; i++) if (!(T[i] > 17.0 && T[i] < 26.0)) bad = 1;
    /* 4. tables and getters */
    double tau[3], taue[6], sw[9], shat[6], stilde[18], semb[12];
    if (or_mrsdc_weights(3, 2, 0.0, 1.0, tau, taue, sw, shat, stilde, semb)) return 1;
    const int64_t nnz = or_vol_nnz(o);
    int64_t *rp = malloc(sizeof(int64_t) * (n + 1));
    int32_t *col = malloc(sizeof(int32_t) * nnz);
    double *A = malloc(sizeof(double) * nnz), *B = malloc(sizeof(double) * nnz);
    double *ML = malloc(sizeof(double) * n), *be = malloc(sizeof(double) * n);
    or_get_volume(o, rp, col, A, B, ML, be);
    if (or_assemble_interface(o, 0.01, 0.0, 0.0, 500.0)) return 1;
    const int64_t inz = or_iface_nnz(o);
    int64_t *irp = malloc(sizeof(int64_t) * (n + 1));
    int32_t *icol = malloc(sizeof(int32_t) * (inz > 0 ? inz : 1));
    double *ival = malloc(sizeof(double) * (inz > 0 ? inz : 1)), *bG = malloc(sizeof(double) * n), area = 0.0;
    or_get_interface(o, irp, icol, ival, bG, &area);
    if (fabs(area - 0.29 * 0.2) > 1e-12) { printf("area %.15g\n", area); bad = 1; }   /* footprint shifted 0.01 m */
    double *y = malloc(sizeof(double) * n), res[4], bnorm = 0.0;
    or_apply_system(o, 1.0, T, y);
    const int64_t rows[4] = {0, 1, n / 2, n - 1};
    if (or_ie_residual_rows(o, 1.0, 0.01, 0.0, 0.0, 500.0, T, T, 4, rows, res, &bnorm)) return 1;
    free(rp); free(col); free(A); free(B); free(ML); free(be); free(irp); free(icol); free(ival); free(bG); free(y);
    free(T);
    or_destroy(o);
    free(f.xyz); free(f.tets); free(f.faces); free(f.tags);
    free(s.xyz); free(s.tets); free(s.faces); free(s.tags);
    if (bad) { printf("oracle_sanitize FAILED\n"); return 1; }
    printf("oracle_sanitize ok\n");
    return 0;
}
