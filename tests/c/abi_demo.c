/*
 * abi_demo.c -- the C ABI of include/thermo.h used from plain C99, without Python.
 *
 * Builds two stacked slabs with non-matching Kuhn tetrahedral lattices (rail 0.3 x 0.2 x 0.1 m
 * with 6x4x2 cells, stock on top with 5x3x4 cells), Robin floor (50 W/m^2K, 24 C) and cooled
 * top (200, 18), contact alpha = 1000 and friction eta = 500, then
 *   1. computes the coupled stationary state (thermo_stationary) and checks it
 *      against the analytic piecewise-linear two-slab profile (bottom 22.5, rail top 22.35,
 *      stock bottom 22.025, top 20.875 C; derived in tests/test_oracle_stepping.py);
 *   2. takes 5 implicit-Euler steps with a huge dt (thermo_step) from the uniform state and
 *      checks the same profile (dt -> infinity);
 *   3. checks the error paths (bad n -> THERMO_EINVAL).
 * Exit code 0 and "abi_demo ok" on success.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "thermo.h"
#include "box_mesh.h"

static int check_profile(thermo_ctx *ctx, const mesh_t *f, const mesh_t *s, const char *what) {
    const double Tbot = 22.5, T1 = 22.35, T2 = 22.025, Ttop = 20.875;   /* analytic, H1 = H2 = 0.1 */
    int n = f->nn + s->nn;
    double *T = malloc(sizeof(double) * n);
    if (thermo_get_T(ctx, 0, -1, T, n, 0)) { fprintf(stderr, "get_T: %s\n", thermo_last_error(ctx)); return 1; }
    double err = 0.0;
    for (int i = 0; i < f->nn; i++) {
        double z = f->xyz[3 * i + 2];
        err = fmax(err, fabs(T[i] - (Tbot + (T1 - Tbot) * z / 0.1)));
    }
    for (int i = 0; i < s->nn; i++) {
        double z = s->xyz[3 * i + 2];
        err = fmax(err, fabs(T[f->nn + i] - (T2 + (Ttop - T2) * (z - 0.1) / 0.1)));
    }
    free(T);
    printf("%s: max |T - analytic| = %.3e\n", what, err);
    return err < 1e-9 ? 0 : 1;
}

int main(void) {
    mesh_t f, s;
    make_box(&f, 6, 4, 2, 0.3, 0.2, 0.1, 0.0, 3, 4);   /* floor 3, contact 4 */
    make_box(&s, 5, 3, 4, 0.3, 0.2, 0.1, 0.1, 4, 2);   /* contact 4, cooled top 2 */
    thermo_mesh mf = {f.nn, f.xyz, f.nt, f.tets, f.nf, f.faces, f.tags};
    thermo_mesh ms = {s.nn, s.xyz, s.nt, s.tets, s.nf, s.faces, s.tags};
    thermo_scenario sc = {0.0, 0.0, 1.0, {1.0, 0.0, 0.0}, 500.0, 0.0, 1.0};
    thermo_ctx *ctx = NULL;
    int rc = thermo_create_mesh(&ctx, &mf, &ms, 4, 4, 50.0, 3.6e6, 1000.0, 1, &sc, 24.0, NULL);
    if (rc) { fprintf(stderr, "create: %d %s\n", rc, thermo_last_error(NULL)); return 1; }
    const double g0[3] = {0.0, 0.0, 0.0};
    if (thermo_set_bc(ctx, 0, 3, 50.0, 24.0, g0) || thermo_set_bc(ctx, 1, 2, 200.0, 18.0, g0)) {
        fprintf(stderr, "set_bc: %s\n", thermo_last_error(ctx));
        return 1;
    }
    int bad = 0;
    if (thermo_stationary(ctx, 0.0, 1)) { fprintf(stderr, "stationary: %s\n", thermo_last_error(ctx)); return 1; }
    bad |= check_profile(ctx, &f, &s, "stationary");
    double *T0 = malloc(sizeof(double) * (f.nn + s.nn));
    for (int i = 0; i < f.nn + s.nn; i++) T0[i] = 24.0;
    if (thermo_set_T(ctx, 0, -1, T0, f.nn + s.nn, 0) || thermo_step(ctx, 0.0, 1e7, 5)) {
        fprintf(stderr, "step: %s\n", thermo_last_error(ctx));
        return 1;
    }
    bad |= check_profile(ctx, &f, &s, "implicit Euler, dt = 1e7 s");
    thermo_stats st;
    if (thermo_get_stats(ctx, &st) || st.steps_done != 5 || st.failed_step != -1) bad = 1;
    if (thermo_get_T(ctx, 0, -1, T0, 3, 0) != THERMO_EINVAL) bad = 1;   /* wrong n */
    if (thermo_set_guess(ctx, 3) != THERMO_EINVAL || thermo_set_guess(ctx, 0) != THERMO_OK) bad = 1;
    thermo_destroy(ctx);
    free(T0);
    if (bad) { printf("abi_demo FAILED\n"); return 1; }
    printf("abi_demo ok\n");
    return 0;
}
