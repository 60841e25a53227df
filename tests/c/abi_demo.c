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

typedef struct {
    int nn, nt, nf;
    double *xyz;
    int32_t *tets, *faces, *tags;
} mesh_t;

static double det3(const double *a, const double *b, const double *c, const double *d) {
    double u[3], v[3], w[3];
    for (int k = 0; k < 3; k++) { u[k] = b[k] - a[k]; v[k] = c[k] - a[k]; w[k] = d[k] - a[k]; }
    return u[0] * (v[1] * w[2] - v[2] * w[1]) - u[1] * (v[0] * w[2] - v[2] * w[0]) + u[2] * (v[0] * w[1] - v[1] * w[0]);
}

static int cmp3(const void *a, const void *b) {
    const int32_t *x = a, *y = b;
    for (int k = 0; k < 3; k++) if (x[k] != y[k]) return x[k] < y[k] ? -1 : 1;
    return 0;
}

/* box [0,L]^3-ish lattice of nx x ny x nz cells at height z0, Kuhn split (6 tets per cell along
 * the (0,0,0)-(1,1,1) diagonal); boundary faces = tet faces seen once; tag by position */
static void make_box(mesh_t *m, int nx, int ny, int nz, double Lx, double Ly, double Lz, double z0,
                     int tag_bottom, int tag_top) {
    m->nn = (nx + 1) * (ny + 1) * (nz + 1);
    m->nt = 6 * nx * ny * nz;
    m->xyz = malloc(sizeof(double) * 3 * m->nn);
    m->tets = malloc(sizeof(int32_t) * 4 * m->nt);
#define NID(i, j, k) ((i) + (nx + 1) * ((j) + (ny + 1) * (k)))
    for (int k = 0; k <= nz; k++)
        for (int j = 0; j <= ny; j++)
            for (int i = 0; i <= nx; i++) {
                double *p = m->xyz + 3 * NID(i, j, k);
                p[0] = Lx * i / nx; p[1] = Ly * j / ny; p[2] = z0 + Lz * k / nz;
            }
    static const int perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    int t = 0;
    for (int k = 0; k < nz; k++)
        for (int j = 0; j < ny; j++)
            for (int i = 0; i < nx; i++)
                for (int p = 0; p < 6; p++) {
                    int c[3] = {0, 0, 0}, v[4];
                    v[0] = NID(i, j, k);
                    for (int s = 0; s < 3; s++) {
                        c[perm[p][s]] = 1;
                        v[s + 1] = NID(i + c[0], j + c[1], k + c[2]);
                    }
                    if (det3(m->xyz + 3 * v[0], m->xyz + 3 * v[1], m->xyz + 3 * v[2], m->xyz + 3 * v[3]) < 0) {
                        int tmp = v[1]; v[1] = v[2]; v[2] = tmp;
                    }
                    memcpy(m->tets + 4 * t++, v, sizeof v);
                }
#undef NID
    /* all tet faces (sorted vertex triple + the oriented triple), boundary = seen once */
    int32_t *all = malloc(sizeof(int32_t) * 6 * 4 * m->nt);
    static const int fv[4][3] = {{1, 2, 3}, {0, 3, 2}, {0, 1, 3}, {0, 2, 1}};   /* outward for det > 0 */
    for (int e = 0; e < m->nt; e++)
        for (int f = 0; f < 4; f++) {
            int32_t *r = all + 6 * (4 * e + f);
            for (int s = 0; s < 3; s++) r[3 + s] = m->tets[4 * e + fv[f][s]];
            int32_t a = r[3], b = r[4], cc = r[5], tmp;
            if (a > b) { tmp = a; a = b; b = tmp; }
            if (b > cc) { tmp = b; b = cc; cc = tmp; }
            if (a > b) { tmp = a; a = b; b = tmp; }
            r[0] = a; r[1] = b; r[2] = cc;
        }
    qsort(all, 4 * (size_t)m->nt, sizeof(int32_t) * 6, cmp3);
    m->faces = malloc(sizeof(int32_t) * 3 * 4 * m->nt);
    m->tags = malloc(sizeof(int32_t) * 4 * m->nt);
    m->nf = 0;
    for (int q = 0; q < 4 * m->nt;) {
        int r = q + 1;
        while (r < 4 * m->nt && cmp3(all + 6 * q, all + 6 * r) == 0) r++;
        if (r - q == 1) {
            const int32_t *o = all + 6 * q + 3;
            double zc = (m->xyz[3 * o[0] + 2] + m->xyz[3 * o[1] + 2] + m->xyz[3 * o[2] + 2]) / 3.0;
            memcpy(m->faces + 3 * m->nf, o, sizeof(int32_t) * 3);
            m->tags[m->nf++] = fabs(zc - z0) < 1e-12 ? tag_bottom : (fabs(zc - z0 - Lz) < 1e-12 ? tag_top : 0);
        }
        q = r;
    }
    free(all);
}

static int check_profile(void *ctx, const mesh_t *f, const mesh_t *s, const char *what) {
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
    void *ctx = NULL;
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
