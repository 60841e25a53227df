/*
 * box_mesh.h -- Kuhn-split box lattices for the plain-C test programs (abi_demo.c,
 * oracle_sanitize.c): nodes, positively oriented tetrahedra, boundary faces tagged by height.
 */
#ifndef BOX_MESH_H
#define BOX_MESH_H
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

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


#endif
