// assemble.cu -- one-time device assembly of the volume operator.
//
// Row-owner formulation: every node i gathers the contributions of its incident
// tetrahedra (and boundary faces) in ascending element order, so each matrix row is a
// sequential, deterministic sum and no atomics touch floating-point data.
//
// Layout: sliced ELL with slice height 32 (one warp per slice),
// column-major inside a slice: entry k of row i lives at slice_ptr[i/32] + 32 k + i%32.
// Short rows are padded with (col = i, value 0).
#include <cub/cub.cuh>

#include <cstdio>

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

// ------------------------------------------------------------------------------ geometry

// Gradients of the barycentric coordinates of a tet; returns det J.
__device__ __forceinline__ double tet_grad(const double *xyz, const int32_t *t, double g[4][3]) {
    double x0[3], e[3][3];
#pragma unroll
    for (int d = 0; d < 3; ++d) x0[d] = xyz[3 * t[0] + d];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int d = 0; d < 3; ++d) e[a][d] = xyz[3 * t[a + 1] + d] - x0[d];
    // cofactor rows: (e1 x e2), (e2 x e0), (e0 x e1) divided by det
    double c0[3] = {e[1][1] * e[2][2] - e[1][2] * e[2][1], e[1][2] * e[2][0] - e[1][0] * e[2][2],
                    e[1][0] * e[2][1] - e[1][1] * e[2][0]};
    double det = e[0][0] * c0[0] + e[0][1] * c0[1] + e[0][2] * c0[2];
    double c1[3] = {e[2][1] * e[0][2] - e[2][2] * e[0][1], e[2][2] * e[0][0] - e[2][0] * e[0][2],
                    e[2][0] * e[0][1] - e[2][1] * e[0][0]};
    double c2[3] = {e[0][1] * e[1][2] - e[0][2] * e[1][1], e[0][2] * e[1][0] - e[0][0] * e[1][2],
                    e[0][0] * e[1][1] - e[0][1] * e[1][0]};
    double inv = 1.0 / det;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        g[1][d] = c0[d] * inv;
        g[2][d] = c1[d] * inv;
        g[3][d] = c2[d] * inv;
        g[0][d] = -(g[1][d] + g[2][d] + g[3][d]);
    }
    return det;
}

__global__ void k_tet_check(const double *xyz, const int32_t *tets, int64_t ntets, int64_t N,
                            int *bad) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= ntets) return;
    int32_t t[4];
    for (int a = 0; a < 4; ++a) {
        t[a] = tets[4 * e + a];
        if (t[a] < 0 || t[a] >= N) { atomicOr(bad, 1); return; }
    }
    double g[4][3];
    double det = tet_grad(xyz, t, g);
    if (!(det > 0.0)) atomicOr(bad, 2);
}

// ------------------------------------------------------------------------------ incidence

__global__ void k_count(const int32_t *el, int arity, int64_t nel, int64_t *cnt) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= nel) return;
    for (int a = 0; a < arity; ++a) atomicAdd((unsigned long long *)&cnt[el[arity * e + a]], 1ull);
}

__global__ void k_fill(const int32_t *el, int arity, int64_t nel, const int64_t *ptr,
                       unsigned long long *cursor, int32_t *ids) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= nel) return;
    for (int a = 0; a < arity; ++a) {
        int32_t v = el[arity * e + a];
        unsigned long long pos = atomicAdd(&cursor[v], 1ull);
        ids[ptr[v] + (int64_t)pos] = (int32_t)e;
    }
}

__global__ void k_sort_lists(const int64_t *ptr, int32_t *ids, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t b = ptr[i], e = ptr[i + 1];
    for (int64_t k = b + 1; k < e; ++k) {
        int32_t v = ids[k];
        int64_t m = k - 1;
        while (m >= b && ids[m] > v) { ids[m + 1] = ids[m]; --m; }
        ids[m + 1] = v;
    }
}

// Build a node -> element incidence CSR with ascending element ids per node.
static int build_incidence(Ctx &c, const int32_t *d_el, int arity, int64_t nel, int64_t n,
                           int64_t **d_ptr, int32_t **d_ids) {
    cudaStream_t st = c.stream;
    int64_t *cnt = nullptr;
    unsigned long long *cursor = nullptr;
    CK(cudaMalloc(&cnt, sizeof(int64_t) * (n + 1)));
    CK(cudaMalloc(&cursor, sizeof(unsigned long long) * (n + 1)));
    CK(cudaMalloc(d_ptr, sizeof(int64_t) * (n + 1)));
    CK(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (n + 1), st));
    CK(cudaMemsetAsync(cursor, 0, sizeof(unsigned long long) * (n + 1), st));
    int64_t blocks = (nel + 255) / 256;
    if (nel > 0) k_count<<<(unsigned)blocks, 256, 0, st>>>(d_el, arity, nel, cnt);
    CK(cudaGetLastError());
    size_t tmp_bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, *d_ptr, n + 1, st));
    void *tmp = nullptr;
    CK(cudaMalloc(&tmp, tmp_bytes));
    CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, *d_ptr, n + 1, st));
    CK(cudaMalloc(d_ids, sizeof(int32_t) * (size_t)(arity * nel + 1)));
    if (nel > 0) k_fill<<<(unsigned)blocks, 256, 0, st>>>(d_el, arity, nel, *d_ptr, cursor, *d_ids);
    CK(cudaGetLastError());
    k_sort_lists<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(*d_ptr, *d_ids, n);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    cudaFree(tmp);
    cudaFree(cnt);
    cudaFree(cursor);
    return 0;
}

// ------------------------------------------------------------------------------ pattern

// Sorted unique vertices of the tets incident to node i (includes i).  Returns the count,
// or -1 if more than THERMO_MAX_ROW.
__device__ int row_neighbours(const int64_t *tptr, const int32_t *tinc, const int32_t *tets,
                              int64_t i, int32_t *nb) {
    int n = 0;
    for (int64_t k = tptr[i]; k < tptr[i + 1]; ++k) {
        const int32_t *t = tets + 4 * (int64_t)tinc[k];
        for (int a = 0; a < 4; ++a) {
            int32_t v = t[a];
            int p = n;
            while (p > 0 && nb[p - 1] > v) --p;
            if (p > 0 && nb[p - 1] == v) continue;
            if (n == THERMO_MAX_ROW) return -1;
            for (int q = n; q > p; --q) nb[q] = nb[q - 1];
            nb[p] = v;
            ++n;
        }
    }
    return n;
}

__global__ void k_row_len(const int64_t *tptr, const int32_t *tinc, const int32_t *tets, int64_t N,
                          int32_t *len, int *bad) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    int32_t nb[THERMO_MAX_ROW];
    int n = row_neighbours(tptr, tinc, tets, i, nb);
    if (n < 0) { atomicOr(bad, 4); n = 0; }
    len[i] = n;
}

__global__ void k_slice_width(const int32_t *len, int64_t N, int64_t nslices, int64_t *w32) {
    int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s > nslices) return;
    if (s == nslices) { w32[s] = 0; return; }
    int w = 0;
    for (int l = 0; l < 32; ++l) {
        int64_t i = 32 * s + l;
        if (i < N) w = max(w, len[i]);
    }
    w32[s] = 32 * (int64_t)w;
}

// Columns (padded), diagonal position, stiffness values A = -nu int grad phi . grad phi and
// lumped mass rho Cp V/4 per incident tet, row-owner, ascending tet order.
__global__ void k_row_fill(const int64_t *tptr, const int32_t *tinc, const int32_t *tets,
                           const double *xyz, int64_t N, const int64_t *slice_ptr, double nu,
                           double rho_cp, int32_t *col, double *A, double *R, int64_t *diagpos,
                           double *ML) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t nslices = (N + 31) / 32;
    if (i >= nslices * 32) return;
    int64_t s = i >> 5;
    int lane = (int)(i & 31);
    int64_t base = slice_ptr[s] + lane;
    int w = (int)((slice_ptr[s + 1] - slice_ptr[s]) >> 5);
    if (i >= N) {   // lanes past the last row: harmless padding
        for (int k = 0; k < w; ++k) { col[base + 32 * k] = 0; A[base + 32 * k] = 0.0; R[base + 32 * k] = 0.0; }
        return;
    }
    int32_t nb[THERMO_MAX_ROW];
    double acc[THERMO_MAX_ROW];
    int n = row_neighbours(tptr, tinc, tets, i, nb);
    if (n < 0) n = 0;
    for (int k = 0; k < n; ++k) acc[k] = 0.0;
    double ml = 0.0;
    for (int64_t m = tptr[i]; m < tptr[i + 1]; ++m) {
        const int32_t *t = tets + 4 * (int64_t)tinc[m];
        double g[4][3];
        double det = tet_grad(xyz, t, g);
        double V = det / 6.0;
        int a = 0;
        while (t[a] != i) ++a;
        ml += rho_cp * V * 0.25;
        for (int b = 0; b < 4; ++b) {
            double gab = g[a][0] * g[b][0] + g[a][1] * g[b][1] + g[a][2] * g[b][2];
            int lo = 0, hi = n - 1, pos = 0;
            while (lo <= hi) {   // binary search of column t[b]
                int mid = (lo + hi) >> 1;
                if (nb[mid] == t[b]) { pos = mid; break; }
                if (nb[mid] < t[b]) lo = mid + 1; else hi = mid - 1;
            }
            acc[pos] += -nu * V * gab;
        }
    }
    // entry 0 of every row is its diagonal (the solve reads D from there), then the other
    // columns ascending; short rows are padded with (i, 0)
    int d = 0;
    while (d < n && nb[d] != i) ++d;
    for (int k = 0; k < w; ++k) {
        int64_t e = base + 32 * (int64_t)k;
        const int src = k == 0 ? d : (k <= d ? k - 1 : k);   // sorted position of entry k
        if (k < n && d < n) {
            col[e] = nb[src];
            A[e] = acc[src];
        } else {
            col[e] = (int32_t)i;
            A[e] = 0.0;
        }
        R[e] = 0.0;
    }
    diagpos[i] = base;
    ML[i] = ml;
}

// ------------------------------------------------------------------------------ Robin

// Row-owner Robin assembly: for each face f at node i with Robin data (alpha,
// T_a = T_ref + g.x): R[i, f_b] -= alpha S/12 (1 + d_ab), benv[i] += alpha S/12 (1+d_ab) T_a(x_b)
// (exact: consistent P1 surface mass, T_a linear).  tab[k] = {key, alpha, T_ref, g0, g1, g2}.
__global__ void k_robin(const int64_t *fptr, const int32_t *finc, const int32_t *faces,
                        const int32_t *fkey, const double *xyz, int64_t N, const int64_t *slice_ptr,
                        const int32_t *col, const double *tab, int ntab, double *R, double *benv) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    double b = 0.0;
    int64_t s = i >> 5;
    int lane = (int)(i & 31);
    int64_t base = slice_ptr[s] + lane;
    int w = (int)((slice_ptr[s + 1] - slice_ptr[s]) >> 5);
    for (int64_t m = fptr[i]; m < fptr[i + 1]; ++m) {
        int64_t f = finc[m];
        int key = fkey[f];
        const double *r = nullptr;
        for (int k = 0; k < ntab; ++k)
            if ((int)tab[8 * k] == key) r = tab + 8 * k;
        if (!r || r[1] == 0.0) continue;
        const int32_t *v = faces + 3 * f;
        double u[3], q[3];
        for (int d = 0; d < 3; ++d) {
            u[d] = xyz[3 * v[1] + d] - xyz[3 * v[0] + d];
            q[d] = xyz[3 * v[2] + d] - xyz[3 * v[0] + d];
        }
        double cx = u[1] * q[2] - u[2] * q[1], cy = u[2] * q[0] - u[0] * q[2], cz = u[0] * q[1] - u[1] * q[0];
        double S = 0.5 * sqrt(cx * cx + cy * cy + cz * cz);
        int a = 0;
        while (v[a] != i) ++a;
        for (int bb = 0; bb < 3; ++bb) {
            double Ms = S / 12.0 * (a == bb ? 2.0 : 1.0);
            const double *x = xyz + 3 * (int64_t)v[bb];
            double Ta = r[2] + r[3] * x[0] + r[4] * x[1] + r[5] * x[2];
            b += r[1] * Ms * Ta;
            for (int k = 0; k < w; ++k) {
                int64_t e = base + 32 * (int64_t)k;
                if (col[e] == v[bb]) { R[e] -= r[1] * Ms; break; }
            }
        }
    }
    benv[i] = b;
}

__global__ void k_zero(double *p, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = 0.0;
}

// K~_vol = M_L - dt (A + R); the padding entries stay 0.
__global__ void k_build_vals(const double *A, const double *R, int64_t n, double dt, double *val) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e < n) val[e] = -dt * (A[e] + R[e]);
}

__global__ void k_build_diag(const int64_t *diagpos, const double *ML, double mu, int64_t N, double *val,
                             double *Dvol, double *Dinv, double *Dinv_vol) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    int64_t e = diagpos[i];
    double d = val[e] + mu * ML[i];
    val[e] = d;
    Dvol[i] = d;
    Dinv[i] = 1.0 / d;
    Dinv_vol[i] = 1.0 / d;
}

// f^I operator values A + B_env (MRSDC)
__global__ void k_build_kv(const double *A, const double *R, int64_t n, double *KV) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e < n) KV[e] = A[e] + R[e];
}

// ------------------------------------------------------------------------------ host side

static inline unsigned nb(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

int assemble_create(Ctx &c, const double *xyz, const int32_t *tets, const int32_t *faces,
                    const int32_t *fkey) {
    cudaStream_t st = c.stream;
    const int64_t N = c.N;
    CK(cudaMalloc(&c.d_xyz, sizeof(double) * 3 * N));
    CK(cudaMalloc(&c.d_tets, sizeof(int32_t) * 4 * (c.ntets + 1)));
    CK(cudaMalloc(&c.d_faces, sizeof(int32_t) * 3 * (c.nfaces + 1)));
    CK(cudaMalloc(&c.d_fkey, sizeof(int32_t) * (c.nfaces + 1)));
    CK(cudaMemcpyAsync(c.d_xyz, xyz, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(c.d_tets, tets, sizeof(int32_t) * 4 * c.ntets, cudaMemcpyHostToDevice, st));
    if (c.nfaces) {
        CK(cudaMemcpyAsync(c.d_faces, faces, sizeof(int32_t) * 3 * c.nfaces, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(c.d_fkey, fkey, sizeof(int32_t) * c.nfaces, cudaMemcpyHostToDevice, st));
    }
    int *d_bad = nullptr;
    CK(cudaMalloc(&d_bad, sizeof(int)));
    CK(cudaMemsetAsync(d_bad, 0, sizeof(int), st));
    if (c.ntets) k_tet_check<<<nb(c.ntets), 256, 0, st>>>(c.d_xyz, c.d_tets, c.ntets, N, d_bad);
    CK(cudaGetLastError());
    int bad = 0;
    CK(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (bad & 1) { c.err = "tetrahedron vertex index out of range"; cudaFree(d_bad); return -1; }
    if (bad & 2) { c.err = "tetrahedron with non-positive det J (inverted or degenerate)"; cudaFree(d_bad); return -1; }

    int rc = build_incidence(c, c.d_tets, 4, c.ntets, N, &c.d_tinc_ptr, &c.d_tinc);
    if (rc) return rc;
    rc = build_incidence(c, c.d_faces, 3, c.nfaces, N, &c.d_finc_ptr, &c.d_finc);
    if (rc) return rc;

    // pattern: row lengths -> slice widths -> slice pointers
    c.nslices = (N + 31) / 32;
    int32_t *d_len = nullptr;
    int64_t *d_w = nullptr;
    CK(cudaMalloc(&d_len, sizeof(int32_t) * N));
    CK(cudaMalloc(&d_w, sizeof(int64_t) * (c.nslices + 1)));
    CK(cudaMalloc(&c.d_slice_ptr, sizeof(int64_t) * (c.nslices + 1)));
    k_row_len<<<nb(N, 128), 128, 0, st>>>(c.d_tinc_ptr, c.d_tinc, c.d_tets, N, d_len, d_bad);
    CK(cudaGetLastError());
    k_slice_width<<<nb(c.nslices + 1), 256, 0, st>>>(d_len, N, c.nslices, d_w);
    CK(cudaGetLastError());
    size_t tmp_bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_w, c.d_slice_ptr, c.nslices + 1, st));
    void *tmp = nullptr;
    CK(cudaMalloc(&tmp, tmp_bytes));
    CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, d_w, c.d_slice_ptr, c.nslices + 1, st));
    int64_t nnz_pad = 0;
    CK(cudaMemcpyAsync(&nnz_pad, c.d_slice_ptr + c.nslices, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    // true nnz = sum of row lengths
    int64_t *d_nnz = nullptr;
    CK(cudaMalloc(&d_nnz, sizeof(int64_t)));
    size_t tmp2 = 0;
    CK(cub::DeviceReduce::Sum(nullptr, tmp2, d_len, d_nnz, N, st));
    void *tmpr = nullptr;
    CK(cudaMalloc(&tmpr, tmp2));
    CK(cub::DeviceReduce::Sum(tmpr, tmp2, d_len, d_nnz, N, st));
    CK(cudaMemcpyAsync(&c.nnz, d_nnz, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    cudaFree(tmp); cudaFree(tmpr); cudaFree(d_nnz); cudaFree(d_w); cudaFree(d_len);
    if (bad & 4) { c.err = "node with more than THERMO_MAX_ROW neighbours"; cudaFree(d_bad); return -1; }
    cudaFree(d_bad);
    c.nnz_pad = nnz_pad;

    CK(cudaMalloc(&c.d_col, sizeof(int32_t) * (nnz_pad + 1)));
    CK(cudaMalloc(&c.d_A, sizeof(double) * (nnz_pad + 1)));
    CK(cudaMalloc(&c.d_R, sizeof(double) * (nnz_pad + 1)));
    CK(cudaMalloc(&c.d_val, sizeof(double) * (nnz_pad + 1)));
    CK(cudaMalloc(&c.d_diagpos, sizeof(int64_t) * N));
    CK(cudaMalloc(&c.d_ML, sizeof(double) * (N + 16)));   // +16: 16-byte bulk copies of row ranges
    CK(cudaMalloc(&c.d_benv, sizeof(double) * (N + 16)));
    CK(cudaMalloc(&c.d_Dvol, sizeof(double) * (N + 16)));
    CK(cudaMalloc(&c.d_Dinv, sizeof(double) * (N + 16)));
    CK(cudaMemsetAsync(c.d_benv, 0, sizeof(double) * N, st));
    k_row_fill<<<nb(c.nslices * 32, 128), 128, 0, st>>>(c.d_tinc_ptr, c.d_tinc, c.d_tets, c.d_xyz, N,
                                                        c.d_slice_ptr, c.nu, c.rho_cp, c.d_col, c.d_A,
                                                        c.d_R, c.d_diagpos, c.d_ML);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return 0;
}

int assemble_robin(Ctx &c) {
    cudaStream_t st = c.stream;
    std::vector<double> tab;
    for (auto &r : c.robin) {
        double row[8] = {(double)(r.part * 65536 + r.tag), r.alpha, r.T_ref, r.g[0], r.g[1], r.g[2], 0, 0};
        tab.insert(tab.end(), row, row + 8);
    }
    if (c.d_robin_tab) { cudaFree(c.d_robin_tab); c.d_robin_tab = nullptr; }
    CK(cudaMalloc(&c.d_robin_tab, sizeof(double) * (tab.size() + 8)));
    if (!tab.empty())
        CK(cudaMemcpyAsync(c.d_robin_tab, tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice, st));
    k_zero<<<nb(c.nnz_pad), 256, 0, st>>>(c.d_R, c.nnz_pad);
    CK(cudaGetLastError());
    k_robin<<<nb(c.N, 128), 128, 0, st>>>(c.d_finc_ptr, c.d_finc, c.d_faces, c.d_fkey, c.d_xyz, c.N,
                                          c.d_slice_ptr, c.d_col, c.d_robin_tab, (int)c.robin.size(),
                                          c.d_R, c.d_benv);
    CK(cudaGetLastError());
    c.robin_dirty = false;
    c.built_dt = -1.0;
    return 0;
}

int build_operator(Ctx &c, double dt, double mu) {
    cudaStream_t st = c.stream;
    c.spec_valid = false;   // the Jacobi vectors are rewritten below
    k_build_vals<<<nb(c.nnz_pad), 256, 0, st>>>(c.d_A, c.d_R, c.nnz_pad, dt, c.d_val);
    CK(cudaGetLastError());
    if (!c.d_Dinv_vol) CK(cudaMalloc(&c.d_Dinv_vol, sizeof(double) * c.N));
    k_build_diag<<<nb(c.N), 256, 0, st>>>(c.d_diagpos, c.d_ML, mu, c.N, c.d_val, c.d_Dvol, c.d_Dinv, c.d_Dinv_vol);
    CK(cudaGetLastError());
    // overlap mode: the second interface buffer set carries its own Jacobi vector (the interface
    // kernels rewrite its interface rows every other step; all other rows are the volume ones)
    if (c.d_Dinv_b) CK(cudaMemcpyAsync(c.d_Dinv_b, c.d_Dinv, sizeof(double) * c.N, cudaMemcpyDeviceToDevice, st));
    if (!c.d_KV) CK(cudaMalloc(&c.d_KV, sizeof(double) * (c.nnz_pad + 1)));
    k_build_kv<<<nb(c.nnz_pad), 256, 0, st>>>(c.d_A, c.d_R, c.nnz_pad, c.d_KV);
    CK(cudaGetLastError());
    ++c.op_ver;   // the interface rows' Jacobi diagonals assembled ahead (ahead mode) are stale
    c.built_dt = mu == 1.0 ? dt : -1.0;   // anything but the implicit-Euler operator: rebuild next step
    return 0;
}

}  // namespace thermo
