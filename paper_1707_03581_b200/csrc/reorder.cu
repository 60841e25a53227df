// reorder.cu -- internal node numbering and the state transfers that hide it.
//
// The paper's meshes are CAD-derived and meshed independently, so the caller's
// node numbering is arbitrary.  The bandwidth-bound solve (cg.cu, KIND 2) streams each chunk
// of 256 rows together with a "column window" of the gathered vector: at most CG_MAXR
// contiguous runs totalling <= 65,535 entries.  A banded numbering (lattice order, or the
// level structure of a breadth-first order) meets that; a scattered one does not.  At create
// the library therefore probes the caller's numbering with the same window test and, when it
// fails, renumbers each part by reverse Cuthill-McKee on the volume pattern (breadth-first
// level sets from a pseudo-peripheral node, neighbours by increasing degree; a variant rooted
// at the interface nodes is selectable).  Fixed nodes stay in [0, nf) and moving ones in [nf, N).
//
// The ABI keeps the caller's numbering: thermo_set_T / thermo_get_T / thermo_get_T_async
// scatter and gather through the permutation (and, for S > 1 scenarios, between the state block
// [SP / CW][N][CW] and one contiguous field per scenario), and thermo_get_interface maps
// its row and column indices back.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
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

// Window test of the current volume pattern with the default solve's chunking (W = 8 slices,
// run gap 32): *good = every chunk fits the windowed kernel.
int order_probe(Ctx &c, bool *good, int *max_runs, int *max_window) {
    const int W = 8;
    const int64_t nchunks = (c.nslices + W - 1) / W;
    int2 *runs = nullptr;
    int32_t *nruns = nullptr, *lown = nullptr;
    uint16_t *lcol = nullptr;
    int *d_stats = nullptr;
    cudaError_t e = cudaMalloc(&runs, sizeof(int2) * nchunks * 32);
    if (e == cudaSuccess) e = cudaMalloc(&nruns, sizeof(int32_t) * nchunks);
    if (e == cudaSuccess) e = cudaMalloc(&lown, sizeof(int32_t) * nchunks);
    if (e == cudaSuccess) e = cudaMalloc(&lcol, sizeof(uint16_t) * c.nnz_pad);
    if (e == cudaSuccess) e = cudaMalloc(&d_stats, sizeof(int) * 4);
    int stats[4] = {0, 0, 0, 0};
    if (e == cudaSuccess) e = cudaMemsetAsync(d_stats, 0, sizeof(int) * 4, c.stream);
    if (e == cudaSuccess) {
        chunk_windows_launch(c, W, 32, runs, nruns, lown, lcol, d_stats);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(stats, d_stats, sizeof stats, cudaMemcpyDeviceToHost, c.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
    for (void *p : {(void *)runs, (void *)nruns, (void *)lown, (void *)lcol, (void *)d_stats})
        if (p) cudaFree(p);
    CK(e);
    *max_window = stats[0];
    *max_runs = stats[1];
    *good = !stats[2] && stats[1] <= 32;
    return 0;
}

// Cuthill-McKee numbering of each part from the device volume pattern (breadth-first level
// sets, neighbours by increasing degree).
//   rooted = false (default): reverse Cuthill-McKee from a pseudo-peripheral node (George-Liu).
//     Narrow levels: every 256-row chunk's column window fits the windowed kernel (KIND 2).
//   rooted = true: level 0 = the part's interface nodes (ordered by a Cuthill-McKee sweep of the
//     surface graph), then the levels away from the interface; the interface rows form one
//     contiguous block as in lattice order, but the levels are wider (shells around the rail
//     top) and the windows of cfg 2/3 exceed the KIND 2 stage budget (KIND 1 is chosen).
//     Measured (random numbering, B200, per CG iteration vs lattice order): default cfg 2
//     1.17x / cfg 3 1.09x (KIND 2); rooted 1.10x / 1.09x (KIND 1).  DESIGN.md §6.
// new_to_old[i] = the caller's (coupled) index of internal node i.
int rcm_order(Ctx &c, const std::vector<char> &is_iface, bool rooted, std::vector<int32_t> &new_to_old) {
    const int64_t N = c.N;
    std::vector<int64_t> sp(c.nslices + 1);
    std::vector<int32_t> col(c.nnz_pad);
    CK(cudaMemcpyAsync(sp.data(), c.d_slice_ptr, sizeof(int64_t) * sp.size(), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaMemcpyAsync(col.data(), c.d_col, sizeof(int32_t) * col.size(), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    // neighbours of row i: entries k < width of its slice, padding (col == i) skipped
    auto width = [&](int64_t i) { return (int)((sp[i / 32 + 1] - sp[i / 32]) / 32); };
    auto nb = [&](int64_t i, int k) { return col[sp[i / 32] + 32 * (int64_t)k + i % 32]; };
    std::vector<int32_t> deg(N, 0);
    for (int64_t i = 0; i < N; ++i) {
        const int w = width(i);
        int d = 0;
        for (int k = 0; k < w; ++k) d += nb(i, k) != (int32_t)i;
        deg[i] = d;
    }
    auto by_degree = [&](int32_t a, int32_t b) { return deg[a] != deg[b] ? deg[a] < deg[b] : a < b; };
    std::vector<int32_t> level(N, -1), order;
    order.reserve(N);
    // breadth-first levels from r over the nodes with allowed(v) (marks `level`; the visited
    // nodes go to `seen` so the marks can be reset); returns the eccentricity, `last` = last level
    auto bfs_levels = [&](int32_t r, auto allowed, std::vector<int32_t> &seen, std::vector<int32_t> &last) {
        seen.clear();
        seen.push_back(r);
        level[r] = 0;
        int L = 0;
        for (size_t head = 0; head < seen.size(); ++head) {
            const int32_t u = seen[head];
            L = level[u];
            const int w = width(u);
            for (int k = 0; k < w; ++k) {
                const int32_t v = nb(u, k);
                if (v != u && level[v] < 0 && allowed(v)) {
                    level[v] = level[u] + 1;
                    seen.push_back(v);
                }
            }
        }
        last.clear();
        for (int32_t v : seen)
            if (level[v] == L) last.push_back(v);
        return L;
    };
    // pseudo-peripheral node of r's component (restricted to allowed)
    auto peripheral = [&](int32_t r, auto allowed) {
        std::vector<int32_t> seen, last;
        int ecc = bfs_levels(r, allowed, seen, last);
        for (int rep = 0; rep < 8; ++rep) {
            int32_t x = last[0];
            for (int32_t v : last)
                if (by_degree(v, x)) x = v;
            for (int32_t v : seen) level[v] = -1;
            const int e2 = bfs_levels(x, allowed, seen, last);
            if (e2 <= ecc) break;
            r = x;
            ecc = e2;
        }
        for (int32_t v : seen) level[v] = -1;
        return r;
    };
    std::vector<char> done(N, 0);
    std::vector<int32_t> nbuf;
    // Cuthill-McKee sweep: order[head..] grows by the unvisited allowed neighbours of each node
    auto sweep = [&](size_t head, auto allowed) {
        for (; head < order.size(); ++head) {
            const int32_t u = order[head];
            nbuf.clear();
            const int w = width(u);
            for (int k = 0; k < w; ++k) {
                const int32_t v = nb(u, k);
                if (v != u && !done[v] && allowed(v)) {
                    done[v] = 1;
                    nbuf.push_back(v);
                }
            }
            std::sort(nbuf.begin(), nbuf.end(), by_degree);
            order.insert(order.end(), nbuf.begin(), nbuf.end());
        }
    };
    auto any = [](int32_t) { return true; };
    auto on_iface = [&](int32_t v) { return is_iface[v] != 0; };
    for (int part = 0; part < 2; ++part) {
        const int64_t lo = part ? c.nf : 0, hi = part ? N : c.nf;
        const size_t part_begin = order.size();
        if (rooted) {   // level 0: the interface nodes, surface component by surface component
            for (int64_t s = lo; s < hi; ++s) {
                if (done[s] || !is_iface[s]) continue;
                const int32_t r = peripheral((int32_t)s, on_iface);
                const size_t b = order.size();
                order.push_back(r);
                done[r] = 1;
                sweep(b, on_iface);
            }
            sweep(part_begin, any);   // levels away from the interface
        }
        for (int64_t s = lo; s < hi; ++s) {   // (remaining) components from a pseudo-peripheral node
            if (done[s]) continue;
            const int32_t r = peripheral((int32_t)s, any);
            const size_t b = order.size();
            order.push_back(r);
            done[r] = 1;
            sweep(b, any);
        }
        if ((int64_t)(order.size() - part_begin) != hi - lo) {
            c.err = "reordering: volume pattern couples the two parts";
            return -1;
        }
        if (!rooted) std::reverse(order.begin() + part_begin, order.end());   // reverse Cuthill-McKee
    }
    new_to_old.swap(order);
    return 0;
}

// Element (row i, scenario s) of a block vector with the layout [SP / CW][N][CW].
__device__ __forceinline__ int64_t blk(int64_t N, int CW, int64_t i, int s) {
    return ((int64_t)(s / CW) * N + i) * CW + s % CW;
}

// out[k] = T[map(off + k), scen], map = int_of_ext (nullptr: identity)
__global__ void k_gather_T(const double *__restrict__ T, int64_t N, int CW, int scen, const int32_t *__restrict__ map,
                           int64_t off, int64_t cnt, double *__restrict__ out) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= cnt) return;
    const int64_t e = off + k;
    out[k] = T[blk(N, CW, map ? map[e] : e, scen)];
}

// T[map(off + k), scen] = in[k]
__global__ void k_scatter_T(double *__restrict__ T, int64_t N, int CW, int scen, const int32_t *__restrict__ map,
                            int64_t off, int64_t cnt, const double *__restrict__ in) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= cnt) return;
    const int64_t e = off + k;
    T[blk(N, CW, map ? map[e] : e, scen)] = in[k];
}

// All scenarios at once: out[s][e] = T[map(e), s] for e < N, s < S (a transpose of the block
// through 32 x 32 shared-memory tiles; identity map: both sides coalesced)
__global__ void k_gather_all(const double *__restrict__ T, int S, int CW, const int32_t *__restrict__ map, int64_t N,
                             double *__restrict__ out) {
    __shared__ double tile[32][33];
    const int64_t e0 = blockIdx.x * 32ll;
    const int s0 = blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        const int64_t e = e0 + r;
        const int s = s0 + tx;
        if (e < N && s < S) tile[r][tx] = T[blk(N, CW, map ? (int64_t)map[e] : e, s)];
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int s = s0 + r;
        const int64_t e = e0 + tx;
        if (e < N && s < S) out[(int64_t)s * N + e] = tile[tx][r];
    }
}

int gather_T(Ctx &c, int scen, int64_t off, int64_t cnt, const double *T, double *out, cudaStream_t st) {
    if (cnt <= 0) return 0;
    k_gather_T<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(T, c.N, c.CW, scen, c.d_int_of_ext, off, cnt, out);
    CK(cudaGetLastError());
    return 0;
}

int scatter_T(Ctx &c, int scen, int64_t off, int64_t cnt, double *T, const double *in, cudaStream_t st) {
    if (cnt <= 0) return 0;
    k_scatter_T<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(T, c.N, c.CW, scen, c.d_int_of_ext, off, cnt, in);
    CK(cudaGetLastError());
    return 0;
}

int gather_all(Ctx &c, const double *T, double *out, cudaStream_t st) {
    dim3 grid((unsigned)((c.N + 31) / 32), (unsigned)((c.S + 31) / 32)), block(32, 8);
    k_gather_all<<<grid, block, 0, st>>>(T, c.S, c.CW, c.d_int_of_ext, c.N, out);
    CK(cudaGetLastError());
    return 0;
}

}  // namespace thermo
