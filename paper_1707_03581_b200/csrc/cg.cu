// cg.cu -- the implicit-Euler solve (M_L - dt K(t')) T^{n+1} = M_L T^n + dt (b_env + b_G)
// by Jacobi-preconditioned CG, one persistent cooperative kernel per
// time step.
//
// Schedule per CG iteration, z-primary Jacobi-PCG:
//   S: q = K~ p (sliced-ELL volume part + per-step interface rows, p the only gathered
//      vector), q' = D^{-1} q; partials of p.q and of the expansions of the next r.z, r.r
//   -- grid barrier; alpha = rho / p.q, beta = r.z_new / rho, convergence test on r.r
//   U: x += alpha p ; z -= alpha q' ; p = z + beta p   (streams, no reduction)
//   -- grid barrier
// Every value of every reduction is combined in a fixed order (deterministic, identical in
// all CTAs), so all CTAs take the same control-flow decisions.
//
// Sliced-ELL sweeps (phase 0 and S) come in three kinds:
//  KIND 0  register streaming: every warp streams its slices with L1-bypassing,
//          L2-evict-first loads and gathers the vector entries from L1/L2 (fallback).
//  KIND 1  TMA matrix ring: a producer warp streams chunks of W consecutive slices (values +
//          int32 columns, contiguous in HBM) into an NS-stage shared-memory ring with
//          cp.async.bulk (mbarrier complete_tx); NG groups of W consumer warps take every
//          NG-th chunk and gather the vector entries from L1/L2.
//  KIND 2  TMA matrix + vector windows: as KIND 1, but the columns are stored as 16-bit
//          indices local to the chunk, and the producer also bulk-copies the chunk's column
//          window (<= 32 contiguous runs of the gathered vectors, precomputed at setup) into
//          shared memory, so every gather is a shared-memory load.  10 instead of 12 bytes
//          per stored entry, and no gather latency on the critical path.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <vector>

#include "ctx.h"
#include "cg_params.h"

namespace cg = cooperative_groups;

namespace thermo {

#define CK(x)                                                                    \
    do {                                                                         \
        cudaError_t e_ = (x);                                                    \
        if (e_ != cudaSuccess) {                                                 \
            c.err = std::string("CUDA: ") + cudaGetErrorString(e_) + " at " #x; \
            return -3;                                                           \
        }                                                                        \
    } while (0)

#define CG_HDR 128      // stage header bytes (int32): [0..W] slice offsets, [16..16+W] interface
                        // ranges, [30] end-marker position, [31] chunk id (< 0: end marker)
#define CG_MAXR 32      // max window runs per chunk (one per producer lane)
#define CG_GAP 32       // column gaps up to this size are bridged inside one run; N > 2^22: CG_GAP_LARGE
#define CG_GAP_LARGE 512  // fewer, longer window copies: cfg 3 403 -> 399 us per iteration, while
                          // cfg 2 is 1 % slower with them (55.3 -> 56.0 us)

// CGParams: cg_params.h


// Prefetch into L2 the leading edge of the column window of a chunk whose largest column
// index is hi_col: rows [hi_col - len + 1, hi_col] of each vector in pf (len = rows of the
// chunk, 16-B aligned).  hi_col < 0: nothing.
template <int W>
__device__ __forceinline__ void prefetch_edge(const CGParams &P, int hi_col) {
    if (hi_col < 0) return;
    const int64_t rows = (int64_t)W * 32;
    int64_t hi = (int64_t)hi_col + 1;
    int64_t lo = hi - rows;
    if (lo < 0) lo = 0;
    lo &= ~(int64_t)1;
    hi = (hi + 1) & ~(int64_t)1;
    if (hi > P.N) hi = P.N & ~(int64_t)1;
    if (hi <= lo) return;
#pragma unroll
    for (int v = 0; v < 4; ++v)
        if (v < P.npf) bulk_prefetch_l2(P.pf[v] + lo, (uint32_t)((hi - lo) * 8));
}

// Producer-side metadata of one chunk, loaded one chunk ahead of its use so that the
// producer never waits on global-memory latency (lane l holds slice offset l, interface
// range l and window run l).
struct ChunkMeta {
    int64_t ptr;
    int sif, nruns, hi_own, hi_pf, lown;
    int2 run;
};

template <int KIND, int W>
__device__ __forceinline__ ChunkMeta load_meta(const CGParams &P, int64_t ch, int lane, int G) {
    ChunkMeta m;
    m.ptr = 0; m.sif = 0; m.nruns = 0; m.hi_own = -1; m.hi_pf = -1; m.lown = 0;
    m.run = make_int2(0, 0);
    if (ch >= P.nchunks) return m;
    const int64_t s0 = ch * W, s1 = min(s0 + (int64_t)W, P.nslices);
    const int64_t sl = min(s0 + lane, s1);
    if (lane <= W) {
        m.ptr = P.slice_ptr[sl];
        m.sif = P.slice_if[sl];
    }
    if (KIND == 2) {
        m.nruns = P.chunk_nruns[ch];
        m.lown = P.chunk_lown[ch];
        m.run = P.chunk_runs[ch * CG_MAXR + lane];   // lanes >= nruns ignore theirs
    }
    if (lane == 0) {
        // leading edge of the column window two chunk waves ahead (and the chunk itself
        // during the first waves)
        if (ch < 2 * G) m.hi_own = P.chunk_hi[ch];
        if (ch + 2 * G < P.nchunks) m.hi_pf = P.chunk_hi[ch + 2 * G];
    }
    return m;
}

// Interface index of the row owned by this lane (-1 if none), given the slice's range
// [b, e) in if_rows.  Warp-uniform call.
__device__ __forceinline__ int iface_index_r(const CGParams &P, int b, int e, int64_t i, int lane) {
    if (b == e) return -1;
    const int m = e - b;
    const int mine = lane < m ? P.if_rows[b + lane] : -1;
    int ik = -1;
    for (int j = 0; j < m; ++j) {
        int rj = __shfl_sync(0xffffffffu, mine, j);
        if (rj == (int)i) ik = b + j;
    }
    return ik;
}

// Interface rows: entries in rounds of IB -- every column / value load of a round issued, then
// every gather, then the sums in ascending entry order (the same order as one at a time), so a
// row costs two dependent round trips per round instead of two per entry.
#define IB 8
template <bool kTwo>
__device__ __forceinline__ double ell_row(const CGParams &P, int ik, const double *x1, const double *x2,
                                          double beta, int64_t row = -1, double *self = nullptr) {
    const int cnt = P.ell_cnt[ik];
    double acc = 0.0;
    for (int c0 = 0; c0 < cnt; c0 += IB) {
        int j[IB];
        double v[IB], y[IB];
#pragma unroll
        for (int u = 0; u < IB; ++u) {
            const int64_t e = (int64_t)min(c0 + u, cnt - 1) * P.n_if + ik;
            j[u] = P.ell_col[e];
            v[u] = P.ell_val[e];
        }
#pragma unroll
        for (int u = 0; u < IB; ++u) {
            y[u] = x1[j[u]];
            if (kTwo) y[u] = fma(beta, x2[j[u]], y[u]);
        }
#pragma unroll
        for (int u = 0; u < IB; ++u)
            if (c0 + u < cnt) {
                acc = fma(v[u], y[u], acc);
                if (self && j[u] == row) *self += v[u];   // the interface part of the diagonal
            }
    }
    return acc;
}

// FUSED: interface row applied to p_new = beta p + (z - alpha q') (the owner's formula)
__device__ __forceinline__ double ell_row3(const CGParams &P, int ik, const double *z, const double *q,
                                           const double *p, double alpha, double beta, int64_t row, double *self) {
    const int cnt = P.ell_cnt[ik];
    double acc = 0.0;
    for (int c0 = 0; c0 < cnt; c0 += IB) {
        int j[IB];
        double v[IB], y[IB];
#pragma unroll
        for (int u = 0; u < IB; ++u) {
            const int64_t e = (int64_t)min(c0 + u, cnt - 1) * P.n_if + ik;
            j[u] = P.ell_col[e];
            v[u] = P.ell_val[e];
        }
#pragma unroll
        for (int u = 0; u < IB; ++u) y[u] = fma(beta, p[j[u]], fma(-alpha, q[j[u]], z[j[u]]));
#pragma unroll
        for (int u = 0; u < IB; ++u)
            if (c0 + u < cnt) {
                acc = fma(v[u], y[u], acc);
                if (j[u] == row) *self += v[u];
            }
    }
    return acc;
}
#undef IB

// ---------------------------------------------------------------------------------
// row sources: sum_k val_k * (x1[col_k] + beta * x2[col_k]) over one sliced-ELL row whose
// entries sit at stride 32.  All sources add in the same order (k ascending, fused
// multiply-add), so the three kinds produce bitwise-identical row sums.
// ---------------------------------------------------------------------------------
struct SrcGlobal {   // KIND 0: matrix streamed from HBM, gathers from L1/L2
    const int32_t *cp;
    const double *vp;
    uint64_t pol;
    // FUSED kernels are KIND 2 only; these keep the generic sweep body compilable
    __device__ __forceinline__ double ownw(int) const { return 0.0; }
    __device__ __forceinline__ double dot3(int, double, double) const { return 0.0; }
    // own-row value of the first / second gathered vector
    __device__ __forceinline__ double own1(const double *g, int64_t i) const { return g[i]; }
    __device__ __forceinline__ double own2(const double *g, int64_t i) const { return g[i]; }
    // value of the row's entry 0 = its diagonal (assembly order)
    __device__ __forceinline__ double first() const { return ld_stream(vp, pol); }
    template <bool kTwo>
    __device__ __forceinline__ double dot(int w, const double *x1, const double *x2, double beta) const {
        double acc = 0.0;
        int k = 0;
        for (; k + 8 <= w; k += 8) {
            int c[8];
            double v[8], y[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) c[u] = ld_stream(cp + 32 * (k + u), pol);
#pragma unroll
            for (int u = 0; u < 8; ++u) y[u] = kTwo ? fma(beta, x2[c[u]], x1[c[u]]) : x1[c[u]];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = ld_stream(vp + 32 * (k + u), pol);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = fma(v[u], y[u], acc);
        }
        for (; k < w; ++k) {
            const int c0 = ld_stream(cp + 32 * k, pol);
            const double y0 = kTwo ? fma(beta, x2[c0], x1[c0]) : x1[c0];
            acc = fma(ld_stream(vp + 32 * k, pol), y0, acc);
        }
        return acc;
    }
};

struct SrcRing {     // KIND 1: matrix in the shared-memory ring, gathers from L1/L2
    const int32_t *cp;
    const double *vp;
    // FUSED kernels are KIND 2 only; these keep the generic sweep body compilable
    __device__ __forceinline__ double ownw(int) const { return 0.0; }
    __device__ __forceinline__ double dot3(int, double, double) const { return 0.0; }
    __device__ __forceinline__ double own1(const double *g, int64_t i) const { return g[i]; }
    __device__ __forceinline__ double own2(const double *g, int64_t i) const { return g[i]; }
    __device__ __forceinline__ double first() const { return vp[0]; }
    template <bool kTwo>
    __device__ __forceinline__ double dot(int w, const double *x1, const double *x2, double beta) const {
        constexpr int B = 16;
        double acc = 0.0;
        for (int k = 0; k < w; k += B) {
            int c[B];
            double y[B];
#pragma unroll
            for (int u = 0; u < B; ++u) c[u] = (k + u < w) ? cp[32 * (k + u)] : -1;
#pragma unroll
            for (int u = 0; u < B; ++u) y[u] = c[u] >= 0 ? (kTwo ? fma(beta, x2[c[u]], x1[c[u]]) : x1[c[u]]) : 0.0;
#pragma unroll
            for (int u = 0; u < B; ++u)
                if (k + u < w) acc = fma(vp[32 * (k + u)], y[u], acc);
        }
        return acc;
    }
};

struct SrcWin {      // KIND 2: matrix and gathered vectors in shared memory
    const uint16_t *lp;
    const double *vp;
    const double *w1;    // window slot 0 (slots 1, 2 at +wstride, +2 wstride: FUSED)
    const double *wo;    // own-row block (ownv)
    int lown;            // window-local index of this lane's own row (the chunk's rows form
                         // one contiguous block of its column set)
    int lown2;           // index of this lane's own row in the own-row block (ownv)
    int wstride;         // window slot stride (entries)
    __device__ __forceinline__ double own1(const double *, int64_t) const { return w1[lown]; }
    __device__ __forceinline__ double own2(const double *, int64_t) const { return wo[lown2]; }
    __device__ __forceinline__ double ownw(int slot) const { return w1[slot * wstride + lown]; }
    __device__ __forceinline__ double first() const { return vp[0]; }
    template <bool kTwo>
    __device__ __forceinline__ double dot(int w, const double *, const double *, double beta) const {
        const double *w2 = w1 + wstride;
        double acc = 0.0;
        int k = 0;
        for (; k + 8 <= w; k += 8) {
            int c[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) c[u] = lp[32 * (k + u)];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const double y = kTwo ? fma(beta, w2[c[u]], w1[c[u]]) : w1[c[u]];
                acc = fma(vp[32 * (k + u)], y, acc);
            }
        }
        for (; k < w; ++k) {
            const int c0 = lp[32 * k];
            const double y = kTwo ? fma(beta, w2[c0], w1[c0]) : w1[c0];
            acc = fma(vp[32 * k], y, acc);
        }
        return acc;
    }
    // FUSED: sum_k val_k * p_new[col_k] with p_new = beta p + (z - alpha q') formed from the
    // windows of z (slot 0), q' (slot 1), p (slot 2) -- the owner's formula, bit for bit
    __device__ __forceinline__ double dot3(int w, double alpha, double beta) const {
        const double *w2 = w1 + wstride, *w3 = w1 + 2 * wstride;
        double acc = 0.0;
        int k = 0;
        for (; k + 8 <= w; k += 8) {
            int c[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) c[u] = lp[32 * (k + u)];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const double y = fma(beta, w3[c[u]], fma(-alpha, w2[c[u]], w1[c[u]]));
                acc = fma(vp[32 * (k + u)], y, acc);
            }
        }
        for (; k < w; ++k) {
            const int c0 = lp[32 * k];
            const double y = fma(beta, w3[c0], fma(-alpha, w2[c0], w1[c0]));
            acc = fma(vp[32 * k], y, acc);
        }
        return acc;
    }
};

// ---------------------------------------------------------------------------------
// TMA ring
// ---------------------------------------------------------------------------------
struct Ring {
    uint64_t *full, *empty;
    unsigned char *stage;   // NS stages of [header | values | columns | windows]
    size_t stage_bytes, col_off, win_off;
    uint32_t n;             // stages passed through the ring so far (same count in every warp)
    // producer: metadata of the CTA's first three chunks, loaded by the first sweep and reused by
    // every later one (the chunk set of a CTA never changes), so a sweep starts without a
    // global-memory round trip
    bool meta_ok;
    ChunkMeta m0, m1, m2;
};

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

// Bytes of the own-row copy of chunk ch (rows rounded up to even: 16-byte bulk copies; the
// vectors carry padding past N).
__device__ __forceinline__ uint32_t own_bytes(const CGParams &P, int64_t ch, int W) {
    const int64_t r0 = ch * W * 32;
    const int64_t rows = min((int64_t)W * 32, P.N - r0);
    return (uint32_t)(((rows + 1) & ~(int64_t)1) * 8);
}

// Sweep over all slices: calls body(s, src, w, ib, ie) for every slice owned by this warp.
// TMA kinds: CTA b takes chunks b, b + G, b + 2G, ... (static order: every CTA's dot-product
// partial -- and so every result bit -- is reproducible); the chunk id travels in the stage
// header; an id < 0 is the end marker (one per consumer group).
template <int KIND, int W, int NG, class Body>
__device__ __forceinline__ void sweep(const CGParams &P, Ring &R, Body &&body) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t NS = (uint32_t)P.nstages;
    if (KIND == 0) {
        const int nw = blockDim.x >> 5;
        const int gw = blockIdx.x * nw + warp;
        const int TW = gridDim.x * nw;
        const uint64_t pol = policy_evict_first();
        for (int64_t s = gw; s < P.nslices; s += TW) {
            const int64_t b0 = P.slice_ptr[s], b1 = P.slice_ptr[s + 1];
            SrcGlobal src{P.col + b0 + lane, P.val + b0 + lane, pol};
            body(s, src, (int)((b1 - b0) >> 5), P.slice_if[s], P.slice_if[s + 1]);
        }
        return;
    }
    const int G = gridDim.x;
    if (warp == W * NG) {   // ---------------- producer warp
        const uint64_t pol = policy_evict_first();
        int64_t ch = blockIdx.x;
        // metadata pipeline: chunk ch + d*G was requested d iterations ago (d = 1, 2)
        if (!R.meta_ok) {
            R.m0 = load_meta<KIND, W>(P, ch, lane, G);
            R.m1 = load_meta<KIND, W>(P, ch + G, lane, G);
            R.m2 = load_meta<KIND, W>(P, ch + 2 * G, lane, G);
            R.meta_ok = true;
        }
        ChunkMeta cur = R.m0;
        ChunkMeta m1 = R.m1;
        ChunkMeta m2 = R.m2;
        while (true) {
            const uint32_t st = R.n % NS, ph = (R.n / NS) & 1u;
            if (ch >= P.nchunks) {   // end markers for every consumer group
                const uint32_t m0 = R.n;
                for (int q = 0; q < NG; ++q) {
                    const uint32_t sq = R.n % NS, pq = (R.n / NS) & 1u;
                    if (lane == 0) {
                        mbar_wait(&R.empty[sq], pq ^ 1u);
                        int *hdr = reinterpret_cast<int *>(R.stage + (size_t)sq * R.stage_bytes);
                        hdr[31] = -1;
                        hdr[30] = (int)m0;
                        mbar_arrive(&R.full[sq]);
                    }
                    __syncwarp();
                    ++R.n;
                }
                break;
            }
            const ChunkMeta m3 = load_meta<KIND, W>(P, ch + 3 * G, lane, G);   // in flight meanwhile
            const int nruns = KIND == 2 ? (lane < cur.nruns ? 1 : 0) : 0;
            int woff = 0, wtot = 0;
            if (KIND == 2) {   // exclusive scan of the run lengths -> window offsets
                const int len = nruns ? cur.run.y : 0;
                int x = len;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                woff = x - len;
                wtot = __shfl_sync(0xffffffffu, x, 31);
            }
            const int64_t e0 = __shfl_sync(0xffffffffu, cur.ptr, 0);
            const int64_t e1 = __shfl_sync(0xffffffffu, cur.ptr, W);
            if (lane == 0) mbar_wait(&R.empty[st], ph ^ 1u);
            __syncwarp();
            // the consumers' generic-proxy reads of this stage (released through the empty
            // barrier) before this warp's async-proxy bulk writes into it: without the fence a
            // copy can land while a consumer's shared-memory load of the previous chunk is still
            // outstanding (seen as rare stale values in the batched kernel, cg_spmm.cu)
            fence_proxy_async_smem();
            unsigned char *sb = R.stage + (size_t)st * R.stage_bytes;
            int *hdr = reinterpret_cast<int *>(sb);
            if (lane <= W) {
                hdr[lane] = (int)(cur.ptr - e0);
                hdr[16 + lane] = cur.sif;
            }
            if (lane == 0) {
                hdr[31] = (int)ch;
                hdr[29] = cur.lown;
            }
            const uint32_t cnt = (uint32_t)(e1 - e0);
            __syncwarp();
            if (lane == 0) {
                const uint32_t cbytes = KIND == 2 ? cnt * 2u : cnt * 4u;
                uint32_t wbytes = KIND == 2 && !(P.debug & 2) ? (uint32_t)P.nwv * (uint32_t)wtot * 8u : 0u;
                if (KIND == 2 && P.ownv && !(P.debug & 2)) wbytes += own_bytes(P, ch, W);
                mbar_arrive_expect_tx(&R.full[st], cnt * 8u + cbytes + wbytes);
                bulk_g2s(sb + CG_HDR, P.val + e0, cnt * 8u, &R.full[st], pol);
                if (KIND == 2) bulk_g2s(sb + R.col_off, P.lcol + e0, cbytes, &R.full[st], pol);
                else bulk_g2s(sb + R.col_off, P.col + e0, cbytes, &R.full[st], pol);
            }
            __syncwarp();
            if (KIND == 2 && nruns && !(P.debug & 2)) {
#pragma unroll
                for (int v = 0; v < 3; ++v)
                    if (v < P.nwv)
                        bulk_g2s_nohint(sb + R.win_off + ((size_t)v * P.win_cap + woff) * 8, P.wv[v] + cur.run.x,
                                        (uint32_t)cur.run.y * 8u, &R.full[st]);
            }
            if (KIND == 2 && P.ownv && lane == 1 && !(P.debug & 2))   // own rows only, second slot
                bulk_g2s_nohint(sb + R.win_off + (size_t)P.nwin * P.win_cap * 8, P.ownv + ch * W * 32,
                                own_bytes(P, ch, W), &R.full[st]);
            if (lane == 0 && !(P.debug & 4)) {
                prefetch_edge<W>(P, cur.hi_own);
                prefetch_edge<W>(P, cur.hi_pf);
            }
            __syncwarp();
            ++R.n;
            ch += G;
            cur = m1;
            m1 = m2;
            m2 = m3;
        }
        return;
    }
    // ---------------- consumer warps: group g takes every NG-th stage
    const int g = warp / W, wg = warp % W;
    while (true) {
        const uint32_t st = R.n % NS, ph = (R.n / NS) & 1u;
        if ((int)(R.n % NG) == g) {
            mbar_wait(&R.full[st], ph);
            const unsigned char *sb = R.stage + (size_t)st * R.stage_bytes;
            const int *hdr = reinterpret_cast<const int *>(sb);
            const int ch = hdr[31];
            if (ch < 0) {
                const uint32_t m0 = (uint32_t)hdr[30];
                __syncwarp();
                if (lane == 0) mbar_arrive(&R.empty[st]);
                R.n = m0 + NG;
                break;
            }
            const int64_t s = (int64_t)ch * W + wg;
            if (s < P.nslices && !(P.debug & 1)) {
                const double *vals = reinterpret_cast<const double *>(sb + CG_HDR);
                const int o0 = hdr[wg], o1 = hdr[wg + 1];
                if (KIND == 2) {
                    const uint16_t *lc = reinterpret_cast<const uint16_t *>(sb + R.col_off);
                    const double *w1 = reinterpret_cast<const double *>(sb + R.win_off);
                    // own row in the window; rows past N (padding lanes of the last slice) read
                    // row N - 1 instead, whose value they discard
                    const int64_t irow = 32 * s + lane;
                    const int pad = irow > P.N - 1 ? (int)(irow - (P.N - 1)) : 0;
                    SrcWin src{lc + o0 + lane, vals + o0 + lane, w1, w1 + (size_t)P.nwin * P.win_cap,
                               hdr[29] + 32 * wg + lane - pad, 32 * wg + lane - pad, P.win_cap};
                    body(s, src, (o1 - o0) >> 5, hdr[16 + wg], hdr[17 + wg]);
                } else {
                    const int32_t *cols = reinterpret_cast<const int32_t *>(sb + R.col_off);
                    SrcRing src{cols + o0 + lane, vals + o0 + lane};
                    body(s, src, (o1 - o0) >> 5, hdr[16 + wg], hdr[17 + wg]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&R.empty[st]);
        }
        ++R.n;
    }
}

// Update phase through the TMA ring (TMA kinds): the producer bulk-copies chunks of UR rows
// of the four input streams (p, D^{-1} q, x, z) into a ring stage; consumer threads update
// their rows from shared memory and store x, z.  No L1 involvement: with most of the shared
// memory taken by the ring, L1-allocating loads would be limited by the small L1.
// body(row, p, q', x, z) for every row of this CTA's chunks; static chunk order.
template <int W, int NG, class Body>
__device__ __forceinline__ void sweep_u(const CGParams &P, Ring &R, const double *const (&src)[4], Body &&body) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t NS = (uint32_t)P.nstages;
    const int G = gridDim.x;
    const int64_t UR = P.u_rows;
    const int64_t nch = (P.N + UR - 1) / UR;
    if (warp == W * NG) {   // producer
        int64_t ch = blockIdx.x;
        while (true) {
            const uint32_t st = R.n % NS, ph = (R.n / NS) & 1u;
            if (ch >= nch) {
                const uint32_t m0 = R.n;
                for (int q = 0; q < NG; ++q) {
                    const uint32_t sq = R.n % NS, pq = (R.n / NS) & 1u;
                    if (lane == 0) {
                        mbar_wait(&R.empty[sq], pq ^ 1u);
                        int *hdr = reinterpret_cast<int *>(R.stage + (size_t)sq * R.stage_bytes);
                        hdr[31] = -1;
                        hdr[30] = (int)m0;
                        mbar_arrive(&R.full[sq]);
                    }
                    __syncwarp();
                    ++R.n;
                }
                break;
            }
            if (lane == 0) {
                mbar_wait(&R.empty[st], ph ^ 1u);
                fence_proxy_async_smem();   // consumers' reads of the stage before the bulk writes
                unsigned char *sb = R.stage + (size_t)st * R.stage_bytes;
                int *hdr = reinterpret_cast<int *>(sb);
                hdr[31] = (int)ch;
                const int64_t r0 = ch * UR;
                const int64_t rows = min(UR, P.N - r0);
                const uint32_t bytes = (uint32_t)(((rows + 1) & ~(int64_t)1) * 8);   // 16-B multiple
                mbar_arrive_expect_tx(&R.full[st], 4u * bytes);
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    bulk_g2s_nohint(sb + CG_HDR + (size_t)v * UR * 8, src[v] + r0, bytes, &R.full[st]);
            }
            __syncwarp();
            ++R.n;
            ch += G;
        }
        return;
    }
    const int g = warp / W, tid = threadIdx.x - g * W * 32;
    while (true) {
        const uint32_t st = R.n % NS, ph = (R.n / NS) & 1u;
        if ((int)(R.n % NG) == g) {
            mbar_wait(&R.full[st], ph);
            const unsigned char *sb = R.stage + (size_t)st * R.stage_bytes;
            const int ch = reinterpret_cast<const int *>(sb)[31];
            if (ch < 0) {
                const uint32_t m0 = (uint32_t)reinterpret_cast<const int *>(sb)[30];
                __syncwarp();
                if (lane == 0) mbar_arrive(&R.empty[st]);
                R.n = m0 + NG;
                break;
            }
            const double *base = reinterpret_cast<const double *>(sb + CG_HDR);
            const int64_t r0 = (int64_t)ch * UR;
            const int rows = (int)min(UR, P.N - r0);
            for (int r = tid; r < rows; r += W * 32)
                body(r0 + r, base[r], base[UR + r], base[2 * UR + r], base[3 * UR + r]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&R.empty[st]);
        }
        ++R.n;
    }
}

__host__ __device__ constexpr int cg_threads(int kind, int W, int NG) { return kind == 0 ? THERMO_BLOCK : (W * NG + 1) * 32; }

template <int KIND, int W, int NG, bool FUSED = false>
__global__ void __launch_bounds__(cg_threads(KIND, W, NG), KIND == 0 ? 2 : 1) k_cg_step(CGParams P) {
    const int NS = P.nstages;
    __shared__ double red_smem[THERMO_RED_SMEM];
    extern __shared__ __align__(128) unsigned char ring_raw[];
    // an earlier step failed, or the interface of this or an earlier step overflowed
    if (P.status[0] || (P.status[1] && P.status[4] <= P.step)) {   // an earlier step failed or the interface overflowed
        if (!P.status[0] && blockIdx.x == 0 && threadIdx.x == 0) {
            P.status[0] = 2;
            P.status[2] = P.step;
        }
        return;
    }
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const int G = gridDim.x;
    const int64_t N = P.N;

    Ring R;
    R.n = 0;
    R.meta_ok = false;
    if (KIND != 0) {
        R.full = reinterpret_cast<uint64_t *>(ring_raw);
        R.empty = R.full + NS;
        R.stage = ring_raw + 128;
        R.col_off = CG_HDR + (size_t)P.stage_entries * 8;
        R.win_off = align16(R.col_off + (size_t)P.stage_entries * (KIND == 2 ? 2 : 4));
        R.stage_bytes = align16(R.win_off + (KIND == 2 ? (size_t)(P.nwin * P.win_cap + 32 * W) * 8 : 0));
        if (threadIdx.x == 0) {
            for (int s = 0; s < NS; ++s) {
                mbar_init(&R.full[s], 1);
                mbar_init(&R.empty[s], W);
            }
            fence_mbar_init();
        }
        __syncthreads();
    }

    // ---- r0 = b - K~ x0, b = M_L T^n + dt (b_env + b_G); z0 = D^{-1} r0, p0 = z0.  x0 = T^n, or
    // the extrapolation X0 from earlier steps (then T^n's own rows come as the own-row block)
    const bool tr_on = P.trace && blockIdx.x == 0 && threadIdx.x == 0;
    int ntr = 0;
    if (tr_on) P.trace[ntr++] = gtimer();
    double red0[4] = {0.0, 0.0, 0.0, 0.0};   // b.b, r.r, r.z, |Gamma_R|
    P.pf[0] = P.T_in; P.pf[1] = P.ML; P.pf[2] = P.benv; P.pf[3] = P.Dinv;
    P.npf = P.prefetch ? 4 : 0;
    const double *const x0 = P.X0 ? P.X0 : P.T_in;
    P.wv[0] = x0;
    P.nwv = 1;
    P.ownv = P.X0 ? P.T_in : nullptr;
    sweep<KIND, W, NG>(P, R, [&](int64_t s, const auto &src, int w, int ib, int ie) {
        const int64_t i = 32 * s + lane;
        const int64_t ii = i < N ? i : N - 1;
        // own-row loads first: their latency overlaps the row sum
        const double be = P.benv[ii], ml = P.ML[ii], dv = P.Dinv[ii];
        const double Ti = P.X0 ? src.own2(P.T_in, ii) : src.own1(P.T_in, ii);
        const int ik = iface_index_r(P, ib, ie, i, lane);
        // ahead mode: the Jacobi diagonal of an interface row comes with its step's slot
        const double di = ik >= 0 && P.if_dinv_s ? P.if_dinv_s[ik] : dv;
        double ax = src.template dot<false>(w, x0, nullptr, 0.0);
        if (ik >= 0) ax += ell_row<false>(P, ik, x0, nullptr, 0.0);
        if (i < N) {
            double bi = be;
            if (ik >= 0) bi += P.if_b[ik];
            bi = P.rhs ? P.rhs[i] : fma(ml, Ti, P.dt * bi);
            const double r = bi - ax;
            const double zi = di * r;
            P.z[i] = zi;
            P.pa[i] = zi;   // p_0 = z_0
            red0[0] = fma(bi, bi, red0[0]);
            red0[1] = fma(r, r, red0[1]);
            red0[2] = fma(r, zi, red0[2]);
            if (ik >= 0 && ik < P.nA) red0[3] += P.if_phi[ik];
        }
    });
    P.ownv = nullptr;
    cta_reduce_store<4>(red0, red_smem, P.partials, 0);
    fence_proxy_async_global();   // plain stores before the next TMA reads
    grid.sync();
    if (tr_on) P.trace[ntr++] = gtimer();
    double tot0[4];
    grid_total<4>(P.partials, G, 0, red_smem, tot0);
    const double tol2 = P.rtol2 * tot0[0];
    double rho = tot0[2], rr = tot0[1];
    bool conv = rr <= tol2 && !P.debug;   // debug runs: fixed iteration count
    const double *xsrc = x0;
    double *const p = P.pa;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)G * blockDim.x;
    int it = 0;
    if constexpr (FUSED) {
        // One grid barrier per iteration: S(k) gathers the iteration-(k-1) state z, q', p of
        // buffer set (k-1)&1 and forms p_k = beta p + (z - alpha q') for every column itself,
        // so the update of iteration k-1 (x, z, p of its own rows) happens inside S(k); S(k)
        // writes z_k, p_k, q'_k to set k&1 (nobody reads that set during S(k)).  The CTA
        // partials alternate between two slot groups (a fast CTA's S(k+1) must not overwrite
        // what a slow CTA still reads).  Same formulas, same order: bitwise the unfused result.
        double alpha = 0.0, beta = 0.0;
        const bool fine = tr_on && P.trace_fine;   // THERMO_CG_TRACE=2: 4 stamps per iteration
        while (!conv && it < P.maxit) {
            if (fine && ntr < 1000) P.trace[ntr++] = gtimer();
            const bool first = it == 0;
            const int sn = it & 1;   // state set written (read: the other one)
            const double *const zr = sn ? P.z : P.z2, *const qr = sn ? P.q : P.q2, *const pr = sn ? P.pa : P.pb;
            double *const zw = sn ? P.z2 : P.z, *const qw = sn ? P.q2 : P.q, *const pw = sn ? P.pb : P.pa;
            double red[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            P.npf = 0;
            if (first) {
                P.wv[0] = P.pa;   // p_0 = z_0; z_0's own rows come as the own-row block
                P.nwv = 1;
                P.ownv = P.z;
            } else {
                P.wv[0] = zr; P.wv[1] = qr; P.wv[2] = pr;
                P.nwv = 3;
                P.ownv = xsrc;
            }
            sweep<KIND, W, NG>(P, R, [&](int64_t s, const auto &src, int w, int ib, int ie) {
                const int64_t i = 32 * s + lane;
                const int64_t ii = i < N ? i : N - 1;
                double zo, pi, xn = 0.0;
                if (first) {
                    pi = src.own1(nullptr, ii);
                    zo = src.own2(nullptr, ii);
                } else {
                    const double z0 = src.ownw(0), q0 = src.ownw(1), p0 = src.ownw(2), x0v = src.own2(nullptr, ii);
                    zo = fma(-alpha, q0, z0);
                    pi = fma(beta, p0, zo);
                    xn = fma(alpha, p0, x0v);
                }
                const int ik = iface_index_r(P, ib, ie, i, lane);
                double dg = src.first();
                double acc;
                if (first) {
                    acc = src.template dot<false>(w, nullptr, nullptr, 0.0);
                    if (ik >= 0) acc += ell_row<false>(P, ik, P.pa, nullptr, 0.0, ii, &dg);
                } else {
                    acc = src.dot3(w, alpha, beta);
                    if (ik >= 0) acc += ell_row3(P, ik, zr, qr, pr, alpha, beta, ii, &dg);
                }
                if (i < N) {
                    const double qv = acc / dg;
                    const double zd = zo * dg;
                    qw[i] = qv;
                    if (!first) {
                        zw[i] = zo;
                        pw[i] = pi;
                        P.T_out[i] = xn;
                    }
                    red[0] = fma(pi, acc, red[0]);
                    red[1] = fma(zo, zd, red[1]);
                    red[2] = fma(zo, acc, red[2]);
                    red[3] = fma(acc, qv, red[3]);
                    red[4] = fma(zd, zd, red[4]);
                    red[5] = fma(zd, acc, red[5]);
                    red[6] = fma(acc, acc, red[6]);
                }
            });
            P.ownv = nullptr;
            if (fine && ntr < 1000) P.trace[ntr++] = gtimer();
            const int slot = 4 + 7 * sn;
            cta_reduce_store<7>(red, red_smem, P.partials, slot);
            if (fine && ntr < 1000) P.trace[ntr++] = gtimer();
            fence_proxy_async_global();   // plain stores before the next TMA reads
            grid.sync();
            if (tr_on && ntr < 1000) P.trace[ntr++] = gtimer();
            double t7[7];
            grid_total<7>(P.partials, G, slot, red_smem, t7);
            if (!first) xsrc = P.T_out;   // x_it is complete
            if (!first && !P.debug) {
                rr = t7[4];
                if (rr <= tol2) { conv = true; break; }
            }
            const double an = rho / t7[0];
            const double rz_new = fma(an, fma(an, t7[3], -2.0 * t7[2]), t7[1]);
            const double rr_new = fma(an, fma(an, t7[6], -2.0 * t7[5]), t7[4]);
            const double rr_noise = 1e-13 * (t7[4] + fabs(2.0 * an * t7[5]) + an * an * t7[6]);
            beta = rz_new / rho;
            alpha = an;
            rho = rz_new;
            rr = rr_new;
            conv = rr <= tol2 && rr > rr_noise && !P.debug;
            ++it;
            if (conv || it >= P.maxit) {   // the last update x_it = x_{it-1} + alpha p_{it-1} alone
                const double *pl = pw;   // p_{it-1} (p_0 = P.pa)
                for (int64_t i = tid; i < N; i += nthr) P.T_out[i] = fma(alpha, pl[i], xsrc[i]);
                break;
            }
        }
    } else {
        while (!conv && it < P.maxit) {
            // ---- S: q = K~ p (the only gathered vector); q' = D^{-1} q with the diagonal d taken
            // from the row's own entries; partials of p.q and of the expansions of the next r.z and r.r
            //   z_new = z - alpha q', r_new = z_new d:  r.z = z^2 d - 2 alpha z q + alpha^2 q^2 / d,
            //   r.r = (z d)^2 - 2 alpha z d q + alpha^2 q^2,
            // so beta is known before the U phase, which forms the next direction itself
            double red[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            const bool first = it == 0;
            P.pf[0] = p;
            P.npf = P.prefetch ? 1 : 0;
            P.wv[0] = p;
            P.nwv = 1;
            P.ownv = P.z;
            sweep<KIND, W, NG>(P, R, [&](int64_t s, const auto &src, int w, int ib, int ie) {
                const int64_t i = 32 * s + lane;
                const int64_t ii = i < N ? i : N - 1;
                const double pi = src.own1(p, ii);      // issued before the row sum
                const double zo = src.own2(P.z, ii);
                const int ik = iface_index_r(P, ib, ie, i, lane);
                double dg = src.first();   // the diagonal (entry 0) + the interface self term
                double acc = src.template dot<false>(w, p, nullptr, 0.0);
                if (ik >= 0) acc += ell_row<false>(P, ik, p, nullptr, 0.0, ii, &dg);
                if (i < N) {
                    const double qs = acc / dg;
                    const double zd = zo * dg;
                    if (!(P.debug & 8)) P.q[i] = qs;   // debug bit 8: timing without the store
                    red[0] = fma(pi, acc, red[0]);
                    red[1] = fma(zo, zd, red[1]);
                    red[2] = fma(zo, acc, red[2]);
                    red[3] = fma(acc, qs, red[3]);
                    red[4] = fma(zd, zd, red[4]);
                    red[5] = fma(zd, acc, red[5]);
                    red[6] = fma(acc, acc, red[6]);
                }
            });
            P.ownv = nullptr;
            cta_reduce_store<7>(red, red_smem, P.partials, 4);
            fence_proxy_async_global();   // plain stores before the next TMA reads
            grid.sync();
            if (tr_on && ntr < 1000) P.trace[ntr++] = gtimer();
            double t7[7];
            grid_total<7>(P.partials, G, 4, red_smem, t7);
            // t7[4] = sum (z d)^2 is the current r.r computed directly: if an expansion below was
            // too close to its rounding noise to be trusted, the convergence test lands here, one
            // S phase later, before the update
            if (!first && !P.debug) {
                rr = t7[4];
                if (rr <= tol2) { conv = true; break; }
            }
            const double alpha = rho / t7[0];
            const double rz_new = fma(alpha, fma(alpha, t7[3], -2.0 * t7[2]), t7[1]);
            const double rr_new = fma(alpha, fma(alpha, t7[6], -2.0 * t7[5]), t7[4]);
            // rounding noise of the expansion (terms of size r.r of this iteration)
            const double rr_noise = 1e-13 * (t7[4] + fabs(2.0 * alpha * t7[5]) + alpha * alpha * t7[6]);
            const double beta = rz_new / rho;
            // ---- U: x += alpha p, z -= alpha q', p = z + beta p (streams only, no reduction)
            if constexpr (KIND != 0) {
                const double *const usrc[4] = {p, P.q, xsrc, P.z};
                sweep_u<W, NG>(P, R, usrc, [&](int64_t i, double pv, double qv, double xv, double zv) {
                    P.T_out[i] = fma(alpha, pv, xv);
                    const double zn = fma(-alpha, qv, zv);
                    P.z[i] = zn;
                    p[i] = fma(beta, pv, zn);
                });
            } else {   // element pairs with 16-byte loads, two pairs in flight per thread and trip
                const int64_t npair = N >> 1;
                double2 *p2 = reinterpret_cast<double2 *>(p);
                const double2 *q2 = reinterpret_cast<const double2 *>(P.q);
                const double2 *x2 = reinterpret_cast<const double2 *>(xsrc);
                double2 *z2 = reinterpret_cast<double2 *>(P.z);
                double2 *o2 = reinterpret_cast<double2 *>(P.T_out);
                auto upd = [&](double2 pv, double2 qv, double2 xv, double2 zv, int64_t j) {
                    o2[j] = make_double2(fma(alpha, pv.x, xv.x), fma(alpha, pv.y, xv.y));
                    const double2 zn = make_double2(fma(-alpha, qv.x, zv.x), fma(-alpha, qv.y, zv.y));
                    z2[j] = zn;
                    p2[j] = make_double2(fma(beta, pv.x, zn.x), fma(beta, pv.y, zn.y));
                };
                constexpr int UU = 2;
                int64_t j = tid;
                for (; j + (UU - 1) * nthr < npair; j += UU * nthr) {
                    double2 pv[UU], qv[UU], xv[UU], zv[UU];
    #pragma unroll
                    for (int u = 0; u < UU; ++u) {
                        const int64_t jj = j + u * nthr;
                        pv[u] = ld_cg2(p2 + jj); qv[u] = ld_cg2(q2 + jj); xv[u] = ld_cg2(x2 + jj); zv[u] = ld_cg2(z2 + jj);
                    }
    #pragma unroll
                    for (int u = 0; u < UU; ++u) upd(pv[u], qv[u], xv[u], zv[u], j + u * nthr);
                }
                for (; j < npair; j += nthr) upd(p2[j], q2[j], x2[j], z2[j], j);
                if ((N & 1) && tid == nthr - 1) {
                    const int64_t i = N - 1;
                    P.T_out[i] = fma(alpha, p[i], xsrc[i]);
                    const double zn = fma(-alpha, P.q[i], P.z[i]);
                    P.z[i] = zn;
                    p[i] = fma(beta, p[i], zn);
                }
            }
            fence_proxy_async_global();   // plain stores before the next TMA reads
            grid.sync();
            if (tr_on && ntr < 1000) P.trace[ntr++] = gtimer();
            rho = rz_new;
            rr = rr_new;
            // debug runs: fixed iteration count (maxit); an expansion within its noise is not trusted
            conv = rr <= tol2 && rr > rr_noise && !P.debug;
            xsrc = P.T_out;
            ++it;
        }
    }
    if (it == 0) {   // already converged: T^{n+1} = x0
        for (int64_t i = tid; i < N; i += nthr) P.T_out[i] = x0[i];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const double rel = tot0[0] > 0.0 ? sqrt(rr / tot0[0]) : sqrt(rr);
        P.iters_out[P.step] = it;
        P.relres_out[P.step] = rel;
        P.area_out[P.step] = tot0[3];
        if (!conv && !P.debug) {
            P.status[0] = 1;
            P.status[2] = P.step;
            P.status[3] = 0;
            *P.fail_relres = rel;
        }
    }
}

// ---------------------------------------------------------------------------------
// setup
// ---------------------------------------------------------------------------------

// largest column index of every chunk of W slices (warp per chunk)
__global__ void k_chunk_hi(const int64_t *slice_ptr, const int32_t *col, int64_t nslices, int64_t nchunks,
                           int W, int32_t *hi) {
    const int64_t ch = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (ch >= nchunks) return;
    const int64_t s0 = ch * W, s1 = min(s0 + (int64_t)W, nslices);
    int m = 0;
    for (int64_t e = slice_ptr[s0] + lane; e < slice_ptr[s1]; e += 32) m = max(m, col[e]);
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) hi[ch] = m;
}

// Column window of every chunk (block per chunk, KIND 2): the chunk's distinct columns,
// sorted, cut into runs wherever a gap exceeds CG_GAP, runs widened to even bounds (16-byte
// bulk copies); then every entry's chunk-local 16-bit column index.  stats[0] = max window,
// stats[1] = max runs, stats[2] = overflow (window > 65535 or chunk > CW_MAXE entries).
#define CW_MAXE 4096
__global__ void __launch_bounds__(256) k_chunk_windows(const int64_t *slice_ptr, const int32_t *col,
                                                       int64_t nslices, int W, int gap, int2 *runs_out,
                                                       int32_t *nruns_out, int32_t *lown_out, uint16_t *lcol,
                                                       int *stats) {
    __shared__ int key[CW_MAXE];
    __shared__ int rstart[CW_MAXE / 2 + 1], rlast[CW_MAXE / 2 + 1], roff[CW_MAXE / 2 + 2];
    __shared__ int nr_s;
    const int64_t ch = blockIdx.x;
    const int64_t s0 = ch * W, s1 = min(s0 + (int64_t)W, nslices);
    const int64_t e0 = slice_ptr[s0];
    const int E = (int)(slice_ptr[s1] - e0);
    if (E > CW_MAXE) {
        if (threadIdx.x == 0) atomicOr(&stats[2], 1);
        return;
    }
    int n2 = 1;
    while (n2 < E) n2 <<= 1;
    for (int e = threadIdx.x; e < n2; e += blockDim.x) key[e] = e < E ? col[e0 + e] : 0x7fffffff;
    __syncthreads();
    for (int size = 2; size <= n2; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < n2 / 2; i += blockDim.x) {
                const int lo = 2 * stride * (i / stride) + (i % stride), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const int a = key[lo], b = key[hi];
                if ((a > b) == up) { key[lo] = b; key[hi] = a; }
            }
            __syncthreads();
        }
    if (threadIdx.x == 0) {   // runs (serial over <= 4096 sorted keys)
        // at most CG_MAXR runs are recorded (the run arrays hold CW_MAXE / 2 + 1 > CG_MAXR):
        // a chunk with more (a scattered numbering) disqualifies the variant (stats[1])
        int nr = 0;
        bool over = E == 0;
        for (int j = 0; j < E && !over; ++j) {
            if (j == 0 || key[j] - key[j - 1] > gap + 1) {
                if (nr == CG_MAXR) { over = true; break; }
                rstart[nr] = key[j] & ~1;
                if (nr > 0) rlast[nr - 1] = key[j - 1];
                ++nr;
            }
        }
        if (over) {
            atomicMax(&stats[1], CG_MAXR + 1);
            nruns_out[ch] = 0;
            nr_s = 0;
        } else {
            rlast[nr - 1] = key[E - 1];
            roff[0] = 0;
            for (int r = 0; r < nr; ++r) roff[r + 1] = roff[r] + (((rlast[r] + 2) & ~1) - rstart[r]);
            nr_s = nr;
            atomicMax(&stats[0], roff[nr]);
            atomicMax(&stats[1], nr);
            if (roff[nr] > 65535) atomicOr(&stats[2], 2);
            nruns_out[ch] = nr;
            // local index of the chunk's first row (its own rows are one contiguous block)
            const int r0 = (int)(s0 * 32);
            int lo = 0;
            for (int r = 0; r < nr; ++r) if (rstart[r] <= r0) lo = r;
            lown_out[ch] = roff[lo] + (r0 - rstart[lo]);
            for (int r = 0; r < nr; ++r) runs_out[ch * CG_MAXR + r] = make_int2(rstart[r], roff[r + 1] - roff[r]);
        }
    }
    __syncthreads();
    const int nr = nr_s;
    if (nr == 0) return;   // variant rejected (stats); lcol is not used
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        const int c = col[e0 + e];
        int lo = 0, hi = nr - 1;
        while (lo < hi) {   // last run with start <= c
            const int mid = (lo + hi + 1) >> 1;
            if (rstart[mid] <= c) lo = mid; else hi = mid - 1;
        }
        int lc = roff[lo] + (c - rstart[lo]);
        if (c < rstart[lo] || c > rlast[lo] + 1) lc = 0;   // cannot happen: every column is in a run
        lcol[e0 + e] = (uint16_t)lc;
    }
}

void chunk_windows_launch(Ctx &c, int W, int gap, int2 *runs, int32_t *nruns, int32_t *lown, uint16_t *lcol,
                          int *d_stats) {
    const int64_t nchunks = (c.nslices + W - 1) / W;
    k_chunk_windows<<<(unsigned)nchunks, 256, 0, c.stream>>>(c.d_slice_ptr, c.d_col, c.nslices, W, gap, runs, nruns,
                                                            lown, lcol, d_stats);
}

struct Variant {
    int kind, W, NG;
    bool fused;   // one grid barrier per iteration (KIND 2 only)
};
static const Variant kVariants[] = {{0, 8, 1, false}, {1, 8, 2, false}, {2, 8, 1, false}, {2, 8, 2, false},
                                   {2, 6, 1, false},  {2, 6, 2, false}, {2, 4, 2, false}, {2, 4, 1, false},
                                   {2, 8, 1, true},   {2, 6, 1, true},  {2, 4, 1, true}};
#define CG_NVAR 11

template <int KIND, int W, int NG, bool FUSED = false>
static const void *kernel_ptr() { return (const void *)k_cg_step<KIND, W, NG, FUSED>; }

static const void *variant_kernel(int v) {
    switch (v) {
        case 0: return kernel_ptr<0, 8, 1>();
        case 1: return kernel_ptr<1, 8, 2>();
        case 2: return kernel_ptr<2, 8, 1>();
        case 3: return kernel_ptr<2, 8, 2>();
        case 4: return kernel_ptr<2, 6, 1>();
        case 5: return kernel_ptr<2, 6, 2>();
        case 6: return kernel_ptr<2, 4, 2>();
        case 7: return kernel_ptr<2, 4, 1>();
        case 8: return kernel_ptr<2, 8, 1, true>();
        case 9: return kernel_ptr<2, 6, 1, true>();
        default: return kernel_ptr<2, 4, 1, true>();
    }
}

static size_t stage_bytes(const Variant &v, int E, int wc) {
    size_t col_off = CG_HDR + (size_t)E * 8;
    size_t win_off = align16(col_off + (size_t)E * (v.kind == 2 ? 2 : 4));
    return align16(win_off + (v.kind == 2 ? (size_t)((v.fused ? 3 : 1) * wc + 32 * v.W) * 8 : 0));
}

int cg_setup(Ctx &c) {
    const char *env = getenv("THERMO_CG_VARIANT");   // testing / tuning hook
    int want = env ? atoi(env) : -1;
    if (want >= CG_NVAR) want = -1;
    std::vector<int64_t> sp(c.nslices + 1);
    CK(cudaMemcpy(sp.data(), c.d_slice_ptr, sizeof(int64_t) * (c.nslices + 1), cudaMemcpyDeviceToHost));
    auto emax_for = [&](int W) {
        int64_t m = 0;
        for (int64_t s0 = 0; s0 < c.nslices; s0 += W) m = std::max(m, sp[std::min<int64_t>(s0 + W, c.nslices)] - sp[s0]);
        return (int)((m + 31) / 32 * 32);
    };
    // candidate order: the requested variant, then the default preference
    std::vector<int> order;
    if (want >= 0) order.push_back(want);
    // L2-resident problems are latency-bound: the one-barrier kernel (8) saves a grid barrier
    // and a ring pass per iteration (cfg 1: 14.6 -> 13.3 us); beyond that its three vector
    // windows cost more TMA ingress than the update phase it removes (cfg 2: 57 -> 74 us,
    // cfg 3: 405 -> 459 us per iteration), so the two-phase kernel (2) is the default there
    const bool small = c.N <= (int64_t)1 << 18;
    for (int v : {8, 2, 3, 4, 5, 6, 7, 1, 0})
        if (v != want && (small || v != 8)) order.push_back(v);
    int chosen = -1, per_sm = 0;
    for (int vi : order) {
        const Variant &v = kVariants[vi];
        const int E = emax_for(v.W);
        const int64_t nchunks = (c.nslices + v.W - 1) / v.W;
        int wc = 0;
        if (v.kind == 2) {
            if (E > CW_MAXE) continue;
            // windows of every chunk (and the 16-bit local columns) for this chunk size
            if (!c.d_lcol) CK(cudaMalloc(&c.d_lcol, sizeof(uint16_t) * (c.nnz_pad + 8)));
            if (c.d_chunk_runs) { cudaFree(c.d_chunk_runs); cudaFree(c.d_chunk_nruns); }
            CK(cudaMalloc(&c.d_chunk_runs, sizeof(int2) * nchunks * CG_MAXR));
            CK(cudaMalloc(&c.d_chunk_nruns, sizeof(int32_t) * (nchunks + 1)));
            if (c.d_chunk_lown) cudaFree(c.d_chunk_lown);
            CK(cudaMalloc(&c.d_chunk_lown, sizeof(int32_t) * (nchunks + 1)));
            int *d_stats = nullptr;
            CK(cudaMalloc(&d_stats, sizeof(int) * 4));
            CK(cudaMemsetAsync(d_stats, 0, sizeof(int) * 4, c.stream));
            const char *eg = getenv("THERMO_CG_GAP");   // tuning hook: bridged column gap
            const int gap = eg ? std::max(2, atoi(eg)) : (c.N > ((int64_t)1 << 22) ? CG_GAP_LARGE : CG_GAP);
            k_chunk_windows<<<(unsigned)nchunks, 256, 0, c.stream>>>(c.d_slice_ptr, c.d_col, c.nslices, v.W, gap,
                                                                    c.d_chunk_runs, c.d_chunk_nruns, c.d_chunk_lown,
                                                                    c.d_lcol, d_stats);
            CK(cudaGetLastError());
            int stats[4];
            CK(cudaMemcpyAsync(stats, d_stats, sizeof stats, cudaMemcpyDeviceToHost, c.stream));
            CK(cudaStreamSynchronize(c.stream));
            cudaFree(d_stats);
            if (stats[2] || stats[1] > CG_MAXR) continue;
            wc = (stats[0] + 1) & ~1;
            c.cg_max_runs = stats[1];
        }
        const size_t sb = stage_bytes(v, E, wc);
        // ring budget: 210 KB leaves the rest of the 228-KB carve-out to L1 (224 KB, one more
        // stage on cfg 3, measured no faster: the ring is not depth-bound)
        const char *ekb = getenv("THERMO_CG_SMEM_KB");   // tuning hook
        const size_t budget = (size_t)(ekb ? atoi(ekb) : 210) * 1024 - 128;
        int ns = v.kind == 0 ? 1 : (int)std::min<size_t>(8, budget / sb);
        if (const char *e = getenv("THERMO_CG_STAGES")) ns = std::min(ns, std::max(2, atoi(e)));   // tuning hook
        // consumer group g takes ring slots n = g (mod NG), stage n mod ns: with ns a multiple
        // of NG every stage belongs to one group, so a group can never run two phases ahead
        // of a stage's mbarrier (an ns = 3, NG = 2 ring passed a parity wait one phase early
        // and read a stale stage on cfg 3)
        if (v.kind != 0) ns -= ns % v.NG;
        if (v.kind != 0 && ns < std::max(2, v.NG)) continue;   // at least one stage in flight
        const size_t smem = v.kind == 0 ? 0 : 128 + (size_t)ns * sb;
        const void *fn = variant_kernel(vi);
        if (smem > 48 * 1024) CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, cg_threads(v.kind, v.W, v.NG), smem));
        if (per_sm < 1) continue;
        chosen = vi;
        c.cg_smem = smem;
        c.cg_stage_entries = E;
        c.cg_win_cap = wc;
        c.cg_chunk = v.W;
        c.cg_block = cg_threads(v.kind, v.W, v.NG);
        c.cg_nstages = ns;
        c.cg_u_rows = v.kind == 0 ? 0 : (int64_t)((sb - CG_HDR) / 32) & ~(int64_t)31;   // 4 streams
        break;
    }
    if (chosen < 0) { c.err = "no CG kernel variant can be resident"; return -3; }
    if (getenv("THERMO_CG_VERBOSE"))
        fprintf(stderr, "[thermo cg] variant %d (kind %d, W %d, NG %d): stage entries %d, window cap %d, "
                        "stage %zu B, %d stages, smem %zu B\n", chosen, kVariants[chosen].kind, c.cg_chunk,
                kVariants[chosen].NG, c.cg_stage_entries, c.cg_win_cap,
                stage_bytes(kVariants[chosen], c.cg_stage_entries, c.cg_win_cap), c.cg_nstages, c.cg_smem);
    c.cg_variant = chosen;
    c.cg_kind = kVariants[chosen].kind;
    const char *dbg = getenv("THERMO_CG_DEBUG");
    c.cg_debug = dbg ? atoi(dbg) : 0;
    const char *pfe = getenv("THERMO_CG_PREFETCH");
    c.cg_prefetch = pfe ? atoi(pfe) : 0;
    c.cg_tma = kVariants[chosen].kind != 0;
    c.cg_fused = kVariants[chosen].fused;
    if (c.cg_fused && !c.d_z2) {   // second buffer set of z, q' (vectors padded like the others)
        CK(cudaMalloc(&c.d_z2, sizeof(double) * (c.N + 16)));
        CK(cudaMalloc(&c.d_q2, sizeof(double) * (c.N + 16)));
        CK(cudaMemsetAsync(c.d_z2, 0, sizeof(double) * (c.N + 16), c.stream));
        CK(cudaMemsetAsync(c.d_q2, 0, sizeof(double) * (c.N + 16), c.stream));
    }
    const int W = c.cg_chunk;
    const int64_t nchunks = (c.nslices + W - 1) / W;
    CK(cudaMalloc(&c.d_chunk_hi, sizeof(int32_t) * (nchunks + 1)));
    k_chunk_hi<<<(unsigned)((nchunks * 32 + 255) / 256), 256, 0, c.stream>>>(c.d_slice_ptr, c.d_col, c.nslices,
                                                                           nchunks, W, c.d_chunk_hi);
    CK(cudaGetLastError());
    c.cg_grid = (kVariants[chosen].kind == 0 ? per_sm : 1) * c.num_sms;
    if (const char *e = getenv("THERMO_CG_CTAS")) {   // tuning hook: fewer CTAs than SMs
        const int g = atoi(e);
        if (g >= 1 && g < c.cg_grid) c.cg_grid = g;
    }
    CK(cudaMalloc(&c.d_partials, sizeof(double) * THERMO_NRED * c.cg_grid));
    return cl_setup(c);   // small problems: the single-cluster latency solve (cg_cluster.cu)
}

int cg_launch_solve(Ctx &c, const double *x0, double *x, const double *rhs, const double *Dinv, bool iface,
                    int32_t *iters_out, double *relres_out, int slot) {
    CGParams P;
    memset(&P, 0, sizeof P);
    P.N = c.N;
    P.nslices = c.nslices;
    P.nchunks = (c.nslices + c.cg_chunk - 1) / c.cg_chunk;
    P.slice_ptr = c.d_slice_ptr;
    P.col = c.d_col;
    P.lcol = c.d_lcol;
    P.val = c.d_val;
    P.ML = c.d_ML;
    P.benv = c.d_benv;
    P.Dinv = Dinv;
    P.n_if = iface ? c.n_if : 0;
    P.nA = c.nA;
    P.if_rows = c.d_if_rows;
    P.slice_if = iface ? c.d_slice_if : c.d_slice_if_zero;
    P.ell_cnt = c.d_ell_cnt;
    P.ell_col = c.d_ell_col;
    P.ell_val = c.d_ell_val;
    P.if_b = c.d_if_b;
    P.if_phi = c.d_if_phi;
    P.T_in = x0;
    P.rhs = rhs;
    P.T_out = x;
    P.z = c.d_z;
    P.pa = c.d_p[0];
    P.pb = c.d_p[1];
    P.q = c.d_q;
    P.partials = c.d_partials;
    P.status = c.d_status;
    P.fail_relres = c.d_fail_relres;
    P.iters_out = iters_out;
    P.relres_out = relres_out;
    P.area_out = c.d_area;
    P.dt = 0.0;
    P.rtol2 = c.rtol * c.rtol;
    P.maxit = c.maxit > 0 ? c.maxit : (int)std::min<int64_t>(10 * c.N, 10000);
    P.step = slot;
    P.stage_entries = c.cg_stage_entries;
    P.nstages = c.cg_nstages;
    P.u_rows = c.cg_u_rows;
    P.win_cap = c.cg_win_cap;
    P.nwin = c.cg_fused ? 3 : 1;
    P.z2 = c.d_z2;
    P.q2 = c.d_q2;
    P.chunk_hi = c.d_chunk_hi;
    P.chunk_runs = c.d_chunk_runs;
    P.chunk_nruns = c.d_chunk_nruns;
    P.chunk_lown = c.d_chunk_lown;
    P.trace = nullptr;
    if (c.rs_on) return rs_launch(c, P, false, 0);
    if (c.cl_on) return cl_launch(c, P, false, 0);
    void *args[] = {&P};
    CK(cudaLaunchCooperativeKernel(variant_kernel(c.cg_variant), dim3(c.cg_grid), dim3(c.cg_block), args,
                                   c.cg_smem, c.stream));
    return 0;
}

int cg_launch_step(Ctx &c, int step, double dt, const double *x0, int buf, bool ovl, int ah_slot, int xhist,
                   int xguess, int nst) {
    CGParams P;
    memset(&P, 0, sizeof P);
    P.N = c.N;
    P.nslices = c.nslices;
    P.nchunks = (c.nslices + c.cg_chunk - 1) / c.cg_chunk;
    P.slice_ptr = c.d_slice_ptr;
    P.col = c.d_col;
    P.lcol = c.d_lcol;
    P.val = c.d_val;
    P.ML = c.d_ML;
    P.benv = c.d_benv;
    P.Dinv = buf ? c.d_Dinv_b : c.d_Dinv;
    P.n_if = c.n_if;
    P.nA = c.nA;
    P.if_rows = c.d_if_rows;
    P.slice_if = c.d_slice_if;
    P.ell_cnt = buf ? c.d_ell_cnt_b : c.d_ell_cnt;
    P.ell_col = buf ? c.d_ell_col_b : c.d_ell_col;
    P.ell_val = buf ? c.d_ell_val_b : c.d_ell_val;
    P.if_b = buf ? c.d_if_b_b : c.d_if_b;
    P.if_phi = buf ? c.d_if_phi_b : c.d_if_phi;
    P.T_in = c.d_T[(c.cur + step) & 1];
    P.X0 = x0;
    P.T_out = c.d_T[(c.cur + step + 1) & 1];
    P.z = c.d_z;
    P.pa = c.d_p[0];
    P.pb = c.d_p[1];
    P.q = c.d_q;
    P.partials = c.d_partials;
    P.status = c.d_status;
    P.fail_relres = c.d_fail_relres;
    P.iters_out = c.d_iters;
    P.relres_out = c.d_relres;
    P.area_out = c.d_area;
    P.dt = dt;
    P.rtol2 = c.rtol * c.rtol;
    P.maxit = c.cg_debug ? 50 : (c.maxit > 0 ? c.maxit : (int)std::min<int64_t>(10 * c.N, 10000));
    P.step = step;
    P.stage_entries = c.cg_stage_entries;
    P.nstages = c.cg_nstages;
    P.u_rows = c.cg_u_rows;
    P.win_cap = c.cg_win_cap;
    P.nwin = c.cg_fused ? 3 : 1;
    P.z2 = c.d_z2;
    P.q2 = c.d_q2;
    P.chunk_hi = c.d_chunk_hi;
    P.chunk_runs = c.d_chunk_runs;
    P.chunk_nruns = c.d_chunk_nruns;
    P.chunk_lown = c.d_chunk_lown;
    P.trace = c.d_trace;
    P.trace_fine = c.d_trace && getenv("THERMO_CG_TRACE") && atoi(getenv("THERMO_CG_TRACE")) == 2;
    P.debug = c.cg_debug;
    P.prefetch = c.cg_prefetch;
    if (ah_slot >= 0) {   // ahead mode: this step's interface rows sit in slot ah_slot
        const int64_t nif = c.n_if;
        P.ell_cnt = c.d_ah_ell_cnt + ah_slot * nif;
        P.ell_col = c.d_ah_ell_col + (int64_t)ah_slot * c.cap * nif;
        P.ell_val = c.d_ah_ell_val + (int64_t)ah_slot * c.cap * nif;
        P.if_b = c.d_ah_if_b + ah_slot * nif;
        P.if_phi = c.d_ah_if_phi + ah_slot * nif;
        P.if_dinv_s = c.d_ah_dinv + ah_slot * nif;
        P.Dinv = c.d_Dinv_vol;
    }
    if (c.rs_on) {
        P.xhist = xhist;     // extrapolated start formed inside the kernel (no k_extrap launch)
        P.xguess = xguess;
        P.xsave = xguess >= 2 ? 1 : 0;
        P.Th = c.d_Thist;
        P.nst = nst;
        P.Tin_w = c.d_T[(c.cur + step) & 1];
        return rs_launch(c, P, ovl, buf);
    }
    if (c.cl_on) return cl_launch(c, P, ovl, buf);
    void *args[] = {&P};
    if (ovl) {   // cooperative launch that records ev_cg[step & 1] once all of its CTAs have begun
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        at[1].id = cudaLaunchAttributeLaunchCompletionEvent;
        at[1].val.launchCompletionEvent.event = c.ev_cg[buf];   // events follow the buffer sets
        at[1].val.launchCompletionEvent.flags = 0;
        cudaLaunchConfig_t cfg;
        memset(&cfg, 0, sizeof cfg);
        cfg.gridDim = dim3(c.cg_grid_ovl);
        cfg.blockDim = dim3(c.cg_block);
        cfg.dynamicSmemBytes = c.cg_smem;
        cfg.stream = c.stream;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        CK(cudaLaunchKernelExC(&cfg, variant_kernel(c.cg_variant), args));
        return 0;
    }
    CK(cudaLaunchCooperativeKernel(variant_kernel(c.cg_variant), dim3(ovl ? c.cg_grid_ovl : c.cg_grid),
                                   dim3(c.cg_block), args,
                                   c.cg_smem, c.stream));
    return 0;
}

// Overlap mode: a second interface buffer set, a side stream with its events,
// and a CG grid that leaves overlap_sms SMs to the side stream's interface kernels.
int overlap_setup(Ctx &c) {
    if (c.S != 1 || c.n_if == 0) return 0;
    const char *e = getenv("THERMO_OVERLAP");   // 0: off, 1: on, unset: L2-resident sizes only
    const bool want = e ? atoi(e) != 0 : c.N <= (int64_t)1 << 18;
    if (!want) return 0;
    const char *es = getenv("THERMO_OVERLAP_SMS");
    int free_sms = es ? atoi(es) : 24;
    free_sms = std::max(1, std::min(free_sms, c.num_sms / 2));
    const int64_t nif = c.n_if;
    CK(cudaMalloc(&c.d_ell_cnt_b, sizeof(int32_t) * nif));
    CK(cudaMalloc(&c.d_ell_col_b, sizeof(int32_t) * c.cap * nif));
    CK(cudaMalloc(&c.d_ell_val_b, sizeof(double) * c.cap * nif));
    CK(cudaMalloc(&c.d_if_b_b, sizeof(double) * nif));
    CK(cudaMalloc(&c.d_if_phi_b, sizeof(double) * nif));
    CK(cudaMalloc(&c.d_Dinv_b, sizeof(double) * (c.N + 16)));
    CK(cudaMalloc(&c.d_step_sc_spec, sizeof(double) * 4));
    CK(cudaMalloc(&c.d_spec_status, sizeof(int) * 8));
    CK(cudaMemsetAsync(c.d_ell_cnt_b, 0, sizeof(int32_t) * nif, c.stream));
    CK(cudaMemsetAsync(c.d_if_b_b, 0, sizeof(double) * nif, c.stream));
    CK(cudaMemsetAsync(c.d_if_phi_b, 0, sizeof(double) * nif, c.stream));
    CK(cudaStreamCreateWithFlags(&c.if_stream, cudaStreamNonBlocking));
    for (cudaEvent_t *ev : {&c.ev_if[0], &c.ev_if[1], &c.ev_cg[0], &c.ev_cg[1], &c.ev_done[0], &c.ev_done[1], &c.ev_main,
                            &c.ev_side_end})
        CK(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
    c.overlap = true;
    c.overlap_sms = free_sms;
    c.cg_grid_ovl = std::min(c.cg_grid, c.num_sms - free_sms);   // the other solves keep the full grid
    // the solve CTAs claim all of their SMs' shared memory, so no interface block is placed next
    // to them (co-resident interface blocks slowed the latency-bound solve by ~25 % on cfg 1)
    if (c.cg_tma) {
        int dev_max = 0;
        CK(cudaDeviceGetAttribute(&dev_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.dev));
        const size_t claim = (size_t)dev_max - sizeof(double) * THERMO_RED_SMEM;
        if (claim > c.cg_smem) {
            CK(cudaFuncSetAttribute(variant_kernel(c.cg_variant), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)claim));
            c.cg_smem = claim;
        }
    }
    return 0;
}

}  // namespace thermo
