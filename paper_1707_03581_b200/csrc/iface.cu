// iface.cu -- per-step re-integration of the interface terms on Gamma_R(t).
//
// K2a (k_pairs, one launch for both surfaces): a warp takes 4 triangles of one surface, finds
// every triangle of the other surface whose box overlaps (uniform bin grid, each pair visited
// once), cuts the overlap polygon F cap (G + o) by Sutherland-Hodgman (F = rail-top
// triangle, G = stock-bottom triangle, o = in-plane offset of the stock), fans it from
// vertex 0 and integrates the products of the two P1 fields exactly with the P1 mass formula
//   int_tau g h = |tau|/12 (sum_i g_i h_i + sum_i g_i sum_i h_i)
// on every fan triangle tau; the result is one record per overlapping pair and side.
// K2b (k_rows): one warp per interface node sums the records of its star into its row of
// K~_G = -dt [[M_B,fix, C_B], [C_B^T, M_B,mov]] and its friction source
// eta/2 int phi, and refreshes its Jacobi diagonal.
// Every sum runs in a fixed order, so results are deterministic; no floating-point atomics.
//
// Host part (iface_setup): plane and in-plane basis, interface node numbering, stars, bin
// grids, and the per-row capacity of the interface rows (swept over the motion range).
#include <algorithm>
#include <cmath>
#include <cstring>

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

#define IF_MAXV 8    // polygon vertices (a triangle clipped by 3 half-planes has <= 6)

__device__ __forceinline__ double cross2(double ax, double ay, double bx, double by) {
    return ax * by - ay * bx;
}

// Clip triangle F (counter-clockwise) by the counter-clockwise triangle G; inclusive
// inside test.  Returns the vertex count of F cap G.
__device__ int clip_tri(const double2 F[3], const double2 G[3], double2 *out) {
    double2 a[IF_MAXV], b[IF_MAXV];
    int n = 3;
    a[0] = F[0]; a[1] = F[1]; a[2] = F[2];
    double2 *cur = a, *nxt = b;
    for (int e = 0; e < 3; ++e) {
        double2 c1 = G[e], c2 = G[e == 2 ? 0 : e + 1];
        double ex = c2.x - c1.x, ey = c2.y - c1.y;
        int m = 0;
        double2 prev = cur[n - 1];
        double dprev = cross2(ex, ey, prev.x - c1.x, prev.y - c1.y);
        for (int k = 0; k < n; ++k) {
            double2 p = cur[k];
            double dp = cross2(ex, ey, p.x - c1.x, p.y - c1.y);
            if (dp >= 0.0) {
                if (dprev < 0.0 && m < IF_MAXV) {
                    double t = dprev / (dprev - dp);
                    nxt[m++] = make_double2(prev.x + t * (p.x - prev.x), prev.y + t * (p.y - prev.y));
                }
                if (m < IF_MAXV) nxt[m++] = p;
            } else if (dprev >= 0.0 && m < IF_MAXV) {
                double t = dprev / (dprev - dp);
                nxt[m++] = make_double2(prev.x + t * (p.x - prev.x), prev.y + t * (p.y - prev.y));
            }
            prev = p;
            dprev = dp;
        }
        double2 *tmp = cur; cur = nxt; nxt = tmp;
        n = m;
        if (n == 0) break;
    }
    for (int k = 0; k < n; ++k) out[k] = cur[k];
    return n;
}

__device__ __forceinline__ void bary(const double2 T[3], double2 y, double l[3]) {
    double D = cross2(T[1].x - T[0].x, T[1].y - T[0].y, T[2].x - T[0].x, T[2].y - T[0].y);
    double inv = 1.0 / D;
    l[1] = cross2(y.x - T[0].x, y.y - T[0].y, T[2].x - T[0].x, T[2].y - T[0].y) * inv;
    l[2] = cross2(T[1].x - T[0].x, T[1].y - T[0].y, y.x - T[0].x, y.y - T[0].y) * inv;
    l[0] = 1.0 - l[1] - l[2];
}

__device__ __forceinline__ int bin_coord(double v, double v0, double inv_h, int n) {
    int b = (int)floor((v - v0) * inv_h);
    return b < 0 ? 0 : (b >= n ? n - 1 : b);
}

// ------------------------------------------------------------------------------ K2a: pairs

// Integrals over one overlap polygon F cap (G + o) (both triangles given in the fixed frame), for
// both sides at once: ownF = int phi_F,a phi_F,b, ownG = int phi_G,a phi_G,b (symmetric, 00 01 02
// 11 12 22), cross[a*3+b] = int phi_F,a phi_G,b, bF / bG = int phi_F,a / phi_G,a.  The polygon is F
// clipped by G; the G side's cross block is the transpose (x*y == y*x in IEEE arithmetic, so it
// equals bitwise what a G-side evaluation of the same products would give).
__device__ bool pair_integrals(const double2 F[3], const double2 G[3], PairRec &r) {
    double2 poly[IF_MAXV];
    const int nv = clip_tri(F, G, poly);
    if (nv < 3) return false;
    // barycentric maps of both triangles (the same arithmetic as bary(), inverse hoisted)
    const double invF = 1.0 / cross2(F[1].x - F[0].x, F[1].y - F[0].y, F[2].x - F[0].x, F[2].y - F[0].y);
    const double invG = 1.0 / cross2(G[1].x - G[0].x, G[1].y - G[0].y, G[2].x - G[0].x, G[2].y - G[0].y);
    auto bc = [](const double2 T[3], double inv, double2 y, double l[3]) {
        l[1] = cross2(y.x - T[0].x, y.y - T[0].y, T[2].x - T[0].x, T[2].y - T[0].y) * inv;
        l[2] = cross2(T[1].x - T[0].x, T[1].y - T[0].y, y.x - T[0].x, y.y - T[0].y) * inv;
        l[0] = 1.0 - l[1] - l[2];
    };
    double R[27];   // ownF[6] ownG[6] cross[9] bF[3] bG[3]
#pragma unroll
    for (int q = 0; q < 27; ++q) R[q] = 0.0;
    double f0[3], g0[3], f1[3], g1[3], f2[3], g2[3];
    bc(F, invF, poly[0], f0);
    bc(G, invG, poly[0], g0);
    bc(F, invF, poly[1], f1);
    bc(G, invG, poly[1], g1);
    double area = 0.0;
    for (int f = 1; f + 1 < nv; ++f) {
        const double2 p0 = poly[0], p1 = poly[f], p2 = poly[f + 1];
        bc(F, invF, p2, f2);
        bc(G, invG, p2, g2);
        const double ar = 0.5 * cross2(p1.x - p0.x, p1.y - p0.y, p2.x - p0.x, p2.y - p0.y);
        if (ar > 0.0) {
            area += ar;
            const double w12 = ar * (1.0 / 12.0), w3 = ar * (1.0 / 3.0);
            double sf[3], sg[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                sf[a] = f0[a] + f1[a] + f2[a];
                sg[a] = g0[a] + g1[a] + g2[a];
            }
            int q = 0;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                R[21 + a] += w3 * sf[a];
                R[24 + a] += w3 * sg[a];
#pragma unroll
                for (int b = a; b < 3; ++b, ++q) {
                    R[q] += w12 * (f0[a] * f0[b] + f1[a] * f1[b] + f2[a] * f2[b] + sf[a] * sf[b]);
                    R[6 + q] += w12 * (g0[a] * g0[b] + g1[a] * g1[b] + g2[a] * g2[b] + sg[a] * sg[b]);
                }
#pragma unroll
                for (int b = 0; b < 3; ++b)
                    R[12 + a * 3 + b] += w12 * (f0[a] * g0[b] + f1[a] * g1[b] + f2[a] * g2[b] + sf[a] * sg[b]);
            }
        }
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            f1[a] = f2[a];
            g1[a] = g2[a];
        }
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        r.ownF[q] = R[q];
        r.ownG[q] = R[6 + q];
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) r.cross[q] = R[12 + q];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        r.bF[q] = R[21 + q];
        r.bG[q] = R[24 + q];
    }
    return area > 0.0;
}

__device__ __forceinline__ int warp_excl_scan(int v, int lane) {
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x - v;
}

// Warp per (PAIR_TPW consecutive stock-bottom triangles G, scenario s); every overlapping pair is
// clipped once, from the stock side (round 1 clipped it once per side).
//  1. candidates: per G, the rail-top triangles of all bins under its box (in the rail frame) are
//     flattened (bins row-major, ascending ids) and spread over the lanes; box-overlapping ones,
//     each counted in one bin only, are appended to a per-warp shared-memory queue in that order
//     (ballot prefix).
//  2. integrals: the queue is clipped 32 pairs at a time, one pair per lane, so the lanes stay
//     busy across triangles; a hit's record slot is its rank among its own G's hits (records of
//     a G come out in candidate order, the same for every run).  The rail triangle F gets a
//     reference g * pcap + slot appended to its list (an integer atomic: the list order varies,
//     k_refsort sorts it).
#define PAIR_TPW 8
#define PAIR_WPB 4

__global__ void __launch_bounds__(32 * PAIR_WPB, 3) k_pairs(IfaceParams P) {
    extern __shared__ int pair_q_all[];   // [PAIR_WPB][PAIR_TPW * pcap]
    __shared__ int pair_cnt_all[PAIR_WPB][PAIR_TPW];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int nT = P.nTB;
    const int t0 = (blockIdx.x * PAIR_WPB + wib) * PAIR_TPW;
    const int s = blockIdx.y;
    if (t0 >= nT) return;
    int *q = pair_q_all + wib * PAIR_TPW * P.pcap;
    int *qcnt = pair_cnt_all[wib];
    const int qcap = PAIR_TPW * P.pcap;
    const double ox = P.step_sc[4 * s + 0], oy = P.step_sc[4 * s + 1];
    const BinGrid &G = P.binA;
    const int64_t gid0 = (int64_t)s * nT;          // stock triangles of this scenario
    int32_t *rcnt = P.pcnt + (int64_t)s * P.nTA;   // reference counts of its rail triangles
    int32_t *refs = P.refs + (int64_t)s * P.nTA * P.pcap;

    // lane j < PAIR_TPW: query box of stock triangle t0 + j in the rail frame
    double qlx_l = 1.0, qhx_l = 0.0, qly_l = 1.0, qhy_l = 0.0;
    if (lane < PAIR_TPW && t0 + lane < nT) {
        const int4 T = P.triB[t0 + lane];
        const int tv[3] = {T.x, T.y, T.z};
        double lox = 1e300, loy = 1e300, hix = -1e300, hiy = -1e300;
        for (int v = 0; v < 3; ++v) {
            const double2 u = P.uv[tv[v]];
            const double px = u.x + ox, py = u.y + oy;
            lox = fmin(lox, px); hix = fmax(hix, px);
            loy = fmin(loy, py); hiy = fmax(hiy, py);
        }
        qlx_l = lox; qhx_l = hix; qly_l = loy; qhy_l = hiy;
        if (qlx_l > G.hx || qhx_l < G.lx || qly_l > G.hy || qhy_l < G.ly) {   // off the rail top
            qlx_l = 1.0; qhx_l = 0.0;
        }
    }
    // ---- 1. candidates -> queue
    int qn = 0;
    bool ok = true;
    for (int j = 0; j < PAIR_TPW; ++j) {
        const double qlx = __shfl_sync(0xffffffffu, qlx_l, j), qhx = __shfl_sync(0xffffffffu, qhx_l, j);
        const double qly = __shfl_sync(0xffffffffu, qly_l, j), qhy = __shfl_sync(0xffffffffu, qhy_l, j);
        if (lane == 0) qcnt[j] = 0;
        if (!(qlx <= qhx)) continue;   // no triangle / no candidate
        const int bx0 = bin_coord(qlx, G.x0, G.inv_h, G.nx), bx1 = bin_coord(qhx, G.x0, G.inv_h, G.nx);
        const int by0 = bin_coord(qly, G.y0, G.inv_h, G.ny), by1 = bin_coord(qhy, G.y0, G.inv_h, G.ny);
        const int nbx = bx1 - bx0 + 1, nbins = nbx * (by1 - by0 + 1);
        for (int b0 = 0; b0 < nbins; b0 += 32) {   // up to 32 bins per round
            const int bl = b0 + lane;
            int bin = -1, cnt = 0;
            if (bl < nbins) {
                bin = (by0 + bl / nbx) * G.nx + bx0 + bl % nbx;
                cnt = G.ptr[bin + 1] - G.ptr[bin];
            }
            const int off = warp_excl_scan(cnt, lane);
            const int total = __shfl_sync(0xffffffffu, off + cnt, 31);
            for (int base = 0; base < total; base += 32) {
                const int idx = base + lane;
                int qq = 0;   // bin slot holding candidate idx (every lane takes part in the shuffles)
                for (int l = 1; l < 32; ++l) {
                    const int ol = __shfl_sync(0xffffffffu, off, l);
                    if (l < nbins - b0 && ol <= idx) qq = l;
                }
                const int binq = __shfl_sync(0xffffffffu, bin, qq);
                const int offq = __shfl_sync(0xffffffffu, off, qq);
                bool cand = false;
                int u = -1;
                if (idx < total) {
                    u = G.ids[G.ptr[binq] + (idx - offq)];
                    const double4 ub = P.boxA[u];
                    const int bx = bx0 + (b0 + qq) % nbx, by = by0 + (b0 + qq) / nbx;
                    cand = !(ub.x > qhx || ub.z < qlx || ub.y > qhy || ub.w < qly) &&
                           bin_coord(fmax(qlx, ub.x), G.x0, G.inv_h, G.nx) == bx &&
                           bin_coord(fmax(qly, ub.y), G.y0, G.inv_h, G.ny) == by;
                }
                const unsigned m = __ballot_sync(0xffffffffu, cand);
                if (cand) {
                    const int pos = qn + __popc(m & lt);
                    if (pos < qcap) q[pos] = (u << 3) | j; else ok = false;
                }
                qn += __popc(m);
            }
        }
    }
    __syncwarp();
    // ---- 2. integrals, 32 queued pairs per round
    const int nq = min(qn, qcap);
    for (int r0 = 0; r0 < nq; r0 += 32) {
        const int r = r0 + lane;
        const bool valid = r < nq;
        int j = 0, u = 0;
        bool hit = false;
        PairRec rec;
        if (valid) {
            const int e = q[r];
            j = e & 7;
            u = e >> 3;
            const int4 T = P.triB[t0 + j], W = P.triA[u];
            const int tv[3] = {T.x, T.y, T.z}, wv[3] = {W.x, W.y, W.z};
            double2 Gp[3], Fp[3];
            for (int v = 0; v < 3; ++v) {
                const double2 a = P.uv[tv[v]], b = P.uv[wv[v]];
                Gp[v] = make_double2(a.x + ox, a.y + oy);
                Fp[v] = b;
            }
            hit = pair_integrals(Fp, Gp, rec);
        }
        const unsigned hm = __ballot_sync(0xffffffffu, hit);
        const unsigned grp = __match_any_sync(0xffffffffu, valid ? j : 8 + lane);
        if (hit) {
            const int pos = qcnt[j] + __popc(hm & grp & lt);
            if (pos < P.pcap) {
                rec.other = u;
                P.pairs[(gid0 + t0 + j) * P.pcap + pos] = rec;
                const int rp = atomicAdd(&rcnt[u], 1);
                if (rp < P.pcap) refs[(int64_t)u * P.pcap + rp] = (t0 + j) * P.pcap + pos;
                else ok = false;
            } else {
                ok = false;
            }
        }
        __syncwarp();
        if (valid && (grp & lt) == 0) qcnt[j] += __popc(hm & grp);   // group leader
        __syncwarp();
    }
    if (!__all_sync(0xffffffffu, ok) && lane == 0) {
        atomicOr(&P.status[1], 1);
        atomicMin(&P.status[4], P.step + (P.step_per_slot ? (int)blockIdx.y : 0));
    }
    if (lane < PAIR_TPW && t0 + lane < nT) P.pcnt[(int64_t)P.S * P.nTA + gid0 + t0 + lane] = min(qcnt[lane], P.pcap);
}

// Thread per (rail-top triangle F, scenario s): sort F's references ascending (insertion sort,
// <= pcap entries), so that k_rows reads them in an order independent of the atomics' timing.
__global__ void k_refsort(IfaceParams P) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P.nTA) return;
    const int64_t tid = (int64_t)blockIdx.y * P.nTA + t;
    int n = P.pcnt[tid];
    if (n <= 1) return;
    n = min(n, P.pcap);
    P.pcnt[tid] = n;
    int32_t *r = P.refs + tid * P.pcap;
    int v[64];
    if (n > 64) return;   // pcap > 64 is refused at setup
    for (int i = 0; i < n; ++i) v[i] = r[i];
    for (int i = 1; i < n; ++i) {
        const int x = v[i];
        int k = i - 1;
        while (k >= 0 && v[k] > x) {
            v[k + 1] = v[k];
            --k;
        }
        v[k + 1] = x;
    }
    for (int i = 0; i < n; ++i) r[i] = v[i];
}

// ------------------------------------------------------------------------------ K2b: rows

// Warp per (interface node k, scenario s).  The node's contributions (6 per pair record of
// its star: own columns b=0..2, other b=0..2) are streamed in a fixed order -- rounds of 32
// records, then q = 0..5, then lane -- and merged into a shared-memory row:
//  - a column gets its slot on first appearance (new keys ranked by lane within the round),
//    found again through a small shared-memory hash table;
//  - contributions to one slot inside a round are summed in lane order by the group leader,
//    then added to the slot.
// Every floating-point sum therefore runs in a fixed order: deterministic, no FP atomics.
#define ROW_HS 256   // hash table size per warp (power of two, >= 2 x capacity)
#define ROW_WPB 4    // warps per block

struct RowSmem {
    int hkey[ROW_HS], hslot_[ROW_HS];
    int ucol[ROW_HS / 2];
    double val[ROW_HS / 2];
    double tmp[32];
};

__device__ __forceinline__ int hslot(int key) { return (int)(((unsigned)key * 2654435761u) >> 24) & (ROW_HS - 1); }

__global__ void __launch_bounds__(32 * ROW_WPB) k_rows(IfaceParams P) {
    __shared__ RowSmem sm_all[ROW_WPB];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int k = blockIdx.x * ROW_WPB + wib;
    const int s = blockIdx.y;
    if (k >= P.n_if) return;
    RowSmem &W = sm_all[wib];
    const bool sideA = k < P.nA;
    const int nT = sideA ? P.nTA : P.nTB;
    const int64_t base_cnt = sideA ? 0 : (int64_t)P.nTA * P.S;   // pcnt: rail refs | stock records
    const int4 *own_tri = sideA ? P.triA : P.triB;
    const int4 *oth_tri = sideA ? P.triB : P.triA;
    const int32_t row = P.if_rows[k];
    const double scale = P.dt * P.alpha;
    const int st0 = P.star_ptr[k], nstar = P.star_ptr[k + 1] - st0;   // <= 32 (checked at setup)
    const unsigned lt = (1u << lane) - 1u;
    int t_l = 0, np_l = 0, a_l = 0, so_l = 0;
    if (lane < nstar) {
        t_l = P.star_tri[st0 + lane];
        so_l = P.star_own[st0 + lane];
        const int4 T = own_tri[t_l];
        a_l = (T.x == k) ? 0 : ((T.y == k) ? 1 : 2);
        np_l = P.pcnt[base_cnt + (int64_t)s * nT + t_l];
    }
    const int roff = warp_excl_scan(np_l, lane);
    const int R = __shfl_sync(0xffffffffu, roff + np_l, 31);
    // slots [0, n_own): the node's own-surface columns (its star vertices, ascending), fixed;
    // the other surface's columns get the following slots in order of first appearance
    const int o0 = P.own_ptr[k], n_own = R > 0 ? P.own_ptr[k + 1] - o0 : 0;
    if (R > 0) {   // rows without overlap (most of the rail top) skip all of this
        for (int h = lane; h < ROW_HS; h += 32) W.hkey[h] = -1;
        for (int u = lane; u < n_own; u += 32) {
            W.ucol[u] = P.if_rows[P.own_idx[o0 + u]];
            W.val[u] = 0.0;
        }
        __syncwarp();
    }
    int count = n_own;
    bool ok = true;
    double phi = 0.0;
    for (int r0 = 0; r0 < R; r0 += 32) {
        const int r = r0 + lane;
        int q = 0;
        for (int l = 1; l < 32; ++l) {
            const int ol = __shfl_sync(0xffffffffu, roff, l);
            if (l < nstar && ol <= r) q = l;
        }
        const int tq = __shfl_sync(0xffffffffu, t_l, q);
        const int aq = __shfl_sync(0xffffffffu, a_l, q);
        const int oq = __shfl_sync(0xffffffffu, roff, q);
        const int soq = __shfl_sync(0xffffffffu, so_l, q);
        const bool valid = r < R;
        int cc[6];
        double cv[6];
        if (valid) {
            // rail rows reach their pairs through the sorted references, stock rows directly
            int64_t ridx;
            int oth;
            if (sideA) {
                const int key = P.refs[((int64_t)s * P.nTA + tq) * P.pcap + (r - oq)];
                ridx = (int64_t)s * P.nTB * P.pcap + key;
                oth = key / P.pcap;
            } else {
                ridx = ((int64_t)s * P.nTB + tq) * P.pcap + (r - oq);
                oth = P.pairs[ridx].other;
            }
            const PairRec &rec = P.pairs[ridx];
            const int4 Tq = own_tri[tq];
            const int4 Wq = oth_tri[oth];
            const int sym[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
            const int tv[3] = {Tq.x, Tq.y, Tq.z}, wv[3] = {Wq.x, Wq.y, Wq.z};
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                cc[b] = P.if_rows[tv[b]];
                cv[b] = scale * (sideA ? rec.ownF[sym[aq][b]] : rec.ownG[sym[aq][b]]);   // -dt * (-alpha int phi phi)
                cc[3 + b] = P.if_rows[wv[b]];
                cv[3 + b] = -scale * (sideA ? rec.cross[aq * 3 + b] : rec.cross[b * 3 + aq]);   // -dt * (+alpha ...)
            }
            phi += sideA ? rec.bF[aq] : rec.bG[aq];
        }
#pragma unroll
        for (int qq = 0; qq < 6; ++qq) {
            const int key = valid ? cc[qq] : -1;
            int slot = -1;
            if (qq < 3) {   // own-surface column: its slot is known
                slot = valid ? (soq >> (8 * qq)) & 255 : -1;
            } else if (valid) {   // other surface: existing slot?
                int h = hslot(key);
                for (int pr = 0; pr < ROW_HS; ++pr) {
                    const int kk = W.hkey[h];
                    if (kk == key) { slot = W.hslot_[h]; break; }
                    if (kk == -1) break;
                    h = (h + 1) & (ROW_HS - 1);
                }
            }
            // new keys: one leader per distinct key, slots by leader lane order
            const bool isnew = qq >= 3 && valid && slot < 0;
            const unsigned grp = __match_any_sync(0xffffffffu, isnew ? key : (valid ? -2 : -3 - lane));
            const bool leader_new = isnew && (grp & lt) == 0;
            const unsigned lm = __ballot_sync(0xffffffffu, leader_new);
            if (leader_new) {
                slot = count + __popc(lm & lt);
                if (slot < ROW_HS / 2) {
                    W.ucol[slot] = key;
                    W.val[slot] = 0.0;
                    int h = hslot(key);
                    for (int pr = 0; pr < ROW_HS; ++pr) {
                        if (atomicCAS(&W.hkey[h], -1, key) == -1) { W.hslot_[h] = slot; break; }
                        h = (h + 1) & (ROW_HS - 1);
                    }
                }
            }
            count += __popc(lm);
            if (isnew) slot = __shfl_sync(grp, slot, __ffs(grp) - 1);
            __syncwarp();
            // sum per slot in lane order, leader adds to the row
            W.tmp[lane] = valid ? cv[qq] : 0.0;
            __syncwarp();
            const unsigned g2 = __match_any_sync(0xffffffffu, valid ? slot : -3 - lane);
            if (valid && (g2 & lt) == 0 && slot < ROW_HS / 2) {
                double acc = 0.0;
                for (unsigned m = g2; m; m &= m - 1) acc += W.tmp[__ffs(m) - 1];
                W.val[slot] += acc;
            }
            __syncwarp();
        }
    }
    phi = warp_sum(phi);
    if (count > P.cap || count > ROW_HS / 2) ok = false;
    double dself = 0.0;
    if (ok) {
        for (int u = lane; u < count; u += 32) {
            const int64_t idx = ell_index(P, s, u, k);
            P.ell_col[idx] = W.ucol[u];
            P.ell_val[idx] = W.val[u];
            if (W.ucol[u] == row) dself = W.val[u];
        }
    }
    dself = warp_sum(dself);   // exactly one lane holds the diagonal (others add 0)
    if (lane == 0) {
        if (!ok) {
            atomicOr(&P.status[1], 1);
            atomicMin(&P.status[4], P.step + (P.step_per_slot ? s : 0));
        }
        P.ell_cnt[row_index(P, s, k)] = ok ? count : 0;
        P.if_phi[row_index(P, s, k)] = phi;
        P.if_b[row_index(P, s, k)] = 0.5 * P.step_sc[4 * s + 2] * phi;
        const double dinv = 1.0 / (P.Dvol[row] + dself);
        if (P.no_dinv) {
        } else if (P.S == 1) {
            P.Dinv[row] = dinv;
        } else {
            if (P.DinvS) P.DinvS[(int64_t)row * P.SP + s] = dinv;   // gather kernel (cg_batched.cu)
            if (P.if_d) {                                           // windowed SpMM kernel (cg_spmm.cu)
                P.if_dinv[row_index(P, s, k)] = dinv;
                P.if_d[row_index(P, s, k)] = P.Dvol[row] + dself;
            }
        }
    }
}

// Conservative count of overlapping-candidate triangles of the other surface for each
// triangle of `side` at offset o (boxes padded by pad).
__global__ void k_tri_count(IfaceParams P, int side, const double2 *offs, double pad, int *maxcnt) {
    const int nT = side == 0 ? P.nTA : P.nTB;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nT) return;
    const double2 o = offs[blockIdx.y];
    const double4 b = (side == 0 ? P.boxA : P.boxB)[t];
    const double4 *oth_box = side == 0 ? P.boxB : P.boxA;
    const BinGrid &G = side == 0 ? P.binB : P.binA;
    const double sx = side == 0 ? -o.x : o.x, sy = side == 0 ? -o.y : o.y;
    const double lx = b.x + sx - pad, hx = b.z + sx + pad, ly = b.y + sy - pad, hy = b.w + sy + pad;
    const int bx0 = bin_coord(lx, G.x0, G.inv_h, G.nx), bx1 = bin_coord(hx, G.x0, G.inv_h, G.nx);
    const int by0 = bin_coord(ly, G.y0, G.inv_h, G.ny), by1 = bin_coord(hy, G.y0, G.inv_h, G.ny);
    int n = 0;
    for (int by = by0; by <= by1; ++by)
        for (int bx = bx0; bx <= bx1; ++bx) {
            const int bin = by * G.nx + bx;
            for (int m = G.ptr[bin]; m < G.ptr[bin + 1]; ++m) {
                const double4 ub = oth_box[G.ids[m]];
                if (ub.x > hx || ub.z < lx || ub.y > hy || ub.w < ly) continue;
                if (bin_coord(fmax(lx, ub.x), G.x0, G.inv_h, G.nx) != bx ||
                    bin_coord(fmax(ly, ub.y), G.y0, G.inv_h, G.ny) != by) continue;
                ++n;
            }
        }
    atomicMax(maxcnt, n);
}

// Conservative count of the interface entries of row k for an offset o (expanded by pad):
// distinct own-star nodes + distinct nodes of other-surface triangles whose box overlaps.
__global__ void k_iface_count(IfaceParams P, const double2 *offs, double pad, int *maxcnt) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= P.n_if) return;
    const double2 o = offs[blockIdx.y];
    const bool sideA = k < P.nA;
    const int4 *own_tri = sideA ? P.triA : P.triB;
    const int4 *oth_tri = sideA ? P.triB : P.triA;
    const double4 *oth_box = sideA ? P.boxB : P.boxA;
    const BinGrid &G = sideA ? P.binB : P.binA;
    const double sx = sideA ? -o.x : o.x, sy = sideA ? -o.y : o.y;   // own frame -> other frame
    int ids[512];
    int n = 0;
    bool over = false;
    auto add = [&](int v) {
        for (int q = 0; q < n; ++q) if (ids[q] == v) return;
        if (n < 512) ids[n++] = v; else over = true;
    };
    for (int st = P.star_ptr[k]; st < P.star_ptr[k + 1]; ++st) {
        const int4 t = own_tri[P.star_tri[st]];
        add(t.x); add(t.y); add(t.z);
        double lox = 1e300, loy = 1e300, hix = -1e300, hiy = -1e300;
        const int tv[3] = {t.x, t.y, t.z};
        for (int v = 0; v < 3; ++v) {
            double2 u = P.uv[tv[v]];
            lox = fmin(lox, u.x + sx); hix = fmax(hix, u.x + sx);
            loy = fmin(loy, u.y + sy); hiy = fmax(hiy, u.y + sy);
        }
        lox -= pad; loy -= pad; hix += pad; hiy += pad;
        const int bx0 = bin_coord(lox, G.x0, G.inv_h, G.nx), bx1 = bin_coord(hix, G.x0, G.inv_h, G.nx);
        const int by0 = bin_coord(loy, G.y0, G.inv_h, G.ny), by1 = bin_coord(hiy, G.y0, G.inv_h, G.ny);
        for (int by = by0; by <= by1; ++by)
            for (int bx = bx0; bx <= bx1; ++bx) {
                const int bin = by * G.nx + bx;
                for (int m = G.ptr[bin]; m < G.ptr[bin + 1]; ++m) {
                    const double4 ub = oth_box[G.ids[m]];
                    if (ub.x > hix || ub.z < lox || ub.y > hiy || ub.w < loy) continue;
                    const int4 w = oth_tri[G.ids[m]];
                    add(w.x); add(w.y); add(w.z);
                }
            }
    }
    atomicMax(maxcnt, over ? (1 << 30) : n);
}

// ------------------------------------------------------------------------------ host

static void make_bins(const std::vector<double4> &box, std::vector<int32_t> &ptr, std::vector<int32_t> &ids,
                      BinGrid &g) {
    double lx = 1e300, ly = 1e300, hx = -1e300, hy = -1e300, area = 0.0;
    for (auto &b : box) {
        lx = std::min(lx, b.x); ly = std::min(ly, b.y);
        hx = std::max(hx, b.z); hy = std::max(hy, b.w);
        area += (b.z - b.x) * (b.w - b.y);
    }
    int nt = (int)box.size();
    double h = nt ? std::sqrt(std::max(area, 1e-300) / nt) : 1.0;
    if (!(h > 0)) h = 1.0;
    int nx = std::max(1, std::min(4096, (int)std::ceil((hx - lx) / h)));
    int ny = std::max(1, std::min(4096, (int)std::ceil((hy - ly) / h)));
    h = std::max((hx - lx) / nx, (hy - ly) / ny);
    if (!(h > 0)) h = 1.0;
    g.x0 = nt ? lx : 0.0;
    g.y0 = nt ? ly : 0.0;
    g.lx = lx; g.ly = ly; g.hx = hx; g.hy = hy;
    g.inv_h = 1.0 / h;
    g.nx = nx;
    g.ny = ny;
    auto bc = [&](double v, double v0, int n) {
        int b = (int)std::floor((v - v0) * g.inv_h);
        return b < 0 ? 0 : (b >= n ? n - 1 : b);
    };
    std::vector<int32_t> cnt((size_t)nx * ny + 1, 0);
    for (int t = 0; t < nt; ++t)
        for (int by = bc(box[t].y, g.y0, ny); by <= bc(box[t].w, g.y0, ny); ++by)
            for (int bx = bc(box[t].x, g.x0, nx); bx <= bc(box[t].z, g.x0, nx); ++bx) cnt[by * nx + bx + 1]++;
    for (size_t i = 1; i < cnt.size(); ++i) cnt[i] += cnt[i - 1];
    ptr = cnt;
    ids.assign(cnt.back() + 1, 0);
    std::vector<int32_t> pos(cnt.begin(), cnt.end() - 1);
    for (int t = 0; t < nt; ++t)   // ascending t -> ascending ids within each bin
        for (int by = bc(box[t].y, g.y0, ny); by <= bc(box[t].w, g.y0, ny); ++by)
            for (int bx = bc(box[t].x, g.x0, nx); bx <= bc(box[t].z, g.x0, nx); ++bx) ids[pos[by * nx + bx]++] = t;
}

template <class T>
static int upload(Ctx &c, T **d, const std::vector<T> &h) {
    CK(cudaMalloc(d, sizeof(T) * (h.size() + 1)));
    if (!h.empty()) CK(cudaMemcpyAsync(*d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, c.stream));
    return 0;
}

int iface_setup(Ctx &c, const double *X, const std::vector<int32_t> &fA, const std::vector<int32_t> &fB) {
    const int nTA = (int)(fA.size() / 3), nTB = (int)(fB.size() / 3);
    c.nTA = nTA;
    c.nTB = nTB;
    // slice -> interface-row range map (needed even without an interface)
    std::vector<int32_t> rows;
    {
        std::vector<int32_t> ra(fA), rb(fB);
        std::sort(ra.begin(), ra.end());
        ra.erase(std::unique(ra.begin(), ra.end()), ra.end());
        std::sort(rb.begin(), rb.end());
        rb.erase(std::unique(rb.begin(), rb.end()), rb.end());
        for (int32_t r : ra) if (r >= c.nf) { c.err = "interface face of part 0 references a part-1 node"; return -1; }
        for (int32_t r : rb) if (r < c.nf) { c.err = "interface face of part 1 references a part-0 node"; return -1; }
        c.nA = (int)ra.size();
        rows = ra;
        rows.insert(rows.end(), rb.begin(), rb.end());
    }
    c.n_if = (int)rows.size();
    std::vector<int32_t> slice_if(c.nslices + 1);
    for (int64_t s = 0; s <= c.nslices; ++s)
        slice_if[s] = (int32_t)(std::lower_bound(rows.begin(), rows.end(), (int32_t)std::min<int64_t>(32 * s, INT32_MAX)) - rows.begin());
    if (int rc = upload(c, &c.d_slice_if, slice_if)) return rc;
    {
        std::vector<int32_t> zeros(c.nslices + 1, 0);
        if (int rc = upload(c, &c.d_slice_if_zero, zeros)) return rc;
    }
    if (c.n_if == 0) return 0;
    if (nTA == 0 || nTB == 0) { c.err = "interface tag present on only one part"; return -1; }

    // plane of the first rail-top face, in-plane orthonormal basis (e1, e2)
    const double *p0 = X + 3 * (int64_t)fA[0], *p1 = X + 3 * (int64_t)fA[1], *p2 = X + 3 * (int64_t)fA[2];
    double u[3], w[3], n[3];
    for (int d = 0; d < 3; ++d) { u[d] = p1[d] - p0[d]; w[d] = p2[d] - p0[d]; }
    n[0] = u[1] * w[2] - u[2] * w[1];
    n[1] = u[2] * w[0] - u[0] * w[2];
    n[2] = u[0] * w[1] - u[1] * w[0];
    double ln = std::sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
    if (!(ln > 0)) { c.err = "degenerate interface face"; return -1; }
    for (int d = 0; d < 3; ++d) n[d] /= ln;
    int ax = 0;
    for (int d = 1; d < 3; ++d) if (std::fabs(n[d]) < std::fabs(n[ax])) ax = d;
    double e1[3] = {0, 0, 0};
    e1[ax] = 1.0;
    double dn = e1[0] * n[0] + e1[1] * n[1] + e1[2] * n[2];
    for (int d = 0; d < 3; ++d) e1[d] -= dn * n[d];
    double l1 = std::sqrt(e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2]);
    for (int d = 0; d < 3; ++d) e1[d] /= l1;
    double e2[3] = {n[1] * e1[2] - n[2] * e1[1], n[2] * e1[0] - n[0] * e1[2], n[0] * e1[1] - n[1] * e1[0]};
    memcpy(c.plane_n, n, sizeof n);
    memcpy(c.e1, e1, sizeof e1);
    memcpy(c.e2, e2, sizeof e2);

    // interface nodes: coordinates, coplanarity
    std::vector<int32_t> kmap;   // global row -> k, via binary search on `rows`
    auto kof = [&](int32_t r) { return (int32_t)(std::lower_bound(rows.begin(), rows.end(), r) - rows.begin()); };
    std::vector<double2> uv(c.n_if);
    double diam = 0.0;
    for (int k = 0; k < c.n_if; ++k) {
        const double *x = X + 3 * (int64_t)rows[k];
        double d[3] = {x[0] - p0[0], x[1] - p0[1], x[2] - p0[2]};
        uv[k] = make_double2(d[0] * e1[0] + d[1] * e1[1] + d[2] * e1[2], d[0] * e2[0] + d[1] * e2[1] + d[2] * e2[2]);
        diam = std::max(diam, std::fabs(uv[k].x) + std::fabs(uv[k].y));
    }
    for (int k = 0; k < c.n_if; ++k) {
        const double *x = X + 3 * (int64_t)rows[k];
        double dist = (x[0] - p0[0]) * n[0] + (x[1] - p0[1]) * n[1] + (x[2] - p0[2]) * n[2];
        if (std::fabs(dist) > 1e-9 * std::max(1.0, diam)) { c.err = "interface faces are not coplanar"; return -1; }
    }
    // triangles (counter-clockwise in (e1, e2)), boxes, stars, min edge
    auto mk = [&](const std::vector<int32_t> &f, int nt, std::vector<int4> &tri, std::vector<double4> &box) -> int {
        tri.resize(nt);
        box.resize(nt);
        for (int t = 0; t < nt; ++t) {
            int k0 = kof(f[3 * t]), k1 = kof(f[3 * t + 1]), k2 = kof(f[3 * t + 2]);
            double ar = (uv[k1].x - uv[k0].x) * (uv[k2].y - uv[k0].y) - (uv[k1].y - uv[k0].y) * (uv[k2].x - uv[k0].x);
            if (ar == 0.0) { c.err = "degenerate interface triangle"; return -1; }
            if (ar < 0) std::swap(k1, k2);
            tri[t] = make_int4(k0, k1, k2, 0);
            int kk[3] = {k0, k1, k2};
            double4 b = make_double4(1e300, 1e300, -1e300, -1e300);
            for (int v = 0; v < 3; ++v) {
                b.x = std::min(b.x, uv[kk[v]].x); b.y = std::min(b.y, uv[kk[v]].y);
                b.z = std::max(b.z, uv[kk[v]].x); b.w = std::max(b.w, uv[kk[v]].y);
                double2 q = uv[kk[(v + 1) % 3]];
                double le = std::hypot(q.x - uv[kk[v]].x, q.y - uv[kk[v]].y);
                if (c.min_edge == 0.0 || le < c.min_edge) c.min_edge = le;
            }
            box[t] = b;
        }
        return 0;
    };
    std::vector<int4> triA, triB;
    std::vector<double4> boxA, boxB;
    if (mk(fA, nTA, triA, boxA) || mk(fB, nTB, triB, boxB)) return -1;
    std::vector<int32_t> sptr(c.n_if + 1, 0), stri;
    for (auto &t : triA) { sptr[t.x + 1]++; sptr[t.y + 1]++; sptr[t.z + 1]++; }
    for (auto &t : triB) { sptr[t.x + 1]++; sptr[t.y + 1]++; sptr[t.z + 1]++; }
    for (int k = 0; k < c.n_if; ++k) sptr[k + 1] += sptr[k];
    stri.assign(sptr[c.n_if] + 1, 0);
    {
        std::vector<int32_t> pos(sptr.begin(), sptr.end() - 1);
        for (int t = 0; t < nTA; ++t) { stri[pos[triA[t].x]++] = t; stri[pos[triA[t].y]++] = t; stri[pos[triA[t].z]++] = t; }
        for (int t = 0; t < nTB; ++t) { stri[pos[triB[t].x]++] = t; stri[pos[triB[t].y]++] = t; stri[pos[triB[t].z]++] = t; }
    }
    // own-column lists of the rows: the sorted star vertices of every node, and per star entry
    // the slots of its triangle's three vertices in that list (k_rows adds these without hashing)
    std::vector<int32_t> optr(c.n_if + 1, 0), oidx, sown(stri.size(), 0);
    {
        std::vector<int32_t> verts;
        for (int k = 0; k < c.n_if; ++k) {
            verts.clear();
            const bool sa = k < c.nA;
            for (int e = sptr[k]; e < sptr[k + 1]; ++e) {
                const int4 t = sa ? triA[stri[e]] : triB[stri[e]];
                verts.push_back(t.x); verts.push_back(t.y); verts.push_back(t.z);
            }
            std::sort(verts.begin(), verts.end());
            verts.erase(std::unique(verts.begin(), verts.end()), verts.end());
            if (verts.size() > 255) { c.err = "interface node with more than 255 star vertices"; return -1; }
            optr[k + 1] = optr[k] + (int32_t)verts.size();
            oidx.insert(oidx.end(), verts.begin(), verts.end());
            for (int e = sptr[k]; e < sptr[k + 1]; ++e) {
                const int4 t = sa ? triA[stri[e]] : triB[stri[e]];
                const int tv[3] = {t.x, t.y, t.z};
                int packed = 0;
                for (int b = 0; b < 3; ++b) {
                    const int pos = (int)(std::lower_bound(verts.begin(), verts.end(), tv[b]) - verts.begin());
                    packed |= pos << (8 * b);
                }
                sown[e] = packed;
            }
        }
    }
    std::vector<int32_t> bAp, bAi, bBp, bBi;
    make_bins(boxA, bAp, bAi, c.binA);
    make_bins(boxB, bBp, bBi, c.binB);
    if (upload(c, &c.d_if_rows, rows) || upload(c, &c.d_uv, uv) || upload(c, &c.d_star_ptr, sptr) ||
        upload(c, &c.d_star_tri, stri) || upload(c, &c.d_star_own, sown) || upload(c, &c.d_own_ptr, optr) ||
        upload(c, &c.d_own_idx, oidx) || upload(c, &c.d_triA, triA) || upload(c, &c.d_triB, triB) ||
        upload(c, &c.d_boxA, boxA) || upload(c, &c.d_boxB, boxB) || upload(c, &c.d_binA_ptr, bAp) ||
        upload(c, &c.d_binA_ids, bAi) || upload(c, &c.d_binB_ptr, bBp) || upload(c, &c.d_binB_ids, bBi))
        return -3;
    c.binA.ptr = c.d_binA_ptr; c.binA.ids = c.d_binA_ids;
    c.binB.ptr = c.d_binB_ptr; c.binB.ids = c.d_binB_ids;

    // in-plane motion of every scenario; the offset must stay in the plane
    for (auto &sc : c.scen) {
        double dnn = sc.dir[0] * n[0] + sc.dir[1] * n[1] + sc.dir[2] * n[2];
        double dl = std::fabs(sc.dir[0]) + std::fabs(sc.dir[1]) + std::fabs(sc.dir[2]);
        if (std::fabs(dnn) > 1e-12 * std::max(1.0, dl)) { c.err = "motion direction leaves the interface plane"; return -1; }
        sc.d2[0] = sc.dir[0] * e1[0] + sc.dir[1] * e1[1] + sc.dir[2] * e1[2];
        sc.d2[1] = sc.dir[0] * e2[0] + sc.dir[1] * e2[1] + sc.dir[2] * e2[2];
    }

    // capacity: sweep every scenario's motion range [s0 - |amp|, s0 + |amp|] in steps of
    // min_edge / 2 with boxes padded by the step (conservative superset at any offset)
    const double step = 0.5 * c.min_edge;
    std::vector<double2> offs;
    for (auto &sc : c.scen) {
        double lo = sc.s0 - std::fabs(sc.amp), hi = sc.s0 + std::fabs(sc.amp);
        int64_t ns = std::min<int64_t>(200000, (int64_t)std::ceil((hi - lo) / step) + 1);
        for (int64_t i = 0; i < ns; ++i) {
            double s = ns == 1 ? lo : lo + (hi - lo) * (double)i / (double)(ns - 1);
            double2 o = make_double2(s * sc.d2[0], s * sc.d2[1]);
            bool dup = false;
            for (size_t q = offs.size() > 64 ? offs.size() - 64 : 0; q < offs.size(); ++q)
                if (offs[q].x == o.x && offs[q].y == o.y) { dup = true; break; }
            if (!dup) offs.push_back(o);
        }
    }
    if (offs.size() > 400000) offs.resize(400000);
    double2 *d_offs = nullptr;
    int *d_max = nullptr;
    if (upload(c, &d_offs, offs)) return -3;
    CK(cudaMalloc(&d_max, sizeof(int)));
    CK(cudaMemsetAsync(d_max, 0, sizeof(int), c.stream));
    IfaceParams P;
    memset(&P, 0, sizeof P);
    iface_params(c, P, nullptr, 0.0);
    for (size_t b0 = 0; b0 < offs.size(); b0 += 60000) {
        unsigned ny = (unsigned)std::min<size_t>(60000, offs.size() - b0);
        dim3 grid((unsigned)((c.n_if + 127) / 128), ny);
        k_iface_count<<<grid, 128, 0, c.stream>>>(P, d_offs + b0, step, d_max);
        CK(cudaGetLastError());
    }
    int *d_pmax = nullptr;
    CK(cudaMalloc(&d_pmax, sizeof(int)));
    CK(cudaMemsetAsync(d_pmax, 0, sizeof(int), c.stream));
    for (int side = 0; side < 2; ++side) {
        const int nT = side == 0 ? c.nTA : c.nTB;
        for (size_t b0 = 0; b0 < offs.size(); b0 += 60000) {
            unsigned ny = (unsigned)std::min<size_t>(60000, offs.size() - b0);
            dim3 grid((unsigned)((nT + 127) / 128), ny);
            k_tri_count<<<grid, 128, 0, c.stream>>>(P, side, d_offs + b0, step, d_pmax);
            CK(cudaGetLastError());
        }
    }
    int mx = 0, pmx = 0;
    CK(cudaMemcpyAsync(&pmx, d_pmax, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaMemcpyAsync(&mx, d_max, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    cudaFree(d_offs);
    cudaFree(d_max);
    cudaFree(d_pmax);
    if (mx > 2048) { c.err = "interface rows too dense (capacity > 2048)"; return -5; }
    c.cap = ((mx + 4) + 3) / 4 * 4;
    c.pcap = pmx + 2;
    if ((size_t)PAIR_WPB * PAIR_TPW * c.pcap * sizeof(int) > 48 * 1024) {
        c.err = "interface triangles overlap too many triangles of the other surface";
        return -5;
    }
    // contributions per row: 6 per record, records <= star size x pcap
    int max_star = 0;
    for (int k = 0; k < c.n_if; ++k) max_star = std::max(max_star, sptr[k + 1] - sptr[k]);
    if (max_star > 32) { c.err = "interface node with more than 32 surface triangles"; return -1; }
    if (c.cap > ROW_HS / 2) { c.err = "interface rows too dense for the row merge (capacity > 128)"; return -5; }
    c.cmax = 6 * max_star * c.pcap;
    if (c.pcap > 64) { c.err = "interface triangles overlap too many triangles of the other surface (> 62)"; return -5; }
    CK(cudaMalloc(&c.d_pairs, sizeof(PairRec) * (size_t)c.S * c.nTB * c.pcap));
    CK(cudaMalloc(&c.d_refs, sizeof(int32_t) * (size_t)c.S * c.nTA * c.pcap));
    CK(cudaMalloc(&c.d_pcnt, sizeof(int32_t) * (size_t)c.S * (c.nTA + c.nTB)));

    const int64_t S = c.S, nif = c.n_if;
    CK(cudaMalloc(&c.d_ell_cnt, sizeof(int32_t) * S * nif));
    CK(cudaMalloc(&c.d_ell_col, sizeof(int32_t) * S * c.cap * nif));
    CK(cudaMalloc(&c.d_ell_val, sizeof(double) * S * c.cap * nif));
    CK(cudaMalloc(&c.d_if_b, sizeof(double) * S * nif));
    CK(cudaMalloc(&c.d_if_phi, sizeof(double) * S * nif));
    CK(cudaMalloc(&c.d_if_dinv, sizeof(double) * S * nif));
    CK(cudaMemsetAsync(c.d_ell_cnt, 0, sizeof(int32_t) * S * nif, c.stream));
    CK(cudaMemsetAsync(c.d_if_b, 0, sizeof(double) * S * nif, c.stream));
    CK(cudaMemsetAsync(c.d_if_phi, 0, sizeof(double) * S * nif, c.stream));
    return 0;
}

void iface_params(Ctx &c, IfaceParams &P, const double *step_sc, double dt, int buf) {
    P.nTA = c.nTA;
    P.nTB = c.nTB;
    P.pcap = c.pcap;
    P.pairs = c.d_pairs;
    P.pcnt = c.d_pcnt;
    P.refs = c.d_refs;
    P.cmax = c.cmax;
    P.n_if = c.n_if;
    P.nA = c.nA;
    P.S = c.S;
    P.cap = c.cap;
    P.if_rows = c.d_if_rows;
    P.uv = c.d_uv;
    P.star_ptr = c.d_star_ptr;
    P.star_tri = c.d_star_tri;
    P.star_own = c.d_star_own;
    P.own_ptr = c.d_own_ptr;
    P.own_idx = c.d_own_idx;
    P.triA = c.d_triA;
    P.triB = c.d_triB;
    P.boxA = c.d_boxA;
    P.boxB = c.d_boxB;
    P.binA = c.binA;
    P.binB = c.binB;
    P.alpha = c.alpha;
    P.dt = dt;
    P.step_sc = step_sc;
    P.Dvol = c.d_Dvol;
    P.ell_cnt = buf ? c.d_ell_cnt_b : c.d_ell_cnt;
    P.ell_col = buf ? c.d_ell_col_b : c.d_ell_col;
    P.ell_val = buf ? c.d_ell_val_b : c.d_ell_val;
    P.if_b = buf ? c.d_if_b_b : c.d_if_b;
    P.if_phi = buf ? c.d_if_phi_b : c.d_if_phi;
    P.Dinv = buf ? c.d_Dinv_b : c.d_Dinv;
    P.if_dinv = c.d_if_dinv;
    P.if_d = c.sb_on ? c.d_if_d : nullptr;   // per-scenario d, 1/d of the windowed SpMM kernel
    P.DinvS = c.d_DinvS;
    P.SP = c.SP;
    P.status = c.d_status;
}

int iface_launch(Ctx &c, const IfaceParams &P, cudaStream_t stream) {
    if (c.n_if == 0) return 0;
    const int tpb = PAIR_WPB * PAIR_TPW;
    const size_t qsm = sizeof(int) * (size_t)PAIR_WPB * PAIR_TPW * c.pcap;
    cudaStream_t st = stream ? stream : c.stream;
    // blockIdx.y = scenario (batched mode) or node time (the slots of the SDC methods): P.S of them
    CK(cudaMemsetAsync(P.pcnt, 0, sizeof(int32_t) * (size_t)P.S * c.nTA, st));   // rail reference counts
    const int nbB = (c.nTB + tpb - 1) / tpb;
    k_pairs<<<dim3((unsigned)nbB, (unsigned)P.S), 32 * PAIR_WPB, qsm, st>>>(P);
    CK(cudaGetLastError());
    k_refsort<<<dim3((unsigned)((c.nTA + 127) / 128), (unsigned)P.S), 128, 0, st>>>(P);
    CK(cudaGetLastError());
    k_rows<<<dim3((unsigned)((c.n_if + ROW_WPB - 1) / ROW_WPB), (unsigned)P.S), 32 * ROW_WPB, 0, st>>>(P);
    CK(cudaGetLastError());
    return 0;
}

}  // namespace thermo
