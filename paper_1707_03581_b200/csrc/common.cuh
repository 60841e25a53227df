// common.cuh -- shared device helpers and parameter blocks of the thermo library.
// Part of the CUDA product path; never includes anything from oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#ifndef THERMO_BLOCK
#define THERMO_BLOCK 256
#endif
#define THERMO_WARPS (THERMO_BLOCK / 32)
#define THERMO_NRED 24  // reduction slots per CTA (phase 0: 0-3, S: 4-10, fused S of odd iterations: 11-17)

namespace thermo {

// ---------------------------------------------------------------------------------
// memory helpers
// ---------------------------------------------------------------------------------

// L2 eviction policy for data streamed once per sweep (matrix values / columns).
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// Streaming read: non-coherent path, no L1 allocation, L2 evict-first policy.
__device__ __forceinline__ double ld_stream(const double *p, uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int ld_stream(const int *p, uint64_t pol) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

// Coherent load that bypasses L1 (cached in L2 only): streams that are read once per phase
// but written by other CTAs earlier in the same kernel.  Keeps L1 miss slots free when most
// of the shared memory is taken by a TMA ring.
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ double ld_cg1(const double *p) {
    double v;
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

// order this thread's generic-proxy shared-memory accesses before later async-proxy (TMA)
// accesses of the same memory (and vice versa)
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// order this thread's generic-proxy global writes before async-proxy (TMA bulk copy) reads of the
// same memory issued after a later barrier (every grid barrier after which vectors written by
// plain stores are streamed by cp.async.bulk)
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ double2 ld_cg2(const double2 *p) {
    double2 v;
    asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

// ---------------------------------------------------------------------------------
// mbarrier + bulk-copy (TMA engine) helpers
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy on the TMA engine, completion signalled on `bar` (tx bytes)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                         uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s_nohint(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// L2 prefetch of a contiguous range on the TMA engine (16-byte aligned, size % 16 == 0)
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// ---------------------------------------------------------------------------------
// deterministic reductions: xor-butterfly inside a warp (every lane ends with the same
// bits), fixed-order combination across warps and CTAs.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// smem scratch of the reductions: >= 144 doubles (warp partials [0, 32*NV), totals at 136).
#define THERMO_RED_SMEM 160

// Reduce NV values over the CTA and store them to partials[blockIdx.x * THERMO_NRED + slot + j].
template <int NV>
__device__ __forceinline__ void cta_reduce_store(double (&v)[NV], double *smem, double *partials,
                                                 int slot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = warp_sum(v[j]);
    if (lane == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) smem[warp * NV + j] = v[j];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            double x = lane < nwarps ? smem[lane * NV + j] : 0.0;
            x = warp_sum(x);
            if (lane == 0) partials[blockIdx.x * THERMO_NRED + slot + j] = x;
        }
    }
    __syncthreads();
}

// Sum the per-CTA partials of G CTAs (fixed order); every thread of every CTA returns the
// identical value.  Must be called by all threads of the CTA after a grid-wide barrier.
template <int NV>
__device__ __forceinline__ void grid_total(const double *partials, int G, int slot, double *smem,
                                           double (&out)[NV]) {
    // warp w sums value j = w (w + nwarps, ...): lane l takes CTAs l, l + 32, ... with all of its
    // loads in flight together (one L2 round trip for G <= 256), adds them in ascending CTA
    // order, then the xor butterfly -- a fixed order, so every CTA gets the identical bits
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int j = warp; j < NV; j += nw) {
        double x = 0.0;
        int g0 = 0;
        for (; g0 + 32 * 8 <= G; g0 += 32 * 8) {
            double a[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] = ld_cg1(partials + (g0 + 32 * u + lane) * THERMO_NRED + slot + j);
#pragma unroll
            for (int u = 0; u < 8; ++u) x += a[u];
        }
        double a[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int g = g0 + 32 * u + lane;
            // through L2: the partials are rewritten by other CTAs every reduction of the launch, and an
            // L1 line of this SM could still hold the previous reduction's value
            a[u] = g < G ? ld_cg1(partials + g * THERMO_NRED + slot + j) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) x += a[u];
        x = warp_sum(x);
        if (lane == 0) smem[136 + j] = x;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NV; ++j) out[j] = smem[136 + j];
    __syncthreads();
}

// ---------------------------------------------------------------------------------
// parameter blocks
// ---------------------------------------------------------------------------------

struct BinGrid {      // uniform bin grid over one surface triangulation (2-D, own frame)
    double x0, y0, inv_h;
    double lx, ly, hx, hy;   // union box of the surface's triangles
    int nx, ny;
    const int32_t *ptr;   // [nx*ny + 1]
    const int32_t *ids;   // triangle ids, ascending within a bin
};

struct PairRec {       // one overlapping (rail-top F, stock-bottom G) triangle pair, both sides' view
    int other;         // the rail-top triangle F (records are listed under their stock triangle G)
    int pad_;
    double ownF[6];    // int phi_F,a phi_F,b over F cap G, symmetric 3x3 (00 01 02 11 12 22)
    double ownG[6];    // int phi_G,a phi_G,b
    double cross[9];   // int phi_F,a phi_G,b, [a*3 + b]
    double bF[3];      // int phi_F,a
    double bG[3];      // int phi_G,a
};

struct IfaceParams {
    int nTA, nTB;         // rail-top / stock-bottom triangles
    int pcap;             // pair records per triangle
    int cmax;             // contributions per interface row (6 x records of its star)
    PairRec *pairs;       // [S*nTB * pcap] records of each stock-bottom triangle (one per pair)
    int32_t *pcnt;        // [S*nTA + S*nTB]: rail side: refs of each rail-top triangle; stock side: records
    int32_t *refs;        // [S*nTA * pcap] per rail-top triangle: its pairs' record indices g*pcap + slot
                          // (within the scenario), ascending after k_refsort
    int n_if;             // interface rows: [0, nA) rail top (fixed), [nA, n_if) stock bottom
    int nA;
    int S;                // scenarios
    int cap;              // ELL capacity per row
    const int32_t *if_rows;   // [n_if] global row of each interface node
    const double2 *uv;        // [n_if] in-plane coordinates (fixed frame / stock reference frame)
    const int32_t *star_ptr;  // [n_if + 1]
    const int32_t *star_tri;  // own-surface triangles around each node, ascending
    const int32_t *star_own;  // per star entry: the slots of the triangle's 3 vertices in the
                              // node's own-column list (3 x 8 bits)
    const int32_t *own_ptr;   // [n_if + 1] own-column lists (sorted interface-node indices
    const int32_t *own_idx;   //   of the node's star vertices)
    const int4 *triA;         // [nTA] (k0, k1, k2, -) interface-row indices, counter-clockwise
    const int4 *triB;
    const double4 *boxA;      // [nTA] (lo.x, lo.y, hi.x, hi.y)
    const double4 *boxB;
    BinGrid binA, binB;
    double alpha, dt;
    const double *step_sc;    // [S][4] this step: (o.x, o.y, eta, s)
    const double *Dvol;       // [N] volume diagonal of K~
    // outputs, per scenario s: ell_cnt[s*n_if + k], ell_col/val[(s*cap + c)*n_if + k]
    int32_t *ell_cnt;
    int32_t *ell_col;
    double *ell_val;
    double *if_b;             // [S][n_if] dt-free friction source eta/2 int phi
    double *if_phi;           // [S][n_if] int_{Gamma_R} phi
    double *Dinv;             // S == 1: [N] Jacobi inverse diagonal, interface rows rewritten
    double *if_dinv;          // S > 1: [k][s] per-scenario Jacobi inverse diagonal of the interface rows
    double *if_d;             // S > 1: [k][s] per-scenario Jacobi diagonal of the interface rows
    int step;                 // time step of this assembly: an overflow records the first one in
                              // status[4] (the overlap mode assembles one step ahead of the solve)
    double *DinvS;            // S > 1: [N][SP] per-scenario Jacobi inverse diagonal
    int SP;                   // S > 1: row stride of the block vectors (even, >= S)
    int no_dinv;              // 1: leave the Jacobi diagonal alone (MRSDC: f^E is explicit)
    int slot_major;           // 1: batch index = node-time slot, arrays laid out slot by slot
                              // ([s][c][k], [s][k]) so per-slot row loops stay coalesced
    int step_per_slot;        // 1: batch entry s belongs to time step `step + s` (the ahead mode assembles
                              // the interfaces of consecutive steps in one launch set)
    int *status;              // status[1] |= overflow
};

// ELL slot c of interface row k, scenario s.  S == 1: slot-major [c][k] (coalesced across the
// rows of a slice); S > 1: [k][c][s] (coalesced across the scenarios of one row).
// ell_cnt, if_b, if_phi are indexed [k * S + s].
__host__ __device__ __forceinline__ int64_t ell_index(const IfaceParams &P, int s, int c, int k) {
    if (P.slot_major) return ((int64_t)s * P.cap + c) * P.n_if + k;
    return P.S == 1 ? (int64_t)c * P.n_if + k : ((int64_t)k * P.cap + c) * P.S + s;
}
// per-row entries (ell_cnt, if_b, if_phi) of row k, batch index s
__host__ __device__ __forceinline__ int64_t row_index(const IfaceParams &P, int s, int k) {
    return P.slot_major ? (int64_t)s * P.n_if + k : (int64_t)k * P.S + s;
}

}  // namespace thermo
