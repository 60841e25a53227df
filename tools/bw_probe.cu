// bw_probe.cu -- attainable HBM bandwidth for the access patterns of the CG kernel phases
// (measurement aid for DESIGN.md section 7.1; not part of the library).
//
//   read_ldg   : every thread streams 16-byte loads (ld.global.nc, L1 no-allocate), sums them
//   read_tma   : the S-phase pattern: one producer warp per CTA bulk-copies (cp.async.bulk)
//                CHUNK-byte pieces into an NS-stage shared-memory ring, 8 consumer warps
//                touch every 8-byte word of a stage and release it
//   copy_ldg   : 16-byte load + store (the MEASURED_PEAKS copy pattern)
//   u_pattern  : 4 streams read, 3 written (the U phase)
//
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bw_probe tools/bw_probe.cu
// ./tools/bw_probe [GB]
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t err_ = (x); if (err_ != cudaSuccess) { printf("CUDA %s at %s\n", cudaGetErrorString(err_), #x); exit(1); } } while (0)

__device__ __forceinline__ double2 ldnc(const double2 *p) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

__global__ void read_ldg(const double2 *a, int64_t n, double *out) {
    double s = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
        double2 v0 = ldnc(a + i), v1 = ldnc(a + i + stride), v2 = ldnc(a + i + 2 * stride), v3 = ldnc(a + i + 3 * stride);
        s += v0.x + v0.y + v1.x + v1.y + v2.x + v2.y + v3.x + v3.y;
    }
    for (; i < n; i += stride) { double2 v = ldnc(a + i); s += v.x + v.y; }
    if (s == 1.2345) out[0] = s;
}

__global__ void copy_ldg(const double2 *a, double2 *b, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) b[i] = ldnc(a + i);
}

__global__ void u_pattern(const double2 *p, const double2 *q, double2 *x, double2 *z, double2 *pw, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        double2 pv = ldnc(p + i), qv = ldnc(q + i), xv = ldnc(x + i), zv = ldnc(z + i);
        x[i] = make_double2(xv.x + 0.5 * pv.x, xv.y + 0.5 * pv.y);
        double2 zn = make_double2(zv.x - 0.5 * qv.x, zv.y - 0.5 * qv.y);
        z[i] = zn;
        pw[i] = make_double2(zn.x + 0.25 * pv.x, zn.y + 0.25 * pv.y);
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t ph) {
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(smem_u32(b)),
                 "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// chunk c of `chunk` bytes goes to CTA c % G (static round robin, as the CG kernel)
__global__ void __launch_bounds__(288, 1) read_tma(const char *a, int64_t nchunks, int chunk, int NS, double *out,
                                                   int ncopies) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *full = (uint64_t *)sm, *empty = full + NS;
    unsigned char *stage = sm + 128;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t n = 0;
    if (warp == 8) {
        if (lane == 0) {
            for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++n) {
                const uint32_t s = n % NS, ph = (n / NS) & 1u;
                mbar_wait(&empty[s], ph ^ 1u);
                mbar_expect(&full[s], (uint32_t)chunk);
                if (ncopies == 1) {
                    bulk(stage + (size_t)s * chunk, a + c * chunk, chunk, &full[s]);
                } else {
                    // values + columns (+ a 2-KB own-row block) of a CG chunk
                    const uint32_t tail = ncopies >= 3 ? 2048u : 0u;
                    const uint32_t a0 = (uint32_t)((chunk - tail) * 4 / 5) & ~15u;
                    bulk(stage + (size_t)s * chunk, a + c * chunk, a0, &full[s]);
                    bulk(stage + (size_t)s * chunk + a0, a + c * chunk + a0, chunk - tail - a0, &full[s]);
                    if (tail) bulk(stage + (size_t)s * chunk + chunk - tail, a + c * chunk + chunk - tail, tail, &full[s]);
                }
            }
        }
        return;
    }
    double acc = 0.0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++n) {
        const uint32_t s = n % NS, ph = (n / NS) & 1u;
        mbar_wait(&full[s], ph);
        const double *v = (const double *)(stage + (size_t)s * chunk);
        for (int k = threadIdx.x; k < chunk / 8; k += 256) acc += v[k];
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 1.2345) out[0] = acc;
}

int main(int argc, char **argv) {
    const double gb = argc > 1 ? atof(argv[1]) : 2.0;
    const int64_t bytes = (int64_t)(gb * 1e9) & ~(int64_t)((1 << 20) - 1);
    char *a, *b, *c, *d, *e;
    double *out;
    CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
    const int64_t vb = bytes / 8;   // U-pattern vectors
    CK(cudaMalloc(&c, vb)); CK(cudaMalloc(&d, vb)); CK(cudaMalloc(&e, vb));
    CK(cudaMalloc(&out, 8));
    CK(cudaMemset(a, 0, bytes)); CK(cudaMemset(b, 0, bytes));
    CK(cudaMemset(c, 0, vb)); CK(cudaMemset(d, 0, vb)); CK(cudaMemset(e, 0, vb));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    auto timeit = [&](auto launch, double moved, const char *name) {
        for (int w = 0; w < 2; ++w) launch();
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int r = 0; r < 10; ++r) {
            CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
            float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
            if (ms < best) best = ms;
        }
        CK(cudaGetLastError());
        printf("%-34s %8.1f GB/s  (%.3f ms, %.2f GB)\n", name, moved / (best * 1e-3) / 1e9, best, moved / 1e9);
    };
    const int64_t n2 = bytes / 16;
    for (int per : {4, 8}) {
        char nm[64]; snprintf(nm, sizeof nm, "read_ldg (%d CTAs/SM x 256)", per);
        timeit([&] { read_ldg<<<sms * per, 256>>>((const double2 *)a, n2, out); }, (double)bytes, nm);
    }
    timeit([&] { copy_ldg<<<sms * 8, 256>>>((const double2 *)a, (double2 *)b, n2); }, 2.0 * bytes, "copy_ldg");
    const int64_t nv = vb / 16;
    timeit([&] { u_pattern<<<sms * 8, 256>>>((const double2 *)a, (const double2 *)b, (double2 *)c, (double2 *)d, (double2 *)e, nv); },
           7.0 * vb, "u_pattern (4 read, 3 written)");
    for (int nc : {1, 2, 3}) for (int chunk : {40960}) for (int NS : {3, 4}) {
        const size_t smem = 128 + (size_t)NS * chunk;
        if (smem > 227 * 1024) continue;
        CK(cudaFuncSetAttribute(read_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const int64_t nch = bytes / chunk;
        char nm[64]; snprintf(nm, sizeof nm, "read_tma %d copies, %d B x %d stages", nc, chunk, NS);
        timeit([&] { read_tma<<<sms, 288, smem>>>(a, nch, chunk, NS, out, nc); }, (double)nch * chunk, nm);
    }
    return 0;
}
