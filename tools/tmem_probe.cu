// tmem_probe.cu -- diagnostics (not the product): can tensor memory (TMEM) serve the
// apply path's per-level code-word loads off the shared-memory data path?
//
// One CTA per SM (148), W warps.  Each warp reads 32-bit words of its sub-partition's
// 32 TMEM lanes (tcgen05.ld.32x32b.xN, warp-uniform column) or of shared memory (LDS.32,
// conflict-free), K loads per wait, and we report bytes per SM clock.  Mode "mix": even
// warps TMEM, odd warps LDS (do the two paths add up?).  Mode "lat": one warp, dependent
// tcgen05.ld.x1 + wait chain (latency in cycles).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tmem_probe tools/tmem_probe.cu
//   build/tmem_probe
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
extern __shared__ __align__(1024) uint8_t sm[];

template <int N>
__device__ __forceinline__ void ldtm(uint32_t taddr, uint32_t (&r)[N]);
template <>
__device__ __forceinline__ void ldtm<1>(uint32_t taddr, uint32_t (&r)[1])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(taddr));
}
template <>
__device__ __forceinline__ void ldtm<2>(uint32_t taddr, uint32_t (&r)[2])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(taddr));
}
template <>
__device__ __forceinline__ void ldtm<4>(uint32_t taddr, uint32_t (&r)[4])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// mode 0: TMEM xN, mode 1: LDS, mode 2: mix (even warps TMEM x1, odd LDS), mode 3: latency
template <int N, int K>
__global__ void __launch_bounds__(512, 1) probe(int mode, int iters, unsigned long long *cyc, uint32_t *sink)
{
    __shared__ uint32_t taddr_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    uint32_t *s = reinterpret_cast<uint32_t *>(sm);
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) s[i] = i * 2654435761u;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16);
    // fill this warp's lanes, its quarter of the columns (every warp of a sub-partition)
    for (int c = (warp >> 2); c < 512; c += (blockDim.x >> 7)) {
        uint32_t v = c * 131u + lane;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tbase + c), "r"(v));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");

    uint32_t acc = 0;
    unsigned long long t0 = clock64();
    const bool use_tm = mode == 0 || mode == 3 || (mode == 2 && (warp & 1) == 0);
    if (mode == 3) {
        if (warp == 0) {
            uint32_t col = 5;
            for (int it = 0; it < iters; ++it) {
                uint32_t r[1];
                ldtm<1>(tbase + col, r);
                wait_ld();
                col = (__shfl_sync(0xffffffffu, r[0], 0) + it) & 255u;  // dependent, warp-uniform
                acc += r[0];
            }
        }
    } else if (mode >= 4) {  // 4: TMEM x1, 5: LDS, 6: half TMEM + half LDS per warp; fixed addresses
        uint32_t ta[8], la[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            ta[k] = tbase + ((k * 61 + warp * 7) & 511);
            la[k] = sa(sm) + ((((k * 61 + warp * 7) & 511) * 32 + lane) * 4 & 65535);
        }
        for (int it = 0; it < iters; ++it) {
            uint32_t r[8];
            if (mode == 4) {
#pragma unroll
                for (int k = 0; k < 8; ++k) { uint32_t q[1]; ldtm<1>(ta[k], q); r[k] = q[0]; }
                wait_ld();
            } else if (mode == 5) {
#pragma unroll
                for (int k = 0; k < 8; ++k) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r[k]) : "r"(la[k]));
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) { uint32_t q[1]; ldtm<1>(ta[k], q); r[k] = q[0]; }
#pragma unroll
                for (int k = 4; k < 8; ++k) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r[k]) : "r"(la[k]));
                wait_ld();
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) acc += r[k];
        }
    } else if (use_tm) {
        for (int it = 0; it < iters; ++it) {
            uint32_t r[K][N];
#pragma unroll
            for (int k = 0; k < K; ++k) ldtm<N>(tbase + (((it * 37 + k * 61 + warp * 7) * N) & 511), r[k]);
            wait_ld();
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int n = 0; n < N; ++n) acc ^= r[k][n];
        }
    } else {
        for (int it = 0; it < iters; ++it) {
            uint32_t r[K * N];
#pragma unroll
            for (int k = 0; k < K * N; ++k) {
                const uint32_t a = sa(sm) + ((((it * 37 + k * 61 + warp * 7) & 511) * 32 + lane) * 4 & 65535);
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r[k]) : "r"(a));
            }
#pragma unroll
            for (int k = 0; k < K * N; ++k) acc ^= r[k];
        }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

template <int N, int K>
void run(const char *name, int mode, int warps, int iters)
{
    unsigned long long *cyc;
    uint32_t *sink;
    cudaMalloc(&cyc, 148 * 8);
    cudaMalloc(&sink, 148 * 512 * 4);
    cudaFuncSetAttribute(probe<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    fprintf(stderr, "start %s w=%d\n", name, warps);
    probe<N, K><<<148, warps * 32, 160 * 1024>>>(mode, iters, cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < 148; ++i) mean += h[i] / 148.0;
    if (mode == 3) {
        printf("{\"probe\": \"%s\", \"cycles_per_dependent_load\": %.1f}\n", name, mean / iters);
    } else {
        const double bytes = (double)warps * 32 * 4 * N * K * iters;
        printf("{\"probe\": \"%s\", \"warps\": %d, \"bytes_per_clk_per_sm\": %.1f, \"loads_per_clk_per_sm\": %.3f}\n",
               name, warps, bytes / mean, (double)warps * K * iters / mean);
    }
    fflush(stdout);
    cudaFree(cyc);
    cudaFree(sink);
}

int main()
{
    const int it = 4096;
    for (int w : {16}) {
        run<1, 8>("tmem_x1", 0, w, it);
        run<2, 8>("tmem_x2", 0, w, it);
        run<4, 8>("tmem_x4", 0, w, it);
        run<1, 8>("lds_u32", 1, w, it);
        run<1, 8>("mix_tmem_x1_lds", 2, w, it);
    }
    for (int w : {8, 16}) {
        run<1, 8>("fixed_tmem_x1", 4, w, it);
        run<1, 8>("fixed_lds_u32", 5, w, it);
        run<1, 8>("fixed_half_tmem_half_lds", 6, w, it);
    }
    run<1, 16>("tmem_x1_k16", 0, 16, it);
    run<1, 4>("tmem_x1_k4", 0, 16, it);
    run<1, 1>("tmem_x1_k1", 0, 16, it);
    // (a dependent-load latency probe, mode 3, hung the box: left out)
    return 0;
}
