// stream_probe.cu -- diagnostics (not the product): how fast can one persistent
// CTA per SM stream a doc-major fp32 [D x F] matrix through a TMA ring of S slots
// of B boxes (ROWS docs x 32 factors, 128B swizzle) when the consumers do no work?
// This is the factor stream of the fused kernel in isolation.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/stream_probe tools/stream_probe.cu -lcuda
//   build/stream_probe D F S B ROWS
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
extern __shared__ __align__(1024) uint8_t sm[];

__global__ void __launch_bounds__(544, 1) probe(const __grid_constant__ CUtensorMap tm, int n_tiles, int n_sub,
                                                 int S, int B, int rows, float *sink)
{
    const uint32_t box = rows * 128;
    const uint32_t slot = B * box;
    uint32_t bars = S * slot;
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(sm + bars + 16 * s)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 16;" ::"r"(sa(sm + bars + 16 * s + 8)));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int jobs = (n_sub + B - 1) / B;
    if (warp == 16) {
        if (lane) return;
        uint32_t st = 0, ph = 0;
        for (int t = blockIdx.x; t < n_tiles; t += gridDim.x)
            for (int j = 0; j < jobs; ++j) {
                uint32_t full = sa(sm + bars + 16 * st), empty = full + 8;
                asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" ::"r"(empty), "r"(ph ^ 1));
                int nb = min(B, n_sub - j * B);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full), "r"(nb * box));
                for (int b = 0; b < nb; ++b)
                    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                                 ::"r"(sa(sm + st * slot + b * box)), "l"(&tm), "r"((j * B + b) * 32), "r"(t * rows), "r"(full) : "memory");
                if (++st == (uint32_t)S) { st = 0; ph ^= 1; }
            }
        return;
    }
    uint32_t st = 0, ph = 0;
    float acc = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x)
        for (int j = 0; j < jobs; ++j) {
            uint32_t full = sa(sm + bars + 16 * st), empty = full + 8;
            asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" ::"r"(full), "r"(ph) : "memory");
            acc += *(volatile float *)(sm + st * slot + threadIdx.x * 4);
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty) : "memory");
            if (++st == (uint32_t)S) { st = 0; ph ^= 1; }
        }
    if (acc == 12345.f) sink[0] = acc;
}

int main(int argc, char **argv)
{
    long D = atol(argv[1]), F = atol(argv[2]);
    int S = atoi(argv[3]), B = atoi(argv[4]), rows = atoi(argv[5]);
    float *x, *sink;
    cudaMalloc(&x, D * F * 4);
    cudaMalloc(&sink, 4);
    cudaMemset(x, 0, D * F * 4);
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)F, (cuuint64_t)D};
    cuuint64_t str[1] = {(cuuint64_t)F * 4};
    cuuint32_t boxd[2] = {32, (cuuint32_t)rows}, es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims, str, boxd, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode %d\n", r); return 1; }
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    size_t smem = (size_t)S * B * rows * 128 + 16 * S + 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int n_tiles = (D + rows - 1) / rows, n_sub = (F + 31) / 32;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    std::vector<float> ts;
    for (int i = 0; i < 25; ++i) {
        cudaEventRecord(e0);
        probe<<<nsm, 544, smem>>>(tm, n_tiles, n_sub, S, B, rows, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (i >= 5) ts.push_back(ms);
    }
    cudaError_t e = cudaGetLastError();
    std::sort(ts.begin(), ts.end());
    float ms = ts[ts.size() / 2];
    printf("{\"D\":%ld,\"F\":%ld,\"S\":%d,\"B\":%d,\"rows\":%d,\"smem\":%zu,\"ms\":%.4f,\"GBs\":%.1f,\"err\":\"%s\"}\n", D, F, S, B,
           rows, smem, ms, D * F * 4 / ms / 1e6, cudaGetErrorString(e));
    return 0;
}
