// Micro-benchmark: tcgen05.ld throughput (bytes/clk/SM) vs warps and shape.
#include "../../paper_1506_08938_b200/csrc/tcgen05.cuh"
#include <cstdio>
using namespace nmfb;
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,"
        "%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
          "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
          "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
__global__ void k(long long *out, int iters, int shape) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&slot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t t = slot + ((uint32_t)((warp & 3) * 32) << 16);
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const uint32_t col = (uint32_t)((i * 32 + (warp >> 2) * 64) & 511);
        if (shape == 16) {
            uint32_t v[16];
            tmem_ld16(t + col, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int q = 0; q < 16; ++q) acc += v[q];
        } else {
            uint32_t v[32];
            ld32(t + col, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int q = 0; q < 32; ++q) acc += v[q];
        }
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = acc; }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512));
}
int main() {
    long long *d, h[2];
    cudaMalloc(&d, 16);
    for (int shape : {16, 32})
        for (int warps : {4, 8, 16, 32}) {
            const int iters = 4096;
            k<<<1, warps * 32>>>(d, iters, shape);
            k<<<1, warps * 32>>>(d, iters, shape);
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            double bytes = (double)warps * 32 * shape * 4 * iters;
            printf("x%d warps=%2d: %.1f B/clk/SM (%lld clk)\n", shape, warps, bytes / h[0], h[0]);
        }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
