// Micro-benchmark: tcgen05.mma kind::tf32 issue/complete rate on one SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//   -I include tests/micro/mma_rate.cu -lcuda -o /tmp/mma_rate
#include "../../paper_1506_08938_b200/csrc/tc_gemm.cu"
namespace nmfb {
int launch_status() { return cudaGetLastError() == cudaSuccess ? 0 : -1; }
}

namespace nmfb {
__device__ __forceinline__ long long gt() {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void umma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc));
}
__device__ __forceinline__ void umma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc));
}
// mode 0: one accumulator; 1: 4 rotating accumulators; 2: commit+wait every 4
// kind 0: tf32, 1: bf16; M = 128
__global__ void mma_rate(long long *out, int N, int iters, int mode, int kind, int sw64) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t *sm = (uint8_t *)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((float *)sm)[i] = 0.f;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&slot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t fmt = kind == 0 ? 2u : (kind == 1 ? 1u : 0u);
        const uint32_t cfmt = kind == 2 ? 2u : 1u;
        const uint32_t idesc = (cfmt << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(N >> 3) << 17) |
                               ((uint32_t)(128 >> 4) << 24);
        uint64_t a = umma_desc_sw128(sm), b = umma_desc_sw128(sm + 16384);
        if (sw64) {  // SWIZZLE_64B K-major: layout 4, SBO = 8 rows x 64 B
            a = (a & ~(((uint64_t)0x3FFF << 32) | ((uint64_t)7 << 61))) | ((uint64_t)(512 >> 4) << 32) | ((uint64_t)4 << 61);
            b = (b & ~(((uint64_t)0x3FFF << 32) | ((uint64_t)7 << 61))) | ((uint64_t)(512 >> 4) << 32) | ((uint64_t)4 << 61);
        }
        uint32_t ph = 0;
        long long t0 = gt();
        for (int it = 0; it < iters; ++it) {
            const uint32_t d = tmem + (mode == 1 ? (uint32_t)((it & 3) * (N <= 128 ? N : 0)) : 0u);
            const uint64_t dk = (uint64_t)((it & 3) * 2);
            if (kind == 0)
                umma_tf32(d, a + dk, b + dk, idesc, 1u);
            else if (kind == 1)
                umma_f16(d, a + dk, b + dk, idesc);
            else
                umma_i8(d, a + dk, b + dk, idesc);
            if (mode == 2 && (it & 3) == 3) {
                umma_commit(&bar);
                mbar_wait(&bar, ph);
                ph ^= 1u;
            }
        }
        long long t1 = gt();
        umma_commit(&bar);
        mbar_wait(&bar, ph);
        long long t2 = gt();
        out[0] = t1 - t0;
        out[1] = t2 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}
}  // namespace nmfb

int main() {
    long long *d, h[2];
    cudaMalloc(&d, 16);
    cudaFuncSetAttribute(nmfb::mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int iters = 4096;
    for (int kind = 0; kind < 3; ++kind)
        for (int mode = 0; mode < 2; ++mode)
            for (int N : {16, 32, 64, 80, 128, 256})
              for (int sw64 = 0; sw64 < 2; ++sw64) {
                nmfb::mma_rate<<<1, 128, 100 * 1024>>>(d, N, iters, mode, kind, sw64);
                nmfb::mma_rate<<<1, 128, 100 * 1024>>>(d, N, iters, mode, kind, sw64);
                cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
                double ns = (double)h[1] / iters;
                double flops = 2.0 * 128 * N * (kind == 0 ? 8 : (kind == 1 ? 16 : 32));
                printf("%s sw%d mode=%d N=%3d: issue %.1f ns/mma, complete %.1f ns/mma, %.1f TFLOP/s/SM "
                       "(x148 = %.0f TF/s)\n",
                       kind == 0 ? "tf32" : (kind == 1 ? "bf16" : "u8  "), sw64 ? 64 : 128, mode, N, (double)h[0] / iters, ns,
                       flops / ns / 1e3, flops / ns / 1e3 * 148);
            }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
