// Micro-benchmark: CUDA-core FMA peaks on the box ("measure
// FFMA/DFMA peaks"), the denominator of the NNLS roofline.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tests/micro/fma_peak.cu -o /tmp/fma_peak
// Prints one JSON line: fp32 FFMA, packed FFMA2 and fp64 DFMA TFLOP/s, each
// the best of 5 launches of a register-resident kernel with 8 (16 for the
// packed form) independent FMA chains per thread, grid = 148 SMs x 8 CTAs.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void __launch_bounds__(256) ffma_kernel(float *out, int iters, float a, float b) {
    float acc[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3f + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) acc[c] = fmaf(acc[c], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[c];
    if (s == 1234.5f) out[threadIdx.x] = s;
}

template <int CH>
__global__ void __launch_bounds__(256) ffma2_kernel(float *out, int iters, float a, float b) {
    float2 acc[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = make_float2(threadIdx.x * 1e-3f + c, c + 0.5f);
    const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) acc[c] = __ffma2_rn(acc[c], a2, b2);
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[c].x + acc[c].y;
    if (s == 1234.5f) out[threadIdx.x] = s;
}

template <int CH>
__global__ void __launch_bounds__(256) dfma_kernel(double *out, int iters, double a, double b) {
    double acc[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[c];
    if (s == 1234.5) out[threadIdx.x] = s;
}

template <typename K>
static float best_ms(K launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int t = 0; t < 5; ++t) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    float *fo;
    double *dout;
    cudaMalloc(&fo, 1024 * sizeof(float));
    cudaMalloc(&dout, 1024 * sizeof(double));
    const dim3 grid(sms * 8), block(256);
    const double threads = (double)grid.x * block.x;
    const int it = 1 << 16, itd = 1 << 12;
    float t1 = best_ms([&] { ffma_kernel<8><<<grid, block>>>(fo, it, 0.999f, 1e-3f); });
    float t2 = best_ms([&] { ffma2_kernel<8><<<grid, block>>>(fo, it, 0.999f, 1e-3f); });
    float t3 = best_ms([&] { dfma_kernel<8><<<grid, block>>>(dout, itd, 0.999, 1e-3); });
    const double f1 = threads * it * 8 * 2 / (t1 * 1e-3) / 1e12;
    const double f2 = threads * it * 16 * 2 / (t2 * 1e-3) / 1e12;
    const double f3 = threads * itd * 8 * 2 / (t3 * 1e-3) / 1e12;
    printf("{\"ffma_tflops\": %.2f, \"ffma2_tflops\": %.2f, \"dfma_tflops\": %.3f, \"sms\": %d, "
           "\"attr_clock_mhz\": %d, \"err\": \"%s\"}\n",
           f1, f2, f3, sms, clk / 1000, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
