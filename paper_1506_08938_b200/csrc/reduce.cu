// Deterministic fp64 reductions for the objective terms
// (nmf.py:152-165: mu1*sum|F| + beta1*sum|G| + mu2*sum F^2 + beta2*sum G^2;
// matrix.py:246-253 trace-identity cross term <G, Y^T>).  Fixed grid and a
// fixed tree, so results do not depend on timing or device.
#include "common.cuh"
#include "nmfb_internal.h"

namespace nmfb {

constexpr int DOT_BLOCKS = 592;  // 4 x 148 SMs, fixed for determinism

// BAD: slot 0 counts entries that are negative or not finite (data check)
template <typename TA, typename TB, bool BAD = false>
__global__ void __launch_bounds__(256) dot3_kernel(const TA *__restrict__ a,
                                                   const TB *__restrict__ b, int64_t len,
                                                   double *__restrict__ part) {
    __shared__ double red[3][256];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < len;
         i += (int64_t)gridDim.x * 256) {
        double x = (double)a[i];
        if (BAD)
            s0 += (x < 0.0 || !isfinite(x)) ? 1.0 : 0.0;
        else if (b)
            s0 += x * (double)b[i];
        s1 += fabs(x);
        s2 += x * x;
    }
    red[0][threadIdx.x] = s0;
    red[1][threadIdx.x] = s1;
    red[2][threadIdx.x] = s2;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            red[0][threadIdx.x] += red[0][threadIdx.x + o];
            red[1][threadIdx.x] += red[1][threadIdx.x + o];
            red[2][threadIdx.x] += red[2][threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x < 3) part[threadIdx.x * gridDim.x + blockIdx.x] = red[threadIdx.x][0];
}

__global__ void dot3_final_kernel(const double *__restrict__ part, int nb,
                                  double *__restrict__ out) {
    __shared__ double red[3][256];
    for (int k = 0; k < 3; ++k) {
        double s = 0.0;
        for (int i = threadIdx.x; i < nb; i += 256) s += part[k * nb + i];
        red[k][threadIdx.x] = s;
    }
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            for (int k = 0; k < 3; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x < 3) out[threadIdx.x] = red[threadIdx.x][0];
}

size_t dot_workspace_bytes(int64_t) { return sizeof(double) * 3 * DOT_BLOCKS; }

template <typename TA>
static void dot_launch_a(const TA *a, const void *b, int b_dtype, int64_t len, double *part,
                         cudaStream_t st) {
    if (b_dtype == NMFB_F64)
        dot3_kernel<TA, double><<<DOT_BLOCKS, 256, 0, st>>>(a, (const double *)b, len, part);
    else
        dot3_kernel<TA, float><<<DOT_BLOCKS, 256, 0, st>>>(a, (const float *)b, len, part);
}

int dot_launch(const void *a, int a_dtype, const void *b, int b_dtype, int64_t len, double *out,
               void *ws, cudaStream_t st) {
    double *part = (double *)ws;
    if (a_dtype == NMFB_F64)
        dot_launch_a<double>((const double *)a, b, b_dtype, len, part, st);
    else
        dot_launch_a<float>((const float *)a, b, b_dtype, len, part, st);
    dot3_final_kernel<<<1, 256, 0, st>>>(part, DOT_BLOCKS, out);
    return launch_status();
}

// One pass over the data matrix: out = {#negative-or-nonfinite, sum|x|, sum x^2}
// (require_nonnegative, matrix.py:169-178, and the init scale's mean).
int data_stats_launch(const void *a, int a_dtype, int64_t len, double *out, void *ws,
                      cudaStream_t st) {
    double *part = (double *)ws;
    if (a_dtype == NMFB_F64)
        dot3_kernel<double, double, true><<<DOT_BLOCKS, 256, 0, st>>>((const double *)a, nullptr,
                                                                      len, part);
    else
        dot3_kernel<float, float, true><<<DOT_BLOCKS, 256, 0, st>>>((const float *)a, nullptr,
                                                                    len, part);
    dot3_final_kernel<<<1, 256, 0, st>>>(part, DOT_BLOCKS, out);
    return launch_status();
}

// out[i] = sum_{s < S} parts[s * len + i] (split-K partials of a data
// product summed before a collective; float32).  The summation order is the
// NNLS prologue's (fast_h, nnls_fast.cuh: four interleaved accumulators), so a
// world-1 collective path reproduces the single-GPU linear terms bit for bit.
__global__ void sum_parts_f32_kernel(const float *__restrict__ parts, int S, int64_t len,
                                     float *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= len) return;
    const float *p = parts + i;
    float s0 = p[0], s1 = 0.f, s2 = 0.f, s3 = 0.f;
    int k = 1;
    for (; k + 3 < S; k += 4) {
        s0 += p[(int64_t)k * len];
        s1 += p[(int64_t)(k + 1) * len];
        s2 += p[(int64_t)(k + 2) * len];
        s3 += p[(int64_t)(k + 3) * len];
    }
    for (; k < S; ++k) s0 += p[(int64_t)k * len];
    out[i] = (s0 + s1) + (s2 + s3);
}

int sum_parts_launch(const float *parts, int S, int64_t len, float *out, cudaStream_t st) {
    if (len <= 0) return NMFB_OK;
    if (S < 1) return NMFB_ERR_ARG;
    sum_parts_f32_kernel<<<(unsigned)((len + 255) / 256), 256, 0, st>>>(parts, S, len, out);
    return launch_status();
}

// dst[i] += src[i] (exact elementwise add; used to accumulate drop-in outputs)
template <typename T>
__global__ void axpy1_kernel(T *__restrict__ dst, const T *__restrict__ src, int64_t len,
                             int upper_r) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= len) return;
    if (upper_r > 0) {  // r x r: upper triangle only (kernels.py:275-280)
        int64_t a = i / upper_r, b = i % upper_r;
        if (b < a) return;
    }
    dst[i] = Exact<T>::add(dst[i], src[i]);
}

int add_into_launch(int dtype, void *dst, const void *src, int64_t len, int upper_r,
                    cudaStream_t st) {
    if (len <= 0) return NMFB_OK;
    dim3 grid((unsigned)((len + 255) / 256));
    if (dtype == NMFB_F64)
        axpy1_kernel<double><<<grid, 256, 0, st>>>((double *)dst, (const double *)src, len,
                                                   upper_r);
    else
        axpy1_kernel<float><<<grid, 256, 0, st>>>((float *)dst, (const float *)src, len, upper_r);
    return launch_status();
}

}  // namespace nmfb
