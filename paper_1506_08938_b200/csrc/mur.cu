// Multiplicative-update baseline on the device (reference baselines.py:41-85):
//   F <- F * (G'V) / (G'G F + floor),   G <- G * (V F') / (G (F F') + floor)
// The data products G'V and V F' come from the same kernels as the
// alternating-NNLS step (tcgen05 GEMM partials, CSC/CSR SpMM, reference-order
// linear terms), in the NNLS kernel's linear-term convention
//   h = h_base - sum_{s < S} parts[s]   (S >= 1),   h = parts   (S == 0),
// so the numerator is -h (the callers pass h_base = 0).  One warp per
// problem row x (r values): the row is staged in shared memory (the update
// is in place), every lane forms den_i = sum_k Q[i][k] x_k + floor for its
// coordinates in fp64 against the raw Gram Q (fp64, r x r, L1-resident), and
// x_i <- x_i * (num_i / den_i) in the reference's operation order.
#include "common.cuh"
#include "nmfb_internal.h"

namespace nmfb {

namespace {

constexpr int MUR_WARPS = 8;

template <typename T, typename TH>
__global__ void __launch_bounds__(32 * MUR_WARPS)
    mur_update_kernel(const double *__restrict__ Q, int r, const TH *__restrict__ hp, int S,
                      int64_t h_ld, int64_t h_pstride, double h_base, T *__restrict__ x,
                      int64_t count, double floor_, unsigned long long *stats) {
    extern __shared__ double xs_all[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *xs = xs_all + (size_t)warp * r;
    const int64_t nw = (int64_t)gridDim.x * MUR_WARPS;
    for (int64_t j = (int64_t)blockIdx.x * MUR_WARPS + warp; j < count; j += nw) {
        T *row = x + j * r;
        for (int i = lane; i < r; i += 32) xs[i] = (double)row[i];
        __syncwarp();
        for (int i = lane; i < r; i += 32) {
            const double *q = Q + (int64_t)i * r;
            double den = 0.0;
            for (int k = 0; k < r; ++k) den = fma(q[k], xs[k], den);
            den += floor_;
            const TH *p = hp + j * h_ld + i;
            double h;
            if (S == 0) {
                h = (double)p[0];
            } else {
                TH s = p[0];
                for (int t = 1; t < S; ++t) s += p[(int64_t)t * h_pstride];
                h = h_base - (double)s;
            }
            const T num = (T)(-h);
            const T ratio = num / (T)den;
            row[i] = (T)xs[i] * ratio;
        }
        __syncwarp();
    }
    if (stats && blockIdx.x == 0 && threadIdx.x == 0)
        atomicAdd(&stats[0], (unsigned long long)count);  // one update per subproblem
}

template <typename T, typename TH>
int mur_go(const double *Q, int r, const void *h, int S, int64_t h_ld, int64_t h_pstride,
           double h_base, void *x, int64_t count, double floor_, uint64_t *stats,
           cudaStream_t st) {
    int64_t blocks = (count + MUR_WARPS - 1) / MUR_WARPS;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    const size_t smem = sizeof(double) * MUR_WARPS * r;
    auto kern = mur_update_kernel<T, TH>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)smem);
    kern<<<(unsigned)blocks, 32 * MUR_WARPS, smem, st>>>(
        Q, r, (const TH *)h, S, h_ld, h_pstride, h_base, (T *)x, count, floor_,
        (unsigned long long *)stats);
    return launch_status();
}

}  // namespace

int mur_update_launch(int dtype, const double *Q, int r, const void *h, int h_dtype, int S,
                      int64_t h_ld, int64_t h_pstride, double h_base, void *x, int64_t count,
                      double floor_, uint64_t *stats, cudaStream_t st) {
    if (r <= 0 || count < 0 || S < 0 || !Q || (count > 0 && (!h || !x)) ||
        (dtype != NMFB_F32 && dtype != NMFB_F64) || (h_dtype != NMFB_F32 && h_dtype != NMFB_F64))
        return NMFB_ERR_ARG;
    if (count == 0) return NMFB_OK;
    if (dtype == NMFB_F64)
        return h_dtype == NMFB_F64
                   ? mur_go<double, double>(Q, r, h, S, h_ld, h_pstride, h_base, x, count, floor_,
                                            stats, st)
                   : mur_go<double, float>(Q, r, h, S, h_ld, h_pstride, h_base, x, count, floor_,
                                           stats, st);
    return h_dtype == NMFB_F64
               ? mur_go<float, double>(Q, r, h, S, h_ld, h_pstride, h_base, x, count, floor_,
                                       stats, st)
               : mur_go<float, float>(Q, r, h, S, h_ld, h_pstride, h_base, x, count, floor_,
                                      stats, st);
}

}  // namespace nmfb
