// Gram products A^T A (G^T G for the coefficient step, F F^T for the
// component step; matrix.py:181-197, kernels.py:276-280) and the fused
// anti-lopsided rescale epilogue (nqp.py:116-131, parallel.py:87-91,104,196).
//
// Gram: CTA = 64x64 output tile x one row chunk; 256 threads each own a 4x4
// register block; rows are staged 32 at a time in shared memory.  fp32 inputs
// accumulate each 32-row slab in fp32 and fold it into fp64 accumulators
// (products of fp32 values are exact in fp64 anyway); fp64 inputs accumulate
// in fp64.  Chunk partials are summed in chunk order by a second kernel, so
// the result is deterministic.  HBM roofline: reads rows*r*sizeof(T) once.
#include <cmath>

#include "common.cuh"
#include "nmfb_internal.h"

namespace nmfb {

constexpr int GT = 64;      // output tile
constexpr int GROWS = 32;   // rows per smem slab

template <typename T>
__global__ void __launch_bounds__(256) gram_partial_kernel(const T *__restrict__ A, int64_t rows,
                                                           int r, int64_t lda, int64_t chunk,
                                                           double *__restrict__ part) {
    // blockIdx.x: tile pair (ti <= tj) index, blockIdx.y: row chunk
    const int ntile = (r + GT - 1) / GT;
    int t = blockIdx.x, ti = 0;
    while (t >= ntile - ti) {
        t -= ntile - ti;
        ++ti;
    }
    const int tj = ti + t;
    const bool diag = (ti == tj);  // diagonal tile: one operand serves both sides
    const int64_t row0 = (int64_t)blockIdx.y * chunk;
    const int64_t row1 = min(rows, row0 + chunk);
    __shared__ __align__(16) T Ai[GROWS][GT];
    __shared__ __align__(16) T Aj[GROWS][GT];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;

    // software pipeline: the next slab's global loads are in flight in
    // registers while the current slab is multiplied from shared memory
    constexpr int PER = GROWS * GT / 256;  // elements per thread per operand
    T pa[PER], pb[PER];
    auto fetch = [&](int64_t rb) {
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int idx = threadIdx.x + q * 256;
            const int rr = idx / GT, c = idx % GT;
            const int64_t row = rb + rr;
            const int ci = ti * GT + c, cj = tj * GT + c;
            const bool okr = row < row1;
            pa[q] = (okr && ci < r) ? A[row * lda + ci] : T(0);
            if (!diag) pb[q] = (okr && cj < r) ? A[row * lda + cj] : T(0);
        }
    };
    if (row0 < row1) fetch(row0);
    for (int64_t rb = row0; rb < row1; rb += GROWS) {
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int idx = threadIdx.x + q * 256;
            Ai[idx / GT][idx % GT] = pa[q];
            if (!diag) Aj[idx / GT][idx % GT] = pb[q];
        }
        __syncthreads();
        if (rb + GROWS < row1) fetch(rb + GROWS);
        const T(*Bj)[GT] = diag ? Ai : Aj;
        T s[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) s[u][v] = T(0);
#pragma unroll 8
        for (int rr = 0; rr < GROWS; ++rr) {
            T a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) a[u] = Ai[rr][ty * 4 + u];
#pragma unroll
            for (int v = 0; v < 4; ++v) b[v] = Bj[rr][tx * 4 + v];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) s[u][v] = fma(a[u], b[v], s[u][v]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] += (double)s[u][v];
        __syncthreads();
    }
    double *out = part + (int64_t)blockIdx.y * r * r;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        int a = ti * GT + ty * 4 + u;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            int b = tj * GT + tx * 4 + v;
            if (a < r && b < r && a <= b) out[a * r + b] = acc[u][v];
        }
    }
}

// out[a][b] = out[b][a] = sum_c part[c][a][b] (a <= b).  One CTA per 32
// consecutive entries: warp w sums the chunks c = w (mod 8) in increasing c
// (coalesced 256-byte rows), then the 8 warp sums are added in warp order --
// a fixed order, so the result is deterministic.
__global__ void __launch_bounds__(256) gram_reduce_kernel(const double *__restrict__ part,
                                                          int nchunk, int r,
                                                          double *__restrict__ out) {
    __shared__ double sh[8][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int idx = blockIdx.x * 32 + lane;
    const int a = idx / r, b = idx % r;
    const bool upper = idx < r * r && a <= b;
    double s = 0.0;
    if (upper)
        for (int c = warp; c < nchunk; c += 8) s += part[(int64_t)c * r * r + idx];
    sh[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && upper) {
        double t = sh[0][lane];
#pragma unroll
        for (int w = 1; w < 8; ++w) t += sh[w][lane];
        out[a * r + b] = t;
        out[b * r + a] = t;
    }
}

// tensor-core partials for fp32 factors (gram_tc.cu)
bool gram_tc_ok(const void *A, int64_t rows, int r, int64_t lda);
int gram_tc_partial_launch(const float *A, int64_t rows, int r, int64_t lda, double *part,
                           int64_t *nunit, cudaStream_t st);

static int64_t gram_chunk(int64_t rows) {
    // ~2 chunks per SM (148 SMs), each a whole number of GROWS-row slabs; the
    // reduce is parallel over entries, so many chunks cost little
    int64_t target = 296;
    int64_t chunk = (rows + target - 1) / target;
    chunk = ((chunk + GROWS - 1) / GROWS) * GROWS;
    if (chunk < GROWS) chunk = GROWS;
    return chunk;
}

// Workspace for any call with at most `rows` rows: the chunk count is at most
// min(ceil(rows / GROWS), 296) -- monotone in rows (the actual count is not:
// fewer rows can mean more, smaller chunks), so one workspace sized for the
// largest operand serves the Grams of both factors.
size_t gram_workspace_bytes(int64_t rows, int r) {
    int64_t nchunk = rows > 0 ? (rows + GROWS - 1) / GROWS : 1;
    if (nchunk > 296) nchunk = 296;
    return (size_t)nchunk * r * r * sizeof(double) + 64;  // + the fused-rescale ticket
}

int gram_launch(int dtype, const void *A, int64_t rows, int r, int64_t lda, double *out,
                void *ws, cudaStream_t st) {
    if (r <= 0 || rows < 0) return NMFB_ERR_ARG;
    int64_t chunk = gram_chunk(rows);
    int64_t nchunk = rows > 0 ? (rows + chunk - 1) / chunk : 1;
    double *part = (double *)ws;
    int ntile = (r + GT - 1) / GT;
    dim3 grid(ntile * (ntile + 1) / 2, (unsigned)nchunk);
    if (rows == 0) {
        cudaMemsetAsync(part, 0, sizeof(double) * r * r, st);
    } else if (dtype == NMFB_F32 && gram_tc_ok(A, rows, r, lda)) {
        int rc = gram_tc_partial_launch((const float *)A, rows, r, lda, part, &nchunk, st);
        if (rc != NMFB_OK) return rc;
    } else if (dtype == NMFB_F64) {
        gram_partial_kernel<double><<<grid, 256, 0, st>>>((const double *)A, rows, r, lda, chunk,
                                                          part);
    } else {
        gram_partial_kernel<float><<<grid, 256, 0, st>>>((const float *)A, rows, r, lda, chunk,
                                                         part);
    }
    gram_reduce_kernel<<<(r * r + 31) / 32, 256, 0, st>>>(part, (int)nchunk, r, out);
    return launch_status();
}

// ---------------------------------------------------------------------------
// Rescale (single CTA): bit-exact restatement of nqp.rescale_arrays on
// H = G + diag_add * I, compacted to the active dims (parallel.py:87-91).
// ---------------------------------------------------------------------------
// Rescale body, run by one CTA: bit-exact restatement of nqp.rescale_arrays
// on H = G + diag_add * I, compacted to the active dims (parallel.py:87-91).
// smem: 2 r doubles + r ints.  G is read with L2 (cg) loads so a CTA that did
// not write it still sees the values other CTAs published before a fence.
template <typename T>
__device__ void rescale_body(const double *__restrict__ G, int r, double diag_add, T *Qa,
                             T *scale_a, int32_t *act_idx, uint8_t *active, int32_t *ra_dev,
                             double *full_scale, double *sh) {
    double *diag = sh;                         // r
    double *sq = sh + r;                       // r: sqrt(diag)
    int *pos = (int *)(sh + 2 * r);            // r: compact position or -1
    __shared__ double s_delta;
    __shared__ int s_ra;
    const int tid = threadIdx.x;
    for (int i = tid; i < r; i += blockDim.x) {
        // H = Q_g + (2.0 * mu2) * np.eye(r): the identity term adds diag_add * 1.0
        const double d = __dadd_rn(__ldcg(G + i * r + i), __dmul_rn(diag_add, 1.0));
        diag[i] = d;
        sq[i] = __dsqrt_rn(d);
    }
    __syncthreads();
    if (tid == 0) {
        // np.max over the diagonal (NaN propagates)
        double mx = diag[0];
        bool nan = false;
        for (int i = 0; i < r; ++i) {
            if (isnan(diag[i])) nan = true;
            if (diag[i] > mx) mx = diag[i];
        }
        if (nan) mx = __longlong_as_double(0x7ff8000000000000ULL);
        s_delta = __dmul_rn(1e-12, mx);
        int k = 0;
        for (int i = 0; i < r; ++i) {
            bool act = diag[i] > s_delta;
            active[i] = act ? 1 : 0;
            pos[i] = act ? k : -1;
            if (act) act_idx[k++] = i;
        }
        s_ra = k;
        *ra_dev = k;
    }
    __syncthreads();
    const int ra = s_ra;
    for (int i = tid; i < r; i += blockDim.x) {
        if (full_scale) full_scale[i] = sq[i];
        if (pos[i] >= 0) scale_a[pos[i]] = (T)sq[i];
    }
    // eight entries per thread per pass: the L2 loads of a pass are issued
    // together (a load -> divide -> store chain per entry left one load in
    // flight per thread: ~65 us at r = 200)
    constexpr int U = 8;
    const int step = (int)blockDim.x;
    for (int base = tid; base < r * r; base += U * step) {
        double g[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int idx = base + u * step;
            g[u] = idx < r * r ? __ldcg(G + idx) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int idx = base + u * step;
            if (idx >= r * r) continue;
            const int i = idx / r, j = idx - i * r;
            const int pi = pos[i], pj = pos[j];
            if (pi < 0 || pj < 0) continue;
            double v;
            if (i == j) {
                v = 1.0;
            } else {
                // off-diagonal of H = G + diag_add * eye: G_ij + 0.0
                v = __ddiv_rn(__dadd_rn(g[u], 0.0), __dmul_rn(sq[i], sq[j]));
            }
            Qa[pi * ra + pj] = (T)v;
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(1024) rescale_kernel(const double *__restrict__ G, int r,
                                                       double diag_add, T *Qa, T *scale_a,
                                                       int32_t *act_idx, uint8_t *active,
                                                       int32_t *ra_dev, double *full_scale) {
    extern __shared__ double sh[];
    rescale_body<T>(G, r, diag_add, Qa, scale_a, act_idx, active, ra_dev, full_scale, sh);
}

// The multi-GPU H_f: sum the per-source r x r slots in source order (as
// sum_slots_f64) into H, then rescale it -- one single-CTA launch.
template <typename T>
__global__ void __launch_bounds__(1024) sum_slots_rescale_kernel(
    const double *__restrict__ slots, int S, int64_t stride, double *H, int r, double diag_add,
    T *Qa, T *scale_a, int32_t *act_idx, uint8_t *active, int32_t *ra_dev) {
    extern __shared__ double sh[];
    for (int i = threadIdx.x; i < r * r; i += blockDim.x) {
        double acc = slots[i];
        for (int s = 1; s < S; ++s) acc += slots[(int64_t)s * stride + i];
        H[i] = acc;
    }
    __syncthreads();
    rescale_body<T>(H, r, diag_add, Qa, scale_a, act_idx, active, ra_dev, nullptr, sh);
}

// Gram reduce with the rescale fused into its epilogue: the CTA that finishes
// last (ticket) runs the rescale on the completed Gram -- one launch and no
// host round trip between the Gram and the rescaled Q (north star (2)).
template <typename T>
__global__ void __launch_bounds__(256) gram_reduce_rescale_kernel(
    const double *__restrict__ part, int nchunk, int r, double *__restrict__ out,
    unsigned *ticket, double diag_add, T *Qa, T *scale_a, int32_t *act_idx, uint8_t *active,
    int32_t *ra_dev) {
    extern __shared__ double sh[];
    __shared__ double red[8][32];
    __shared__ bool last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int idx = blockIdx.x * 32 + lane;
    const int a = idx / r, b = idx % r;
    const bool upper = idx < r * r && a <= b;
    double s = 0.0;
    if (upper)
        for (int c = warp; c < nchunk; c += 8) s += part[(int64_t)c * r * r + idx];
    red[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && upper) {
        double t = red[0][lane];
#pragma unroll
        for (int w = 1; w < 8; ++w) t += red[w][lane];
        out[a * r + b] = t;
        out[b * r + a] = t;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    rescale_body<T>(out, r, diag_add, Qa, scale_a, act_idx, active, ra_dev, nullptr, sh);
    if (threadIdx.x == 0) *ticket = 0u;  // ready for the next launch
}

int gram_rescale_launch(int dtype, const void *A, int64_t rows, int r, int64_t lda, double *out,
                        void *ws, double diag_add, void *Qa, void *scale_a, int32_t *act_idx,
                        uint8_t *active, int32_t *ra_dev, cudaStream_t st) {
    if (r <= 0 || rows < 0 || r > 4096) return NMFB_ERR_ARG;
    int64_t chunk = gram_chunk(rows);
    int64_t nchunk = rows > 0 ? (rows + chunk - 1) / chunk : 1;
    double *part = (double *)ws;
    // the ticket sits past the largest partial area this workspace can hold
    unsigned *ticket = (unsigned *)((char *)ws + gram_workspace_bytes(rows, r) - 64);
    cudaMemsetAsync(ticket, 0, sizeof(unsigned), st);
    int ntile = (r + GT - 1) / GT;
    dim3 grid(ntile * (ntile + 1) / 2, (unsigned)nchunk);
    if (rows == 0) {
        cudaMemsetAsync(part, 0, sizeof(double) * r * r, st);
    } else if (dtype == NMFB_F32 && gram_tc_ok(A, rows, r, lda)) {
        int rc = gram_tc_partial_launch((const float *)A, rows, r, lda, part, &nchunk, st);
        if (rc != NMFB_OK) return rc;
    } else if (dtype == NMFB_F64)
        gram_partial_kernel<double><<<grid, 256, 0, st>>>((const double *)A, rows, r, lda, chunk,
                                                          part);
    else
        gram_partial_kernel<float><<<grid, 256, 0, st>>>((const float *)A, rows, r, lda, chunk,
                                                         part);
    const size_t smem = 2 * r * sizeof(double) + r * sizeof(int);
    const unsigned nb = (unsigned)((r * r + 31) / 32);
    if (smem > 48 * 1024) {
        cudaFuncSetAttribute(gram_reduce_rescale_kernel<double>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(gram_reduce_rescale_kernel<float>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    if (dtype == NMFB_F64)
        gram_reduce_rescale_kernel<double><<<nb, 256, smem, st>>>(
            part, (int)nchunk, r, out, ticket, diag_add, (double *)Qa, (double *)scale_a, act_idx,
            active, ra_dev);
    else
        gram_reduce_rescale_kernel<float><<<nb, 256, smem, st>>>(
            part, (int)nchunk, r, out, ticket, diag_add, (float *)Qa, (float *)scale_a, act_idx,
            active, ra_dev);
    return launch_status();
}

int rescale_launch(int dtype, const double *G, int r, double diag_add, void *Qa, void *scale_a,
                   int32_t *act_idx, uint8_t *active, int32_t *ra_dev, double *full_scale,
                   cudaStream_t st) {
    if (r <= 0 || r > 4096) return NMFB_ERR_ARG;
    size_t smem = 2 * r * sizeof(double) + r * sizeof(int);
    if (smem > 48 * 1024) {
        cudaFuncSetAttribute(rescale_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        cudaFuncSetAttribute(rescale_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    }
    if (dtype == NMFB_F64)
        rescale_kernel<double><<<1, 1024, smem, st>>>(G, r, diag_add, (double *)Qa,
                                                     (double *)scale_a, act_idx, active, ra_dev,
                                                     full_scale);
    else
        rescale_kernel<float><<<1, 1024, smem, st>>>(G, r, diag_add, (float *)Qa,
                                                    (float *)scale_a, act_idx, active, ra_dev,
                                                    full_scale);
    return launch_status();
}

int sum_slots_rescale_launch(int dtype, const double *slots, int S, int64_t stride, double *H,
                             int r, double diag_add, void *Qa, void *scale_a, int32_t *act_idx,
                             uint8_t *active, int32_t *ra_dev, cudaStream_t st) {
    if (r <= 0 || r > 4096 || S < 1 || !slots || !H) return NMFB_ERR_ARG;
    size_t smem = 2 * r * sizeof(double) + r * sizeof(int);
    if (smem > 48 * 1024) {
        cudaFuncSetAttribute(sum_slots_rescale_kernel<double>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(sum_slots_rescale_kernel<float>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    if (dtype == NMFB_F64)
        sum_slots_rescale_kernel<double><<<1, 1024, smem, st>>>(
            slots, S, stride, H, r, diag_add, (double *)Qa, (double *)scale_a, act_idx, active,
            ra_dev);
    else
        sum_slots_rescale_kernel<float><<<1, 1024, smem, st>>>(
            slots, S, stride, H, r, diag_add, (float *)Qa, (float *)scale_a, act_idx, active,
            ra_dev);
    return launch_status();
}

}  // namespace nmfb
