// Sparse data products for CSC/CSR data (kernels.py:251-258 linear terms,
// kernels.py:270-274 Y^T accumulator).  Warp per data column (CSC) or row
// (CSR); lanes own components i = lane + 32c, so every G / F^T row gather is
// one coalesced r-float read.  Nonzeros are fetched 32 at a time by the lanes
// and broadcast by shuffles.  Each output is a sequential sum over the
// column's / row's nonzeros in storage order: in NMFB_MODE_REFERENCE with
// unfused arithmetic that is exactly the reference's order (bit-exact fp64).
// HBM roofline per pass: nnz*(4 + sizeof(T)) + (m or n + 1)*8 bytes of index
// data + the gathered rows (L2-resident at C3).
#include "common.cuh"
#include "nmfb_internal.h"

namespace nmfb {

template <typename T, bool EXACT, int C>
__global__ void __launch_bounds__(128) csc_linear_kernel(const int64_t *__restrict__ indptr,
                                                         const int32_t *__restrict__ rowidx,
                                                         const T *__restrict__ vals,
                                                         int64_t col_lo, int64_t col_hi,
                                                         const T *__restrict__ G, int r, T mu1,
                                                         T *__restrict__ h) {
    const int64_t col = col_lo + (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (col >= col_hi) return;
    const int lane = threadIdx.x & 31;
    T acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = mu1;
    const int64_t p0 = indptr[col], p1 = indptr[col + 1];
    for (int64_t base = p0; base < p1; base += 32) {
        const int cnt = (int)min((int64_t)32, p1 - base);
        int myrow = 0;
        T myv = T(0);
        if (lane < cnt) {
            myrow = rowidx[base + lane];
            myv = vals[base + lane];
        }
#pragma unroll 4
        for (int u = 0; u < cnt; ++u) {
            const int row = __shfl_sync(NMFB_FULL_MASK, myrow, u);
            const T v = __shfl_sync(NMFB_FULL_MASK, myv, u);
            const T *grow = G + (int64_t)row * r;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const int i = lane + 32 * c;
                if (i < r) {
                    if (EXACT)
                        acc[c] = Exact<T>::msub(acc[c], grow[i], v);
                    else
                        acc[c] = fma(-grow[i], v, acc[c]);
                }
            }
        }
    }
    T *out = h + (col - col_lo) * r;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int i = lane + 32 * c;
        if (i < r) out[i] = acc[c];
    }
}

struct SparseShards {
    int64_t b[NMFB_MAX_WORKERS + 1];
    int w;
};

// YT[row][i] = sum over the row's entries (ascending column) FT[col][i] * v.
// With shards: per-worker partial sums, added in worker order (the reference
// reduce, parallel.py:150-156).
template <typename T, typename TY, bool EXACT, int C>
__global__ void __launch_bounds__(128) csr_yt_kernel(const int64_t *__restrict__ rowptr,
                                                     const int32_t *__restrict__ colidx,
                                                     const T *__restrict__ vals, int64_t n,
                                                     const T *__restrict__ FT, int r,
                                                     SparseShards sh, TY *__restrict__ YT) {
    const int64_t row = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (row >= n) return;
    const int lane = threadIdx.x & 31;
    TY total[C], acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) total[c] = acc[c] = TY(0);
    int w = 0;
    int64_t whi = sh.b[1];
    const int64_t p0 = rowptr[row], p1 = rowptr[row + 1];
    for (int64_t base = p0; base < p1; base += 32) {
        const int cnt = (int)min((int64_t)32, p1 - base);
        int mycol = 0;
        T myv = T(0);
        if (lane < cnt) {
            mycol = colidx[base + lane];
            myv = vals[base + lane];
        }
        for (int u = 0; u < cnt; ++u) {
            const int col = __shfl_sync(NMFB_FULL_MASK, mycol, u);
            const T v = __shfl_sync(NMFB_FULL_MASK, myv, u);
            if (EXACT) {
                while (col >= whi && w + 1 < sh.w) {  // next worker shard
#pragma unroll
                    for (int c = 0; c < C; ++c) {
                        total[c] = Exact<TY>::add(total[c], acc[c]);
                        acc[c] = TY(0);
                    }
                    ++w;
                    whi = sh.b[w + 1];
                }
            }
            const T *f = FT + (int64_t)col * r;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const int i = lane + 32 * c;
                if (i < r) {
                    if (EXACT)
                        acc[c] = Exact<TY>::madd(acc[c], (TY)f[i], (TY)v);
                    else
                        acc[c] = fma((TY)f[i], (TY)v, acc[c]);
                }
            }
        }
    }
    TY *out = YT + row * r;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int i = lane + 32 * c;
        if (i < r) out[i] = EXACT ? Exact<TY>::add(total[c], acc[c]) : acc[c];
    }
}

// ---------------------------------------------------------------------------
// Fast-path gathers with 16-byte vector loads (r % 4 == 0, r <= 128): lane l
// of the warp owns components 4l..4l+3 of the output row, so each nonzero is
// one 128-bit L2 load per active lane (r / 4 lanes) instead of ceil(r/32)
// scalar loads; unrolled 8 deep for memory-level parallelism.  Same
// per-component summation order as the scalar kernels (nonzeros in order).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) csc_linear_v4_kernel(const int64_t *__restrict__ indptr,
                                                            const int32_t *__restrict__ rowidx,
                                                            const float *__restrict__ vals,
                                                            int64_t col_lo, int64_t col_hi,
                                                            const float *__restrict__ G, int r,
                                                            float mu1, float *__restrict__ h) {
    const int64_t col = col_lo + (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (col >= col_hi) return;
    const int lane = threadIdx.x & 31;
    const bool act = lane < (r >> 2);
    float4 acc = make_float4(mu1, mu1, mu1, mu1);
    const int64_t p0 = indptr[col], p1 = indptr[col + 1];
    for (int64_t base = p0; base < p1; base += 32) {
        const int cnt = (int)min((int64_t)32, p1 - base);
        int myrow = 0;
        float myv = 0.f;
        if (lane < cnt) {
            myrow = rowidx[base + lane];
            myv = vals[base + lane];
        }
#pragma unroll 8
        for (int u = 0; u < cnt; ++u) {
            const int row = __shfl_sync(NMFB_FULL_MASK, myrow, u);
            const float v = __shfl_sync(NMFB_FULL_MASK, myv, u);
            if (act) {
                const float4 g = __ldg(reinterpret_cast<const float4 *>(G + (int64_t)row * r) + lane);
                acc.x = fmaf(-g.x, v, acc.x);
                acc.y = fmaf(-g.y, v, acc.y);
                acc.z = fmaf(-g.z, v, acc.z);
                acc.w = fmaf(-g.w, v, acc.w);
            }
        }
    }
    if (act) reinterpret_cast<float4 *>(h + (col - col_lo) * r)[lane] = acc;
}

template <typename TY>
__global__ void __launch_bounds__(128) csr_yt_chunk_v4_kernel(const int64_t *__restrict__ chunks,
                                                              int64_t nchunks,
                                                              const int32_t *__restrict__ colidx,
                                                              const float *__restrict__ vals,
                                                              const float *__restrict__ FT, int r,
                                                              TY *__restrict__ YT,
                                                              TY *__restrict__ part) {
    const int64_t ch = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (ch >= nchunks) return;
    const int lane = threadIdx.x & 31;
    const bool act = lane < (r >> 2);
    const int64_t row = chunks[ch * 4 + 0], p0 = chunks[ch * 4 + 1], p1 = chunks[ch * 4 + 2];
    const int64_t slot = chunks[ch * 4 + 3];
    TY a0 = TY(0), a1 = TY(0), a2 = TY(0), a3 = TY(0);
    for (int64_t base = p0; base < p1; base += 32) {
        const int cnt = (int)min((int64_t)32, p1 - base);
        int mycol = 0;
        float myv = 0.f;
        if (lane < cnt) {
            mycol = colidx[base + lane];
            myv = vals[base + lane];
        }
#pragma unroll 8
        for (int u = 0; u < cnt; ++u) {
            const int col = __shfl_sync(NMFB_FULL_MASK, mycol, u);
            const float v = __shfl_sync(NMFB_FULL_MASK, myv, u);
            if (act) {
                const float4 f = __ldg(reinterpret_cast<const float4 *>(FT + (int64_t)col * r) + lane);
                a0 = fma((TY)f.x, (TY)v, a0);
                a1 = fma((TY)f.y, (TY)v, a1);
                a2 = fma((TY)f.z, (TY)v, a2);
                a3 = fma((TY)f.w, (TY)v, a3);
            }
        }
    }
    if (act) {
        TY *out = ((slot < 0) ? (YT + row * r) : (part + slot * r)) + 4 * lane;
        out[0] = a0;
        out[1] = a1;
        out[2] = a2;
        out[3] = a3;
    }
}

bool sparse_vec_ok(int r, const void *a, const void *b);
int csc_linear_vec_launch(const int64_t *indptr, const int64_t *seg, int nblk,
                          const int32_t *rowidx, const float *vals, int64_t lo, int64_t hi,
                          const float *G, int r, double mu1, float *h, cudaStream_t st);
int csr_yt_chunked_vec_launch(const int64_t *chunks, int64_t nchunks, const int64_t *heavy,
                              int64_t nheavy, const int64_t *seg, int nblk, const int32_t *colidx,
                              const float *vals, const float *FT, int r, int yt_dtype, void *YT,
                              void *part, cudaStream_t st);

static bool v4_ok(int r, const void *a) {
    return r % 4 == 0 && r <= 128 && ((uintptr_t)a % 16) == 0;
}

template <typename T, bool EXACT>
static int csc_linear_dispatch(const int64_t *indptr, const int32_t *rowidx, const void *vals,
                               int64_t lo, int64_t hi, const void *G, int r, double mu1, void *h,
                               cudaStream_t st) {
    dim3 grid((unsigned)((hi - lo + 3) / 4));
    const T *v = (const T *)vals;
    const T *g = (const T *)G;
    T *o = (T *)h;
    if (!EXACT && sizeof(T) == 4 && sparse_vec_ok(r, G, h))  // 16-byte gathers, r <= 256
        return csc_linear_vec_launch(indptr, nullptr, 1, rowidx, (const float *)vals, lo, hi,
                                     (const float *)G, r, mu1, (float *)h, st);
#define NMFB_CSC(Cc) \
    csc_linear_kernel<T, EXACT, Cc><<<grid, 128, 0, st>>>(indptr, rowidx, v, lo, hi, g, r, (T)mu1, o)
    if (r <= 32)
        NMFB_CSC(1);
    else if (r <= 64)
        NMFB_CSC(2);
    else if (r <= 128)
        NMFB_CSC(4);
    else if (r <= 256)
        NMFB_CSC(8);
    else
        return NMFB_ERR_ARG;
#undef NMFB_CSC
    return launch_status();
}

int csc_linear_launch(int dtype, int mode, const int64_t *indptr, const int32_t *rowidx,
                      const void *vals, int64_t lo, int64_t hi, const void *G, int r, double mu1,
                      void *h, cudaStream_t st) {
    if (hi <= lo) return NMFB_OK;
    bool exact = (mode == NMFB_MODE_REFERENCE);
    if (dtype == NMFB_F64)
        return exact ? csc_linear_dispatch<double, true>(indptr, rowidx, vals, lo, hi, G, r, mu1,
                                                         h, st)
                     : csc_linear_dispatch<double, false>(indptr, rowidx, vals, lo, hi, G, r,
                                                          mu1, h, st);
    return exact ? csc_linear_dispatch<float, true>(indptr, rowidx, vals, lo, hi, G, r, mu1, h, st)
                 : csc_linear_dispatch<float, false>(indptr, rowidx, vals, lo, hi, G, r, mu1, h,
                                                     st);
}

template <typename T, typename TY, bool EXACT>
static int csr_yt_dispatch(const int64_t *rowptr, const int32_t *colidx, const void *vals,
                           int64_t n, const void *FT, int r, const SparseShards &sh, void *YT,
                           cudaStream_t st) {
    dim3 grid((unsigned)((n + 3) / 4));
    const T *v = (const T *)vals;
    const T *f = (const T *)FT;
    TY *o = (TY *)YT;
#define NMFB_CSR(Cc) \
    csr_yt_kernel<T, TY, EXACT, Cc><<<grid, 128, 0, st>>>(rowptr, colidx, v, n, f, r, sh, o)
    if (r <= 32)
        NMFB_CSR(1);
    else if (r <= 64)
        NMFB_CSR(2);
    else if (r <= 128)
        NMFB_CSR(4);
    else if (r <= 256)
        NMFB_CSR(8);
    else
        return NMFB_ERR_ARG;
#undef NMFB_CSR
    return launch_status();
}

int csr_yt_launch(int dtype, int mode, const int64_t *rowptr, const int32_t *colidx,
                  const void *vals, int64_t n, const void *FT, int r, int yt_dtype,
                  const int64_t *bounds, int workers, void *YT, cudaStream_t st) {
    if (n <= 0) return NMFB_OK;
    SparseShards sh;
    if (workers < 1 || workers > NMFB_MAX_WORKERS) return NMFB_ERR_ARG;
    sh.w = workers;
    for (int i = 0; i <= workers; ++i) sh.b[i] = bounds ? bounds[i] : (i == 0 ? 0 : INT64_MAX);
    bool exact = (mode == NMFB_MODE_REFERENCE);
    if (dtype == NMFB_F64) {
        if (yt_dtype != NMFB_F64) return NMFB_ERR_ARG;
        return exact ? csr_yt_dispatch<double, double, true>(rowptr, colidx, vals, n, FT, r, sh,
                                                             YT, st)
                     : csr_yt_dispatch<double, double, false>(rowptr, colidx, vals, n, FT, r, sh,
                                                              YT, st);
    }
    if (yt_dtype == NMFB_F64)
        return exact ? csr_yt_dispatch<float, double, true>(rowptr, colidx, vals, n, FT, r, sh, YT,
                                                            st)
                     : csr_yt_dispatch<float, double, false>(rowptr, colidx, vals, n, FT, r, sh,
                                                             YT, st);
    return exact ? csr_yt_dispatch<float, float, true>(rowptr, colidx, vals, n, FT, r, sh, YT, st)
                 : csr_yt_dispatch<float, float, false>(rowptr, colidx, vals, n, FT, r, sh, YT,
                                                        st);
}

// Load-balanced Y^T pass (production): Zipf row popularity makes a few rows
// hold 10^4+ nonzeros, so rows are cut into chunks of <= NMFB_CSR_CHUNK
// entries (plan built once per matrix).  A warp sums one chunk (fp64 or fp32
// accumulator); single-chunk rows are written directly, multi-chunk ("heavy")
// rows go through partial slots that a second kernel folds in chunk order
// (deterministic).  chunks: [nchunks][4] = (row, lo, hi, slot or -1);
// heavy: [nheavy][3] = (row, first slot, count).
template <typename T, typename TY, int C>
__global__ void __launch_bounds__(128) csr_yt_chunk_kernel(const int64_t *__restrict__ chunks,
                                                           int64_t nchunks,
                                                           const int32_t *__restrict__ colidx,
                                                           const T *__restrict__ vals,
                                                           const T *__restrict__ FT, int r,
                                                           TY *__restrict__ YT,
                                                           TY *__restrict__ part) {
    const int64_t ch = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (ch >= nchunks) return;
    const int lane = threadIdx.x & 31;
    const int64_t row = chunks[ch * 4 + 0], p0 = chunks[ch * 4 + 1], p1 = chunks[ch * 4 + 2];
    const int64_t slot = chunks[ch * 4 + 3];
    TY acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = TY(0);
    for (int64_t base = p0; base < p1; base += 32) {
        const int cnt = (int)min((int64_t)32, p1 - base);
        int mycol = 0;
        T myv = T(0);
        if (lane < cnt) {
            mycol = colidx[base + lane];
            myv = vals[base + lane];
        }
#pragma unroll 4
        for (int u = 0; u < cnt; ++u) {
            const int col = __shfl_sync(NMFB_FULL_MASK, mycol, u);
            const T v = __shfl_sync(NMFB_FULL_MASK, myv, u);
            const T *f = FT + (int64_t)col * r;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const int i = lane + 32 * c;
                if (i < r) acc[c] = fma((TY)f[i], (TY)v, acc[c]);
            }
        }
    }
    TY *out = (slot < 0) ? (YT + row * r) : (part + slot * r);
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int i = lane + 32 * c;
        if (i < r) out[i] = acc[c];
    }
}

template <typename TY>
__global__ void csr_yt_fold_kernel(const int64_t *__restrict__ heavy, int64_t nheavy, int r,
                                   const TY *__restrict__ part, TY *__restrict__ YT) {
    const int64_t h = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (h >= nheavy) return;
    const int lane = threadIdx.x & 31;
    const int64_t row = heavy[h * 3 + 0], first = heavy[h * 3 + 1], count = heavy[h * 3 + 2];
    // same per-element slot order as a plain loop (0 + p0 + p1 + ...), with
    // eight elements per lane and four slots unrolled so the loads overlap
    for (int i0 = 0; i0 < r; i0 += 256) {
        TY s[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) s[q] = TY(0);
#pragma unroll 4
        for (int64_t k = 0; k < count; ++k) {
            const TY *p = part + (first + k) * r;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int i = i0 + lane + 32 * q;
                if (i < r) s[q] += p[i];
            }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int i = i0 + lane + 32 * q;
            if (i < r) YT[row * r + i] = s[q];
        }
    }
}

template <typename T, typename TY>
static int csr_yt_chunked_dispatch(const int64_t *chunks, int64_t nchunks, const int64_t *heavy,
                                   int64_t nheavy, const int32_t *colidx, const void *vals,
                                   const void *FT, int r, void *YT, void *part, cudaStream_t st) {
    dim3 grid((unsigned)((nchunks + 3) / 4));
    const T *v = (const T *)vals;
    const T *f = (const T *)FT;
    TY *o = (TY *)YT, *pp = (TY *)part;
    if (sizeof(T) == 4 && sparse_vec_ok(r, FT, FT))  // 16-byte gathers, r <= 256
        return csr_yt_chunked_vec_launch(chunks, nchunks, heavy, nheavy, nullptr, 1, colidx,
                                         (const float *)vals, (const float *)FT, r,
                                         sizeof(TY) == 8 ? NMFB_F64 : NMFB_F32, YT, part, st);
#define NMFB_CSRC(Cc) \
    csr_yt_chunk_kernel<T, TY, Cc><<<grid, 128, 0, st>>>(chunks, nchunks, colidx, v, f, r, o, pp)
    if (r <= 32)
        NMFB_CSRC(1);
    else if (r <= 64)
        NMFB_CSRC(2);
    else if (r <= 128)
        NMFB_CSRC(4);
    else if (r <= 256)
        NMFB_CSRC(8);
    else
        return NMFB_ERR_ARG;
#undef NMFB_CSRC
    if (nheavy > 0)
        csr_yt_fold_kernel<TY><<<(unsigned)((nheavy + 3) / 4), 128, 0, st>>>(heavy, nheavy, r, pp,
                                                                             o);
    return launch_status();
}

int csr_yt_chunked_launch(int dtype, const int64_t *chunks, int64_t nchunks, const int64_t *heavy,
                          int64_t nheavy, const int32_t *colidx, const void *vals, const void *FT,
                          int r, int yt_dtype, void *YT, void *part, cudaStream_t st) {
    if (nchunks <= 0) return NMFB_OK;
    if (dtype == NMFB_F64)
        return yt_dtype == NMFB_F64
                   ? csr_yt_chunked_dispatch<double, double>(chunks, nchunks, heavy, nheavy,
                                                             colidx, vals, FT, r, YT, part, st)
                   : NMFB_ERR_ARG;
    return yt_dtype == NMFB_F64
               ? csr_yt_chunked_dispatch<float, double>(chunks, nchunks, heavy, nheavy, colidx,
                                                        vals, FT, r, YT, part, st)
               : csr_yt_chunked_dispatch<float, float>(chunks, nchunks, heavy, nheavy, colidx,
                                                       vals, FT, r, YT, part, st);
}

// Drop-in (nmfb_estep_sparse) accumulator: YT[row][i] += x[col][i] * v for the
// shard's columns in column order -- one thread per component walks the
// shard's nonzeros serially, which keeps the reference's per-entry order
// (kernels.py:270-274).  Check/drop-in path only; fit() uses csr_yt_kernel.
template <typename T>
__global__ void csc_scatter_yt_kernel(const int64_t *__restrict__ indptr,
                                      const int32_t *__restrict__ rowidx,
                                      const T *__restrict__ vals, int64_t lo, int64_t hi,
                                      const T *__restrict__ FT, int r, T *__restrict__ YT) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= r) return;
    for (int64_t col = lo; col < hi; ++col) {
        const T x = FT[col * r + i];
        for (int64_t t = indptr[col]; t < indptr[col + 1]; ++t) {
            T *dst = YT + (int64_t)rowidx[t] * r + i;
            *dst = Exact<T>::madd(*dst, x, vals[t]);
        }
    }
}

int csc_scatter_yt_launch(int dtype, const int64_t *indptr, const int32_t *rowidx,
                          const void *vals, int64_t lo, int64_t hi, const void *FT, int r,
                          void *YT, cudaStream_t st) {
    if (hi <= lo) return NMFB_OK;
    dim3 grid((unsigned)((r + 63) / 64));
    if (dtype == NMFB_F64)
        csc_scatter_yt_kernel<double><<<grid, 64, 0, st>>>(indptr, rowidx, (const double *)vals,
                                                          lo, hi, (const double *)FT, r,
                                                          (double *)YT);
    else
        csc_scatter_yt_kernel<float><<<grid, 64, 0, st>>>(indptr, rowidx, (const float *)vals, lo,
                                                         hi, (const float *)FT, r, (float *)YT);
    return launch_status();
}

}  // namespace nmfb
