// Sparse data products for large factors: 16-byte gathers up to r = 256 and
// L2 cache blocking of the gathered factor (at config 5 the
// gathers are 4 nnz r = 80 GB per pass, and G = 800 MB does not fit the
// 126 MB L2, so every pass streams the factor rows from HBM at random).
//
// Blocking: the factor's rows are cut into `nblk` blocks of `blk_rows` rows
// (each a few tens of MB, L2-resident while its pass runs).  Pass b walks,
// for every output (a CSC column for G^T X, a CSR row chunk for X F^T), only
// the entries whose gathered row lies in block b.  Storage keeps row indices
// ascending within a column (CSC) and column indices ascending within a row
// (CSR), so block b's entries of an output are ONE contiguous sub-range,
// located once per matrix by binary search (`seg`, (nout) x (nblk + 1)
// offsets).  The running sum of an output is carried between passes through
// its fp32 (or fp64) output slot: storing and reloading an accumulator of the
// same type is exact, so the blocked result is bit-identical to one
// sequential pass over the output's entries in storage order.
#include "common.cuh"
#include "nmfb_internal.h"

namespace nmfb {

namespace {

// seg[o * (nblk + 1) + b] = first entry of output o whose index >= b * blk
// (entries [ptr_lo(o), ptr_hi(o)) ascending); seg[..+nblk] = ptr_hi(o)
__global__ void segments_kernel(int64_t nout, const int64_t *__restrict__ lo_of,
                                int lo_stride, const int64_t *__restrict__ hi_of, int hi_stride,
                                const int32_t *__restrict__ idx, int64_t blk, int nblk,
                                int64_t *__restrict__ seg) {
    const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= nout) return;
    const int64_t p0 = lo_of[o * lo_stride], p1 = hi_of[o * hi_stride];
    int64_t *s = seg + o * (nblk + 1);
    s[0] = p0;
    int64_t at = p0;
    for (int b = 1; b < nblk; ++b) {
        const int64_t key = (int64_t)b * blk;
        int64_t a = at, z = p1;  // lower bound of key in [at, p1)
        while (a < z) {
            const int64_t mid = (a + z) >> 1;
            if ((int64_t)idx[mid] < key) a = mid + 1;
            else z = mid;
        }
        s[b] = at = a;
    }
    s[nblk] = p1;
}

// Streaming hints: the sparse indices / values and the h / Y^T rows are
// touched once per pass -- load / store them evict-first so they do not push
// the reused factor rows (G block, F^T) out of L2.
#ifndef NMFB_SPMM_STREAM_HINTS
#define NMFB_SPMM_STREAM_HINTS 1
#endif
// The outputs only when they exceed L2 (config 5's h / Y^T: 160 / 800 MB);
// an L2-sized output (config 3) is better left for the NNLS that reads it next.
#if NMFB_SPMM_STREAM_HINTS
#define NMFB_LDS_(p) __ldcs(p)
#define NMFB_STO_(p, v)       \
    do {                      \
        if (stream_out)       \
            __stcs((p), (v)); \
        else                  \
            *(p) = (v);       \
    } while (0)
#define NMFB_LDO_(p) (stream_out ? __ldcs(p) : *(p))
#else
#define NMFB_LDS_(p) (*(p))
#define NMFB_STO_(p, v) (*(p) = (v))
#define NMFB_LDO_(p) (*(p))
#endif
constexpr int64_t kStreamOutBytes = 64ll << 20;

#ifndef NMFB_CSC_MINB
#define NMFB_CSC_MINB 12  // <= 40 registers: C5 G^T X 5.85 -> 5.67 ms (16: spills, 8.1)
#endif
template <int NV>
__global__ void __launch_bounds__(128, NMFB_CSC_MINB) csc_linear_v4x_kernel(
    const int64_t *__restrict__ indptr, const int64_t *__restrict__ seg, int nblk, int b,
    const int32_t *__restrict__ rowidx, const float *__restrict__ vals, int64_t col_lo,
    int64_t col_hi, const float *__restrict__ G, int r, float mu1, float *__restrict__ h,
    bool stream_out) {
    const int64_t col = col_lo + (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (col >= col_hi) return;
    const int lane = threadIdx.x & 31;
    const int nq = r >> 2;
    float4 acc[NV];
    float4 *out = reinterpret_cast<float4 *>(h + (col - col_lo) * r);
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        const int c = lane + 32 * q;
        acc[q] = (b > 0 && c < nq) ? NMFB_LDO_(out + c) : make_float4(mu1, mu1, mu1, mu1);
    }
    int64_t p0, p1;
    if (seg) {
        p0 = seg[col * (nblk + 1) + b];
        p1 = seg[col * (nblk + 1) + b + 1];
    } else {
        p0 = indptr[col];
        p1 = indptr[col + 1];
    }
    for (int64_t base = p0; base < p1; base += 32) {
        const int cnt = (int)min((int64_t)32, p1 - base);
        int myrow = 0;
        float myv = 0.f;
        if (lane < cnt) {
            myrow = NMFB_LDS_(rowidx + base + lane);
            myv = NMFB_LDS_(vals + base + lane);
        }
#pragma unroll 8
        for (int u = 0; u < cnt; ++u) {
            const int row = __shfl_sync(NMFB_FULL_MASK, myrow, u);
            const float v = __shfl_sync(NMFB_FULL_MASK, myv, u);
            const float4 *g4 = reinterpret_cast<const float4 *>(G + (int64_t)row * r);
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                const int c = lane + 32 * q;
                if (c < nq) {
                    const float4 g = __ldg(g4 + c);
                    acc[q].x = fmaf(-g.x, v, acc[q].x);
                    acc[q].y = fmaf(-g.y, v, acc[q].y);
                    acc[q].z = fmaf(-g.z, v, acc[q].z);
                    acc[q].w = fmaf(-g.w, v, acc[q].w);
                }
            }
        }
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        const int c = lane + 32 * q;
        if (c < nq) NMFB_STO_(out + c, acc[q]);
    }
}

// TA: accumulation type (the heavy-row chunk partials too), TY: the Y^T
// output (fp32 Y^T is accumulated in fp64 and rounded once)
#ifndef NMFB_CSR_MINB
#define NMFB_CSR_MINB 10  // <= 48 registers: C5 X F^T 9.07 -> 6.70 ms (occupancy; 8: 7.24)
#endif
template <typename TA, typename TY, int NV>
__global__ void __launch_bounds__(128, NMFB_CSR_MINB) csr_yt_chunk_v4x_kernel(
    const int64_t *__restrict__ chunks, int64_t nchunks, const int64_t *__restrict__ seg, int nblk,
    int b, const int32_t *__restrict__ colidx, const float *__restrict__ vals,
    const float *__restrict__ FT, int r, TY *__restrict__ YT, TA *__restrict__ part,
    bool stream_out) {
    const int64_t ch = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (ch >= nchunks) return;
    const int lane = threadIdx.x & 31;
    const int nq = r >> 2;
    const int64_t row = chunks[ch * 4 + 0];
    const int64_t slot = chunks[ch * 4 + 3];
    int64_t p0 = chunks[ch * 4 + 1], p1 = chunks[ch * 4 + 2];
    if (seg) {
        p0 = seg[ch * (nblk + 1) + b];
        p1 = seg[ch * (nblk + 1) + b + 1];
    }
    TY *outy = YT + row * r;
    TA *outp = part + slot * r;
    TA a[NV][4];
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        const int c = lane + 32 * q;
#pragma unroll
        for (int t = 0; t < 4; ++t)
            a[q][t] = (b > 0 && c < nq) ? (slot < 0 ? (TA)outy[4 * c + t] : outp[4 * c + t])
                                        : TA(0);
    }
    for (int64_t base = p0; base < p1; base += 32) {
        const int cnt = (int)min((int64_t)32, p1 - base);
        int mycol = 0;
        float myv = 0.f;
        if (lane < cnt) {
            mycol = NMFB_LDS_(colidx + base + lane);
            myv = NMFB_LDS_(vals + base + lane);
        }
        if constexpr (sizeof(TY) == 8) {
            // fp64 Y^T (check / blocked passes): every product accumulated in fp64
#pragma unroll 8
            for (int u = 0; u < cnt; ++u) {
                const int col = __shfl_sync(NMFB_FULL_MASK, mycol, u);
                const float v = __shfl_sync(NMFB_FULL_MASK, myv, u);
                const float4 *f4 = reinterpret_cast<const float4 *>(FT + (int64_t)col * r);
#pragma unroll
                for (int q = 0; q < NV; ++q) {
                    const int c = lane + 32 * q;
                    if (c < nq) {
                        const float4 f = __ldg(f4 + c);
                        a[q][0] = fma((TA)f.x, (TA)v, a[q][0]);
                        a[q][1] = fma((TA)f.y, (TA)v, a[q][1]);
                        a[q][2] = fma((TA)f.z, (TA)v, a[q][2]);
                        a[q][3] = fma((TA)f.w, (TA)v, a[q][3]);
                    }
                }
            }
            continue;
        }
        // fp32 Y^T (production): up to 32 nonzeros summed in fp32 (packed
        // FFMA2), then folded into the fp64 running sums -- one conversion + DADD
        // per 32 products instead of per product (the batch sum is within 32
        // ulps; Y^T is stored fp32)
        float2 bsum[NV][2];
#pragma unroll
        for (int q = 0; q < NV; ++q) bsum[q][0] = bsum[q][1] = make_float2(0.f, 0.f);
#pragma unroll 8
        for (int u = 0; u < cnt; ++u) {
            const int col = __shfl_sync(NMFB_FULL_MASK, mycol, u);
            const float v = __shfl_sync(NMFB_FULL_MASK, myv, u);
            const float4 *f4 = reinterpret_cast<const float4 *>(FT + (int64_t)col * r);
            const float2 v2 = make_float2(v, v);
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                const int c = lane + 32 * q;
                if (c < nq) {
                    const float4 f = __ldg(f4 + c);
                    bsum[q][0] = __ffma2_rn(make_float2(f.x, f.y), v2, bsum[q][0]);
                    bsum[q][1] = __ffma2_rn(make_float2(f.z, f.w), v2, bsum[q][1]);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            a[q][0] += (TA)bsum[q][0].x;
            a[q][1] += (TA)bsum[q][0].y;
            a[q][2] += (TA)bsum[q][1].x;
            a[q][3] += (TA)bsum[q][1].y;
        }
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        const int c = lane + 32 * q;
        if (c < nq) {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                if (slot < 0)
                    NMFB_STO_(outy + 4 * c + t, (TY)a[q][t]);
                else
                    outp[4 * c + t] = a[q][t];
            }
        }
    }
}

template <typename TA, typename TY>
__global__ void csr_fold_kernel(const int64_t *__restrict__ heavy, int64_t nheavy, int r,
                                const TA *__restrict__ part, TY *__restrict__ YT) {
    const int64_t hv = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (hv >= nheavy) return;
    const int lane = threadIdx.x & 31;
    const int64_t row = heavy[hv * 3 + 0], s0 = heavy[hv * 3 + 1], ns = heavy[hv * 3 + 2];
    // slots summed in slot order per element (deterministic); eight elements
    // per lane and four slots unrolled keep ~32 independent loads in flight
    // instead of one dependent load per slot
    for (int i0 = 0; i0 < r; i0 += 256) {
        TA s[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int i = i0 + lane + 32 * q;
            s[q] = i < r ? part[s0 * r + i] : TA(0);
        }
        int64_t k = 1;
        for (; k + 4 <= ns; k += 4) {
            // all 32 loads issued before the first add consumes one
            TA v[4][8];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int i = i0 + lane + 32 * q;
                    v[u][q] = i < r ? __ldg(part + (s0 + k + u) * r + i) : TA(0);
                }
            asm volatile("" ::: "memory");  // keep the loads ahead of the adds
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int q = 0; q < 8; ++q) s[q] += v[u][q];
        }
        for (; k < ns; ++k) {
            TA v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int i = i0 + lane + 32 * q;
                v[q] = i < r ? __ldg(part + (s0 + k) * r + i) : TA(0);
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) s[q] += v[q];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int i = i0 + lane + 32 * q;
            if (i < r) YT[row * r + i] = (TY)s[q];
        }
    }
}

inline bool vec_ok(int r, const void *a) {
    return r % 4 == 0 && r <= 256 && ((uintptr_t)a % 16) == 0;
}

}  // namespace

// true when the vectorised kernels below apply (fp32 data, r % 4 == 0, r <= 256)
bool sparse_vec_ok(int r, const void *a, const void *b) { return vec_ok(r, a) && vec_ok(r, b); }

int csc_segments_launch(const int64_t *indptr, const int32_t *rowidx, int64_t m, int64_t blk,
                        int nblk, int64_t *seg, cudaStream_t st) {
    if (m <= 0) return NMFB_OK;
    if (nblk < 1 || blk < 1 || !indptr || !seg) return NMFB_ERR_ARG;
    segments_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(m, indptr, 1, indptr + 1, 1,
                                                                rowidx, blk, nblk, seg);
    return launch_status();
}

int chunk_segments_launch(const int64_t *chunks, int64_t nchunks, const int32_t *colidx,
                          int64_t blk, int nblk, int64_t *seg, cudaStream_t st) {
    if (nchunks <= 0) return NMFB_OK;
    if (nblk < 1 || blk < 1 || !chunks || !seg) return NMFB_ERR_ARG;
    segments_kernel<<<(unsigned)((nchunks + 255) / 256), 256, 0, st>>>(
        nchunks, chunks + 1, 4, chunks + 2, 4, colidx, blk, nblk, seg);
    return launch_status();
}

int csc_linear_vec_launch(const int64_t *indptr, const int64_t *seg, int nblk,
                          const int32_t *rowidx, const float *vals, int64_t lo, int64_t hi,
                          const float *G, int r, double mu1, float *h, cudaStream_t st) {
    if (hi <= lo) return NMFB_OK;
    if (!sparse_vec_ok(r, G, h) || nblk < 1 || (seg && lo != 0)) return NMFB_ERR_ARG;
    const dim3 grid((unsigned)((hi - lo + 3) / 4));
    const bool so = (hi - lo) * r * (int64_t)sizeof(float) > kStreamOutBytes;
    for (int b = 0; b < (seg ? nblk : 1); ++b) {
        if (r <= 128)
            csc_linear_v4x_kernel<1><<<grid, 128, 0, st>>>(indptr, seg, nblk, b, rowidx, vals, lo,
                                                           hi, G, r, (float)mu1, h, so);
        else
            csc_linear_v4x_kernel<2><<<grid, 128, 0, st>>>(indptr, seg, nblk, b, rowidx, vals, lo,
                                                           hi, G, r, (float)mu1, h, so);
    }
    return launch_status();
}

template <typename TY>
static int csr_vec_go(const int64_t *chunks, int64_t nchunks, const int64_t *heavy, int64_t nheavy,
                      const int64_t *seg, int nblk, const int32_t *colidx, const float *vals,
                      const float *FT, int r, TY *YT, double *part, cudaStream_t st) {
    const dim3 grid((unsigned)((nchunks + 3) / 4));
    // (the chunk count bounds the row count from above)
    const bool so = nchunks * r * (int64_t)sizeof(TY) > kStreamOutBytes;
    for (int b = 0; b < (seg ? nblk : 1); ++b) {
        if (r <= 128)
            csr_yt_chunk_v4x_kernel<double, TY, 1><<<grid, 128, 0, st>>>(
                chunks, nchunks, seg, nblk, b, colidx, vals, FT, r, YT, part, so);
        else
            csr_yt_chunk_v4x_kernel<double, TY, 2><<<grid, 128, 0, st>>>(
                chunks, nchunks, seg, nblk, b, colidx, vals, FT, r, YT, part, so);
    }
    if (nheavy > 0)
        csr_fold_kernel<double, TY><<<(unsigned)((nheavy + 3) / 4), 128, 0, st>>>(
            heavy, nheavy, r, part, YT);
    return launch_status();
}

int csr_yt_chunked_vec_launch(const int64_t *chunks, int64_t nchunks, const int64_t *heavy,
                              int64_t nheavy, const int64_t *seg, int nblk, const int32_t *colidx,
                              const float *vals, const float *FT, int r, int yt_dtype, void *YT,
                              void *part, cudaStream_t st) {
    if (nchunks <= 0) return NMFB_OK;
    if (!sparse_vec_ok(r, FT, FT) || nblk < 1) return NMFB_ERR_ARG;
    // fp64 accumulation (and fp64 heavy-row partials) for either output type
    if (yt_dtype == NMFB_F64)
        return csr_vec_go<double>(chunks, nchunks, heavy, nheavy, seg, nblk, colidx, vals, FT, r,
                                  (double *)YT, (double *)part, st);
    return csr_vec_go<float>(chunks, nchunks, heavy, nheavy, seg, nblk, colidx, vals, FT, r,
                             (float *)YT, (double *)part, st);
}

}  // namespace nmfb
