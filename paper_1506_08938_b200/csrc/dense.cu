// Dense data products of the alternation (kernels.py:251-258/306-313 linear
// terms G^T X, kernels.py:270-274/325-329 accumulator Y^T = X F^T), their
// reference-order check-mode twins, the F F^T accumulator in reference order
// (kernels.py:276-280 + parallel.py:127-128, 150-156) and the dense residual
// objective (matrix.py:254-260) without materialising G F.
#include <cfloat>

#include "common.cuh"
#include "nmfb_internal.h"

namespace nmfb {

// ---------------------------------------------------------------------------
// Split-K tall-skinny SIMT GEMM (fp32 FFMA).  C[s] = A(:, Ks) * B(Ks, :).
// BM=128 x BN=64 tile, BK=16, 256 threads, 8x4 register block per thread,
// register-prefetched double buffer.  X is streamed once per pass (the HBM
// term); B (G or F^T, K x r) is L2-resident.
// ---------------------------------------------------------------------------
constexpr int BM = 128, BN = 64, BK = 16;

template <bool AK, bool VEC>
__global__ void __launch_bounds__(256) gemm_tall_kernel(const float *__restrict__ A, int64_t M,
                                                        int64_t K, int64_t lda,
                                                        const float *__restrict__ B, int N,
                                                        int64_t ldb, float *__restrict__ C,
                                                        int64_t kchunk) {
    __shared__ __align__(16) float As[2][BK][BM + 4];
    __shared__ __align__(16) float Bs[2][BK][BN];
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int64_t m0 = (int64_t)blockIdx.x * BM;
    const int n0 = blockIdx.y * BN;
    const int64_t k0 = (int64_t)blockIdx.z * kchunk;
    const int64_t k1 = min(K, k0 + kchunk);
    float *Cs = C + (int64_t)blockIdx.z * M * N;

    float acc[8][4];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.f;

    float ra[8], rb[4];
    auto load_tile = [&](int64_t kb) {
        if (AK) {
            // A(i, k) = A[i*lda + k]; thread: rows (tid>>2) + 64q, k quad (tid&3)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                int row = (tid >> 2) + 64 * q;
                int kq = (tid & 3) * 4;
                int64_t gi = m0 + row, gk = kb + kq;
                if (VEC && gi < M && gk + 3 < k1) {
                    float4 v = *reinterpret_cast<const float4 *>(A + gi * lda + gk);
                    ra[q * 4 + 0] = v.x;
                    ra[q * 4 + 1] = v.y;
                    ra[q * 4 + 2] = v.z;
                    ra[q * 4 + 3] = v.w;
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        ra[q * 4 + c] = (gi < M && gk + c < k1) ? A[gi * lda + gk + c] : 0.f;
                }
            }
        } else {
            // A(i, k) = A[k*lda + i]; thread: k (tid>>5) + 8q, i quad (tid&31)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                int kk = (tid >> 5) + 8 * q;
                int iq = (tid & 31) * 4;
                int64_t gi = m0 + iq, gk = kb + kk;
                if (VEC && gk < k1 && gi + 3 < M) {
                    float4 v = *reinterpret_cast<const float4 *>(A + gk * lda + gi);
                    ra[q * 4 + 0] = v.x;
                    ra[q * 4 + 1] = v.y;
                    ra[q * 4 + 2] = v.z;
                    ra[q * 4 + 3] = v.w;
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        ra[q * 4 + c] = (gk < k1 && gi + c < M) ? A[gk * lda + gi + c] : 0.f;
                }
            }
        }
        // B tile BK x BN: thread loads 4 consecutive columns of one k row
        {
            int kk = tid >> 4;
            int c0 = (tid & 15) * 4;
            int64_t gk = kb + kk;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                int gc = n0 + c0 + c;
                rb[c] = (gk < k1 && gc < N) ? B[gk * ldb + gc] : 0.f;
            }
        }
    };
    auto store_tile = [&](int buf) {
        if (AK) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                int row = (tid >> 2) + 64 * q;
                int kq = (tid & 3) * 4;
#pragma unroll
                for (int c = 0; c < 4; ++c) As[buf][kq + c][row] = ra[q * 4 + c];
            }
        } else {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                int kk = (tid >> 5) + 8 * q;
                int iq = (tid & 31) * 4;
                *reinterpret_cast<float4 *>(&As[buf][kk][iq]) =
                    make_float4(ra[q * 4 + 0], ra[q * 4 + 1], ra[q * 4 + 2], ra[q * 4 + 3]);
            }
        }
        int kk = tid >> 4;
        int c0 = (tid & 15) * 4;
        *reinterpret_cast<float4 *>(&Bs[buf][kk][c0]) = make_float4(rb[0], rb[1], rb[2], rb[3]);
    };

    if (k0 < k1) {
        load_tile(k0);
        store_tile(0);
        __syncthreads();
        int buf = 0;
        for (int64_t kb = k0; kb < k1; kb += BK) {
            const bool more = kb + BK < k1;
            if (more) load_tile(kb + BK);
#pragma unroll
            for (int kk = 0; kk < BK; ++kk) {
                float4 a0 = *reinterpret_cast<const float4 *>(&As[buf][kk][ty * 8]);
                float4 a1 = *reinterpret_cast<const float4 *>(&As[buf][kk][ty * 8 + 4]);
                float4 b0 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][tx * 4]);
                float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                float bv[4] = {b0.x, b0.y, b0.z, b0.w};
#pragma unroll
                for (int u = 0; u < 8; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(av[u], bv[v], acc[u][v]);
            }
            if (more) {
                store_tile(buf ^ 1);
                __syncthreads();
                buf ^= 1;
            }
        }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        int64_t gi = m0 + ty * 8 + u;
        if (gi >= M) continue;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            int gc = n0 + tx * 4 + v;
            if (gc < N) Cs[gi * N + gc] = acc[u][v];
        }
    }
}

int gemm_tall_launch(const float *A, int a_kmajor, int64_t M, int64_t K, int64_t lda,
                     const float *B, int N, int64_t ldb, float *C, int splits, cudaStream_t st) {
    if (M < 0 || K < 0 || N <= 0 || splits < 1) return NMFB_ERR_ARG;
    if (M == 0) return NMFB_OK;
    int64_t kchunk = (K + splits - 1) / splits;
    kchunk = ((kchunk + BK - 1) / BK) * BK;
    if (kchunk == 0) kchunk = BK;
    dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((N + BN - 1) / BN), (unsigned)splits);
    bool vec = (lda % 4 == 0) && ((uintptr_t)A % 16 == 0);
    if (K == 0 || (int64_t)(splits - 1) * kchunk >= K) {
        // empty chunks still write zeros: handled by the kernel (k0 >= k1)
    }
    if (a_kmajor) {
        if (vec)
            gemm_tall_kernel<true, true><<<grid, 256, 0, st>>>(A, M, K, lda, B, N, ldb, C, kchunk);
        else
            gemm_tall_kernel<true, false><<<grid, 256, 0, st>>>(A, M, K, lda, B, N, ldb, C, kchunk);
    } else {
        if (vec)
            gemm_tall_kernel<false, true><<<grid, 256, 0, st>>>(A, M, K, lda, B, N, ldb, C, kchunk);
        else
            gemm_tall_kernel<false, false><<<grid, 256, 0, st>>>(A, M, K, lda, B, N, ldb, C,
                                                                 kchunk);
    }
    return launch_status();
}

// ---------------------------------------------------------------------------
// Reference-order dense products (check mode).  Warp per data column, lanes
// over components; every sum in the reference's index order, no contraction.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void dense_linear_ref_kernel(const T *__restrict__ VT, int64_t n, int64_t col_lo,
                                        int64_t col_hi, const T *__restrict__ G, int r, T mu1,
                                        T *__restrict__ h) {
    using O = Exact<T>;
    int64_t col = col_lo + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (col >= col_hi) return;
    const int lane = threadIdx.x & 31;
    const T *v = VT + col * n;
    for (int i0 = 0; i0 < r; i0 += 32) {
        int i = i0 + lane;
        T acc = mu1;
        for (int64_t row = 0; row < n; ++row) {
            T vv = v[row];
            if (vv != T(0) && i < r) acc = O::msub(acc, G[row * r + i], vv);
        }
        if (i < r) h[(col - col_lo) * r + i] = acc;
    }
}

struct Shards {
    int64_t b[NMFB_MAX_WORKERS + 1];
    int w;
};

template <typename T>
__global__ void dense_yt_ref_kernel(const T *__restrict__ VT, int64_t m, int64_t n,
                                    const T *__restrict__ FT, int r, Shards sh,
                                    T *__restrict__ YT) {
    using O = Exact<T>;
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * r) return;
    int64_t row = idx / r;
    int i = (int)(idx % r);
    T total = T(0);
    for (int w = 0; w < sh.w; ++w) {
        T acc = T(0);
        for (int64_t col = sh.b[w]; col < sh.b[w + 1]; ++col) {
            T v = VT[col * n + row];
            if (v != T(0)) acc = O::madd(acc, FT[col * r + i], v);
        }
        total = O::add(total, acc);
    }
    YT[idx] = total;
}

template <typename T>
__global__ void hp_ref_kernel(const T *__restrict__ FT, int64_t m, int r, Shards sh,
                              T *__restrict__ HF) {
    using O = Exact<T>;
    int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= r * r) return;
    int a = idx / r, b = idx % r;
    if (b < a) return;
    T total = T(0);
    for (int w = 0; w < sh.w; ++w) {
        T acc = T(0);
        for (int64_t col = sh.b[w]; col < sh.b[w + 1]; ++col) {
            T xa = FT[col * r + a];
            if (xa != T(0)) acc = O::madd(acc, xa, FT[col * r + b]);
        }
        total = O::add(total, acc);
    }
    HF[a * r + b] = total;
    HF[b * r + a] = total;
}

static bool make_shards(const int64_t *bounds, int workers, Shards &sh) {
    if (workers < 1 || workers > NMFB_MAX_WORKERS) return false;
    sh.w = workers;
    for (int i = 0; i <= workers; ++i) sh.b[i] = bounds[i];
    return true;
}

int dense_linear_ref_launch(int dtype, const void *VT, int64_t n, int64_t col_lo, int64_t col_hi,
                            const void *G, int r, double mu1, void *h, cudaStream_t st) {
    int64_t cols = col_hi - col_lo;
    if (cols <= 0) return NMFB_OK;
    dim3 grid((unsigned)((cols + 3) / 4));
    if (dtype == NMFB_F64)
        dense_linear_ref_kernel<double><<<grid, 128, 0, st>>>((const double *)VT, n, col_lo,
                                                              col_hi, (const double *)G, r, mu1,
                                                              (double *)h);
    else
        dense_linear_ref_kernel<float><<<grid, 128, 0, st>>>((const float *)VT, n, col_lo, col_hi,
                                                             (const float *)G, r, (float)mu1,
                                                             (float *)h);
    return launch_status();
}

int dense_yt_ref_launch(int dtype, const void *VT, int64_t m, int64_t n, const void *FT, int r,
                        const int64_t *bounds, int workers, void *YT, cudaStream_t st) {
    Shards sh;
    if (!make_shards(bounds, workers, sh)) return NMFB_ERR_ARG;
    int64_t tot = n * r;
    if (tot == 0) return NMFB_OK;
    dim3 grid((unsigned)((tot + 255) / 256));
    if (dtype == NMFB_F64)
        dense_yt_ref_kernel<double><<<grid, 256, 0, st>>>((const double *)VT, m, n,
                                                          (const double *)FT, r, sh, (double *)YT);
    else
        dense_yt_ref_kernel<float><<<grid, 256, 0, st>>>((const float *)VT, m, n,
                                                         (const float *)FT, r, sh, (float *)YT);
    return launch_status();
}

int hp_ref_launch(int dtype, const void *FT, int64_t m, int r, const int64_t *bounds,
                  int workers, void *HF, cudaStream_t st) {
    Shards sh;
    if (!make_shards(bounds, workers, sh)) return NMFB_ERR_ARG;
    dim3 grid((unsigned)((r * r + 255) / 256));
    if (dtype == NMFB_F64)
        hp_ref_kernel<double><<<grid, 256, 0, st>>>((const double *)FT, m, r, sh, (double *)HF);
    else
        hp_ref_kernel<float><<<grid, 256, 0, st>>>((const float *)FT, m, r, sh, (float *)HF);
    return launch_status();
}

// ---------------------------------------------------------------------------
// Dense residual 0.5 ||X - G F||^2, X as XT (m, n).  Tile 64 (m) x 64 (n),
// K = r streamed through shared memory in slabs of 16; 256 threads, 4x4 per
// thread; residual squared-summed in fp32 per thread then fp64 per CTA.
// ---------------------------------------------------------------------------
constexpr int RT = 64, RK = 16;

template <typename T>
__global__ void __launch_bounds__(256) residual_kernel(const T *__restrict__ XT, int64_t m,
                                                       int64_t n, const T *__restrict__ G,
                                                       const T *__restrict__ FT, int r,
                                                       double *__restrict__ part) {
    __shared__ T Fs[RK][RT + 1];
    __shared__ T Gs[RK][RT + 1];
    __shared__ double red[256];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t j0 = (int64_t)blockIdx.y * RT;   // m (columns of X)
    const int64_t r0 = (int64_t)blockIdx.x * RT;   // n (rows of X)
    T acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = T(0);
    for (int kb = 0; kb < r; kb += RK) {
        for (int idx = tid; idx < RK * RT; idx += 256) {
            int t = idx / RK, kk = idx % RK;
            int64_t gj = j0 + t, gr = r0 + t;
            int gk = kb + kk;
            Fs[kk][t] = (gj < m && gk < r) ? FT[gj * r + gk] : T(0);
            Gs[kk][t] = (gr < n && gk < r) ? G[gr * r + gk] : T(0);
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < RK; ++kk) {
            T a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) a[u] = Fs[kk][ty * 4 + u];
#pragma unroll
            for (int v = 0; v < 4; ++v) b[v] = Gs[kk][tx + 16 * v];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
        }
        __syncthreads();
    }
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        int64_t gj = j0 + ty * 4 + u;
        T su = T(0);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            int64_t gr = r0 + tx + 16 * v;
            if (gj < m && gr < n) {
                T d = XT[gj * n + gr] - acc[u][v];
                su = fma(d, d, su);
            }
        }
        s += (double)su;
    }
    red[tid] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (tid < o) red[tid] += red[tid + o];
        __syncthreads();
    }
    if (tid == 0) part[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = red[0];
}

// fp32 production residual: CTA tile 128 (m, columns of X) x 128 (n, rows of
// X), 256 threads with an 8x8 register block each, K = r staged through
// shared memory 32 at a time ([k][j] layouts -> float4 reads).  FFMA-bound:
// 2*n*m*r flops; the residual itself is formed and squared in fp32
// (round-to-nearest, unbiased) and summed in fp64 per CTA.
constexpr int R2T = 128, R2K = 32;

// Operands are the k-major copies the tensor-core passes already keep:
// Gt (r x n) = G^T and Ft (r x m) = F, so every smem fill is a coalesced,
// bank-conflict-free row copy.
__global__ void __launch_bounds__(256, 2) residual_f32_kernel(const float *__restrict__ XT,
                                                              int64_t m, int64_t n,
                                                              const float *__restrict__ Gt,
                                                              const float *__restrict__ Ft,
                                                              int r, double *__restrict__ part) {
    __shared__ __align__(16) float Fs[R2K][R2T];
    __shared__ __align__(16) float Gs[R2K][R2T];
    __shared__ double red[8];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t j0 = (int64_t)blockIdx.y * R2T;  // m
    const int64_t r0 = (int64_t)blockIdx.x * R2T;  // n
    // warm L2 with this CTA's X tile (128 rows x 512 B) so the epilogue's
    // reads do not pay HBM latency after the k-loop
    for (int l = tid; l < R2T * 4; l += 256) {
        const int64_t gj = j0 + (l >> 2), gr = r0 + (l & 3) * 32;
        if (gj < m && gr < n) asm volatile("prefetch.global.L2 [%0];" ::"l"(XT + gj * n + gr));
    }
    float acc[8][8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[u][v] = 0.f;
    for (int kb = 0; kb < r; kb += R2K) {
        // float4 row copies (4 per thread per operand); scalar tail guards
        for (int idx = tid; idx < R2K * (R2T / 4); idx += 256) {
            const int kk = idx >> 5, t4 = (idx & 31) * 4;
            const int gk = kb + kk;
            const int64_t gj = j0 + t4, gr = r0 + t4;
            float4 fv = make_float4(0.f, 0.f, 0.f, 0.f), gv = fv;
            if (gk < r) {
                const float *fp = Ft + (int64_t)gk * m + gj;
                const float *gp = Gt + (int64_t)gk * n + gr;
                if ((m % 4) == 0 && gj + 3 < m) {
                    fv = *reinterpret_cast<const float4 *>(fp);
                } else {
                    fv.x = (gj < m) ? fp[0] : 0.f;
                    fv.y = (gj + 1 < m) ? fp[1] : 0.f;
                    fv.z = (gj + 2 < m) ? fp[2] : 0.f;
                    fv.w = (gj + 3 < m) ? fp[3] : 0.f;
                }
                if ((n % 4) == 0 && gr + 3 < n) {
                    gv = *reinterpret_cast<const float4 *>(gp);
                } else {
                    gv.x = (gr < n) ? gp[0] : 0.f;
                    gv.y = (gr + 1 < n) ? gp[1] : 0.f;
                    gv.z = (gr + 2 < n) ? gp[2] : 0.f;
                    gv.w = (gr + 3 < n) ? gp[3] : 0.f;
                }
            }
            *reinterpret_cast<float4 *>(&Fs[kk][t4]) = fv;
            *reinterpret_cast<float4 *>(&Gs[kk][t4]) = gv;
        }
        __syncthreads();
        const int kmax = min(R2K, r - kb);
#pragma unroll 4
        for (int kk = 0; kk < kmax; ++kk) {
            const float4 a0 = *reinterpret_cast<const float4 *>(&Fs[kk][ty * 8]);
            const float4 a1 = *reinterpret_cast<const float4 *>(&Fs[kk][ty * 8 + 4]);
            // thread columns {4tx..4tx+3} u {64+4tx..}: 16 lanes read 256
            // contiguous bytes per float4 load (no 32-byte-stride conflicts)
            const float4 b0 = *reinterpret_cast<const float4 *>(&Gs[kk][tx * 4]);
            const float4 b1 = *reinterpret_cast<const float4 *>(&Gs[kk][64 + tx * 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float2 b2[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w),
                                  make_float2(b1.x, b1.y), make_float2(b1.z, b1.w)};
            // sm_100 packed FFMA2: two round-to-nearest FMAs per instruction
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const float2 au = make_float2(a[u], a[u]);
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    float2 c = make_float2(acc[u][2 * v], acc[u][2 * v + 1]);
                    c = __ffma2_rn(au, b2[v], c);
                    acc[u][2 * v] = c.x;
                    acc[u][2 * v + 1] = c.y;
                }
            }
        }
        __syncthreads();
    }
    double s = 0.0;
    auto colof = [&](int v) { return r0 + (v < 4 ? tx * 4 + v : 64 + tx * 4 + (v - 4)); };
    const bool vec = (n % 4 == 0) && (colof(7) < n);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int64_t gj = j0 + ty * 8 + u;
        if (gj >= m) continue;
        const float *xrow = XT + gj * n;
        float x[8];
        if (vec) {
            const float4 x0 = *reinterpret_cast<const float4 *>(xrow + colof(0));
            const float4 x1 = *reinterpret_cast<const float4 *>(xrow + colof(4));
            x[0] = x0.x; x[1] = x0.y; x[2] = x0.z; x[3] = x0.w;
            x[4] = x1.x; x[5] = x1.y; x[6] = x1.z; x[7] = x1.w;
        } else {
#pragma unroll
            for (int v = 0; v < 8; ++v) x[v] = (colof(v) < n) ? xrow[colof(v)] : 0.f;
        }
        float su = 0.f;
#pragma unroll
        for (int v = 0; v < 8; ++v) {
            if (colof(v) < n) {
                const float d = x[v] - acc[u][v];
                su = fmaf(d, d, su);
            }
        }
        s += (double)su;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(NMFB_FULL_MASK, s, o);
    if ((tid & 31) == 0) red[tid >> 5] = s;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        part[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

__global__ void sum_parts_kernel(const double *__restrict__ part, int64_t np, double scale,
                                 double *__restrict__ out) {
    __shared__ double red[256];
    double s = 0.0;
    // fixed per-thread strided order + fixed tree => deterministic
    for (int64_t i = threadIdx.x; i < np; i += 256) s += part[i];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out += scale * red[0];
}

size_t residual_workspace_bytes(int64_t m, int64_t n) {
    // sized for the smaller (fp64) tile, which has the most CTAs
    return (size_t)((m + RT - 1) / RT) * (size_t)((n + RT - 1) / RT) * sizeof(double);
}

int dense_residual_launch(int dtype, const void *XT, int64_t m, int64_t n, const void *G,
                          const void *FT, int r, double *out, void *ws, cudaStream_t st) {
    if (m <= 0 || n <= 0) return NMFB_OK;
    double *part = (double *)ws;
    int64_t gx = (n + RT - 1) / RT, gy = (m + RT - 1) / RT;
    if (gy > 65535) return NMFB_ERR_ARG;
    dim3 grid((unsigned)gx, (unsigned)gy);
    if (dtype == NMFB_F64)
        residual_kernel<double><<<grid, 256, 0, st>>>((const double *)XT, m, n,
                                                      (const double *)G, (const double *)FT, r,
                                                      part);
    else
        residual_kernel<float><<<grid, 256, 0, st>>>((const float *)XT, m, n, (const float *)G,
                                                     (const float *)FT, r, part);
    sum_parts_kernel<<<1, 256, 0, st>>>(part, gx * gy, 0.5, out);
    return launch_status();
}

int dense_residual_kmajor_launch(const float *XT, int64_t m, int64_t n, const float *Gt,
                                 const float *Ft, int r, double *out, void *ws,
                                 cudaStream_t st) {
    if (m <= 0 || n <= 0) return NMFB_OK;
    double *part = (double *)ws;
    int64_t gx = (n + R2T - 1) / R2T, gy = (m + R2T - 1) / R2T;
    if (gy > 65535) return NMFB_ERR_ARG;
    residual_f32_kernel<<<dim3((unsigned)gx, (unsigned)gy), 256, 0, st>>>(XT, m, n, Gt, Ft, r,
                                                                          part);
    sum_parts_kernel<<<1, 256, 0, st>>>(part, gx * gy, 0.5, out);
    return launch_status();
}

}  // namespace nmfb
