// Dense objective 0.5 ||X - G F||_F^2 on the int8 tensor cores, EXACTLY
// (matrix.py:227-260 frobenius_objective; nmf.py:152-165).
//
// Why not tf32: the tensor core's fp32 accumulate truncates, so a 3xTF32 G F
// is biased low by ~1e-6 relative, and the residual X - G F is ~2e-3 of X at
// a good fit -- the objective would be biased by ~1e-3.  Integer MMAs are
// exact, so G F is formed from 8-bit slices (Ozaki-style splitting):
//
//   G[i][k] = s_i (g0 2^-8 + g1 2^-16 + g2 2^-24),   s_i = 2^e, G/s_i in [0,1)
//   F[k][j] = t_j (f0 2^-8 + f1 2^-16 + f2 2^-24)    (G, F >= 0: NNLS outputs)
//   (G F)[i][j] = s_i t_j 2^-16 (A0 + 2^-8 A1 + 2^-16 A2) + O(2^-24)
//   A0 = g0.f0,  A1 = g0.f1 + g1.f0,  A2 = g0.f2 + g1.f1 + g2.f0
//
// Six u8 x u8 -> s32 products (tcgen05.mma kind::i8, exact), one TMEM
// accumulator per order.  The epilogue combines the orders into one unsigned
// integer (2^8 A0 + A1 + round(2^-8 A2) < 2^32), converts it once
// (round-to-nearest: unbiased), subtracts from the X tile, squares in fp32 and
// sums in fp64.  Accuracy ~2^-24 relative on G F, unbiased -- at least as
// good as an fp32 FFMA dot product, at tensor-core speed.
//
// Persistent kernel, one CTA per SM, tiles of 128 rows (i, n-dim) x 80
// columns (j, m-dim) walked in row-major order in equal runs per CTA:
//   warp 0     TMA: G slices of the row block (48 KB, reloaded when the row
//              block changes), F slices per tile (30 KB, 2 stages), X tile
//              (128 x 84 fp32, 2 stages; 84-float rows keep the epilogue's
//              float4 reads conflict-free)
//   warp 1     MMA: 6 products x ceil(r/32) k-steps into the tile's 3
//              accumulators (2 x 3 x 80 = 480 TMEM columns, double-buffered)
//   warps 4-23 epilogue: TMEM lanes = rows of the tile, five warps per lane
//              quarter (16 columns each); the three orders are combined in
//              integer arithmetic, converted once, and consumed with packed
//              FP32x2 math
// Bound: HBM reads of X (4 B per element, 0.12 ms per 2e8 elements at the
// measured peak) against ~93 ns per u8 MMA (12 per 128 x 80 tile) and the
// epilogue's issue rate; the FFMA kernel needs 2r flops per element
// (0.27 ms at the fp32 peak for r = 50).
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "nmfb_internal.h"
#include "tcgen05.cuh"

namespace nmfb {

constexpr int RQ_BM = 128;     // rows of X per tile (TMEM lanes)
constexpr int RQ_BN = 80;      // columns of X per tile (MMA N)
constexpr int RQ_XLD = 84;     // smem row pitch of the X tile (floats)
constexpr int RQ_KB = 128;     // max bytes per slice row (r <= 128); 64 when r <= 64
constexpr int RQ_CW = 16;        // epilogue columns per warp (one x16 TMEM load per order)
constexpr int RQ_EPW = RQ_BN / RQ_CW;  // epilogue warps per TMEM lane quarter (5)
constexpr int RQ_EPI = 128 * RQ_EPW;  // epilogue threads
constexpr int RQ_THREADS = 128 + RQ_EPI;  // TMA, MMA, 2 idle, epilogue warps

// ---------------------------------------------------------------------------
// slicing: one warp per row of A (rows x r fp32, lda), r <= 128.
// S: 3 slices, each rows x 128 bytes (zero beyond r); scale[row] = 2^e.
// ---------------------------------------------------------------------------
__global__ void slice_u8_kernel(const float *__restrict__ A, int64_t rows, int r, int64_t lda,
                                int kb, uint8_t *__restrict__ S, float *__restrict__ scale) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    float v[4];
    float mx = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int k = lane * 4 + q;
        // NNLS outputs are >= 0; anything else is clamped (never produced)
        v[q] = k < r ? fmaxf(A[row * lda + k], 0.f) : 0.f;
        mx = fmaxf(mx, v[q]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    int e = 0;
    if (mx > 0.f) frexpf(mx, &e);  // mx = f 2^e, f in [0.5, 1) -> v / 2^e < 1
    const float inv = ldexpf(1.f, -e);
    uint32_t w0 = 0, w1 = 0, w2 = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        float t = v[q] * inv * 256.f;  // exact (power-of-two scaling)
        float d0 = floorf(t);
        t = (t - d0) * 256.f;           // exact
        float d1 = floorf(t);
        t = (t - d1) * 256.f;
        float d2 = rintf(t);            // last slice rounded to nearest (unbiased)
        if (d2 == 256.f) {              // carry; d0 < 255 here since v < 2^e
            d2 = 0.f;
            d1 += 1.f;
            if (d1 == 256.f) {
                d1 = 0.f;
                d0 += 1.f;
            }
        }
        w0 |= (uint32_t)d0 << (8 * q);
        w1 |= (uint32_t)d1 << (8 * q);
        w2 |= (uint32_t)d2 << (8 * q);
    }
    if (lane * 4 < kb) {
        uint32_t *s0 = reinterpret_cast<uint32_t *>(S + row * kb);
        uint32_t *s1 = reinterpret_cast<uint32_t *>(S + (rows + row) * kb);
        uint32_t *s2 = reinterpret_cast<uint32_t *>(S + (2 * rows + row) * kb);
        s0[lane] = w0;
        s1[lane] = w1;
        s2[lane] = w2;
    }
    if (lane == 0) scale[row] = ldexpf(1.f, e);
}

__device__ __forceinline__ void umma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// issued by one elected lane of a converged warp
__device__ __forceinline__ void umma_i8_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p, e;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}

// K-major u8 operand, KB-byte rows: SWIZZLE_64B (layout 4, 8-row atoms of
// 512 B) for KB = 64, SWIZZLE_128B (layout 2, 1024 B atoms) for KB = 128
template <int KB>
__device__ __forceinline__ uint64_t desc_u8(const void *p) {
    uint64_t d = (uint64_t)((smem_u32(p) & 0x3FFFFu) >> 4);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)((8 * KB) >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)(KB == 64 ? 4 : 2) << 61;
    return d;
}

__device__ __forceinline__ long long gtime() {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

struct RqSched {
    int row_blocks, col_tiles;
    int64_t T;  // row_blocks * col_tiles
    int G;      // grid
};
__device__ __forceinline__ int64_t rq_start(const RqSched &s, int b) {
    return (int64_t)b * s.T / s.G;
}

template <int KB, int NF, int NX, int KS>
__global__ void __launch_bounds__(RQ_THREADS, 1)
    residual_i8_kernel(const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmF,
                       const __grid_constant__ CUtensorMap tmX, const float *__restrict__ sg,
                       const float *__restrict__ sf, int64_t n, int64_t m,
                       const RqSched sched, double *__restrict__ part, int dbg) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    constexpr uint32_t g_slice = RQ_BM * KB;                   // 8 / 16 KB
    constexpr uint32_t f_slice = RQ_BN * KB;                   // 5 / 10 KB
    constexpr uint32_t g_bytes = 3 * g_slice;
    constexpr uint32_t f_bytes = 3 * f_slice;
    constexpr uint32_t f_pitch = f_bytes;
    constexpr uint32_t x_bytes = RQ_BM * RQ_XLD * 4;           // 42 KB
    uint8_t *gs = smem;
    uint8_t *fs = gs + g_bytes;                                // NF stages
    float *xs = reinterpret_cast<float *>(fs + NF * f_pitch);  // NX stages
    uint64_t *bars = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(xs) + NX * x_bytes);
    uint64_t *g_full = bars, *g_empty = bars + 1;
    uint64_t *f_full = bars + 2, *f_empty = f_full + NF;
    uint64_t *x_full = f_empty + NF, *x_empty = x_full + NX;
    uint64_t *acc_full = x_empty + NX, *acc_empty = acc_full + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + 2);
    __shared__ double red[4 * RQ_EPW];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        if (lane == 0) {
            mbar_init(g_full, 1);
            mbar_init(g_empty, 1);
            for (int s = 0; s < NF; ++s) {
                mbar_init(&f_full[s], 1);
                mbar_init(&f_empty[s], 1);
            }
            for (int s = 0; s < NX; ++s) {
                mbar_init(&x_full[s], 1);
                mbar_init(&x_empty[s], RQ_EPI);
            }
            for (int s = 0; s < 2; ++s) {
                mbar_init(&acc_full[s], 1);
                mbar_init(&acc_empty[s], RQ_EPI);
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const int64_t t0 = rq_start(sched, blockIdx.x), t1 = rq_start(sched, blockIdx.x + 1);

    if (warp == 0) {
        if (lane == 0) {
            int gl = 0, prev_rb = -1;
            // X tiles beyond the 2-stage ring prefetched into L2, pd tiles
            // ahead (NMFB_RQ_PREFETCH, 0 = off)
            const int pd = (dbg >> 8) & 0xFF;
            for (int64_t t = t0; t < t1; ++t) {
                const int it = (int)(t - t0), sf_ = it % NF, sx = it % NX;
                const int rb = (int)(t / sched.col_tiles), ct = (int)(t % sched.col_tiles);
                if (pd > NX) {
                    for (int q = (it == 0 ? NX : pd); q <= pd; ++q) {
                        const int64_t tq = t + q;
                        if (tq < t1)
                            tma_prefetch_2d(&tmX, (int)(tq % sched.col_tiles) * RQ_BN,
                                            (int)(tq / sched.col_tiles) * RQ_BM);
                    }
                }
                if (rb != prev_rb) {
                    // previous row block's MMAs must be done with the G slices
                    mbar_wait(g_empty, ((uint32_t)gl & 1u) ^ 1u);
                    mbar_expect_tx(g_full, g_bytes);
                    for (int a = 0; a < 3; ++a)
                        tma_load_2d(&tmG, g_full, gs + a * g_slice, 0,
                                    (int)(a * n + (int64_t)rb * RQ_BM));
                    prev_rb = rb;
                    ++gl;
                }
                mbar_wait(&f_empty[sf_], ((uint32_t)(it / NF) & 1u) ^ 1u);
                mbar_expect_tx(&f_full[sf_], f_bytes);
                for (int b = 0; b < 3; ++b)
                    tma_load_2d(&tmF, &f_full[sf_], fs + sf_ * f_pitch + b * f_slice, 0,
                                (int)(b * m + (int64_t)ct * RQ_BN));
                mbar_wait(&x_empty[sx], ((uint32_t)(it / NX) & 1u) ^ 1u);
                mbar_expect_tx(&x_full[sx], x_bytes);
                tma_load_2d(&tmX, &x_full[sx], xs + sx * (x_bytes / 4), ct * RQ_BN, rb * RQ_BM);
                if ((dbg & 64) && blockIdx.x == 0 && it < 64) part[256 + it] = (double)gtime();
            }
        }
    } else if (warp == 1) {
        // s32 accumulate (c_format 2), u8 x u8 (a/b format 0), M = 128, N = 80.
        // The whole warp runs the loop (converged); one elected lane issues
        // each tcgen05 instruction, so no per-instruction divergence loop.
        constexpr uint32_t idesc =
            (2u << 4) | ((uint32_t)(RQ_BN >> 3) << 17) | ((uint32_t)(RQ_BM >> 4) << 24);
        int gl = 0, prev_rb = -1;
        for (int64_t t = t0; t < t1; ++t) {
            const int it = (int)(t - t0), s = it & 1, sf_ = it % NF;
            const int rb = (int)(t / sched.col_tiles);
            if (rb != prev_rb) {
                if (prev_rb >= 0) umma_commit_elect(g_empty);  // after the previous tiles' MMAs
                mbar_wait(g_full, (uint32_t)gl & 1u);
                prev_rb = rb;
                ++gl;
            }
            mbar_wait(&acc_empty[s], ((uint32_t)(it >> 1) & 1u) ^ 1u);
            mbar_wait(&f_full[sf_], (uint32_t)(it / NF) & 1u);
            if ((dbg & 64) && blockIdx.x == 0 && it < 64 && lane == 0)
                part[320 + it] = (double)gtime();
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t d = tmem + (uint32_t)(s * 3 * RQ_BN);
            uint64_t ga[3], fb[3];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                ga[q] = desc_u8<KB>(gs + q * g_slice);
                fb[q] = desc_u8<KB>(fs + sf_ * f_pitch + q * f_slice);
            }
            if (!(dbg & 2)) {
                // order o accumulates sum_{a+b=o} g_a . f_b
#pragma unroll
                for (int o = 0; o < 3; ++o) {
#pragma unroll
                    for (int q = 0; q <= o; ++q) {
#pragma unroll
                        for (int k = 0; k < KS; ++k) {
                            const uint64_t dk = (uint64_t)((k * 32) >> 4);
                            umma_i8_elect(d + (uint32_t)(o * RQ_BN), ga[q] + dk, fb[o - q] + dk,
                                          idesc, (q == 0 && k == 0) ? 0u : 1u);
                        }
                    }
                }
            }
            umma_commit_elect(&f_empty[sf_]);
            umma_commit_elect(&acc_full[s]);
            if ((dbg & 64) && blockIdx.x == 0 && it < 64 && lane == 0)
                part[384 + it] = (double)gtime();
        }
        __syncwarp();
    } else if (warp >= 4) {
        // 8 epilogue warps: warp w reads TMEM lane quarter w % 4 and half
        // (w - 4) / 4 of the tile's 80 columns
        const int quarter = warp & 3;
        const int cpart = (warp - 4) >> 2;  // column chunks c = cpart (mod RQ_EPW)
        const int row_in_tile = quarter * 32 + lane;
        const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
        double total = 0.0;
        for (int64_t t = t0; t < t1; ++t) {
            const int it = (int)(t - t0), s = it & 1, sx = it % NX, sf_ = it % NF;
            const int rb = (int)(t / sched.col_tiles), ct = (int)(t % sched.col_tiles);
            const int64_t i = (int64_t)rb * RQ_BM + row_in_tile;
            const int64_t j0 = (int64_t)ct * RQ_BN;
            const bool row_ok = i < n;
            const float si = row_ok ? sg[i] * (1.f / 16777216.f) : 0.f;
            const float2 nsi = make_float2(-si, -si);
            // this warp's column scales, fetched before the waits (latency hidden);
            // columns past m get scale 0 so their (garbage) G F drops out
            float4 sfr[RQ_BN / RQ_CW / RQ_EPW][RQ_CW / 4];
#pragma unroll
            for (int u = 0; u < RQ_BN / RQ_CW / RQ_EPW; ++u) {
#pragma unroll
                for (int q = 0; q < RQ_CW / 4; ++q) {
                    const int64_t jj = j0 + RQ_CW * (cpart + u * RQ_EPW) + 4 * q;
                    if (jj + 4 <= m) {
                        sfr[u][q] = __ldg(reinterpret_cast<const float4 *>(sf + jj));
                    } else {
                        sfr[u][q].x = jj < m ? sf[jj] : 0.f;
                        sfr[u][q].y = jj + 1 < m ? sf[jj + 1] : 0.f;
                        sfr[u][q].z = jj + 2 < m ? sf[jj + 2] : 0.f;
                        sfr[u][q].w = jj + 3 < m ? sf[jj + 3] : 0.f;
                    }
                }
            }
            mbar_wait(&acc_full[s], (uint32_t)(it >> 1) & 1u);
            mbar_wait(&x_full[sx], (uint32_t)(it / NX) & 1u);
            if ((dbg & 64) && blockIdx.x == 0 && it < 64 && threadIdx.x == 128)
                part[448 + it] = (double)gtime();
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const float *xrow = xs + sx * (x_bytes / 4) + row_in_tile * RQ_XLD;
            const uint32_t base = tmem + lane_base + (uint32_t)(s * 3 * RQ_BN);
            float2 acc = make_float2(0.f, 0.f);
            if (!(dbg & 1)) {
                // this warp's 16 columns; U = 2^8 A0 + A1 + round(2^-8 A2) is an
                // unsigned integer < 2^32 (A0 <= 32 ks 255^2), converted once with
                // round-to-nearest (relative 2^-24, unbiased): G F = s_i t_j 2^-24 U
                const int c0 = RQ_CW * cpart;
                uint32_t a0[RQ_CW], a1[RQ_CW], a2[RQ_CW];
                tmem_ld16(base + (uint32_t)c0, a0);
                tmem_ld16(base + (uint32_t)(RQ_BN + c0), a1);
                tmem_ld16(base + (uint32_t)(2 * RQ_BN + c0), a2);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                float u[RQ_CW];
#pragma unroll
                for (int q = 0; q < RQ_CW; ++q)
                    u[q] = __uint2float_rn((a0[q] << 8) + a1[q] + ((a2[q] + 128u) >> 8));
                const float4 *sfq = sfr[0];
#pragma unroll
                for (int q = 0; q < RQ_CW / 4; ++q) {
                    const float4 x4 = *reinterpret_cast<const float4 *>(xrow + c0 + 4 * q);
                    const float4 f4 = sfq[q];
                    const float2 s0 = __fmul2_rn(nsi, make_float2(f4.x, f4.y));
                    const float2 s1 = __fmul2_rn(nsi, make_float2(f4.z, f4.w));
                    // X - G F with one rounding, squared into the running sum
                    const float2 d0 = __ffma2_rn(make_float2(u[4 * q], u[4 * q + 1]), s0,
                                                 make_float2(x4.x, x4.y));
                    const float2 d1 = __ffma2_rn(make_float2(u[4 * q + 2], u[4 * q + 3]), s1,
                                                 make_float2(x4.z, x4.w));
                    acc = __ffma2_rn(d0, d0, acc);
                    acc = __ffma2_rn(d1, d1, acc);
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            mbar_arrive(&acc_empty[s]);
            mbar_arrive(&x_empty[sx]);
            if ((dbg & 64) && blockIdx.x == 0 && it < 64 && threadIdx.x == 128)
                part[512 + it] = (double)gtime();
            // rows past n contribute zeros only if masked: their X is 0 but
            // G F (garbage slice rows) is not
            if (row_ok) total += (double)acc.x + (double)acc.y;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
        if (lane == 0) red[warp - 4] = total;
        asm volatile("bar.sync 1, %0;" ::"n"(RQ_EPI) : "memory");
        if (warp == 4 && lane == 0) {
            double t = 0.0;
            for (int w = 0; w < 4 * RQ_EPW; ++w) t += red[w];
            part[blockIdx.x] = t;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

__global__ void rq_sum_kernel(const double *__restrict__ part, int np, double *__restrict__ out) {
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < np; ++i) s += part[i];
        *out += 0.5 * s;
    }
}

static int rq_sms() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0, v = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
            sms = v;
        else
            sms = 148;
    }
    return sms;
}

static int slice_kb(int r) { return r <= 64 ? 64 : RQ_KB; }

size_t slice_bytes(int64_t rows, int r) {
    // + 512 B: the per-tile scale copies may read up to 79 floats past the end
    return (size_t)3 * rows * slice_kb(r) + (size_t)rows * 4 + 512;
}

int slice_u8_launch(const float *A, int64_t rows, int r, int64_t lda, void *out,
                    cudaStream_t st) {
    if (rows <= 0) return NMFB_OK;
    if (r <= 0 || r > RQ_KB) return NMFB_ERR_ARG;
    const int kb = slice_kb(r);
    uint8_t *S = (uint8_t *)out;
    float *scale = (float *)(S + (size_t)3 * rows * kb);
    slice_u8_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(A, rows, r, lda, kb, S, scale);
    return launch_status();
}

size_t residual_i8_workspace_bytes() { return (size_t)std::max(rq_sms(), 640) * sizeof(double) + 64; }

template <int KB, int NF, int NX, int KS>
static void launch_rq(const CUtensorMap &tg, const CUtensorMap &tf, const CUtensorMap &tx,
                      const float *sg, const float *sf, int64_t n, int64_t m, const RqSched &s,
                      double *part, int dbg, cudaStream_t st) {
    const size_t smem = (size_t)3 * RQ_BM * KB + (size_t)NF * 3 * RQ_BN * KB +
                        (size_t)NX * RQ_BM * RQ_XLD * 4 + (2 * NF + 2 * NX + 8) * 8 + 1024;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(residual_i8_kernel<KB, NF, NX, KS>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    residual_i8_kernel<KB, NF, NX, KS>
        <<<s.G, RQ_THREADS, smem, st>>>(tg, tf, tx, sg, sf, n, m, s, part, dbg);
}

int residual_i8_launch(const float *X, int64_t n, int64_t m, const void *Gsl, const void *Fsl,
                       int r, double *out, void *ws, cudaStream_t st) {
    if (n <= 0 || m <= 0) return NMFB_OK;
    if (r <= 0 || r > RQ_KB || m % 4 != 0 || ((uintptr_t)X % 16) != 0) return NMFB_ERR_ARG;
    if (3 * n > INT32_MAX || 3 * m > INT32_MAX) return NMFB_ERR_ARG;
    const int kb = slice_kb(r);
    const uint8_t *gs = (const uint8_t *)Gsl, *fs = (const uint8_t *)Fsl;
    const float *sg = (const float *)(gs + (size_t)3 * n * kb);
    const float *sf = (const float *)(fs + (size_t)3 * m * kb);
    const CUtensorMapSwizzle sw = kb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
    CUtensorMap tg, tf, tx;
    if (!make_map_2d(&tg, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, gs, 3 * n, kb, kb, RQ_BM, sw) ||
        !make_map_2d(&tf, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, fs, 3 * m, kb, kb, RQ_BN, sw) ||
        !make_map_2d(&tx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, X, n, m, RQ_XLD, RQ_BM,
                     CU_TENSOR_MAP_SWIZZLE_NONE))
        return NMFB_ERR_CUDA;
    RqSched s;
    s.row_blocks = (int)((n + RQ_BM - 1) / RQ_BM);
    s.col_tiles = (int)((m + RQ_BN - 1) / RQ_BN);
    s.T = (int64_t)s.row_blocks * s.col_tiles;
    s.G = (int)std::min<int64_t>(s.T, rq_sms());
    double *part = (double *)ws;
    const int ksteps = (r + 31) / 32;
    // NMFB_RQ_DEBUG: 1 = skip epilogue math, 2 = skip MMAs (tuning aid only)
    static const int dbg = (getenv("NMFB_RQ_DEBUG") ? atoi(getenv("NMFB_RQ_DEBUG")) : 0) |
                           ((getenv("NMFB_RQ_PREFETCH") ? atoi(getenv("NMFB_RQ_PREFETCH")) : 0)
                            & 0xFF) << 8;
    if (ksteps == 1)
        launch_rq<64, 4, 3, 1>(tg, tf, tx, sg, sf, n, m, s, part, dbg, st);
    else if (ksteps == 2)
        launch_rq<64, 4, 3, 2>(tg, tf, tx, sg, sf, n, m, s, part, dbg, st);
    else if (ksteps == 3)
        launch_rq<128, 2, 2, 3>(tg, tf, tx, sg, sf, n, m, s, part, dbg, st);
    else
        launch_rq<128, 2, 2, 4>(tg, tf, tx, sg, sf, n, m, s, part, dbg, st);
    rq_sum_kernel<<<1, 32, 0, st>>>(part, s.G, out);
    return launch_status();
}

}  // namespace nmfb
