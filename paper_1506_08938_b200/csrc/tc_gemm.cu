// Tensor-core data products of the alternation on sm_100a (tcgen05 + TMA +
// TMEM), the dense passes over X:
//     pass 1 (coefficient step, kernels.py:306-313):  HT = X^T G   (m x r)
//     pass 2 (component step,   kernels.py:325-329):  YT = X  F^T  (n x r)
// Both are C[M x N] = A[M x K] * B[N x K]^T with A and B K-major in HBM
// (A = X^T or X -- both orientations of X are kept resident; B = G^T or F,
// r x K), N = r padded to a multiple of 16 (TMA zero-fills the padding).
//
// Precision: fp32 operands through kind::tf32 with the 3xTF32 split
//     a*b ~= a_hi b_hi + a_hi b_lo + a_lo b_hi,   x_hi = tf32(x), x_lo = x - x_hi
// (~2^-21 relative per product, fp32 accumulation in TMEM).  B_lo is
// precomputed per iteration (B is tiny); A_lo is formed in shared memory by
// the split warps from the TMA-loaded A tile, in place of a second HBM read.
//
// CTA = 6 warps, one output tile of 128 rows x BN, a K range (split-K):
//   warp 0     TMA producer (A, B, B_lo tiles, 128B swizzle, mbarrier tx)
//   warp 1     MMA issuer: 3 x (BK/8) tcgen05.mma per k-block, commit frees the stage
//   warps 2-5  A_lo split during the main loop, then the TMEM -> global epilogue
// HBM roofline: bytes = 4*M*K (A, streamed once) + B tiles (L2-resident) + C.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "nmfb_internal.h"
#include "tcgen05.cuh"

namespace nmfb {

constexpr int TC_BM = 128;
constexpr int TC_BK = 32;  // one 128-byte swizzle row of fp32
constexpr int TC_THREADS = 192;

// C[s][row][c] for the s-th K split.
//
// Accumulation precision: the tensor core's fp32 accumulate truncates, so a
// long K run in one TMEM accumulator drifts low (measured 2e-4 relative over
// K = 10^4).  The K range is therefore cut into chunks of `chunk_kb` k-blocks
// accumulated in one of two TMEM buffers (double-buffered); the split warps
// fold each finished chunk into a running sum (third TMEM region) with
// round-to-nearest CUDA-core adds while the MMA warp fills the other buffer.
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmBlo, float *__restrict__ C, int M, int N,
                   int BN, int num_kb, int kb_per_split, int stages, int chunk_kb,
                   int64_t split_stride) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-align the stage ring (SW128 atoms)
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const uint32_t a_bytes = TC_BM * TC_BK * 4;     // 16 KB
    const uint32_t b_bytes = (uint32_t)BN * TC_BK * 4;
    const uint32_t stage_bytes = 2 * a_bytes + 2 * b_bytes;
    uint64_t *bars = (uint64_t *)(smem + (size_t)stages * stage_bytes);
    uint64_t *full = bars, *split_done = bars + stages, *empty = bars + 2 * stages;
    uint64_t *tmem_full = bars + 3 * stages;      // [2]
    uint64_t *tmem_empty = bars + 3 * stages + 2;  // [2]
    uint32_t *tmem_slot = (uint32_t *)(bars + 3 * stages + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile = blockIdx.x, split = blockIdx.y;
    const int kb0 = split * kb_per_split;
    const int kb1 = min(num_kb, kb0 + kb_per_split);
    const int nkb = max(0, kb1 - kb0);
    const int nchunk = (nkb + chunk_kb - 1) / chunk_kb;
    // columns: [0, BN) chunk buffer 0, [BN, 2BN) chunk buffer 1, [2BN, 3BN) running sum
    const uint32_t need = 3u * (uint32_t)BN;
    const uint32_t tmem_cols = need <= 32 ? 32 : need <= 64 ? 64 : need <= 128 ? 128
                               : need <= 256 ? 256 : 512;

    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < stages; ++s) {
                mbar_init(&full[s], 1);
                mbar_init(&split_done[s], 128);
                mbar_init(&empty[s], 1);
            }
            for (int b = 0; b < 2; ++b) {
                mbar_init(&tmem_full[b], 1);
                mbar_init(&tmem_empty[b], 128);
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmA) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmBlo) : "memory");
        }
        __syncwarp();
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            for (int i = 0; i < nkb; ++i) {
                const int s = i % stages;
                const uint32_t ph = (uint32_t)(i / stages) & 1u;
                mbar_wait(&empty[s], ph ^ 1u);
                uint8_t *st = smem + (size_t)s * stage_bytes;
                mbar_expect_tx(&full[s], a_bytes + 2 * b_bytes);
                const int kc = (kb0 + i) * TC_BK;
                tma_load_2d(&tmA, &full[s], st, kc, tile * TC_BM);
                tma_load_2d(&tmB, &full[s], st + 2 * a_bytes, kc, 0);
                tma_load_2d(&tmBlo, &full[s], st + 2 * a_bytes + b_bytes, kc, 0);
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        // instruction descriptor: F32 accumulate, TF32 A/B, both K-major
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) |
                               ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(TC_BM >> 4) << 24);
        if (lane == 0) {
            int i = 0;
            for (int c = 0; c < nchunk; ++c) {
                const int buf = c & 1;
                mbar_wait(&tmem_empty[buf], ((uint32_t)(c >> 1) & 1u) ^ 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t dacc = tmem + (uint32_t)(buf * BN);
                const int iend = min(nkb, i + chunk_kb);
                for (int i0 = i; i < iend; ++i) {
                    const int s = i % stages;
                    const uint32_t ph = (uint32_t)(i / stages) & 1u;
                    mbar_wait(&split_done[s], ph);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    uint8_t *st = smem + (size_t)s * stage_bytes;
                    const uint64_t a_hi = umma_desc_sw128(st);
                    const uint64_t a_lo = umma_desc_sw128(st + a_bytes);
                    const uint64_t b_hi = umma_desc_sw128(st + 2 * a_bytes);
                    const uint64_t b_lo = umma_desc_sw128(st + 2 * a_bytes + b_bytes);
#pragma unroll
                    for (int k = 0; k < TC_BK / 8; ++k) {
                        // advance 32 B (8 tf32) along K inside the 128 B swizzle row
                        const uint64_t dk = (uint64_t)((k * 32) >> 4);
                        const uint32_t acc = (i > i0 || k > 0) ? 1u : 0u;
                        umma_tf32(dacc, a_hi + dk, b_hi + dk, idesc, acc);
                        umma_tf32(dacc, a_hi + dk, b_lo + dk, idesc, 1u);
                        umma_tf32(dacc, a_lo + dk, b_hi + dk, idesc, 1u);
                    }
                    umma_commit(&empty[s]);  // stage reusable once these MMAs have read it
                }
                umma_commit(&tmem_full[buf]);
            }
        }
        __syncwarp();
    } else {
        // ------- split warps: A_lo = A - tf32(A); fold finished chunks; epilogue -------
        const int t = threadIdx.x - 64;  // 0..127
        const int quarter = warp & 3;    // TMEM lane quarter this warp may access
        const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
        auto fold = [&](int c) {
            const int buf = c & 1;
            mbar_wait(&tmem_full[buf], (uint32_t)(c >> 1) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            for (int c0 = 0; c0 < BN; c0 += 16) {
                uint32_t v[16], s[16];
                tmem_ld16(tmem + lane_base + (uint32_t)(buf * BN + c0), v);
                if (c > 0) tmem_ld16(tmem + lane_base + (uint32_t)(2 * BN + c0), s);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (c > 0) {
#pragma unroll
                    for (int u = 0; u < 16; ++u)
                        v[u] = __float_as_uint(__fadd_rn(__uint_as_float(s[u]),
                                                         __uint_as_float(v[u])));
                }
                tmem_st16(tmem + lane_base + (uint32_t)(2 * BN + c0), v);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            mbar_arrive(&tmem_empty[buf]);
        };
        int i = 0;
        for (int c = 0; c < nchunk; ++c) {
            const int iend = min(nkb, i + chunk_kb);
            for (; i < iend; ++i) {
                const int s = i % stages;
                const uint32_t ph = (uint32_t)(i / stages) & 1u;
                mbar_wait(&full[s], ph);
                const float4 *src = (const float4 *)(smem + (size_t)s * stage_bytes);
                float4 *dst = (float4 *)(smem + (size_t)s * stage_bytes + a_bytes);
#pragma unroll
                for (int q = 0; q < (int)(a_bytes / 16 / 128); ++q) {
                    float4 v = src[q * 128 + t];
                    float4 o;
                    o.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
                    o.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
                    o.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
                    o.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
                    dst[q * 128 + t] = o;
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(&split_done[s]);
            }
            if (c > 0) fold(c - 1);
        }
        if (nchunk > 0) fold(nchunk - 1);
        // epilogue: running sum (TMEM region 2) -> C rows of this lane quarter
        const int row = tile * TC_BM + quarter * 32 + lane;
        float *crow = C + (int64_t)split * split_stride + (int64_t)row * N;
        for (int c0 = 0; c0 < BN; c0 += 16) {
            uint32_t v[16];
            if (nchunk > 0) {
                tmem_ld16(tmem + lane_base + (uint32_t)(2 * BN + c0), v);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            } else {
#pragma unroll
                for (int u = 0; u < 16; ++u) v[u] = 0u;
            }
            if (row < M) {
#pragma unroll
                for (int u = 0; u < 16; ++u)
                    if (c0 + u < N) crow[c0 + u] = __uint_as_float(v[u]);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(tmem_cols));
    }
}

// ---------------------------------------------------------------------------
// Persistent balanced kernel (the production path).  One CTA per SM; the
// (tile, k-block) space is cut into equal runs, one per CTA (stream-K style),
// so every SM streams the same number of A bytes regardless of how M and K
// divide by 148 -- no wave quantisation.  A run that crosses a tile boundary
// is split into per-tile segments; segment j of a tile writes partial slot j
// (C[j]), and the segment that finishes a tile zeroes the tile's unused
// slots, so the consumer sums a fixed number of slots in a fixed order.
//
// Roles (320 threads): warp 0 TMA producer, warp 1 MMA issuer, warps 2-5
// split A_lo = A - tf32(A) into TENSOR MEMORY (tcgen05.st; it is the A
// operand of the a_lo*b_hi MMA and never goes back to shared memory),
// warps 6-9 fold finished TMEM chunks into a register-resident running sum
// (round-to-nearest) and write the epilogue.  TMEM read bandwidth (64 B/clk)
// is the scarce resource for the fold, so all three products of a k-step
// land in ONE accumulator and the running sum lives in registers: a fold
// reads BN columns once.
// TMEM columns: [0,BN) and [BN,2BN) chunk buffers, then 32 per stage of A_lo.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
        "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
        "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
        "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]^T
__device__ __forceinline__ void umma_tf32_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t b,
                                             uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate));
}

constexpr int TC2_THREADS = 320;


// Work schedule shared by host and device.
struct TcSched {
    int tiles, num_kb;
    int mode;          // 0: fixed splits (units = tiles * splits); 1: balanced runs
    int kb_per_split;  // mode 0
    int units;         // mode 0
    int64_t W;         // mode 1: tiles * num_kb
    int G;             // grid size
    int parts;         // slots per tile
};

__host__ __device__ inline int64_t run_start(const TcSched &s, int b) {
    return (int64_t)b * s.W / s.G;
}
// CTA whose run contains linear k-block x (mode 1)
__host__ __device__ inline int run_of(const TcSched &s, int64_t x) {
    int b = (int)((x * s.G) / s.W);
    while (b + 1 < s.G && run_start(s, b + 1) <= x) ++b;
    while (b > 0 && run_start(s, b) > x) --b;
    return b;
}

// Calls f(tile, kb0, nkb, slot, zero_tail) for each segment CTA b owns, in order.
template <class F>
__device__ __forceinline__ void for_each_segment(const TcSched &s, int b, F &&f) {
    if (s.mode == 0) {
        for (int u = b; u < s.units; u += s.G) {
            const int tile = u % s.tiles, slot = u / s.tiles;
            const int kb0 = slot * s.kb_per_split;
            const int nkb = max(0, min(s.num_kb, kb0 + s.kb_per_split) - kb0);
            f(tile, kb0, nkb, slot, false);
        }
    } else {
        int64_t w = run_start(s, b);
        const int64_t w1 = run_start(s, b + 1);
        while (w < w1) {
            const int tile = (int)(w / s.num_kb);
            const int kb0 = (int)(w % s.num_kb);
            const int nkb = (int)min((int64_t)(s.num_kb - kb0), w1 - w);
            const int slot = b - run_of(s, (int64_t)tile * s.num_kb);
            f(tile, kb0, nkb, slot, kb0 + nkb == s.num_kb);
            w += nkb;
        }
    }
}

// element offset of row i of partial slot `slot` inside its owner's buffer
// (RowOut layout); *owner receives the destination rank
__device__ __forceinline__ int64_t rowout_off(const RowOut &o, int parts, int slot, int i,
                                              int N, int *owner) {
    const int chunk = (int)o.chunk;  // rows fit in int (M is an int)
    const int g = i / chunk;
    *owner = g;
    return ((int64_t)(o.src * parts + slot) * chunk + (i - g * chunk)) * N;
}

// Store one fold thread's column (factor column fcol of 128 consecutive rows
// row0.., values v(q)) into partial slot `part`.  row0 is a multiple of 128
// and a multi-GPU owner chunk a multiple of 32 (world = 1: one owner), so a
// 32-row group never straddles two owners: the destination base is derived
// once per group and the stores stay a plain strided sequence.
template <class V>
__device__ __forceinline__ void store_col128(const RowOut &out, int parts, int part, int row0,
                                             int M, int N, int fcol, V v) {
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        const int rg = row0 + 32 * g;
        if (rg < M) {
            int o;
            const int64_t off = rowout_off(out, parts, part, rg, N, &o) + fcol;
            float *p = out.dst[o] + off;
#pragma unroll
            for (int q = 0; q < 32; ++q)
                if (rg + q < M) p[(int64_t)q * N] = v(32 * g + q);
        }
    }
}
// Zero fill of an unused slot (rare: the tile's last segment): not unrolled
__device__ __noinline__ void zero_col128(const RowOut &out, int parts, int part, int row0, int M,
                                         int N, int fcol) {
    for (int g = 0; g < 4; ++g) {
        const int rg = row0 + 32 * g;
        if (rg >= M) break;
        int o;
        const int64_t off = rowout_off(out, parts, part, rg, N, &o) + fcol;
        float *p = out.dst[o] + off;
        for (int q = 0; q < 32 && rg + q < M; ++q) p[(int64_t)q * N] = 0.f;
    }
}


template <int BN>
__global__ void __launch_bounds__(TC2_THREADS, 1)
    tc_gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmBlo, const __grid_constant__ RowOut out,
                    int M, int N, const TcSched sched, int NS, int chunk_kb, int dbg) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    constexpr uint32_t a_bytes = TC_BM * TC_BK * 4;
    constexpr uint32_t b_bytes = (uint32_t)BN * TC_BK * 4;
    constexpr uint32_t stage_bytes = a_bytes + 2 * b_bytes;
    uint64_t *bars = (uint64_t *)(smem + (size_t)NS * stage_bytes);
    uint64_t *full = bars, *split_done = bars + NS, *empty = bars + 2 * NS;
    uint64_t *tmem_full = bars + 3 * NS, *tmem_empty = bars + 3 * NS + 2;
    uint32_t *tmem_slot = (uint32_t *)(bars + 3 * NS + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr uint32_t alo_col = 2u * BN;

    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < NS; ++s) {
                mbar_init(&full[s], 1);
                mbar_init(&split_done[s], 128);
                mbar_init(&empty[s], 1);
            }
            for (int b = 0; b < 2; ++b) {
                mbar_init(&tmem_full[b], 1);
                mbar_init(&tmem_empty[b], 128);
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmA) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmBlo) : "memory");
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

    if (warp == 0) {
        // ---------------- TMA producer (runs ahead across segments) ----------------
        if (lane == 0) {
            int i = 0;
            for_each_segment(sched, blockIdx.x, [&](int tile, int kb0, int nkb, int, bool) {
                for (int t = 0; t < nkb; ++t, ++i) {
                    const int s = i % NS;
                    mbar_wait(&empty[s], ((uint32_t)(i / NS) & 1u) ^ 1u);
                    uint8_t *st = smem + (size_t)s * stage_bytes;
                    mbar_expect_tx(&full[s], stage_bytes);
                    const int kc = (kb0 + t) * TC_BK;
                    tma_load_2d(&tmA, &full[s], st, kc, tile * TC_BM);
                    tma_load_2d(&tmB, &full[s], st + a_bytes, kc, 0);
                    tma_load_2d(&tmBlo, &full[s], st + a_bytes + b_bytes, kc, 0);
                }
            });
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) |
                                   ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(TC_BM >> 4) << 24);
        if (lane == 0) {
            int i = 0, g = 0;
            if (dbg & 1) {
                for_each_segment(sched, blockIdx.x, [&](int, int, int nkb, int, bool) {
                    for (int t = 0; t < nkb; ++t, ++i) {
                        const int s = i % NS;
                        mbar_wait(&split_done[s], (uint32_t)(i / NS) & 1u);
                        mbar_arrive(&empty[s]);
                    }
                });
            } else
            for_each_segment(sched, blockIdx.x, [&](int, int, int nkb, int, bool) {
                for (int c0 = 0; c0 < nkb; c0 += chunk_kb, ++g) {
                    const int buf = g & 1;
                    mbar_wait(&tmem_empty[buf], ((uint32_t)(g >> 1) & 1u) ^ 1u);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t d = tmem + (uint32_t)(buf * BN);
                    const int c1 = min(nkb, c0 + chunk_kb);
                    for (int t = c0; t < c1; ++t, ++i) {
                        const int s = i % NS;
                        mbar_wait(&split_done[s], (uint32_t)(i / NS) & 1u);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        uint8_t *st = smem + (size_t)s * stage_bytes;
                        const uint64_t a_hi = umma_desc_sw128(st);
                        const uint64_t b_hi = umma_desc_sw128(st + a_bytes);
                        const uint64_t b_lo = umma_desc_sw128(st + a_bytes + b_bytes);
                        const uint32_t a_lo = tmem + alo_col + (uint32_t)(s * TC_BK);
#pragma unroll
                        for (int k = 0; k < TC_BK / 8; ++k) {
                            const uint64_t dk = (uint64_t)((k * 32) >> 4);
                            umma_tf32(d, a_hi + dk, b_hi + dk, idesc, (t > c0 || k > 0) ? 1u : 0u);
                            if (!(dbg & 8)) umma_tf32(d, a_hi + dk, b_lo + dk, idesc, 1u);
                            if (!(dbg & 4))
                                umma_tf32_ta(d, a_lo + (uint32_t)(k * 8), b_hi + dk, idesc, 1u);
                        }
                        umma_commit(&empty[s]);
                    }
                    umma_commit(&tmem_full[buf]);
                }
            });
        }
        __syncwarp();
    } else if (warp < 6) {
        // ------- split warps 2-5: A_lo = A - tf32(A) -> TMEM -------
        const int quarter = warp & 3;  // TMEM lane quarter this warp may access
        const int row_in_tile = quarter * 32 + lane;
        const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
        int i = 0;
        for_each_segment(sched, blockIdx.x, [&](int, int, int nkb, int, bool) {
            for (int t = 0; t < nkb; ++t, ++i) {
                const int s = i % NS;
                mbar_wait(&full[s], (uint32_t)(i / NS) & 1u);
                if (dbg & 2) {
                    mbar_arrive(&split_done[s]);
                    continue;
                }
                // this thread's row of the swizzled A tile: 16-byte chunk c of
                // row rr sits at rr*128 + ((c ^ (rr & 7)) * 16)
                const uint8_t *rowp = smem + (size_t)s * stage_bytes + row_in_tile * 128;
                uint32_t lo[32];
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const float4 v =
                        *reinterpret_cast<const float4 *>(rowp + ((c ^ (row_in_tile & 7)) * 16));
                    const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        lo[c * 4 + q] = __float_as_uint(
                            vv[q] - __uint_as_float(__float_as_uint(vv[q]) & 0xFFFFE000u));
                }
                tmem_st32(tmem + lane_base + alo_col + (uint32_t)(s * TC_BK), lo);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mbar_arrive(&split_done[s]);
            }
        });
    } else {
        // ------- fold warps 6-9: chunk buffers -> register running sum; epilogue -------
        const int quarter = warp & 3;
        const int row_in_tile = quarter * 32 + lane;
        const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
        int g = 0;
        if (!(dbg & 1))
        for_each_segment(sched, blockIdx.x, [&](int tile, int, int nkb, int slot, bool zero_tail) {
            float run[BN];
#pragma unroll
            for (int q = 0; q < BN; ++q) run[q] = 0.f;
            const int nch = (nkb + chunk_kb - 1) / chunk_kb;
            for (int c = 0; c < nch; ++c, ++g) {
                const int buf = g & 1;
                mbar_wait(&tmem_full[buf], (uint32_t)(g >> 1) & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int c0 = 0; c0 < BN; c0 += 16) {
                    uint32_t v[16];
                    tmem_ld16(tmem + lane_base + (uint32_t)(buf * BN + c0), v);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int q = 0; q < 16; ++q)
                        run[c0 + q] = __fadd_rn(run[c0 + q], __uint_as_float(v[q]));
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mbar_arrive(&tmem_empty[buf]);
            }
            const int row = tile * TC_BM + row_in_tile;
            if (row < M) {
                int o;
                const int64_t off = rowout_off(out, sched.parts, slot, row, N, &o);
                float *crow = out.dst[o] + off;
#pragma unroll
                for (int q = 0; q < BN; ++q)
                    if (q < N) crow[q] = run[q];
                if (zero_tail) {
                    for (int s2 = slot + 1; s2 < sched.parts; ++s2) {
                        float *z = out.dst[o] + rowout_off(out, sched.parts, s2, row, N, &o);
                        for (int q = 0; q < N; ++q) z[q] = 0.f;
                    }
                }
            }
        });
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}


// ---------------------------------------------------------------------------
// Swapped-operand kernel for r <= 64 (the production path for the BASELINE
// ranks).  Measured on B200: a tcgen05.mma kind::tf32 instruction occupies
// the tensor pipe for ~77 ns whatever its N up to 128 (~87 ns at N = 256), so
// a memory-bound tall-skinny product must cover as many X bytes per
// instruction as possible.  Here the SMALL factor is the A operand and X the
// B operand with N = 256 X rows:
//   A = F' = [Bt_hi ; Bt_lo]  (M = 128 TMEM lanes: 64 hi rows, 64 lo rows)
//   D += F' X_tile^T          (tensor core truncates X to tf32 = X_hi)
//   D += F' X_lo^T            (X_lo = X - tf32(X), written to smem by the split warps)
// so lane i < 64 accumulates hi_i.X and lane 64+i accumulates lo_i.X; both are
// written out as separate partial slots (the consumer sums slots anyway).
// 8 instructions per 256 rows x 32 k (32 KB of X) ~ 0.7 us ~ HBM rate.
// Fold warps (8: 2 per TMEM lane quarter, 128 columns each) promote each
// chunk into a register running sum; setmaxnreg moves registers to them.
// Roles (512 threads): warp 0 TMA, warp 1 MMA, warps 4-7 split, 8-15 fold.
// TMEM: two 256-column chunk buffers.
// ---------------------------------------------------------------------------
constexpr int TC3_BM = 256;  // X rows per tile (MMA N)
// tuning aid (NMFB_TC_DEBUG=64): CTA 0 per-k-block timeline
__device__ long long g_tc3_dbg[5][256];
__device__ long long g_tc3_cta[2][160];  // per-CTA start / end (NMFB_TC_DEBUG=64)
__device__ __forceinline__ long long gtime_ns() {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
constexpr int TC3_THREADS = 512;
constexpr int TC3_NX = 4;    // X stages (32 KB, HBM)
constexpr int TC3_NF = 2;    // F' stages (16 KB, L2-resident factor)
constexpr int TC3_NL = 2;    // split buffers (16 KB bf16 X_lo + 8 KB bf16 [F_hi ; 0])

// bf16 correction MMA (kind::f16): D += [bf16(F_hi) ; 0] (M = 128, 64-byte
// K rows, SWIZZLE_64B) x bf16(X_lo)^T (N = 256).  X_lo ~ 2^-10 |X|, so bf16
// (8-bit, round-to-nearest) costs ~2^-19 of a term, unbiased -- far below the
// 3xTF32 target -- and halves the X_lo smem footprint and MMA count.
__device__ __forceinline__ uint64_t desc_sw64(const void *p) {
    uint64_t d = (uint64_t)((smem_u32(p) & 0x3FFFFu) >> 4);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(512 >> 4) << 32;  // 8 rows x 64 B
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)4 << 61;           // SWIZZLE_64B
    return d;
}
__device__ __forceinline__ void umma_bf16_elect(uint32_t tmem_d, uint64_t a, uint64_t b,
                                                uint32_t idesc) {
    asm volatile(
        "{\n"
        ".reg .pred p, e;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "setp.ne.b32 p, 1, 0;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc));
}
// 8 fp32 (two 16-byte chunks) -> x - tf32(x) rounded to bf16, packed
__device__ __forceinline__ uint4 lo_bf16x8(float4 a, float4 b) {
    auto lo = [](float v) { return v - __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); };
    __nv_bfloat162 p0 = __floats2bfloat162_rn(lo(a.x), lo(a.y));
    __nv_bfloat162 p1 = __floats2bfloat162_rn(lo(a.z), lo(a.w));
    __nv_bfloat162 p2 = __floats2bfloat162_rn(lo(b.x), lo(b.y));
    __nv_bfloat162 p3 = __floats2bfloat162_rn(lo(b.z), lo(b.w));
    return make_uint4(*reinterpret_cast<uint32_t *>(&p0), *reinterpret_cast<uint32_t *>(&p1),
                      *reinterpret_cast<uint32_t *>(&p2), *reinterpret_cast<uint32_t *>(&p3));
}
__device__ __forceinline__ uint4 bf16x8(float4 a, float4 b) {
    __nv_bfloat162 p0 = __floats2bfloat162_rn(a.x, a.y);
    __nv_bfloat162 p1 = __floats2bfloat162_rn(a.z, a.w);
    __nv_bfloat162 p2 = __floats2bfloat162_rn(b.x, b.y);
    __nv_bfloat162 p3 = __floats2bfloat162_rn(b.z, b.w);
    return make_uint4(*reinterpret_cast<uint32_t *>(&p0), *reinterpret_cast<uint32_t *>(&p1),
                      *reinterpret_cast<uint32_t *>(&p2), *reinterpret_cast<uint32_t *>(&p3));
}
__device__ __forceinline__ float4 lds128(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

__global__ void __launch_bounds__(TC3_THREADS, 1)
    tc_gemm3_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmBlo, const __grid_constant__ RowOut out,
                    int M, int N, const TcSched sched, int chunk_kb, int dbg) {
    // separate rings: X (HBM, ~2 us TMA latency under load -> deep), F' (L2,
    // shallow) and the split products [X_lo bf16 | F_hi bf16]
    constexpr int NX = TC3_NX, NF = TC3_NF, NL = TC3_NL;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    constexpr uint32_t x_bytes = TC3_BM * TC_BK * 4;   // 32 KB fp32 X tile
    constexpr uint32_t f_bytes = 128 * TC_BK * 4;      // 16 KB ([hi ; lo] 64 + 64 rows)
    constexpr uint32_t xl_bytes = TC3_BM * TC_BK * 2;  // 16 KB bf16 X_lo
    constexpr uint32_t fb_bytes = 128 * TC_BK * 2;     // 8 KB bf16 [F_hi ; 0]
    constexpr uint32_t l_bytes = xl_bytes + fb_bytes;
    uint8_t *xr = smem;
    uint8_t *fr = xr + (size_t)NX * x_bytes;
    uint8_t *lr = fr + (size_t)NF * f_bytes;
    uint64_t *bars = (uint64_t *)(lr + (size_t)NL * l_bytes);
    uint64_t *xfull = bars, *xempty = xfull + NX;
    uint64_t *ffull = xempty + NX, *fempty = ffull + NF;
    uint64_t *xlo_full = fempty + NF, *xlo_free = xlo_full + NL;
    uint64_t *tmem_full = xlo_free + NL, *tmem_empty = tmem_full + 2;
    uint32_t *tmem_slot = (uint32_t *)(tmem_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if ((dbg & 64) && threadIdx.x == 0 && blockIdx.x < 160) g_tc3_cta[0][blockIdx.x] = gtime_ns();
    // rows 64..127 of the bf16 F_hi operands stay zero
    for (int q = threadIdx.x; q < NL * (int)(fb_bytes / 2) / 16; q += TC3_THREADS) {
        const int j = q / (int)(fb_bytes / 2 / 16), w = q % (int)(fb_bytes / 2 / 16);
        *reinterpret_cast<uint4 *>(lr + (size_t)j * l_bytes + xl_bytes + fb_bytes / 2 + w * 16) =
            make_uint4(0, 0, 0, 0);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");

    if (warp == 0) {
        if (lane == 0) {
            // X / F' stages are free once the main MMAs (commit) and the split
            // warps (128 arrivals) are done with them -- not after the X_lo MMAs
            for (int s = 0; s < NX; ++s) {
                mbar_init(&xfull[s], 1);
                mbar_init(&xempty[s], 1 + 128);
            }
            for (int s = 0; s < NF; ++s) {
                mbar_init(&ffull[s], 1);
                mbar_init(&fempty[s], 1 + 128);
            }
            for (int j = 0; j < NL; ++j) {
                mbar_init(&xlo_full[j], 128);
                mbar_init(&xlo_free[j], 1);
            }
            for (int b = 0; b < 2; ++b) {
                mbar_init(&tmem_full[b], 1);
                mbar_init(&tmem_empty[b], 256);
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmX) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmBlo) : "memory");
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

    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
    }
    if (warp == 0) {
        // ---------------- TMA producer (converged warp, elected issue) ----------------
        // X tiles further ahead than the smem ring are prefetched into L2
        // (distance pd k-blocks; NMFB_TC_PREFETCH, 0 = off), so each TMA load
        // of the ring finds its tile in L2 instead of paying HBM latency
        const int pd = (dbg >> 8) & 0xFF;
        int i = 0;
        for_each_segment(sched, blockIdx.x, [&](int tile, int kb0, int nkb, int, bool) {
            for (int t = 0; t < nkb; ++t, ++i) {
                const int sx = i % NX, sf = i % NF;
                const int kc = (kb0 + t) * TC_BK;
                if (pd > NX) {
                    for (int q = (t == 0 ? NX : pd); q <= pd; ++q)
                        if (t + q < nkb) tma_prefetch_2d_elect(&tmX, kc + q * TC_BK, tile * TC3_BM);
                }
                mbar_wait(&xempty[sx], ((uint32_t)(i / NX) & 1u) ^ 1u);
                mbar_expect_tx_elect(&xfull[sx], x_bytes);
                tma_load_2d_elect(&tmX, &xfull[sx], xr + (size_t)sx * x_bytes, kc, tile * TC3_BM);
                if ((dbg & 64) && blockIdx.x == 0 && i < 256 && lane == 0) g_tc3_dbg[0][i] = gtime_ns();
                mbar_wait(&fempty[sf], ((uint32_t)(i / NF) & 1u) ^ 1u);
                mbar_expect_tx_elect(&ffull[sf], f_bytes);
                uint8_t *fs = fr + (size_t)sf * f_bytes;
                tma_load_2d_elect(&tmB, &ffull[sf], fs, kc, 0);
                tma_load_2d_elect(&tmBlo, &ffull[sf], fs + f_bytes / 2, kc, 0);
            }
        });
    } else if (warp == 1) {
        // ---------------- MMA issuer (converged warp, elected issue) ----------------
        constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) |
                                   ((uint32_t)(TC3_BM >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        constexpr uint32_t idesc_bf = (1u << 4) | (1u << 7) | (1u << 10) |
                                      ((uint32_t)(TC3_BM >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        int i = 0, g = 0;
        for_each_segment(sched, blockIdx.x, [&](int, int, int nkb, int, bool) {
            for (int c0 = 0; c0 < nkb; c0 += chunk_kb, ++g) {
                const int buf = g & 1;
                mbar_wait(&tmem_empty[buf], ((uint32_t)(g >> 1) & 1u) ^ 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t d = tmem + (uint32_t)(buf * TC3_BM);
                const int c1 = min(nkb, c0 + chunk_kb);
                for (int t = c0; t < c1; ++t, ++i) {
                    const int sx = i % NX, sf = i % NF, j = i % NL;
                    const uint64_t fa = umma_desc_sw128(fr + (size_t)sf * f_bytes);
                    const uint64_t xb = umma_desc_sw128(xr + (size_t)sx * x_bytes);
                    const uint64_t xl = desc_sw64(lr + (size_t)j * l_bytes);
                    const uint64_t fbd = desc_sw64(lr + (size_t)j * l_bytes + xl_bytes);
                    mbar_wait(&ffull[sf], (uint32_t)(i / NF) & 1u);
                    mbar_wait(&xfull[sx], (uint32_t)(i / NX) & 1u);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    if ((dbg & 64) && blockIdx.x == 0 && i < 256 && lane == 0) g_tc3_dbg[1][i] = gtime_ns();
#pragma unroll
                    for (int k = 0; k < TC_BK / 8; ++k) {
                        const uint64_t dk = (uint64_t)((k * 32) >> 4);
                        umma_tf32_elect(d, fa + dk, xb + dk, idesc, (t > c0 || k > 0) ? 1u : 0u);
                    }
                    umma_commit_elect(&xempty[sx]);
                    umma_commit_elect(&fempty[sf]);
                    mbar_wait(&xlo_full[j], (uint32_t)(i / NL) & 1u);
                    if ((dbg & 64) && blockIdx.x == 0 && i < 256 && lane == 0) g_tc3_dbg[2][i] = gtime_ns();
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    if (!(dbg & 4)) {
#pragma unroll
                        for (int k = 0; k < TC_BK / 16; ++k) {
                            const uint64_t dk = (uint64_t)((k * 32) >> 4);  // 16 bf16 = 32 B
                            umma_bf16_elect(d, fbd + dk, xl + dk, idesc_bf);
                        }
                    }
                    umma_commit_elect(&xlo_free[j]);
                    if ((dbg & 64) && blockIdx.x == 0 && i < 256 && lane == 0) g_tc3_dbg[3][i] = gtime_ns();
                }
                umma_commit_elect(&tmem_full[buf]);
            }
        });
        __syncwarp();
    } else if (warp >= 4 && warp < 8) {
        // ------- split warps: bf16(X - tf32(X)) and bf16(F_hi) into the L ring -------
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
        const int t128 = threadIdx.x - 128;
        int i = 0;
        for_each_segment(sched, blockIdx.x, [&](int, int, int nkb, int, bool) {
            for (int t = 0; t < nkb; ++t, ++i) {
                const int sx = i % NX, sf = i % NF, j = i % NL;
                mbar_wait(&xfull[sx], (uint32_t)(i / NX) & 1u);
                mbar_wait(&ffull[sf], (uint32_t)(i / NF) & 1u);
                mbar_wait(&xlo_free[j], ((uint32_t)(i / NL) & 1u) ^ 1u);
                if ((dbg & 64) && blockIdx.x == 0 && i < 256 && threadIdx.x == 128) g_tc3_dbg[4][i] = gtime_ns();
                const uint32_t xsrc = smem_u32(xr + (size_t)sx * x_bytes);
                const uint32_t fsrc = smem_u32(fr + (size_t)sf * f_bytes);
                const uint32_t ldst = smem_u32(lr + (size_t)j * l_bytes);
                // items (row r, bf16 chunk cb): fp32 chunks 2cb, 2cb+1 of a SW128
                // row (chunk c at r*128 + ((c ^ (r & 7)) << 4)) -> one SW64 chunk
                // (chunk c at r*64 + ((c ^ ((r >> 1) & 3)) << 4))
#pragma unroll 2
                for (int q = t128; q < ((dbg & 2) ? 0 : TC3_BM * 4); q += 128) {
                    const int r = q >> 2, cb = q & 3;
                    const uint32_t rb = xsrc + (uint32_t)r * 128u;
                    const float4 a = lds128(rb + ((uint32_t)((2 * cb) ^ (r & 7)) << 4));
                    const float4 b = lds128(rb + ((uint32_t)((2 * cb + 1) ^ (r & 7)) << 4));
                    sts128(ldst + (uint32_t)r * 64u + ((uint32_t)(cb ^ ((r >> 1) & 3)) << 4),
                           lo_bf16x8(a, b));
                }
                for (int q = t128; q < ((dbg & 2) ? 0 : 64 * 4); q += 128) {
                    const int r = q >> 2, cb = q & 3;
                    const uint32_t rb = fsrc + (uint32_t)r * 128u;
                    const float4 a = lds128(rb + ((uint32_t)((2 * cb) ^ (r & 7)) << 4));
                    const float4 b = lds128(rb + ((uint32_t)((2 * cb + 1) ^ (r & 7)) << 4));
                    sts128(ldst + xl_bytes + (uint32_t)r * 64u +
                               ((uint32_t)(cb ^ ((r >> 1) & 3)) << 4),
                           bf16x8(a, b));
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(&xlo_full[j]);
                mbar_arrive(&xempty[sx]);
                mbar_arrive(&fempty[sf]);
            }
        });
    } else if (warp >= 8) {
        // ------- fold warps: chunk buffer -> register running sum; epilogue -------
        asm volatile("setmaxnreg.inc.sync.aligned.u32 200;\n" ::: "memory");
        const int quarter = warp & 3;               // TMEM lanes [32q, 32q+32)
        const int half = (warp - 8) >> 2;           // columns [128h, 128h+128)
        const int lane_row = quarter * 32 + lane;   // 0..63 hi rows, 64..127 lo rows
        const int fcol = lane_row & 63;             // factor column
        const int lohi = lane_row >> 6;
        const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
        int g = 0;
        for_each_segment(sched, blockIdx.x, [&](int tile, int, int nkb, int slot, bool zero_tail) {
            float run[128];
#pragma unroll
            for (int q = 0; q < 128; ++q) run[q] = 0.f;
            const int nch = (nkb + chunk_kb - 1) / chunk_kb;
            for (int c = 0; c < nch; ++c, ++g) {
                const int buf = g & 1;
                mbar_wait_sleep(&tmem_full[buf], (uint32_t)(g >> 1) & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t base = tmem + lane_base + (uint32_t)(buf * TC3_BM + half * 128);
#pragma unroll
                for (int c0 = 0; c0 < 128; c0 += 32) {
                    uint32_t v[16], w[16];
                    tmem_ld16(base + (uint32_t)c0, v);
                    tmem_ld16(base + (uint32_t)(c0 + 16), w);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        run[c0 + q] = __fadd_rn(run[c0 + q], __uint_as_float(v[q]));
                        run[c0 + 16 + q] = __fadd_rn(run[c0 + 16 + q], __uint_as_float(w[q]));
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mbar_arrive(&tmem_empty[buf]);
            }
            if (fcol < N) {
                const int part = 2 * slot + lohi;
                const int row0 = tile * TC3_BM + half * 128;
                store_col128(out, sched.parts, part, row0, M, N, fcol,
                             [&](int q) { return run[q]; });
                if (zero_tail) {
                    for (int p2 = part + 2; p2 < sched.parts; p2 += 2)
                        zero_col128(out, sched.parts, p2, row0, M, N, fcol);
                }
            }
        });
    }
    if ((dbg & 64) && warp == 8 && lane == 0 && blockIdx.x < 160) g_tc3_cta[1][blockIdx.x] = gtime_ns();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// B (K x r row-major, e.g. G or F^T) -> Bt_hi (r x K) and Bt_lo = Bt - tf32(Bt).
__global__ void split_transpose_kernel(const float *__restrict__ B, int64_t K, int r,
                                       float *__restrict__ hi, float *__restrict__ lo) {
    __shared__ float tile[32][33];
    const int64_t k0 = (int64_t)blockIdx.x * 32;
    const int c0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += 8) {
        int64_t k = k0 + i;
        int c = c0 + threadIdx.x;
        tile[i][threadIdx.x] = (k < K && c < r) ? B[k * r + c] : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += 8) {
        int c = c0 + i;
        int64_t k = k0 + threadIdx.x;
        if (c < r && k < K) {
            float v = tile[threadIdx.x][i];
            hi[(int64_t)c * K + k] = v;
            lo[(int64_t)c * K + k] = v - __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
        }
    }
}

// Out-of-place transpose of X^T (m x n) into X (n x m) -- once per fit, so
// both dense passes stream a K-major operand.
__global__ void transpose_kernel(const float *__restrict__ in, int64_t rows, int64_t cols,
                                 float *__restrict__ out) {
    __shared__ float tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
    for (int i = threadIdx.y; i < 32; i += 8) {
        int64_t r = r0 + i, c = c0 + threadIdx.x;
        tile[i][threadIdx.x] = (r < rows && c < cols) ? in[r * cols + c] : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += 8) {
        int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (c < cols && r < rows) out[c * rows + r] = tile[threadIdx.x][i];
    }
}

// ---------------------------------------------------------------------------
// host side: tensor maps (cached), launch
// ---------------------------------------------------------------------------
// 2-D fp32 row-major tensor (rows x cols), box = (32 cols, box_rows), SW128
static bool make_map(CUtensorMap *map, const float *ptr, int64_t rows, int64_t cols,
                     int box_rows) {
    return make_map_2d(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, ptr, rows, cols, TC_BK, box_rows,
                       CU_TENSOR_MAP_SWIZZLE_128B);
}

size_t tc_gemm_smem_bytes(int BN, int stages) {
    size_t stage = 2 * (size_t)TC_BM * TC_BK * 4 + 2 * (size_t)BN * TC_BK * 4;
    return stages * stage + (3 * stages + 6) * 8 + 1024;
}

static int sm_count_cached() {
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

static bool tc_classic() {
    static const bool classic = getenv("NMFB_TC_CLASSIC") != nullptr;
    return classic;
}

// Work schedule for (M, K, splits); returns the number of partial slots.
// Kernel variant for a product with N = r output columns.
enum { TC_CLASSIC = 1, TC_V2 = 2, TC_V3 = 3 };
static int tc_variant(int N) {
    if (tc_classic()) return TC_CLASSIC;
    static const bool v2 = getenv("NMFB_TC_V2") != nullptr;
    return (N <= 64 && !v2) ? TC_V3 : TC_V2;
}

// Work schedule for (M, K, splits); returns the number of partial slots.
static int tc_plan(int64_t M, int64_t K, int N, int splits, TcSched *out) {
    const int variant = tc_variant(N);
    const int bm = variant == TC_V3 ? TC3_BM : TC_BM;
    TcSched s{};
    s.tiles = (int)((M + bm - 1) / bm);
    s.num_kb = (int)((K + TC_BK - 1) / TC_BK);
    const int sms = sm_count_cached();
    if (splits <= 0 && variant == TC_CLASSIC) {
        // the classic kernel has no balanced schedule: ~8 waves of fixed chunks
        splits = std::max(1, std::min(16, (int)std::lround(8.0 * sms / s.tiles)));
    }
    if (splits > 0) {
        if (splits > s.num_kb) splits = s.num_kb;
        s.mode = 0;
        s.kb_per_split = (s.num_kb + splits - 1) / splits;
        s.parts = (s.num_kb + s.kb_per_split - 1) / s.kb_per_split;
        s.units = s.tiles * s.parts;
        s.G = std::min(s.units, sms);
        s.W = 0;
    } else {
        s.mode = 1;
        s.W = (int64_t)s.tiles * s.num_kb;
        s.G = (int)std::min<int64_t>(s.W, sms);
        int parts = 1;
        for (int t = 0; t < s.tiles; ++t) {
            const int b0 = run_of(s, (int64_t)t * s.num_kb);
            const int b1 = run_of(s, (int64_t)t * s.num_kb + s.num_kb - 1);
            parts = std::max(parts, b1 - b0 + 1);
        }
        s.parts = parts;
    }
    // v3 writes the hi-factor and lo-factor halves as separate slots
    if (variant == TC_V3) s.parts *= 2;
    if (out) *out = s;
    return s.parts;
}

int tc_parts(int64_t M, int64_t K, int N, int splits) {
    if (M <= 0 || K <= 0 || N <= 0) return 0;
    return tc_plan(M, K, N, splits, nullptr);
}

static void launch_tc3(const CUtensorMap &tx, const CUtensorMap &tb, const CUtensorMap &tbl,
                       const RowOut &out, int M, int N, const TcSched &s, int chunk_kb,
                       cudaStream_t st) {
    static bool attr = false;
    const size_t smem = (size_t)TC3_NX * TC3_BM * TC_BK * 4 + (size_t)TC3_NF * 128 * TC_BK * 4 +
                        (size_t)TC3_NL * (TC3_BM + 128) * TC_BK * 2 + 256 + 1024;
    if (!attr) {
        cudaFuncSetAttribute(tc_gemm3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attr = true;
    }
    static const int dbg = (getenv("NMFB_TC_DEBUG") ? atoi(getenv("NMFB_TC_DEBUG")) : 0) |
                           ((getenv("NMFB_TC_PREFETCH") ? atoi(getenv("NMFB_TC_PREFETCH")) : 0)
                            & 0xFF) << 8;
    tc_gemm3_kernel<<<s.G, TC3_THREADS, smem, st>>>(tx, tb, tbl, out, M, N, s, chunk_kb, dbg);
}

template <int BN>
static void launch_tc2(const CUtensorMap &ta, const CUtensorMap &tb, const CUtensorMap &tbl,
                       const RowOut &out, int M, int N, const TcSched &s, int stages,
                       int chunk_kb, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(tc_gemm2_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024);
        attr = true;
    }
    const size_t stage = (size_t)TC_BM * TC_BK * 4 + 2 * (size_t)BN * TC_BK * 4;
    auto smem_of = [&](int ns) { return ns * stage + (3 * ns + 6) * 8 + 1024; };
    int ns = stages > 0 ? stages : 4;
    while (ns > 2 && (2 * BN + 32 * ns > 512 || smem_of(ns) > 227 * 1024)) --ns;
    // at least 116 KB so only one CTA (one 512-column TMEM allocation) fits per SM
    const size_t smem = std::max<size_t>(smem_of(ns), 116 * 1024);
    // NMFB_TC_DEBUG=1: TMA stream only, =2: TMA + A_lo split (no MMA) -- tuning aid
    static const int dbg = getenv("NMFB_TC_DEBUG") ? atoi(getenv("NMFB_TC_DEBUG")) : 0;
    tc_gemm2_kernel<BN><<<s.G, TC2_THREADS, smem, st>>>(ta, tb, tbl, out, M, N, s, ns, chunk_kb,
                                                        dbg);
}

extern "C" int nmfb_debug_tc3_timeline(long long *host_out) {
    return cudaMemcpyFromSymbol(host_out, g_tc3_dbg, sizeof(g_tc3_dbg)) == cudaSuccess ? 0 : 3;
}
extern "C" int nmfb_debug_tc3_cta(long long *host_out) {
    return cudaMemcpyFromSymbol(host_out, g_tc3_cta, sizeof(g_tc3_cta)) == cudaSuccess ? 0 : 3;
}

int tc_gemm_rows_launch(const float *A, int64_t M, int64_t K, const float *Bt_hi,
                        const float *Bt_lo, int N, const RowOut &out, int splits, int stages,
                        cudaStream_t st) {
    if (M <= 0 || K <= 0 || N <= 0 || N > 160) return NMFB_ERR_ARG;
    if (out.world < 1 || out.world > NMFB_MAX_PEERS || out.src < 0 || out.src >= out.world ||
        out.chunk <= 0 || out.chunk * out.world < M || out.chunk > INT32_MAX)
        return NMFB_ERR_ARG;
    // owner chunks are whole 32-row groups (fast-break blocks; the v3
    // epilogue stores 32-row groups)
    if (out.world > 1 && out.chunk % 32 != 0) return NMFB_ERR_ARG;
    for (int o = 0; o < out.world; ++o)
        if (!out.dst[o]) return NMFB_ERR_ARG;
    if ((K * 4) % 16 != 0) return NMFB_ERR_ARG;  // TMA row pitch must be 16-byte aligned
    if (((uintptr_t)A | (uintptr_t)Bt_hi | (uintptr_t)Bt_lo) % 16 != 0) return NMFB_ERR_ARG;
    const int BN = ((N + 15) / 16) * 16;
    const int variant = tc_variant(N);
    CUtensorMap ta, tb, tbl;
    if (variant == TC_V3) {
        if (!make_map(&ta, A, M, K, TC3_BM) || !make_map(&tb, Bt_hi, N, K, 64) ||
            !make_map(&tbl, Bt_lo, N, K, 64))
            return NMFB_ERR_CUDA;
    } else if (!make_map(&ta, A, M, K, TC_BM) || !make_map(&tb, Bt_hi, N, K, BN) ||
               !make_map(&tbl, Bt_lo, N, K, BN)) {
        return NMFB_ERR_CUDA;
    }
    TcSched s;
    tc_plan(M, K, N, splits, &s);
    // k-blocks between promotions of the (truncating) tensor-core accumulator
    // into the round-to-nearest running sum; NMFB_TC_CHUNK overrides for tuning
    static const int chunk_env = getenv("NMFB_TC_CHUNK") ? atoi(getenv("NMFB_TC_CHUNK")) : 0;
    if (variant == TC_V3) {
        launch_tc3(ta, tb, tbl, out, (int)M, N, s, chunk_env > 0 ? chunk_env : 4, st);
        return launch_status();
    }
    if (variant == TC_V2) {
        const int chunk_kb = chunk_env > 0 ? chunk_env : 4;
        switch (BN) {
#define NMFB_TC2_CASE(bn)                                                                  \
    case bn:                                                                               \
        launch_tc2<bn>(ta, tb, tbl, out, (int)M, N, s, stages, chunk_kb, st);              \
        break;
            NMFB_TC2_CASE(16) NMFB_TC2_CASE(32) NMFB_TC2_CASE(48) NMFB_TC2_CASE(64)
            NMFB_TC2_CASE(80) NMFB_TC2_CASE(96) NMFB_TC2_CASE(112) NMFB_TC2_CASE(128)
            NMFB_TC2_CASE(144) NMFB_TC2_CASE(160)
#undef NMFB_TC2_CASE
            default:
                return NMFB_ERR_ARG;
        }
        return launch_status();
    }
    // classic (non-persistent) kernel, kept for comparison (plain layout only)
    if (out.world != 1 || out.chunk != M) return NMFB_ERR_ARG;
    float *C = out.dst[0];
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024);
        attr_set = true;
    }
    if (stages <= 0) stages = 2;
    while (stages > 2 && tc_gemm_smem_bytes(BN, stages) > 227 * 1024) --stages;
    const size_t smem = tc_gemm_smem_bytes(BN, stages);
    const int chunk_kb = chunk_env > 0 ? chunk_env : 2;
    dim3 grid((unsigned)s.tiles, (unsigned)s.parts);
    tc_gemm_kernel<<<grid, TC_THREADS, smem, st>>>(ta, tb, tbl, C, (int)M, N, BN, s.num_kb,
                                                   s.kb_per_split, stages, chunk_kb,
                                                   (int64_t)M * N);
    return launch_status();
}

int tc_gemm_launch(const float *A, int64_t M, int64_t K, const float *Bt_hi, const float *Bt_lo,
                   int N, float *C, int splits, int stages, cudaStream_t st) {
    RowOut out{};
    out.dst[0] = C;
    out.world = 1;
    out.src = 0;
    out.chunk = M > 0 ? M : 1;
    return tc_gemm_rows_launch(A, M, K, Bt_hi, Bt_lo, N, out, splits, stages, st);
}

int tc_effective_splits(int64_t K, int splits) {
    const int num_kb = (int)((K + TC_BK - 1) / TC_BK);
    if (splits > num_kb) splits = num_kb;
    const int kb_per = (num_kb + splits - 1) / splits;
    return (num_kb + kb_per - 1) / kb_per;
}

int split_transpose_launch(const float *B, int64_t K, int r, float *hi, float *lo,
                           cudaStream_t st) {
    dim3 grid((unsigned)((K + 31) / 32), (unsigned)((r + 31) / 32));
    split_transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(B, K, r, hi, lo);
    return launch_status();
}

int transpose_launch(const float *in, int64_t rows, int64_t cols, float *out, cudaStream_t st) {
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
    transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(in, rows, cols, out);
    return launch_status();
}

}  // namespace nmfb
