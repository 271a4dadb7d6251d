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

#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "nmfb_internal.h"

namespace nmfb {

constexpr int TC_BM = 128;
constexpr int TC_BK = 32;  // one 128-byte swizzle row of fp32
constexpr int TC_THREADS = 192;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra.uni WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap *map, uint64_t *bar, void *dst,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ uint64_t umma_desc_sw128(const void *p) {
    // K-major, SWIZZLE_128B (layout 2), version 1 (sm100), SBO = 1024 B
    // (8 rows x 128 B), LBO = 16 B (unused for swizzled K-major), base offset 0
    uint64_t addr = (uint64_t)((smem_u32(p) & 0x3FFFFu) >> 4);
    uint64_t d = addr;
    d |= (uint64_t)1 << 16;              // LBO (16 B units)
    d |= (uint64_t)(1024 >> 4) << 32;    // SBO
    d |= (uint64_t)1 << 46;              // version
    d |= (uint64_t)2 << 61;              // SWIZZLE_128B
    return d;
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
        "r"(v[15])
        : "memory");
}

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
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    });
    return fn;
}

// 2-D fp32 row-major tensor (rows x cols, cols contiguous), box = (32 cols, box_rows)
static bool make_map(CUtensorMap *map, const float *ptr, int64_t rows, int64_t cols,
                     int box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
    cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)ptr, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

size_t tc_gemm_smem_bytes(int BN, int stages) {
    size_t stage = 2 * (size_t)TC_BM * TC_BK * 4 + 2 * (size_t)BN * TC_BK * 4;
    return stages * stage + (3 * stages + 6) * 8 + 1024;
}

int tc_gemm_launch(const float *A, int64_t M, int64_t K, const float *Bt_hi, const float *Bt_lo,
                   int N, float *C, int splits, int stages, cudaStream_t st) {
    // 3 x BN TMEM columns (two chunk buffers + running sum) must fit in 512
    if (M <= 0 || K <= 0 || N <= 0 || N > 160 || splits < 1) return NMFB_ERR_ARG;
    if ((K * 4) % 16 != 0) return NMFB_ERR_ARG;  // TMA row pitch must be 16-byte aligned
    if (((uintptr_t)A | (uintptr_t)Bt_hi | (uintptr_t)Bt_lo) % 16 != 0) return NMFB_ERR_ARG;
    const int BN = ((N + 15) / 16) * 16;
    if (stages <= 0) stages = 2;
    while (stages > 2 && tc_gemm_smem_bytes(BN, stages) > 227 * 1024) --stages;
    size_t smem = tc_gemm_smem_bytes(BN, stages);
    CUtensorMap ta, tb, tbl;
    if (!make_map(&ta, A, M, K, TC_BM) || !make_map(&tb, Bt_hi, N, K, BN) ||
        !make_map(&tbl, Bt_lo, N, K, BN))
        return NMFB_ERR_CUDA;
    const int num_kb = (int)((K + TC_BK - 1) / TC_BK);
    if (splits > num_kb) splits = num_kb;
    const int kb_per = (num_kb + splits - 1) / splits;
    splits = (num_kb + kb_per - 1) / kb_per;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024);
        attr_set = true;
    }
    dim3 grid((unsigned)((M + TC_BM - 1) / TC_BM), (unsigned)splits);
    const int chunk_kb = 2;  // 24 tensor-core accumulations between promotions
    tc_gemm_kernel<<<grid, TC_THREADS, smem, st>>>(ta, tb, tbl, C, (int)M, N, BN, num_kb, kb_per,
                                                   stages, chunk_kb, (int64_t)M * N);
    return launch_status();
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
