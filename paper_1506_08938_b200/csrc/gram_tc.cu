// Tensor-core Gram A^T A for fp32 factors (matrix.py:181-197 -> north star
// (1): "the Gram products ... on tensor cores"), sm_100a tcgen05 + TMA + TMEM.
//
// A is rows x r, row-major (r % 4 == 0, 16 <= r <= 224).  Both MMA operands
// are the SAME shared-memory tile: a TMA box of 32 columns x 32 rows (128 B
// swizzle) is one MN-major UMMA atom column (32 Gram indices x 8..32 input
// rows; 128B swizzle with a 32B base), so the tile of input rows serves as A^T (M side) and as A (N side)
// without a transpose or a second load.
//
// Precision (3xTF32): a = hi + lo, hi = the tf32 the tensor core reads from
// the raw fp32 bits, lo = a - hi (exact, formed in shared memory by the split
// warps);  a_i a_j ~= hi_i hi_j + hi_i lo_j + lo_i hi_j  (~2^-21 per product).
// The tensor core's fp32 accumulate TRUNCATES, a downward bias of about half
// an ulp per accumulation, so
//   * a chunk is 64 input rows (two stages): its 16 lo-term MMAs are issued
//     FIRST, while the accumulator is ~2^-11 of its final size (their
//     truncations are negligible), then the 8 hi*hi MMAs (~2e-7 bias);
//   * each finished chunk is folded by the fold warps into register-resident
//     fp32 running sums with round-to-nearest adds (tcgen05.ld), and the unit's
//     sums are written as fp64 partials, summed in unit order by the same
//     deterministic reduce (+ fused rescale epilogue) as the CUDA-core path.
//
// Output tiles (upper triangle only): tile 0 = Gram rows [0,128) x columns
// [0, N0), N0 = 32 NB, NB = ceil(r / 32); for r > 128 tile 1 = Gram rows
// [32 (NB-4), 32 NB) (the last four atom columns, so every A atom exists) x
// columns [128, N0): rows >= 128 of it are used.  TMEM: D0 at column 0 (N0
// columns), D1 at column N0 (N0 - 128 columns), <= 320 of 512.
//
// CTA = one unit of `unit_rows` input rows (a multiple of 64; rows past the
// end are TMA zero fill); 16 warps in four warpgroups:
//   warp 0      TMA producer (NB boxes per 32-row stage)
//   warp 1      MMA issuer (one elected lane)
//   warps 2-7   split: lo = a - tf32(a) for the stage, in shared memory
//   warps 8-15  fold: TMEM chunk -> register running sums; final fp64 partial
// The fold warps hold up to 160 running sums each: setmaxnreg moves registers
// from warpgroups 0-1 (40 each) to warpgroups 2-3 (216 each).
// HBM roofline: reads rows * r * 4 bytes once.
#include <cuda.h>

#include <cstdlib>

#include "common.cuh"
#include "nmfb_internal.h"
#include "tcgen05.cuh"

namespace nmfb {

constexpr int GTC_THREADS = 512;
constexpr int GTC_STAGE_ROWS = 32;
constexpr int GTC_BOX_BYTES = GTC_STAGE_ROWS * 128;  // 32 rows x 32 fp32
constexpr int GTC_SPLIT_THREADS = 192;
constexpr int GTC_FOLD_THREADS = 256;
constexpr int GTC_MAX_NB = 7;

// MN-major tf32 operands have one legal shared-memory layout: the 128-byte
// swizzle with a 32-byte base (descriptor layout type 1; the TMA side is
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B).  Atoms are 32 MN elements (128 B) x 4
// K rows; LBO = byte stride between atoms along MN (one TMA box), SBO = stride
// between 4-row K groups (512 B: the box keeps its rows 128 B apart).
__device__ __forceinline__ uint64_t umma_desc_mn_sw128(uint32_t saddr, uint32_t lbo_bytes) {
    uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)(lbo_bytes >> 4) << 16;
    d |= (uint64_t)(512 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)1 << 61;
    return d;
}

// the tensor core truncates its fp32 operand to tf32; rounding lo to nearest
// first keeps the operand error unbiased
__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t u;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
    return __uint_as_float(u);
}

__global__ void __maxnreg__(128)
    gram_tc_kernel(const __grid_constant__ CUtensorMap tmA, int r, int NB, int stages,
                   int unit_rows, double *__restrict__ part) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const uint32_t half_bytes = (uint32_t)NB * GTC_BOX_BYTES;  // hi (or lo) tile of a stage
    const uint32_t stage_bytes = 2 * half_bytes;
    // r <= 96: the M = 128 operand reads 4 - NB atom columns past a tile (they
    // feed accumulator rows >= 32 NB, never stored); the last stage's overrun
    // lands in this pad, inside the allocation
    const uint32_t pad_bytes = NB < 4 ? (uint32_t)(4 - NB) * GTC_BOX_BYTES : 0u;
    uint64_t *bars = (uint64_t *)(smem + (size_t)stages * stage_bytes + pad_bytes);
    uint64_t *full = bars, *split_done = bars + stages, *empty = bars + 2 * stages;
    uint64_t *d_full = bars + 3 * stages;       // [2]
    uint64_t *d_empty = bars + 3 * stages + 2;  // [2]
    uint32_t *tmem_slot = (uint32_t *)(bars + 3 * stages + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int unit = blockIdx.x;
    const int nst = unit_rows / GTC_STAGE_ROWS;  // even
    const int nchunk = nst / 2;
    const bool two = NB > 4;
    const int N0 = 32 * NB, N1 = two ? N0 - 128 : 0;

    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < stages; ++s) {
                mbar_init(&full[s], 1);
                mbar_init(&split_done[s], GTC_SPLIT_THREADS);
                mbar_init(&empty[s], 1);
            }
            for (int t = 0; t < 2; ++t) {
                mbar_init(&d_full[t], 1);
                mbar_init(&d_empty[t], GTC_FOLD_THREADS);
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmA) : "memory");
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

    if (warp < 8) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
        if (warp == 0) {
            // ---------------- TMA producer ----------------
            if (lane == 0) {
                const int row0 = unit * unit_rows;
                for (int i = 0; i < nst; ++i) {
                    const int s = i % stages;
                    mbar_wait(&empty[s], (((uint32_t)(i / stages)) & 1u) ^ 1u);
                    uint8_t *st = smem + (size_t)s * stage_bytes;
                    mbar_expect_tx(&full[s], half_bytes);
                    for (int b = 0; b < NB; ++b)
                        tma_load_2d(&tmA, &full[s], st + (size_t)b * GTC_BOX_BYTES, 32 * b,
                                    row0 + i * GTC_STAGE_ROWS);
                }
            }
            __syncwarp();
        } else if (warp == 1) {
            // ---------------- MMA issuer ----------------
            if (lane == 0) {
                // F32 accumulate, TF32 operands, A and B both MN-major, M = 128
                const uint32_t idesc_base = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) |
                                            (1u << 16) | ((uint32_t)(128 >> 4) << 24);
                const uint32_t idesc0 = idesc_base | ((uint32_t)(N0 >> 3) << 17);
                const uint32_t idesc1 = idesc_base | ((uint32_t)(N1 >> 3) << 17);
                const uint32_t smem_base = smem_u32(smem);
                for (int c = 0; c < nchunk; ++c) {
                    const int i0 = 2 * c;
                    uint32_t sb[2];
                    for (int j = 0; j < 2; ++j) {
                        const int i = i0 + j, s = i % stages;
                        mbar_wait(&split_done[s], ((uint32_t)(i / stages)) & 1u);
                        sb[j] = smem_base + (uint32_t)s * stage_bytes;
                    }
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    for (int t = 0; t < (two ? 2 : 1); ++t) {
                        mbar_wait(&d_empty[t], (((uint32_t)c) & 1u) ^ 1u);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        const uint32_t d = tmem + (uint32_t)(t ? N0 : 0);
                        const uint32_t idesc = t ? idesc1 : idesc0;
                        // A atoms: tile 0 boxes 0..3, tile 1 the last four boxes;
                        // B atoms: tile 0 from box 0, tile 1 from box 4
                        const uint32_t a_off = (uint32_t)(t ? (NB - 4) : 0) * GTC_BOX_BYTES;
                        const uint32_t b_off = (uint32_t)(t ? 4 : 0) * GTC_BOX_BYTES;
                        uint32_t acc = 0u;
                        // lo terms first (accumulator still tiny: truncation negligible)
                        for (int j = 0; j < 2; ++j) {
#pragma unroll
                            for (int k = 0; k < GTC_STAGE_ROWS / 8; ++k) {
                                const uint32_t hi = sb[j] + (uint32_t)k * 1024u;
                                const uint32_t lo = hi + half_bytes;
                                umma_tf32(d, umma_desc_mn_sw128(hi + a_off, GTC_BOX_BYTES),
                                          umma_desc_mn_sw128(lo + b_off, GTC_BOX_BYTES), idesc,
                                          acc);
                                acc = 1u;
                                umma_tf32(d, umma_desc_mn_sw128(lo + a_off, GTC_BOX_BYTES),
                                          umma_desc_mn_sw128(hi + b_off, GTC_BOX_BYTES), idesc,
                                          1u);
                            }
                        }
                        for (int j = 0; j < 2; ++j) {
#pragma unroll
                            for (int k = 0; k < GTC_STAGE_ROWS / 8; ++k) {
                                const uint32_t hi = sb[j] + (uint32_t)k * 1024u;
                                umma_tf32(d, umma_desc_mn_sw128(hi + a_off, GTC_BOX_BYTES),
                                          umma_desc_mn_sw128(hi + b_off, GTC_BOX_BYTES), idesc,
                                          1u);
                            }
                        }
                        umma_commit(&d_full[t]);
                    }
                    // both stages are reusable once every MMA above has read them
                    umma_commit(&empty[i0 % stages]);
                    umma_commit(&empty[(i0 + 1) % stages]);
                }
            }
            __syncwarp();
        } else {
            // ---------------- split warps: lo = a - tf32(a) ----------------
            const int t = threadIdx.x - 64;  // 0..191
            const int nvec = NB * (GTC_BOX_BYTES / 16);
            for (int i = 0; i < nst; ++i) {
                const int s = i % stages;
                mbar_wait(&full[s], ((uint32_t)(i / stages)) & 1u);
                const float4 *src = (const float4 *)(smem + (size_t)s * stage_bytes);
                float4 *dst = (float4 *)(smem + (size_t)s * stage_bytes + half_bytes);
                for (int q = t; q < nvec; q += GTC_SPLIT_THREADS) {
                    const float4 v = src[q];
                    float4 o;
                    o.x = tf32_rna(v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u));
                    o.y = tf32_rna(v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u));
                    o.z = tf32_rna(v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u));
                    o.w = tf32_rna(v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u));
                    dst[q] = o;
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(&split_done[s]);
            }
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 216;");
        // ---------------- fold warps ----------------
        const int quarter = warp & 3;     // TMEM lane quarter of this warp
        const int half = (warp - 8) >> 2;  // column half of each tile
        const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
        const int HB0 = NB;                // 16-column blocks per half, tile 0
        const int HB1 = two ? NB - 4 : 0;  // tile 1
        const uint32_t col0 = (uint32_t)(half * 16 * HB0);
        const uint32_t col1 = (uint32_t)(N0 + half * 16 * HB1);
        float s0[GTC_MAX_NB][16], s1[GTC_MAX_NB - 4][16];
#pragma unroll
        for (int b = 0; b < GTC_MAX_NB; ++b)
#pragma unroll
            for (int u = 0; u < 16; ++u) s0[b][u] = 0.f;
#pragma unroll
        for (int b = 0; b < GTC_MAX_NB - 4; ++b)
#pragma unroll
            for (int u = 0; u < 16; ++u) s1[b][u] = 0.f;
        for (int c = 0; c < nchunk; ++c) {
            const uint32_t ph = ((uint32_t)c) & 1u;
            mbar_wait(&d_full[0], ph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            // two 16-column loads in flight per wait
#pragma unroll
            for (int b = 0; b < GTC_MAX_NB; b += 2) {
                if (b < HB0) {
                    uint32_t v[16], w[16];
                    const bool pair = b + 1 < GTC_MAX_NB && b + 1 < HB0;
                    tmem_ld16(tmem + lane_base + col0 + (uint32_t)(b * 16), v);
                    if (pair) tmem_ld16(tmem + lane_base + col0 + (uint32_t)(b * 16 + 16), w);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int u = 0; u < 16; ++u)
                        s0[b][u] = __fadd_rn(s0[b][u], __uint_as_float(v[u]));
                    if (b + 1 < GTC_MAX_NB && pair) {
#pragma unroll
                        for (int u = 0; u < 16; ++u)
                            s0[b + 1 < GTC_MAX_NB ? b + 1 : b][u] = __fadd_rn(
                                s0[b + 1 < GTC_MAX_NB ? b + 1 : b][u], __uint_as_float(w[u]));
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            mbar_arrive(&d_empty[0]);
            if (two) {
                mbar_wait(&d_full[1], ph);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int b = 0; b < GTC_MAX_NB - 4; b += 2) {
                    if (b < HB1) {
                        uint32_t v[16], w[16];
                        const bool pair = b + 1 < GTC_MAX_NB - 4 && b + 1 < HB1;
                        tmem_ld16(tmem + lane_base + col1 + (uint32_t)(b * 16), v);
                        if (pair) tmem_ld16(tmem + lane_base + col1 + (uint32_t)(b * 16 + 16), w);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                        for (int u = 0; u < 16; ++u)
                            s1[b][u] = __fadd_rn(s1[b][u], __uint_as_float(v[u]));
                        if (b + 1 < GTC_MAX_NB - 4 && pair) {
#pragma unroll
                            for (int u = 0; u < 16; ++u)
                                s1[b + 1 < GTC_MAX_NB - 4 ? b + 1 : b][u] =
                                    __fadd_rn(s1[b + 1 < GTC_MAX_NB - 4 ? b + 1 : b][u],
                                              __uint_as_float(w[u]));
                        }
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mbar_arrive(&d_empty[1]);
            }
        }
        // the unit's partial (upper triangle), fp64
        double *out = part + (size_t)unit * r * r;
        {
            const int a = quarter * 32 + lane;
#pragma unroll
            for (int b = 0; b < GTC_MAX_NB; ++b) {
                if (b < HB0 && a < r) {
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        const int j = (int)col0 + b * 16 + u;
                        if (j < r && a <= j) out[(size_t)a * r + j] = (double)s0[b][u];
                    }
                }
                asm volatile("" ::: "memory");  // keep the conversions block by block
            }
        }
        if (two) {
            const int a = 32 * (NB - 4) + quarter * 32 + lane;
#pragma unroll
            for (int b = 0; b < GTC_MAX_NB - 4; ++b) {
                if (b < HB1 && a >= 128 && a < r) {
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        const int j = 128 + half * 16 * HB1 + b * 16 + u;
                        if (j < r && a <= j) out[(size_t)a * r + j] = (double)s1[b][u];
                    }
                }
                asm volatile("" ::: "memory");
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(512));
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static bool gram_tc_enabled() {
    static const bool on = [] {
        const char *e = getenv("NMFB_GRAM_TC");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Eligibility of the tensor-core path (fp32 only; the caller checks dtype).
bool gram_tc_ok(const void *A, int64_t rows, int r, int64_t lda) {
    if (!gram_tc_enabled()) return false;
    if (r < 16 || r > 32 * GTC_MAX_NB || (r & 3) || (lda & 3) || lda < r) return false;
    if (((uintptr_t)A & 15) || rows < 2048 || rows > (int64_t)1 << 30) return false;
    return encode_fn() != nullptr;
}

static int gram_tc_sms() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0, v = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
            sms = v;
        else
            sms = 148;
    }
    return sms > 296 ? 296 : sms;  // the partial workspace holds at most 296 units
}

// One wave: at most one unit per SM (each CTA owns an SM's shared memory and
// TMEM), each a multiple of the 64-row chunk.
static int64_t gram_tc_unit_rows(int64_t rows) {
    const int64_t n = gram_tc_sms();
    int64_t u = (rows + n - 1) / n;
    u = ((u + 63) / 64) * 64;
    return u < 64 ? 64 : u;
}

// Partials of A^T A into part[unit][r][r] (upper triangle); returns the unit
// count through *nunit.  ws sizing: gram_workspace_bytes (units <= 296).
int gram_tc_partial_launch(const float *A, int64_t rows, int r, int64_t lda, double *part,
                           int64_t *nunit, cudaStream_t st) {
    const int NB = (r + 31) / 32;
    const int64_t unit_rows = gram_tc_unit_rows(rows);
    const int64_t units = (rows + unit_rows - 1) / unit_rows;
    *nunit = units;
    CUtensorMap map;
    {
        EncodeTiledFn fn = encode_fn();
        if (!fn) return NMFB_ERR_ARG;
        cuuint64_t dims[2] = {(cuuint64_t)r, (cuuint64_t)rows};
        cuuint64_t strides[1] = {(cuuint64_t)lda * 4};
        cuuint32_t box[2] = {32u, (cuuint32_t)GTC_STAGE_ROWS};
        cuuint32_t estr[2] = {1, 1};
        if (fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)A, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return NMFB_ERR_ARG;
    }
    const size_t stage_bytes = 2 * (size_t)NB * GTC_BOX_BYTES;
    const size_t pad_bytes = NB < 4 ? (size_t)(4 - NB) * GTC_BOX_BYTES : 0;
    const size_t budget = 227 * 1024 - 1024 - 512 - pad_bytes;
    int stages = (int)(budget / stage_bytes);
    if (stages > 8) stages = 8;
    if (stages < 3) return NMFB_ERR_ARG;
    const size_t smem = stages * stage_bytes + pad_bytes + (3 * stages + 6) * 8 + 1024;
    // per device, cheap: set on every call
    if (cudaFuncSetAttribute(gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024) != cudaSuccess)
        return launch_status();
    gram_tc_kernel<<<(unsigned)units, GTC_THREADS, smem, st>>>(map, r, NB, stages, (int)unit_rows,
                                                              part);
    return launch_status();
}

}  // namespace nmfb
