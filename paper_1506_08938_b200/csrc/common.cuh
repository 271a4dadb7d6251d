// Shared helpers for the sm_100a kernels of the alternating-NNLS hot path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define NMFB_FULL_MASK 0xffffffffu

namespace nmfb {

// Arithmetic policy.  Exact<T> never contracts a multiply-add (every product
// is rounded before the sum), matching numba/fastmath=False and the C oracle
// compiled with -ffp-contract=off: with T=double it is bit-exact against the
// reference.  Fast<T> uses fused multiply-add.
template <typename T> struct Exact;
template <> struct Exact<double> {
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
    // a + b*c with two roundings
    static __device__ __forceinline__ double madd(double a, double b, double c) {
        return __dadd_rn(a, __dmul_rn(b, c));
    }
    // a - b*c with two roundings
    static __device__ __forceinline__ double msub(double a, double b, double c) {
        return __dsub_rn(a, __dmul_rn(b, c));
    }
};
template <> struct Exact<float> {
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
    static __device__ __forceinline__ float madd(float a, float b, float c) {
        return __fadd_rn(a, __fmul_rn(b, c));
    }
    static __device__ __forceinline__ float msub(float a, float b, float c) {
        return __fsub_rn(a, __fmul_rn(b, c));
    }
};

template <typename T> struct Fast;
template <> struct Fast<float> {
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
    static __device__ __forceinline__ float madd(float a, float b, float c) {
        return __fmaf_rn(b, c, a);
    }
    static __device__ __forceinline__ float msub(float a, float b, float c) {
        return __fmaf_rn(-b, c, a);
    }
};

// Python's builtin max(a, b) (kernels.py:117): b only when strictly greater.
template <typename T>
__device__ __forceinline__ T py_max(T a, T b) { return (b > a) ? b : a; }

template <typename T> __device__ __forceinline__ T dev_inf();
template <> __device__ __forceinline__ double dev_inf<double>() { return __longlong_as_double(0x7ff0000000000000ULL); }
template <> __device__ __forceinline__ float dev_inf<float>() { return __int_as_float(0x7f800000); }

__device__ __forceinline__ bool is_finite(double v) { return isfinite(v); }
__device__ __forceinline__ bool is_finite(float v) { return isfinite(v); }

// Fast-break bookkeeping (kernels.py:246-248, 266-267, 145): a problem's stop
// test may read max_stop = max(max_stop0, final norms of the earlier problems
// of its 32-aligned block).  Problems iterate in lockstep; a problem whose own
// rule did not fire WAITS (holding its iterate) until that threshold is known
// or a lower bound of it already stops it.  Exactly reproduces the sequential
// stop indices without snapshots.
enum : int { ST_RUNNING = 0, ST_WAITING = 1, ST_DONE = 2 };

// One warp == one fast-break block, lane == position in the block.
// independent == true: every lane is its own scope with threshold m0 (the
// public single-problem solve, nqp.py:217, where StopState is per call).
template <typename T>
__device__ __forceinline__ void resolve_block_warp(int &status, T norm_k, T &final_norm, T m0,
                                                   bool independent = false) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = independent ? 0u : (1u << lane) - 1u;
    while (true) {
        unsigned done = __ballot_sync(NMFB_FULL_MASK, status == ST_DONE);
        T v = (status == ST_DONE) ? final_norm : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T t = __shfl_up_sync(NMFB_FULL_MASK, v, o);
            if (lane >= o) v = (t > v) ? t : v;
        }
        T excl = __shfl_up_sync(NMFB_FULL_MASK, v, 1);
        if (lane == 0 || independent) excl = T(0);
        T P = (excl > m0) ? excl : m0;
        bool changed = false;
        if (status == ST_WAITING) {
            if (norm_k <= P) {
                status = ST_DONE;
                final_norm = norm_k;
                changed = true;
            } else if ((done & lt) == lt) {
                status = ST_RUNNING;
                changed = true;
            }
        }
        if (!__any_sync(NMFB_FULL_MASK, changed)) break;
    }
}

__device__ __forceinline__ void atomic_min_i64(long long *addr, long long v) {
    atomicMin(addr, v);
}

}  // namespace nmfb
