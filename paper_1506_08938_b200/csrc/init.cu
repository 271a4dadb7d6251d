// Seeded initial factors on the device, bit-identical to the reference's
// host draw (nmf.py:115-127):
//     rng = np.random.default_rng(seed)
//     G = rng.uniform(size=(n, r)) * sqrt(mean / r)      (drawn first)
//     F = rng.uniform(size=(r, m)) * sqrt(mean / r);  FT = F.T
// numpy's default generator is PCG64 (128-bit LCG, XSL-RR output): one draw
//     state <- state * MULT + inc;  x = rotr64(hi(state) ^ lo(state), state >> 122)
//     u = (x >> 11) * 2^-53
// The host turns the seed into (state, inc) with numpy's own SeedSequence
// (np.random.PCG64(seed).state); every thread then jumps the LCG ahead to its
// chunk of the stream (affine-map squaring, O(log n) 128-bit multiplies) and
// generates the chunk.  Draw t fills G (t < n r, row-major) or F (C-order,
// written transposed into FT), scaled in fp64 and rounded once to the
// factor's dtype -- exactly what the host path's `u * scale` then `.to(fp32)`
// does.  At config 5 this replaces ~2 s of host PCG64 draws.
#include "common.cuh"
#include "nmfb_internal.h"

namespace nmfb {

namespace {

struct U128 {
    uint64_t hi, lo;
};

__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo * b.lo;
    r.hi = __umul64hi(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
    return r;
}

__device__ __forceinline__ U128 add128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
    return r;
}

__device__ __forceinline__ uint64_t pcg_output(U128 s) {
    const uint64_t x = s.hi ^ s.lo;
    const unsigned rot = (unsigned)(s.hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

constexpr int CHUNK = 64;

template <typename T>
__global__ void pcg64_factors_kernel(U128 state0, U128 inc, int64_t n, int64_t m, int r,
                                     double scale, T *__restrict__ G, T *__restrict__ FT) {
    const U128 mult = {0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull};
    const int64_t total = (n + m) * (int64_t)r;
    const int64_t t0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * CHUNK;
    if (t0 >= total) return;
    // affine map s -> A s + C for t0 steps, by squaring (A, C) of one step
    U128 A = {0, 1}, C = {0, 0};
    U128 a = mult, c = inc;
    for (uint64_t k = (uint64_t)t0; k; k >>= 1) {
        if (k & 1) {
            A = mul128(A, a);
            C = add128(mul128(C, a), c);
        }
        c = mul128(c, add128(a, U128{0, 1}));  // c <- c (a + 1)
        a = mul128(a, a);
    }
    U128 s = add128(mul128(A, state0), C);
    const int64_t nr = n * (int64_t)r;
    const int64_t t1 = (t0 + CHUNK < total) ? t0 + CHUNK : total;
    for (int64_t t = t0; t < t1; ++t) {
        s = add128(mul128(s, mult), inc);
        const double u = (double)(pcg_output(s) >> 11) * (1.0 / 9007199254740992.0);
        const T v = (T)(u * scale);
        if (t < nr) {
            G[t] = v;
        } else {
            const int64_t f = t - nr;          // F[k][j], C-order (r, m)
            const int64_t k = f / m, j = f - k * m;
            FT[j * r + k] = v;
        }
    }
}

}  // namespace

int pcg64_factors_launch(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                         int64_t n, int64_t m, int r, double scale, int dtype, void *G, void *FT,
                         cudaStream_t st) {
    if (n < 0 || m < 0 || r <= 0 || !G || !FT || (dtype != NMFB_F32 && dtype != NMFB_F64))
        return NMFB_ERR_ARG;
    const int64_t total = (n + m) * (int64_t)r;
    if (total == 0) return NMFB_OK;
    const int64_t threads = (total + CHUNK - 1) / CHUNK;
    const unsigned grid = (unsigned)((threads + 255) / 256);
    const U128 s0 = {state_hi, state_lo}, inc = {inc_hi, inc_lo};
    if (dtype == NMFB_F64)
        pcg64_factors_kernel<double><<<grid, 256, 0, st>>>(s0, inc, n, m, r, scale,
                                                           (double *)G, (double *)FT);
    else
        pcg64_factors_kernel<float><<<grid, 256, 0, st>>>(s0, inc, n, m, r, scale, (float *)G,
                                                          (float *)FT);
    return launch_status();
}

}  // namespace nmfb
