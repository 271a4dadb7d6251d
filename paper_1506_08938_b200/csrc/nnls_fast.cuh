// Fast fp32 batched NNLS (warp-group per problem); see nnls.cu.
#pragma once
#include <type_traits>

#include "nnls_common.cuh"

// smallest E (coordinates per lane, L = 8) that uses the warp-shared Q
// product q_times_w4
// exact greedy-CD argmax (kernels.py:119); 0 = truncated-key experiment
#ifndef NMFB_NNLS_EXACT_ARGMAX
#define NMFB_NNLS_EXACT_ARGMAX 1
#endif

#ifndef NMFB_NNLS_DCARRY
#define NMFB_NNLS_DCARRY 0  // measured slower: r=200 1.67 -> 1.82 ms
#endif

#ifndef NMFB_NNLS_YSMEM
#define NMFB_NNLS_YSMEM 0
#endif

#ifndef NMFB_NNLS_W4_MIN_E
#define NMFB_NNLS_W4_MIN_E 13
#endif

namespace nmfb {

// ---------------------------------------------------------------------------
// Fast fp32 kernel: group of L lanes per problem, E coordinates per lane.
// ---------------------------------------------------------------------------
template <int L>
__device__ __forceinline__ float gsum(float v, unsigned gmask) {
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) v += __shfl_xor_sync(gmask, v, o, L);
    return v;
}
template <int L>
__device__ __forceinline__ float gmin(float v, unsigned gmask) {
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(gmask, v, o, L));
    return v;
}
template <int L>
__device__ __forceinline__ bool gany(bool p, unsigned gmask, int gbase) {
    if (L == 1) return p;
    unsigned b = __ballot_sync(gmask, p);
    return ((b >> gbase) & ((L == 32) ? 0xffffffffu : ((1u << L) - 1u))) != 0u;
}

// Shared-memory layout of the compact Q (ra x ra, symmetric), permuted per
// row so that a lane's E coordinates are contiguous: row j holds, for lane
// l, the entries Q[j][e*L + l] (e = 0..E-1) at Qs[j*SP + l*LS + e], LS = E
// rounded up to 4 (zero padded) and then to an odd number of 16-byte quads,
// SP = L*LS.  Both consumers read whole rows with 16-byte loads: the product
// Q*src (all groups of a warp read the same row j -> broadcast) and the
// greedy-CD gradient update with column p (= row p by symmetry).  With LS/4
// odd, the 8 lanes of a quarter-warp start on 8 distinct bank quads:
// conflict-free.
__host__ __device__ constexpr int nnls_ep(int E) { return (E + 3) & ~3; }
__host__ __device__ constexpr int nnls_ls(int E) {
    return ((nnls_ep(E) / 4) & 1) ? nnls_ep(E) : nnls_ep(E) + 4;
}
__host__ __device__ constexpr int nnls_ee(int E) { return (E + 1) & ~1; }

// acc[e] += s * row[e] for e < EE (EE = E rounded up to even), packed FFMA2.
template <int EE, int EP>
__device__ __forceinline__ void axpy_row(float (&acc)[EE], const float *row, float s) {
    const float4 *r4 = reinterpret_cast<const float4 *>(row);
    const float2 s2 = make_float2(s, s);
#pragma unroll
    for (int q = 0; q < EP / 4; ++q) {
        const float4 v = r4[q];
        if (4 * q + 1 < EE) {
            const float2 o = __ffma2_rn(make_float2(v.x, v.y), s2,
                                        make_float2(acc[4 * q], acc[4 * q + 1]));
            acc[4 * q] = o.x;
            acc[4 * q + 1] = o.y;
        }
        if (4 * q + 3 < EE) {
            const float2 o = __ffma2_rn(make_float2(v.z, v.w), s2,
                                        make_float2(acc[4 * q + 2], acc[4 * q + 3]));
            acc[4 * q + 2] = o.x;
            acc[4 * q + 3] = o.y;
        }
    }
}

// acc[e] += sum_j Q[k_e, j] * src(j), src(j) owned by lane (j % L), element
// j / L; the source values come from a functor of the element index (held or
// recomputed: d = passive gradient, delta = step).
//
// The groups of a warp start the source-lane loop at different offsets
// (rot, one per quarter-warp), so the four quarter-warp phases of a 16-byte
// load fetch four different rows instead of the same row four times
// (shared-memory bandwidth, not a broadcast, is what a quarter-warp phase
// costs).  Each problem's summation order is fixed by its slot in the warp
// (its index mod 32), so results do not depend on sharding.
template <int E, int L, int EE, int EP, typename F>
__device__ __forceinline__ void q_times_f(float (&acc)[EE], F src, const float *Qs_l,
                                          unsigned gmask, int rot) {
    constexpr int SP = L * nnls_ls(E);
#pragma unroll 1
    for (int t = 0; t < L; ++t) {
        const int jl = (t + rot) & (L - 1);
#pragma unroll
        for (int je = 0; je < E; ++je) {
            const float mine = src(je);
            const float sj = (L == 1) ? mine : __shfl_sync(gmask, mine, jl, L);
            axpy_row<EE, EP>(acc, Qs_l + (je * L + jl) * SP, sj);
        }
    }
}

// Q * src for the 4 problems of a warp (L = 8) with every Q element loaded
// ONCE per warp and used for all 4 problems: lane l computes rows
// k = e4 * 32 + l of all four problems (accumulators a[e4][p], packed in
// pairs of problems for FFMA2); the four source values of column j are four
// shuffles.  Each Q load is a 32-bit load of the permuted layout
// (bank-conflict-free for LS/4 odd), so a column costs 4 shuffles +
// ceil(R/32) loads instead of E 16-byte loads per group -- 2.6x fewer
// shared-memory wavefronts at r = 200.  The accumulators move between the
// group layout (lane l of group g: rows e*8 + l of problem g) and the warp
// layout 32 rows at a time through `scr` (128 floats per warp): rows
// e4*32 .. e4*32+31 are the elements e = 4 e4 .. 4 e4 + 3 of every group.
// Per row, the j order is the same as q_times_f's, so the result is
// bit-identical to it with rot = 0.
template <int E, int EE, typename F>
__device__ __forceinline__ void q_times_w4(float (&acc)[EE], F src, const float *Qs,
                                           float *scr, int r, int lane) {
    constexpr int L = 8, LS = nnls_ls(E), SP = L * LS;
    constexpr int E4 = (E * L + 31) / 32;
    const int l = lane & 7, g = lane >> 3;
    float2 a[E4][2];  // [e4][problem pair]: (p0, p1), (p2, p3)
#pragma unroll
    for (int e4 = 0; e4 < E4; ++e4) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = 4 * e4 + q;
            if (e < E) scr[g * 32 + q * 8 + l] = acc[e];
        }
        __syncwarp();
        const int k = e4 * 32 + lane;
        float v[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) v[p] = (k < r) ? scr[p * 32 + lane] : 0.f;
        a[e4][0] = make_float2(v[0], v[1]);
        a[e4][1] = make_float2(v[2], v[3]);
        __syncwarp();
    }
    const float *qcol = Qs + (lane & 7) * LS + (lane >> 3);  // + e4 * 4 + j * SP
#pragma unroll 1
    for (int jl = 0; jl < L; ++jl) {
#pragma unroll
        for (int je = 0; je < E; ++je) {
            const float mine = src(je);
            float sp[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) sp[p] = __shfl_sync(NMFB_FULL_MASK, mine, 8 * p + jl);
            const float2 s01 = make_float2(sp[0], sp[1]), s23 = make_float2(sp[2], sp[3]);
            const float *row = qcol + (je * L + jl) * SP;
#pragma unroll
            for (int e4 = 0; e4 < E4; ++e4) {
                const float q = row[e4 * 4];
                const float2 q2 = make_float2(q, q);
                a[e4][0] = __ffma2_rn(q2, s01, a[e4][0]);
                a[e4][1] = __ffma2_rn(q2, s23, a[e4][1]);
            }
        }
    }
#pragma unroll
    for (int e4 = 0; e4 < E4; ++e4) {
        scr[0 * 32 + lane] = a[e4][0].x;
        scr[1 * 32 + lane] = a[e4][0].y;
        scr[2 * 32 + lane] = a[e4][1].x;
        scr[3 * 32 + lane] = a[e4][1].y;
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = 4 * e4 + q;
            // (rows k >= r read back exact zeros: zero sources, zero Q padding)
            if (e < E) acc[e] = scr[g * 32 + q * 8 + l];
        }
        __syncwarp();
    }
}

// Q * src for the problems with `cond`: the warp-shared product for L = 8 at
// larger ranks (called from warp-uniform control flow; skipped only when no
// problem of the warp needs it, zero sources for the others), else per group.
template <int E, int L, int EE, int EP, typename F>
__device__ __forceinline__ void qmul_if(bool cond, float (&acc)[EE], F src, const float *Qs,
                                        const float *Qsl, float *wscr, int r, int lane,
                                        unsigned gmask, int rot) {
    if constexpr (L == 8 && E >= NMFB_NNLS_W4_MIN_E) {
        if (__any_sync(NMFB_FULL_MASK, cond)) {
            auto masked = [&](int e) { return cond ? src(e) : 0.f; };
            q_times_w4<E, EE>(acc, masked, Qs, wscr, r, lane);
        }
    } else {
        if (cond) q_times_f<E, L, EE, EP>(acc, src, Qsl, gmask, rot);
    }
}

// h = h_base - sum of the split-K partials, with independent loads in flight
// (four accumulators) instead of a load -> add dependency chain.
template <typename TH>
__device__ __forceinline__ float fast_h(const NnlsArgs<float, TH> &a, int64_t j, int i) {
    const TH *p = a.hp + j * a.h_ld + i;
    if (a.S == 0) return (float)p[0];
    TH s0 = p[0], s1 = TH(0), s2 = TH(0), s3 = TH(0);
    int k = 1;
#pragma unroll 1
    for (; k + 3 < a.S; k += 4) {
        s0 += p[(int64_t)k * a.h_pstride];
        s1 += p[(int64_t)(k + 1) * a.h_pstride];
        s2 += p[(int64_t)(k + 2) * a.h_pstride];
        s3 += p[(int64_t)(k + 3) * a.h_pstride];
    }
#pragma unroll 1
    for (; k < a.S; ++k) s0 += p[(int64_t)k * a.h_pstride];
    return (float)((TH)a.h_base - ((s0 + s1) + (s2 + s3)));
}

// Occupancy target: ~4E + 48 live registers per thread (y, grad and Q*d per
// coordinate; the passive gradient and step are recomputed) -> CTAs per SM.
#ifndef NMFB_NNLS_REG_SLACK
#define NMFB_NNLS_REG_SLACK 0
#endif
__host__ __device__ constexpr int nnls_regs(int E, int L) {
    return 4 * E + 48 + (L == 1 ? 48 : 0) + NMFB_NNLS_REG_SLACK;
}
__host__ __device__ constexpr int nnls_min_blocks(int E, int L, int threads) {
    return (65536 / (nnls_regs(E, L) * threads)) < 1 ? 1 : (65536 / (nnls_regs(E, L) * threads));
}

// MIRROR: the solution rows are also stored into a.mirror[] (fused
// all-gather of the multi-GPU path) -- a separate instantiation, so the
// single-GPU kernel carries no extra code
template <typename TH, int E, int L, int B, bool MIRROR>
__global__ void __launch_bounds__(32 * L * B, nnls_min_blocks(E, L, 32 * L * B))
    nnls_fast_kernel(NnlsArgs<float, TH> a) {
    constexpr int R = E * L;
    constexpr int EE = nnls_ee(E), EP = nnls_ep(E), LS = nnls_ls(E), SP = L * LS;
    constexpr bool STAGE_H = E < NMFB_NNLS_W4_MIN_E;  // see the prologue
    // y in shared memory during the greedy CD (experiment, default off:
    // r = 200 1.84 -> 2.02 ms -- the per-selection y reload lengthens the
    // dependency chain more than the removed owner select saves)
    constexpr bool YSMEM = NMFB_NNLS_EXACT_ARGMAX && NMFB_NNLS_YSMEM;
    // the winner's step carried through the exact argmax tree (see the CD)
    constexpr bool DCARRY = NMFB_NNLS_EXACT_ARGMAX && (YSMEM || NMFB_NNLS_DCARRY);
    extern __shared__ __align__(16) float smem_f[];
    float *Qs = smem_f;                          // R x SP, permuted rows (see nnls_ep)
    __shared__ float blk_norm[B][32], blk_final[B][32];
    __shared__ int blk_status[B][32];
    __shared__ int blk_any[B];
    __shared__ int act_s[R];      // act_idx / scale_a / active staged once per CTA
    __shared__ unsigned char actv_s[R];
    __shared__ float scl_s[R];

    const int tid = threadIdx.x;
    const int ra = a.ra_dev ? *a.ra_dev : a.ra, r = a.r;
    {
        float4 *q4 = reinterpret_cast<float4 *>(Qs);
        for (int idx = tid; idx < R * SP / 4; idx += blockDim.x)
            q4[idx] = make_float4(0.f, 0.f, 0.f, 0.f);
        __syncthreads();
        // coalesced reads of the compact Q (eight loads in flight per
        // thread), scattered into the permuted rows
        for (int row = tid >> 5; row < ra; row += blockDim.x >> 5) {
            const float *src = a.Qa + (size_t)row * ra;
            for (int k0 = tid & 31; k0 < ra; k0 += 256) {
                float v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = (k0 + 32 * u < ra) ? src[k0 + 32 * u] : 0.f;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int k = k0 + 32 * u;
                    if (k < ra) Qs[row * SP + (k % L) * LS + k / L] = v[u];
                }
            }
        }
        for (int k = tid; k < ra; k += blockDim.x) {
            act_s[k] = a.act_idx[k];
            scl_s[k] = a.scale_a[k];
        }
        for (int i = tid; i < r; i += blockDim.x) actv_s[i] = a.active[i];
    }
    __syncthreads();

    // persistent: each CTA walks groups of B fast-break blocks (Q, act_idx and
    // scale staged once per CTA instead of once per group)
    const int64_t nblk_all = (a.index_base + a.count - 1) / 32 - a.index_base / 32 + 1;
    const int64_t ncta = (nblk_all + B - 1) / B;
    // (E < 13 launches one CTA per group: a single pass, no loop)
    constexpr bool PERSIST = E >= 13;
    for (int64_t cta = blockIdx.x; PERSIST ? cta < ncta : cta == (int64_t)blockIdx.x;
         cta += gridDim.x) {
        const int warp = tid >> 5, lane = tid & 31;
        const int l = lane % L;
        const int gbase = lane - l;
        const unsigned gmask = (L == 32) ? NMFB_FULL_MASK : (((1u << L) - 1u) << gbase);
        const int slot = warp * (32 / L) + lane / L;  // problem slot in CTA
        const int b = slot >> 5, pos = slot & 31;
        const int64_t blk0 = a.index_base / 32;
        const int64_t blk = blk0 + cta * B + b;
        const bool blk_live = (blk * 32 - a.index_base) < a.count;
        const int64_t g = blk * 32 + pos;
        const int64_t j = g - a.index_base;
        const bool valid = blk_live && (g >= a.index_base) && (j < a.count);
        const float m0 = (blk == blk0 && (a.index_base % 32) != 0) ? a.max_stop0 : 0.0f;
        const float *Qsl = Qs + l * LS;  // this lane's block of every row
        // the warp's q_times_w4 exchange buffer (128 floats) and, in the CD
        // phase, this problem's y row (lane l's coordinates at l*LS + e)
        float *wscr = smem_f + R * SP + (size_t)32 * B * r + (size_t)warp * 128;
        float *ys = smem_f + R * SP + (size_t)32 * B * r + (STAGE_H ? 0 : (size_t)128 * L * B) +
                    (size_t)slot * SP + l * LS;
        // q_times source-lane rotation: one offset per quarter-warp (see q_times_f)
        // (measured: pays at E = 25, costs at E <= 13, where the per-lane source
        // lane and row offsets outweigh the saved shared-memory phases)
        const int rot = (E < 20) ? 0 : (L >= 8) ? ((lane >> 3) * (L / 4)) & (L - 1) : (lane >> 3);
        // CD key mask (|dec| bits above the index code), kept in a register so the
        // per-coordinate key is a single LOP3 with the element code as immediate
        // (index_base < 2^62: the OR adds nothing, but ptxas cannot fold it)
#if !NMFB_NNLS_EXACT_ARGMAX
        const unsigned kmask = (0x7FFFFFFFu & ~((1u << ((E * L <= 128) ? 7 : 8)) - 1u)) |
                               (unsigned)(a.index_base >> 62);
#endif

        // register arrays padded to an even length (packed FP32x2 math); the
        // padding coordinates (k >= R) stay exactly zero
        float y[EE], gr[EE], qd[EE];

        int status = ST_DONE;
        bool fail = false, write_x = false;
        int iters = 0;
        float final_norm = 0.f, norm_k = 0.f, threshold = 0.f;

        // ---- prologue: short-circuit, frozen check, compact load, gradient ----
        // The warm-start row is independent of h: its loads go out first (with
        // every dimension active lane l reads x[j][e*L + l]).  The problem's
        // full linear term h (sum of the split-K partials) is staged in its
        // shared-memory row, four rows' loads in flight per lane -- a compact
        // loop, not E inlined copies of the partial sums (the prologue code
        // would otherwise crowd the CD loop out of the instruction cache) --
        // and scanned for the short-circuit / frozen checks; the compact gather
        // h[act_idx[k]] reads it back.
        float xw[EE];
#pragma unroll
        for (int e = 0; e < EE; ++e) {
            const int k = e * L + l;
            xw[e] = (valid && k < ra) ? a.x[j * r + (ra == r ? k : act_s[k])] : 0.f;
        }
        float *hrow = smem_f + R * SP + (size_t)slot * r;
        bool any_neg = false, frozen_neg = false;
        if (valid) {
#pragma unroll 1
            for (int i0 = l; i0 < r; i0 += 4 * L) {
                float hv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = i0 + u * L;
                    hv[u] = (i < r) ? fast_h<TH>(a, j, i) : 0.f;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = i0 + u * L;
                    if (i < r) {
                        hrow[i] = hv[u];
                        if (hv[u] < 0.f) {
                            any_neg = true;
                            if (!actv_s[i]) frozen_neg = true;
                        }
                    }
                }
            }
        }
        __syncwarp(gmask);
        any_neg = gany<L>(any_neg, gmask, gbase);
        frozen_neg = gany<L>(frozen_neg, gmask, gbase);
        if (valid) {
            if (!any_neg) {
                for (int i = l; i < r; i += L) a.x[j * r + i] = 0.f;
            } else if (frozen_neg) {
                fail = true;
            }
        }
        const bool solve = valid && any_neg && !frozen_neg;
        const bool ident = (ra == r);
#pragma unroll
        for (int e = 0; e < EE; ++e) {
            const int k = e * L + l;
            float qv = 0.f, yv = 0.f;
            if (solve && k < ra) {
                const int ik = ident ? k : act_s[k];
                const float sv = scl_s[k];
                qv = __fdiv_rn(hrow[ik], sv);
                yv = xw[e] * sv;
            }
            y[e] = yv;
            gr[e] = qv;
        }
        qmul_if<E, L, EE, EP>(solve, gr, [&](int e) { return y[e]; }, Qs, Qsl, wscr, r, lane, gmask,
                              rot);
        if (solve) {
            float n0 = 0.f;
#pragma unroll
            for (int e = 0; e < E; ++e)
                if (y[e] > 0.f || gr[e] < 0.f) n0 = fmaf(gr[e], gr[e], n0);
            n0 = gsum<L>(n0, gmask);
            write_x = true;
            final_norm = n0;
            if (n0 > 0.f) {
                threshold = a.eps * n0;
                status = ST_RUNNING;
            }
        }

        // ---- lockstep iterations with per-block fast-break resolution ----
        // passive-set gradient component (kernels.py:59-64): g if y > 0 or g < 0
        auto pgrad = [](float yv, float gv) { return (yv > 0.f || gv < 0.f) ? gv : 0.f; };
        while (true) {
            const bool running = (status == ST_RUNNING);
            bool moved = false;
            if constexpr (L == 8 && E >= NMFB_NNLS_W4_MIN_E) {
                // The Q products are issued from warp-uniform control flow (the
                // warp-shared product needs every lane); problems that do not take a
                // step contribute zero sources and keep their accumulators.
                // exact line search over the passive set (kernels.py:57-103)
                float nsq = 0.f;
                if (running) {
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const float d = pgrad(y[e], gr[e]);
                        nsq = fmaf(d, d, nsq);
                    }
                }
                nsq = gsum<L>(nsq, gmask);
                const bool ls = running && nsq > 0.f;
#pragma unroll
                for (int e = 0; e < EE; ++e) qd[e] = 0.f;
                qmul_if<E, L, EE, EP>(ls, qd, [&](int e) { return pgrad(y[e], gr[e]); }, Qs, Qsl, wscr,
                                      r, lane, gmask, rot);
                float alpha = 1.f, step = 1.f;
                bool clamped = false;
                if (ls) {
                    float curv = 0.f;
#pragma unroll
                    for (int e = 0; e < E; ++e) curv = fmaf(pgrad(y[e], gr[e]), qd[e], curv);
                    curv = gsum<L>(curv, gmask);
                    alpha = (curv > 0.f) ? __fdiv_rn(nsq, curv) : 1.f;
#pragma unroll
                    for (int e = 0; e < E; ++e)
                        if (fmaf(-alpha, pgrad(y[e], gr[e]), y[e]) < 0.f) clamped = true;
                    clamped = gany<L>(clamped, gmask, gbase);
                }
                // _take_step (kernels.py:153-175) with the breakpoint fallback: the
                // projected step at alpha, and once more at the breakpoint alpha_bp
                // when the first one increases the objective
                step = alpha;
                auto delta = [&](int e) {
                    return fmaxf(fmaf(-step, pgrad(y[e], gr[e]), y[e]), 0.f) - y[e];
                };
                const bool ts0 = ls && clamped;
                if (ts0) {
#pragma unroll
                    for (int e = 0; e < EE; ++e) qd[e] = 0.f;
                }
                qmul_if<E, L, EE, EP>(ts0, qd, delta, Qs, Qsl, wscr, r, lane, gmask, rot);
                bool ts1 = false;
                if (ts0) {
                    float df = 0.f;
#pragma unroll
                    for (int e = 0; e < E; ++e) df += delta(e) * fmaf(0.5f, qd[e], gr[e]);
                    df = gsum<L>(df, gmask);
                    if (df > 0.f) {
                        float abp = INFINITY;
#pragma unroll
                        for (int e = 0; e < E; ++e) {
                            const float d = pgrad(y[e], gr[e]);
                            if (d > 0.f && y[e] > 0.f) abp = fminf(abp, __fdiv_rn(y[e], d));
                        }
                        abp = gmin<L>(abp, gmask);
                        if (abp < alpha) {
                            step = abp;
                            ts1 = true;
                        }
                    }
                }
                if (ts1) {
#pragma unroll
                    for (int e = 0; e < EE; ++e) qd[e] = 0.f;
                }
                qmul_if<E, L, EE, EP>(ts1, qd, delta, Qs, Qsl, wscr, r, lane, gmask, rot);
                if (ts0) {
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const float v = fmaxf(fmaf(-step, pgrad(y[e], gr[e]), y[e]), 0.f);
                        if (v != y[e]) moved = true;
                        y[e] = v;
                        gr[e] += qd[e];
                    }
                } else if (ls) {
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const float v = fmaf(-alpha, pgrad(y[e], gr[e]), y[e]);
                        if (v != y[e]) moved = true;
                        y[e] = v;
                        gr[e] = fmaf(-alpha, qd[e], gr[e]);
                    }
                }
            } else {
                if (running) {
                    // exact line search over the passive set (kernels.py:57-103)
                    float nsq = 0.f;
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const float d = pgrad(y[e], gr[e]);
                        nsq = fmaf(d, d, nsq);
                    }
                    nsq = gsum<L>(nsq, gmask);
                    if (nsq > 0.f) {
#pragma unroll
                        for (int e = 0; e < EE; ++e) qd[e] = 0.f;
                        q_times_f<E, L, EE, EP>(qd, [&](int e) { return pgrad(y[e], gr[e]); }, Qsl,
                                                gmask, rot);
                        float curv = 0.f;
#pragma unroll
                        for (int e = 0; e < E; ++e) curv = fmaf(pgrad(y[e], gr[e]), qd[e], curv);
                        curv = gsum<L>(curv, gmask);
                        const float alpha = (curv > 0.f) ? __fdiv_rn(nsq, curv) : 1.f;
                        bool clamped = false;
#pragma unroll
                        for (int e = 0; e < E; ++e)
                            if (fmaf(-alpha, pgrad(y[e], gr[e]), y[e]) < 0.f) clamped = true;
                        clamped = gany<L>(clamped, gmask, gbase);
                        if (clamped) {
                            // _take_step (kernels.py:153-175) with the breakpoint fallback
                            float step = alpha;
                            for (int pass = 0; pass < 2; ++pass) {
                                auto delta = [&](int e) {
                                    return fmaxf(fmaf(-step, pgrad(y[e], gr[e]), y[e]), 0.f) - y[e];
                                };
#pragma unroll
                                for (int e = 0; e < EE; ++e) qd[e] = 0.f;
                                q_times_f<E, L, EE, EP>(qd, delta, Qsl, gmask, rot);
                                if (pass == 1) break;
                                float df = 0.f;
#pragma unroll
                                for (int e = 0; e < E; ++e) df += delta(e) * fmaf(0.5f, qd[e], gr[e]);
                                df = gsum<L>(df, gmask);
                                if (!(df > 0.f)) break;
                                float abp = INFINITY;
#pragma unroll
                                for (int e = 0; e < E; ++e) {
                                    const float d = pgrad(y[e], gr[e]);
                                    if (d > 0.f && y[e] > 0.f) abp = fminf(abp, __fdiv_rn(y[e], d));
                                }
                                abp = gmin<L>(abp, gmask);
                                if (!(abp < alpha)) break;
                                step = abp;
                            }
#pragma unroll
                            for (int e = 0; e < E; ++e) {
                                const float v = fmaxf(fmaf(-step, pgrad(y[e], gr[e]), y[e]), 0.f);
                                if (v != y[e]) moved = true;
                                y[e] = v;
                                gr[e] += qd[e];
                            }
                        } else {
#pragma unroll
                            for (int e = 0; e < E; ++e) {
                                const float v = fmaf(-alpha, pgrad(y[e], gr[e]), y[e]);
                                if (v != y[e]) moved = true;
                                y[e] = v;
                                gr[e] = fmaf(-alpha, qd[e], gr[e]);
                            }
                        }
                    }
            }
            }
            if (running) {
                constexpr int LB = (L == 1) ? 0 : (L == 2) ? 1 : (L == 4) ? 2 : (L == 8) ? 3
                                 : (L == 16) ? 4 : 5;
                const unsigned lcode = (unsigned)(L - 1 - l);
                int pp = -1;
                float pdx = 0.f;
                if constexpr (YSMEM) {
                    // y lives in this problem's shared-memory row for the CD
                    // phase: the winner's owner lane updates its coordinate with
                    // one indexed store instead of a select over its E registers
#pragma unroll
                    for (int q = 0; q < EP / 4; ++q)
                        reinterpret_cast<float4 *>(ys)[q] =
                            make_float4(4 * q < EE ? y[4 * q] : 0.f, 4 * q + 1 < EE ? y[4 * q + 1] : 0.f,
                                        4 * q + 2 < EE ? y[4 * q + 2] : 0.f,
                                        4 * q + 3 < EE ? y[4 * q + 3] : 0.f);
                }
                for (int s = 0; s < ra; ++s) {
                    if (s > 0) axpy_row<EE, EP>(gr, Qsl + pp * SP, pdx);
                    int ep, lp;
                    float dwin = 0.f;
#if NMFB_NNLS_EXACT_ARGMAX
                    // Greedy CD (kernels.py:106-132) with the reference's exact
                    // argmax: the largest |dec| wins and equal values go to the
                    // lowest coordinate k = e*L + l (strict >, kernels.py:119).
                    // dec = d (g + d/2) with d = -min(g, y) is <= 0 for every
                    // coordinate, so its raw bit pattern orders by |dec| as an
                    // unsigned integer (+-0 lowest).  In-lane: a pair tree over
                    // (bits, e[, d]) keeping the lower e on equality; across the
                    // group: a max over bits << 32 | code(e, l), lower (e, l) =
                    // higher code.
                    float yv[YSMEM ? EP : 1];
                    if constexpr (YSMEM) {
#pragma unroll
                        for (int q = 0; q < EP / 4; ++q) {
                            const float4 v = reinterpret_cast<const float4 *>(ys)[q];
                            yv[4 * q] = v.x;
                            yv[4 * q + 1] = v.y;
                            yv[4 * q + 2] = v.z;
                            yv[4 * q + 3] = v.w;
                        }
                    }
                    auto ycur = [&](int e) { if constexpr (YSMEM) return yv[e]; else return y[e]; };
                    unsigned key[EE];
                    int ix[EE];
                    float dv[DCARRY ? EE : 1];
#pragma unroll
                    for (int e = 0; e < EE; e += 2) {
                        const float d0 = -fminf(gr[e], ycur(e)), d1 = -fminf(gr[e + 1], ycur(e + 1));
                        const float2 t = __ffma2_rn(make_float2(0.5f, 0.5f), make_float2(d0, d1),
                                                    make_float2(gr[e], gr[e + 1]));
                        const float2 dc = __fmul2_rn(make_float2(d0, d1), t);
                        key[e] = __float_as_uint(dc.x);
                        key[e + 1] = __float_as_uint(dc.y);
                        ix[e] = e;
                        ix[e + 1] = e + 1;
                        if constexpr (DCARRY) {
                            dv[e] = d0;
                            dv[e + 1] = d1;
                        }
                    }
#pragma unroll
                    for (int w = 1; w < EE; w *= 2)
#pragma unroll
                        for (int e = 0; e + w < EE; e += 2 * w) {
                            const bool keep = key[e] >= key[e + w];
                            key[e] = keep ? key[e] : key[e + w];
                            ix[e] = keep ? ix[e] : ix[e + w];
                            if constexpr (DCARRY) dv[e] = keep ? dv[e] : dv[e + w];
                        }
                    if constexpr (DCARRY) dwin = dv[0];
                    unsigned long long kb = ((unsigned long long)key[0] << 32) |
                                            ((unsigned)(EE - 1 - ix[0]) << LB) | lcode;
#pragma unroll
                    for (int o = L / 2; o > 0; o >>= 1) {
                        const unsigned long long other = __shfl_xor_sync(gmask, kb, o, L);
                        kb = other > kb ? other : kb;
                    }
                    if (((unsigned)(kb >> 32) & 0x7FFFFFFFu) == 0u) {
                        pp = -1;
                        break;
                    }
                    ep = (EE - 1) - (int)((unsigned)kb >> LB);
                    lp = (L - 1) - (int)((unsigned)kb & (unsigned)(L - 1));
#else
                    // truncated-key argmax (experiment): |dec| with its low IB bits
                    // replaced by an index code -- decreases within ~2^-15 of each
                    // other resolve to the lower index
                    constexpr int IB = (R <= 128) ? 7 : 8;
                    constexpr unsigned IMASK = (1u << IB) - 1u;
                    constexpr int EB = IB - LB;
                    constexpr unsigned EMAXC = (1u << EB) - 1u;
                    static_assert(EE <= (1 << EB), "index code does not fit the key");
                    unsigned key[EE];
#pragma unroll
                    for (int e = 0; e < EE; e += 2) {
                        const float d0 = -fminf(gr[e], y[e]), d1 = -fminf(gr[e + 1], y[e + 1]);
                        const float2 t = __ffma2_rn(make_float2(0.5f, 0.5f), make_float2(d0, d1),
                                                    make_float2(gr[e], gr[e + 1]));
                        const float2 dc = __fmul2_rn(make_float2(d0, d1), t);
                        key[e] = (__float_as_uint(dc.x) & kmask) | ((EMAXC - (unsigned)e) << LB);
                        key[e + 1] = (__float_as_uint(dc.y) & kmask) |
                                     ((EMAXC - (unsigned)(e + 1)) << LB);
                    }
#pragma unroll
                    for (int w = 1; w < EE; w *= 3)
#pragma unroll
                        for (int e = 0; e < EE; e += 3 * w) {
                            if (e + 2 * w < EE)
                                key[e] = __vimax3_u32(key[e], key[e + w], key[e + 2 * w]);
                            else if (e + w < EE)
                                key[e] = max(key[e], key[e + w]);
                        }
                    unsigned kb = key[0] | lcode;
#pragma unroll
                    for (int o = L / 2; o > 0; o >>= 1) kb = max(kb, __shfl_xor_sync(gmask, kb, o, L));
                    if ((kb & ~IMASK) == 0u) {
                        pp = -1;
                        break;
                    }
                    ep = (int)(EMAXC - ((kb & IMASK) >> LB));
                    lp = (int)((unsigned)(L - 1) - (kb & (unsigned)(L - 1)));
#endif
                    if constexpr (YSMEM) {
                        // the winner's step, carried through the argmax tree:
                        // d = -min(g, y) of the winning coordinate
                        pdx = (L == 1) ? dwin : __shfl_sync(gmask, dwin, lp, L);
                        if (l == lp) ys[ep] += pdx;
                    } else if constexpr (DCARRY) {
                        // the winner's step d = -min(g, y) comes with the argmax
                        // (carried through the tree), so the owner's update is
                        // independent per register -- no dependent select chain
                        // on the way to the next selection's row axpy
                        pdx = (L == 1) ? dwin : __shfl_sync(gmask, dwin, lp, L);
                        const int epo = (l == lp) ? ep : -1;
#pragma unroll
                        for (int e = 0; e < E; ++e)
                            if (e == epo) y[e] += pdx;
                    } else {
                        float dxo = 0.f;
#pragma unroll
                        for (int e = 0; e < E; ++e) {
                            if (e == ep && l == lp) {
                                dxo = -fminf(gr[e], y[e]);
                                y[e] += dxo;
                            }
                        }
                        pdx = (L == 1) ? dxo : __shfl_sync(gmask, dxo, lp, L);
                    }
                    moved = true;
                    pp = ep * L + lp;
                }
                if (pp >= 0) axpy_row<EE, EP>(gr, Qsl + pp * SP, pdx);
                if constexpr (YSMEM) {
#pragma unroll
                    for (int q = 0; q < EP / 4; ++q) {
                        const float4 v = reinterpret_cast<const float4 *>(ys)[q];
                        if (4 * q < EE) y[4 * q] = v.x;
                        if (4 * q + 1 < EE) y[4 * q + 1] = v.y;
                        if (4 * q + 2 < EE) y[4 * q + 2] = v.z;
                        if (4 * q + 3 < EE) y[4 * q + 3] = v.w;
                    }
                }
                iters += 1;
                bool finite = true;
                float nk = 0.f;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    if (!(isfinite(y[e]) && isfinite(gr[e]))) finite = false;
                    if (y[e] > 0.f || gr[e] < 0.f) nk = fmaf(gr[e], gr[e], nk);
                }
                finite = !gany<L>(!finite, gmask, gbase);
                nk = gsum<L>(nk, gmask);
                if (!finite) {
                    fail = true;
                    write_x = false;
                    status = ST_DONE;
                    final_norm = 0.f;
                } else {
                    norm_k = nk;
                    moved = gany<L>(moved, gmask, gbase);
                    if (nk <= threshold || !moved || iters >= a.max_inner) {
                        status = ST_DONE;
                        final_norm = nk;
                    } else {
                        status = ST_WAITING;
                    }
                }
            }
            // ---- resolve the fast-break block ----
            if (L == 1) {
                if (!__any_sync(NMFB_FULL_MASK, status != ST_DONE)) break;
                resolve_block_warp<float>(status, norm_k, final_norm, m0);
            } else {
                const int bar = 1 + b;
                if (l == 0) {
                    blk_status[b][pos] = status;
                    blk_norm[b][pos] = norm_k;
                    blk_final[b][pos] = final_norm;
                }
                asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(32 * L) : "memory");
                if (warp == b * L) {
                    int st = blk_status[b][lane];
                    float fn = blk_final[b][lane];
                    resolve_block_warp<float>(st, blk_norm[b][lane], fn, m0);
                    blk_status[b][lane] = st;
                    blk_final[b][lane] = fn;
                    bool any = __any_sync(NMFB_FULL_MASK, st != ST_DONE);
                    if (lane == 0) blk_any[b] = any ? 1 : 0;
                }
                asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(32 * L) : "memory");
                status = blk_status[b][pos];
                final_norm = blk_final[b][pos];
                const bool any = blk_any[b] != 0;
                asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(32 * L) : "memory");
                if (!any) break;
            }
        }

        // ---- epilogue ----
        if (valid) {
            if (write_x) {
                for (int i = l; i < r; i += L) a.x[j * r + i] = 0.f;
                __syncwarp(gmask);
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int k = e * L + l;
                    if (k < ra) a.x[j * r + act_s[k]] = __fdiv_rn(y[e], scl_s[k]);
                }
            }
            if (MIRROR && (write_x || !any_neg)) {
                // fused all-gather: the finished row (read back after the group's
                // stores) goes to the same offset in every mirror (peer GPUs)
                __syncwarp(gmask);
                for (int i = l; i < r; i += L) {
                    const float v = a.x[j * r + i];
                    for (int q = 0; q < a.nmirror; ++q) a.mirror[q][j * r + i] = v;
                }
            }
            if (l == 0) {
                if (a.iters_out) a.iters_out[j] = fail ? -1 : iters;
                if (a.final_out) a.final_out[j] = fail ? 0.f : final_norm;
                if (fail) atomicMin((unsigned long long *)&a.stats[1], (unsigned long long)g);
            }
        }
        unsigned long long it = (valid && !fail && l == 0) ? (unsigned long long)iters : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) it += __shfl_xor_sync(NMFB_FULL_MASK, it, o);
        if (lane == 0 && it) atomicAdd(&a.stats[0], it);
        if (PERSIST) __syncthreads();  // staging rows and block state reused by the next group
    }
}

template <typename TH, int E, int L, int B>
static int launch_fast_variant(const NnlsLaunch &p) {
    auto a = make_args<float, TH>(p);
    constexpr int R = E * L, SP = L * nnls_ls(E);
    // Q (R x SP, permuted rows) + one staged h row (r floats) per problem
    // slot + large E: a 128-float q_times_w4 exchange buffer per warp
    // (+ the YSMEM experiment's y rows)
    constexpr bool STAGE_H = E < NMFB_NNLS_W4_MIN_E;
    constexpr bool YSMEM = NMFB_NNLS_EXACT_ARGMAX && NMFB_NNLS_YSMEM;
    size_t smem = sizeof(float) * ((size_t)R * SP + (size_t)32 * B * p.r +
                                   (STAGE_H ? 0 : (size_t)128 * L * B) +
                                   (YSMEM ? (size_t)32 * B * SP : 0));

    auto kern = nnls_fast_kernel<TH, E, L, B, false>;
    if (p.nmirror > 0) {
        if constexpr (std::is_same<TH, float>::value)
            kern = nnls_fast_kernel<TH, E, L, B, true>;
        else
            return NMFB_ERR_ARG;  // the fused all-gather takes fp32 partials
    }
    {
        // dynamic + static shared memory must fit the opt-in per-block limit
        // (227 KB): larger variants are an argument error, not a launch
        // failure (queried once per instantiation)
        static size_t limit = 0;
        if (limit == 0) {
            cudaFuncAttributes fa;
            int dev = 0, optin = 0;
            if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess ||
                cudaGetDevice(&dev) != cudaSuccess ||
                cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) !=
                    cudaSuccess) {
                launch_status();
                return NMFB_ERR_CUDA;
            }
            limit = (size_t)optin - fa.sharedSizeBytes;
        }
        if (smem > limit) return NMFB_ERR_ARG;
    }
    if (smem > 48 * 1024) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (launch_status() != NMFB_OK) return NMFB_ERR_CUDA;
    }
    int64_t nblk = num_blocks(p);
    int64_t ncta = (nblk + B - 1) / B;
    // persistent grid: at most the resident CTAs of the whole device
    static size_t occ_smem = (size_t)-1;
    static int occ_blocks = 0, sms = 0;
    if (occ_smem != smem) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_blocks, kern, 32 * L * B, smem) !=
                cudaSuccess) {
            launch_status();
            return NMFB_ERR_CUDA;
        }
        occ_smem = smem;
    }
    const int64_t resident = (int64_t)(occ_blocks > 0 ? occ_blocks : 1) * (sms > 0 ? sms : 1);
    // (persistent only at E >= 13: r = 100 -4.6%, r = 200 unchanged; at E = 7
    // the loop costs more than the re-staging it saves, +17% at r = 50)
    dim3 grid((unsigned)((E >= 13 && ncta > resident) ? resident : ncta));
    kern<<<grid, 32 * L * B, smem, p.stream>>>(a);
    return launch_status();
}


}  // namespace nmfb
