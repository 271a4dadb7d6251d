// Fast fp32 batched NNLS (warp-group per problem); see nnls.cu.
#pragma once
#include <type_traits>

#include "nnls_common.cuh"

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

// acc[e] += sum_j Q[k_e, j] * src_j, src_j owned by lane (j % L), element j / L.
template <int E, int L>
__device__ __forceinline__ void q_times(float (&acc)[E], const float (&src)[E], const float *Qrow,
                                        int S, unsigned gmask) {
#pragma unroll 1
    for (int jl = 0; jl < L; ++jl) {
#pragma unroll
        for (int je = 0; je < E; ++je) {
            float sj = (L == 1) ? src[je] : __shfl_sync(gmask, src[je], jl, L);
            const int jcol = je * L + jl;
#pragma unroll
            for (int e = 0; e < E; ++e) acc[e] = fmaf(Qrow[e * L * S + jcol], sj, acc[e]);
        }
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
    for (; k + 3 < a.S; k += 4) {
        s0 += p[(int64_t)k * a.h_pstride];
        s1 += p[(int64_t)(k + 1) * a.h_pstride];
        s2 += p[(int64_t)(k + 2) * a.h_pstride];
        s3 += p[(int64_t)(k + 3) * a.h_pstride];
    }
    for (; k < a.S; ++k) s0 += p[(int64_t)k * a.h_pstride];
    return (float)((TH)a.h_base - ((s0 + s1) + (s2 + s3)));
}

// Same, with the source values produced by a functor of the element index
// (recomputed instead of held in registers: d = passive gradient, delta = step).
template <int E, int L, typename F>
__device__ __forceinline__ void q_times_f(float (&acc)[E], F src, const float *Qrow, int S,
                                          unsigned gmask) {
#pragma unroll 1
    for (int jl = 0; jl < L; ++jl) {
#pragma unroll
        for (int je = 0; je < E; ++je) {
            const float mine = src(je);
            const float sj = (L == 1) ? mine : __shfl_sync(gmask, mine, jl, L);
            const int jcol = je * L + jl;
#pragma unroll
            for (int e = 0; e < E; ++e) acc[e] = fmaf(Qrow[e * L * S + jcol], sj, acc[e]);
        }
    }
}

// Occupancy target: ~4E + 48 live registers per thread (y, grad and Q*d per
// coordinate; the passive gradient and step are recomputed) -> CTAs per SM.
__host__ __device__ constexpr int nnls_regs(int E, int L) { return 4 * E + 48 + (L == 1 ? 48 : 0); }
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
    constexpr int S = R | 1;
    extern __shared__ __align__(16) float smem_f[];
    float *Qs = smem_f;                          // R x S
    __shared__ float blk_norm[B][32], blk_final[B][32];
    __shared__ int blk_status[B][32];
    __shared__ int blk_any[B];

    const int tid = threadIdx.x;
    const int ra = a.ra_dev ? *a.ra_dev : a.ra, r = a.r;
    for (int idx = tid; idx < R * S; idx += blockDim.x) {
        int k = idx / S, c = idx - k * S;
        Qs[idx] = (k < ra && c < ra) ? a.Qa[k * ra + c] : 0.0f;
    }
    __syncthreads();

    const int warp = tid >> 5, lane = tid & 31;
    const int l = lane % L;
    const int gbase = lane - l;
    const unsigned gmask = (L == 32) ? NMFB_FULL_MASK : (((1u << L) - 1u) << gbase);
    const int slot = warp * (32 / L) + lane / L;  // problem slot in CTA
    const int b = slot >> 5, pos = slot & 31;
    const int64_t blk0 = a.index_base / 32;
    const int64_t blk = blk0 + (int64_t)blockIdx.x * B + b;
    const bool blk_live = (blk * 32 - a.index_base) < a.count;
    const int64_t g = blk * 32 + pos;
    const int64_t j = g - a.index_base;
    const bool valid = blk_live && (g >= a.index_base) && (j < a.count);
    const float m0 = (blk == blk0 && (a.index_base % 32) != 0) ? a.max_stop0 : 0.0f;
    const float *Qrow = Qs + l * S;  // row of coordinate e is Qrow + e*L*S

    float y[E], gr[E], qd[E];

    int status = ST_DONE;
    bool fail = false, write_x = false;
    int iters = 0;
    float final_norm = 0.f, norm_k = 0.f, threshold = 0.f;

    // ---- prologue: short-circuit, frozen check, compact load, gradient ----
    // The problem's full linear term h (sum of the split-K partials, loads
    // issued 4 at a time) is staged once in shared memory: the short-circuit
    // scan and the compact gather h[act_idx[k]] both read it from there.
    float *hrow = smem_f + R * S + (size_t)slot * r;
    bool any_neg = false, frozen_neg = false;
    if (valid) {
        for (int i = l; i < r; i += L) {
            const float hv = fast_h<TH>(a, j, i);
            hrow[i] = hv;
            if (hv < 0.f) {
                any_neg = true;
                if (!a.active[i]) frozen_neg = true;
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
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int k = e * L + l;
        float qv = 0.f, yv = 0.f;
        if (solve && k < ra) {
            const int ik = a.act_idx[k];
            const float sv = a.scale_a[k];
            qv = __fdiv_rn(hrow[ik], sv);
            yv = a.x[j * r + ik] * sv;
        }
        y[e] = yv;
        gr[e] = qv;
    }
    if (solve) {
        q_times<E, L>(gr, y, Qrow, S, gmask);
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
        if (status == ST_RUNNING) {
            bool moved = false;
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
                for (int e = 0; e < E; ++e) qd[e] = 0.f;
                q_times_f<E, L>(qd, [&](int e) { return pgrad(y[e], gr[e]); }, Qrow, S, gmask);
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
                        for (int e = 0; e < E; ++e) qd[e] = 0.f;
                        q_times_f<E, L>(qd, delta, Qrow, S, gmask);
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
            constexpr int IB = (R <= 128) ? 7 : 8;
            constexpr unsigned IMASK = (1u << IB) - 1u;
            int pp = -1;
            float pdx = 0.f;
            for (int s = 0; s < ra; ++s) {
                unsigned key[E];
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int k = e * L + l;
                    float gi = gr[e];
                    if (pp >= 0) {
                        gi = fmaf(Qrow[e * L * S + pp], pdx, gi);
                        gr[e] = gi;
                    }
                    const float dxi = -fminf(gi, y[e]);
                    const float dec = dxi * fmaf(0.5f, dxi, gi);
                    key[e] = (__float_as_uint(dec) & (0x7FFFFFFFu & ~IMASK)) | (IMASK - (unsigned)k);
                }
#pragma unroll
                for (int w = 1; w < E; w <<= 1)
#pragma unroll
                    for (int e = 0; e + w < E; e += 2 * w) key[e] = max(key[e], key[e + w]);
                unsigned kb = key[0];
#pragma unroll
                for (int o = L / 2; o > 0; o >>= 1) kb = max(kb, __shfl_xor_sync(gmask, kb, o, L));
                if ((kb & ~IMASK) == 0u) {
                    pp = -1;
                    break;
                }
                const int p = (int)(IMASK - (kb & IMASK));
                float dxo = 0.f;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    if (e * L + l == p) {
                        dxo = -fminf(gr[e], y[e]);
                        y[e] += dxo;
                    }
                }
                moved = true;
                pdx = (L == 1) ? dxo : __shfl_sync(gmask, dxo, p % L, L);
                pp = p;
            }
            if (pp >= 0) {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    gr[e] = fmaf(Qrow[e * L * S + pp], pdx, gr[e]);
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
                if (k < ra) a.x[j * r + a.act_idx[k]] = __fdiv_rn(y[e], a.scale_a[k]);
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
}

template <typename TH, int E, int L, int B>
static int launch_fast_variant(const NnlsLaunch &p) {
    auto a = make_args<float, TH>(p);
    constexpr int R = E * L, S = R | 1;
    // Q (R x S) + one staged h row (r floats) per problem slot
    size_t smem = sizeof(float) * ((size_t)R * S + (size_t)32 * B * p.r);
    auto kern = nnls_fast_kernel<TH, E, L, B, false>;
    if (p.nmirror > 0) {
        if constexpr (std::is_same<TH, float>::value)
            kern = nnls_fast_kernel<TH, E, L, B, true>;
        else
            return NMFB_ERR_ARG;  // the fused all-gather takes fp32 partials
    }
    if (smem > 48 * 1024) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (launch_status() != NMFB_OK) return NMFB_ERR_CUDA;
    }
    int64_t nblk = num_blocks(p);
    dim3 grid((unsigned)((nblk + B - 1) / B));
    kern<<<grid, 32 * L * B, smem, p.stream>>>(a);
    return launch_status();
}


}  // namespace nmfb
