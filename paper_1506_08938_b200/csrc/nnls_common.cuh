// Shared pieces of the batched NNLS kernels (see nnls.cu for the design).
#pragma once
#include <climits>

#include "common.cuh"
#include "nmfb_internal.h"

namespace nmfb {

template <typename T, typename TH>
struct NnlsArgs {
    const T *Qa;             // (ra, ra) compact rescaled Hessian, row-major
    const T *scale_a;        // (ra)
    const int32_t *act_idx;  // (ra) active dims in ascending order
    const uint8_t *active;   // (r)
    int r, ra;
    const int32_t *ra_dev;   // nullable device copy of ra (set by the rescale kernel)
    const TH *hp;            // S partials [S][count][h_ld] (h = h_base - sum), or h itself if S==0
    int S;
    int64_t h_ld, h_pstride;
    double h_base;
    T *x;                    // (count, r): warm start in, solution out
    int64_t count, index_base;
    T eps;
    int max_inner;
    T max_stop0;
    int32_t *iters_out;      // nullable (count)
    T *final_out;            // nullable (count)
    T *hist;                 // nullable (count, hist_ld, 2): per-iteration (norm, objective)
    int hist_ld;             // reference kernel only (nqp.solve histories)
    bool independent;        // every problem its own fast-break scope (nqp.solve)
    bool check_grad;         // reference kernel: nqp.solve(check_gradients=True), nqp.py:295-299
    unsigned long long *stats;  // [0] += inner iterations, [1] = min failing global index
    T *mirror[NMFB_MAX_PEERS];  // fast kernel: solution rows also stored here (peer GPUs)
    int nmirror;
};

template <typename T, typename TH, typename O>
__device__ __forceinline__ T load_h(const NnlsArgs<T, TH> &a, int64_t j, int i) {
    const TH *p = a.hp + j * a.h_ld + i;
    if (a.S == 0) return (T)p[0];
    if (a.S == 1) return (T)O::sub((T)a.h_base, (T)p[0]);
    TH s = p[0];
    for (int k = 1; k < a.S; ++k) s += p[k * a.h_pstride];
    return (T)((TH)a.h_base - s);
}

template <typename T, typename TH>
static NnlsArgs<T, TH> make_args(const NnlsLaunch &p) {
    NnlsArgs<T, TH> a;
    a.Qa = (const T *)p.Qa;
    a.scale_a = (const T *)p.scale_a;
    a.act_idx = p.act_idx;
    a.active = p.active;
    a.r = p.r;
    a.ra = p.ra;
    a.ra_dev = p.ra_dev;
    a.hp = (const TH *)p.h;
    a.S = p.h_parts;
    a.h_ld = p.h_ld;
    a.h_pstride = p.h_pstride;
    a.h_base = p.h_base;
    a.x = (T *)p.x;
    a.count = p.count;
    a.index_base = p.index_base;
    a.eps = (T)p.eps;
    a.max_inner = p.max_inner;
    a.max_stop0 = (T)p.max_stop0;
    a.iters_out = p.iters_out;
    a.final_out = (T *)p.final_out;
    a.hist = (T *)p.hist;
    a.hist_ld = p.hist_ld;
    a.independent = p.independent;
    a.check_grad = p.check_grad;
    a.stats = (unsigned long long *)p.stats;
    a.nmirror = p.nmirror;
    for (int q = 0; q < NMFB_MAX_PEERS; ++q) a.mirror[q] = q < p.nmirror ? (T *)p.mirror[q] : nullptr;
    return a;
}

static int64_t num_blocks(const NnlsLaunch &p) {
    int64_t first = p.index_base / 32;
    int64_t last = (p.index_base + p.count - 1) / 32;
    return last - first + 1;
}

}  // namespace nmfb
