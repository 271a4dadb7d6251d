// Reference-order batched NNLS (thread per problem); see nnls.cu.
#include "nnls_common.cuh"

namespace nmfb {

// ---------------------------------------------------------------------------
// Reference-order kernel (thread per problem).
// ---------------------------------------------------------------------------
template <typename T, typename TH, int MAXR>
__global__ void __launch_bounds__(64) nnls_ref_kernel(NnlsArgs<T, TH> a) {
    using O = Exact<T>;
    const int lane = threadIdx.x & 31;
    const int64_t warp_id = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t blk0 = a.index_base / 32;
    const int64_t blk = blk0 + warp_id;
    if (blk * 32 - a.index_base >= a.count) return;  // warp-uniform
    const int64_t g = blk * 32 + lane;
    const int64_t j = g - a.index_base;
    const bool valid = (g >= a.index_base) && (j < a.count);
    const T m0 = (a.independent || (blk == blk0 && (a.index_base % 32) != 0)) ? a.max_stop0 : T(0);
    const int r = a.r, ra = a.ra_dev ? *a.ra_dev : a.ra;

    T hbuf[MAXR], y[MAXR], grad[MAXR], d[MAXR], ynew[MAXR], delta[MAXR], qd[MAXR];
    int status = ST_DONE;
    bool fail = false, write_x = false, gdrift = false;
    int iters = 0;
    T final_norm = T(0), norm_k = T(0), threshold = T(0);
    const T *Q = a.Qa;
    // per-iteration (norm, objective) history for nqp.solve (nqp.py:285-313);
    // objective 0.5 y'Qy + q'y in the rescaled space, q = h[act] / scale
    auto record = [&](int it, T nrm) {
        if (!a.hist || it >= a.hist_ld) return;
        T f = T(0);
        for (int k = 0; k < ra; ++k) {
            T qy = T(0);
            for (int jj = 0; jj < ra; ++jj) qy = O::madd(qy, Q[k * ra + jj], y[jj]);
            T qk = O::div(hbuf[a.act_idx[k]], a.scale_a[k]);
            f = O::add(f, O::mul(y[k], O::add(O::mul(T(0.5), qy), qk)));
        }
        T *hp = a.hist + ((int64_t)j * a.hist_ld + it) * 2;
        hp[0] = nrm;
        hp[1] = f;
    };

    if (valid) {
        bool all_nonneg = true;
        for (int i = 0; i < r; ++i) {
            hbuf[i] = load_h<T, TH, O>(a, j, i);
            if (hbuf[i] < T(0)) all_nonneg = false;
        }
        if (all_nonneg) {
            // the origin is the exact optimum (kernels.py:189-198)
            for (int i = 0; i < r; ++i) a.x[j * r + i] = T(0);
        } else {
            for (int i = 0; i < r; ++i)
                if (!a.active[i] && hbuf[i] < T(0)) fail = true;  // kernels.py:199-201
            if (!fail) {
                for (int k = 0; k < ra; ++k) {
                    int i = a.act_idx[k];
                    T s = a.scale_a[k];
                    d[k] = O::div(hbuf[i], s);        // q (kept in d until the loop starts)
                    y[k] = O::mul(a.x[j * r + i], s);
                }
                for (int k = 0; k < ra; ++k) {
                    T acc = d[k];
                    for (int jj = 0; jj < ra; ++jj) acc = O::madd(acc, Q[k * ra + jj], y[jj]);
                    grad[k] = acc;
                }
                T norm0 = T(0);
                for (int k = 0; k < ra; ++k)
                    if (y[k] > T(0) || grad[k] < T(0)) norm0 = O::madd(norm0, grad[k], grad[k]);
                write_x = true;
                final_norm = norm0;
                record(0, norm0);
                if (norm0 > T(0)) {
                    threshold = O::mul(a.eps, norm0);
                    status = ST_RUNNING;
                }
            }
        }
    }

    while (__any_sync(NMFB_FULL_MASK, status != ST_DONE)) {
        if (status == ST_RUNNING) {
            bool moved = false;
            // exact line search over the passive set (kernels.py:57-103)
            T nsq = T(0);
            for (int i = 0; i < ra; ++i) {
                if (y[i] > T(0) || grad[i] < T(0)) {
                    d[i] = grad[i];
                    nsq = O::madd(nsq, d[i], d[i]);
                } else {
                    d[i] = T(0);
                }
            }
            if (nsq > T(0)) {
                T curv = T(0);
                for (int i = 0; i < ra; ++i) {
                    T acc = T(0);
                    for (int jj = 0; jj < ra; ++jj) acc = O::madd(acc, Q[i * ra + jj], d[jj]);
                    qd[i] = acc;
                    curv = O::madd(curv, d[i], acc);
                }
                T alpha = (curv > T(0)) ? O::div(nsq, curv) : T(1);
                bool clamped = false;
                for (int i = 0; i < ra; ++i) {
                    T v = O::msub(y[i], alpha, d[i]);
                    if (v < T(0)) {
                        clamped = true;
                        v = T(0);
                    }
                    ynew[i] = v;
                    delta[i] = O::sub(v, y[i]);
                }
                if (!clamped) {
                    for (int i = 0; i < ra; ++i) qd[i] = O::mul(-alpha, qd[i]);
                } else {
                    // _take_step (kernels.py:153-175), at most twice
                    T step = alpha;
                    for (int pass = 0; pass < 2; ++pass) {
                        for (int i = 0; i < ra; ++i) {
                            T v = O::msub(y[i], step, d[i]);
                            if (v < T(0)) v = T(0);
                            ynew[i] = v;
                            delta[i] = O::sub(v, y[i]);
                            qd[i] = T(0);
                        }
                        for (int jj = 0; jj < ra; ++jj) {
                            T dj = delta[jj];
                            if (dj != T(0))
                                for (int i = 0; i < ra; ++i) qd[i] = O::madd(qd[i], Q[i * ra + jj], dj);
                        }
                        if (pass == 1) break;
                        T df = T(0);
                        for (int i = 0; i < ra; ++i)
                            df = O::add(df, O::add(O::mul(grad[i], delta[i]),
                                                   O::mul(O::mul(T(0.5), delta[i]), qd[i])));
                        if (!(df > T(0))) break;
                        T alpha_bp = dev_inf<T>();
                        for (int i = 0; i < ra; ++i) {
                            if (d[i] > T(0) && y[i] > T(0)) {
                                T c = O::div(y[i], d[i]);
                                if (c < alpha_bp) alpha_bp = c;
                            }
                        }
                        if (!(alpha_bp < alpha)) break;
                        step = alpha_bp;
                    }
                }
                for (int i = 0; i < ra; ++i) {
                    if (delta[i] != T(0)) moved = true;
                    y[i] = ynew[i];
                    grad[i] = O::add(grad[i], qd[i]);
                }
            }
            // greedy coordinate descent, r updates (kernels.py:104-132)
            int pending_p = -1;
            T pending_dx = T(0);
            for (int s = 0; s < ra; ++s) {
                T best = T(0), best_dx = T(0);
                int p = -1;
                for (int i = 0; i < ra; ++i) {
                    T gi = grad[i];
                    if (pending_p >= 0) {
                        gi = O::madd(gi, Q[i * ra + pending_p], pending_dx);
                        grad[i] = gi;
                    }
                    T dxi = O::sub(py_max(O::sub(y[i], gi), T(0)), y[i]);
                    T dec = fabs(O::add(O::mul(gi, dxi), O::mul(O::mul(T(0.5), dxi), dxi)));
                    if (dec > best) {
                        best = dec;
                        p = i;
                        best_dx = dxi;
                    }
                }
                pending_p = -1;
                if (p < 0) break;
                y[p] = O::add(y[p], best_dx);
                moved = true;
                pending_p = p;
                pending_dx = best_dx;
            }
            if (pending_p >= 0)
                for (int i = 0; i < ra; ++i) grad[i] = O::madd(grad[i], Q[i * ra + pending_p], pending_dx);
            iters += 1;
            bool finite = true;
            for (int i = 0; i < ra; ++i)
                if (!(is_finite(y[i]) && is_finite(grad[i]))) finite = false;
            bool drift = false;
            if (finite && a.check_grad) {
                // nqp.py:295-299: the incremental gradient against a fresh
                // Q y + q, every iteration
                T ref = T(1), worst = T(0);
                for (int k = 0; k < ra; ++k) {
                    T acc = O::div(hbuf[a.act_idx[k]], a.scale_a[k]);
                    for (int jj = 0; jj < ra; ++jj) acc = O::madd(acc, Q[k * ra + jj], y[jj]);
                    if (fabs(acc) > ref) ref = fabs(acc);
                    const T e = fabs(O::sub(grad[k], acc));
                    if (e > worst) worst = e;
                }
                drift = worst > O::mul(T(1e-9), ref);
            }
            if (!finite || drift) {
                fail = true;
                gdrift = drift;
                write_x = false;
                status = ST_DONE;
                final_norm = T(0);
            } else {
                norm_k = T(0);
                for (int i = 0; i < ra; ++i)
                    if (y[i] > T(0) || grad[i] < T(0)) norm_k = O::madd(norm_k, grad[i], grad[i]);
                record(iters, norm_k);
                if (norm_k <= threshold || !moved || iters >= a.max_inner) {
                    status = ST_DONE;
                    final_norm = norm_k;
                } else {
                    status = ST_WAITING;
                }
            }
        }
        resolve_block_warp<T>(status, norm_k, final_norm, m0, a.independent);
    }

    if (valid) {
        if (write_x) {
            for (int i = 0; i < r; ++i) a.x[j * r + i] = T(0);
            for (int k = 0; k < ra; ++k) a.x[j * r + a.act_idx[k]] = O::div(y[k], a.scale_a[k]);
        }
        // -1: non-finite iterate / frozen-dimension failure; -2: the
        // check_gradients drift test failed (the caller raises AssertionError)
        if (a.iters_out) a.iters_out[j] = fail ? (gdrift ? -2 : -1) : iters;
        if (a.final_out) a.final_out[j] = fail ? T(0) : final_norm;
        if (fail) atomicMin((unsigned long long *)&a.stats[1], (unsigned long long)g);
    }
    // inner-iteration total: integer sum is order independent (deterministic)
    unsigned long long it = (valid && !fail) ? (unsigned long long)iters : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) it += __shfl_xor_sync(NMFB_FULL_MASK, it, o);
    if (lane == 0 && it) atomicAdd(&a.stats[0], it);
}

template <typename T, typename TH>
int launch_ref_impl(const NnlsLaunch &p) {
    auto a = make_args<T, TH>(p);
    int64_t warps = num_blocks(p);
    const int wpb = 2;
    dim3 grid((unsigned)((warps + wpb - 1) / wpb));
    if (p.r <= 16)
        nnls_ref_kernel<T, TH, 16><<<grid, 32 * wpb, 0, p.stream>>>(a);
    else if (p.r <= 64)
        nnls_ref_kernel<T, TH, 64><<<grid, 32 * wpb, 0, p.stream>>>(a);
    else if (p.r <= 256)
        nnls_ref_kernel<T, TH, 256><<<grid, 32 * wpb, 0, p.stream>>>(a);
    else
        return NMFB_ERR_ARG;
    return launch_status();
}

template int launch_ref_impl<double, double>(const NnlsLaunch &);
template int launch_ref_impl<float, float>(const NnlsLaunch &);
template int launch_ref_impl<float, double>(const NnlsLaunch &);

}  // namespace nmfb
