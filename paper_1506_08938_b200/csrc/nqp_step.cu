// The public NQP building blocks as batched device steps (fp64, one thread
// per problem, numpy's evaluation order per element):
//   nqp.exact_line_search_step  nqp.py:151-183
//   nqp.greedy_cd_pass          nqp.py:186-209
// The fit path never calls these (its solver is nnls_ref / nnls_fast); they
// back the Python helpers of the same names.
#include "common.cuh"
#include "nmfb_internal.h"

namespace nmfb {

namespace {

template <int MAXR>
__global__ void __launch_bounds__(64) nqp_line_search_kernel(const double *__restrict__ Q, int r,
                                                             const double *x_in,
                                                             const double *g_in, int64_t count,
                                                             double *x_out, double *g_out) {
    using O = Exact<double>;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= count) return;
    double x[MAXR], g[MAXR], d[MAXR], xn[MAXR], qd[MAXR];
    for (int i = 0; i < r; ++i) {
        x[i] = x_in[j * r + i];
        g[i] = g_in[j * r + i];
    }
    // d = where(passive_mask(x, grad), grad, 0); norm_sq = d @ d
    double nsq = 0.0;
    for (int i = 0; i < r; ++i) {
        d[i] = (x[i] > 0.0 || g[i] < 0.0) ? g[i] : 0.0;
        nsq = O::madd(nsq, d[i], d[i]);
    }
    if (nsq == 0.0) {
        for (int i = 0; i < r; ++i) {
            x_out[j * r + i] = x[i];
            g_out[j * r + i] = g[i];
        }
        return;
    }
    double curv = 0.0;  // d @ (Q @ d)
    for (int i = 0; i < r; ++i) {
        double acc = 0.0;
        for (int k = 0; k < r; ++k) acc = O::madd(acc, Q[i * r + k], d[k]);
        curv = O::madd(curv, d[i], acc);
    }
    const double alpha = curv > 0.0 ? O::div(nsq, curv) : 1.0;
    // take(step): x_new = max(x - step d, 0); q_delta = Q[:, changed] @
    // delta[changed]; df = grad @ delta + 0.5 delta @ q_delta
    auto take = [&](double step) {
        for (int i = 0; i < r; ++i) {
            const double v = O::sub(x[i], O::mul(step, d[i]));
            xn[i] = v > 0.0 ? v : 0.0;
            qd[i] = 0.0;
        }
        for (int k = 0; k < r; ++k) {
            const double dk = O::sub(xn[k], x[k]);
            if (dk != 0.0)
                for (int i = 0; i < r; ++i) qd[i] = O::madd(qd[i], Q[i * r + k], dk);
        }
        double gd = 0.0, dq = 0.0;  // grad @ delta, (0.5 delta) @ q_delta
        for (int i = 0; i < r; ++i) {
            const double di = O::sub(xn[i], x[i]);
            gd = O::madd(gd, g[i], di);
            dq = O::madd(dq, O::mul(0.5, di), qd[i]);
        }
        return O::add(gd, dq);
    };
    double df = take(alpha);
    if (df > 0.0) {
        double abp = INFINITY;
        bool any = false;
        for (int i = 0; i < r; ++i)
            if (d[i] > 0.0 && x[i] > 0.0) {
                any = true;
                const double c = O::div(x[i], d[i]);
                if (c < abp) abp = c;
            }
        if (any && abp < alpha) df = take(abp);
    }
    for (int i = 0; i < r; ++i) {
        x_out[j * r + i] = xn[i];
        g_out[j * r + i] = O::add(g[i], qd[i]);
    }
}

template <int MAXR>
__global__ void __launch_bounds__(64) nqp_greedy_cd_kernel(const double *__restrict__ Q, int r,
                                                           const double *x_in,
                                                           const double *g_in, int64_t count,
                                                           int sweeps, double *x_out,
                                                           double *g_out) {
    using O = Exact<double>;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= count) return;
    double x[MAXR], g[MAXR];
    for (int i = 0; i < r; ++i) {
        x[i] = x_in[j * r + i];
        g[i] = g_in[j * r + i];
    }
    for (int s = 0; s < sweeps; ++s) {
        // dx = max(0, x - grad) - x; decrease = |grad dx + 0.5 dx dx|;
        // p = argmax (first maximum)
        double best = -1.0, bdx = 0.0;
        int p = 0;
        for (int i = 0; i < r; ++i) {
            const double t = O::sub(x[i], g[i]);
            const double dx = O::sub(t > 0.0 ? t : 0.0, x[i]);
            const double dec = fabs(O::add(O::mul(g[i], dx), O::mul(O::mul(0.5, dx), dx)));
            if (dec > best) {
                best = dec;
                p = i;
                bdx = dx;
            }
        }
        if (!(best > 0.0)) break;
        for (int i = 0; i < r; ++i) g[i] = O::add(g[i], O::mul(Q[i * r + p], bdx));
        x[p] = O::add(x[p], bdx);
    }
    for (int i = 0; i < r; ++i) {
        x_out[j * r + i] = x[i];
        g_out[j * r + i] = g[i];
    }
}

template <int MAXR>
int launch_step(int op, const double *Q, int r, const double *x, const double *g, int64_t count,
                int sweeps, double *xo, double *go, cudaStream_t st) {
    const unsigned grid = (unsigned)((count + 63) / 64);
    if (op == NMFB_NQP_LINE_SEARCH)
        nqp_line_search_kernel<MAXR><<<grid, 64, 0, st>>>(Q, r, x, g, count, xo, go);
    else
        nqp_greedy_cd_kernel<MAXR><<<grid, 64, 0, st>>>(Q, r, x, g, count, sweeps, xo, go);
    return launch_status();
}

}  // namespace

int nqp_step_launch(int op, const double *Q, int r, const double *x, const double *g,
                    int64_t count, int sweeps, double *xo, double *go, cudaStream_t st) {
    if ((op != NMFB_NQP_LINE_SEARCH && op != NMFB_NQP_GREEDY_CD) || r <= 0 || r > 256 ||
        count < 0)
        return NMFB_ERR_ARG;
    if (count == 0) return NMFB_OK;
    if (!Q || !x || !g || !xo || !go) return NMFB_ERR_ARG;
    if (sweeps < 0) sweeps = r;
    if (r <= 16) return launch_step<16>(op, Q, r, x, g, count, sweeps, xo, go, st);
    if (r <= 64) return launch_step<64>(op, Q, r, x, g, count, sweeps, xo, go, st);
    return launch_step<256>(op, Q, r, x, g, count, sweeps, xo, go, st);
}

}  // namespace nmfb
