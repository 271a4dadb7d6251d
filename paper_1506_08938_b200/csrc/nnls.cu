// Batched nonnegative quadratic programs sharing one rescaled Hessian:
//   minimize 0.5 y'Qy + q'y, y >= 0,   one problem per data column / row.
//
// Semantics follow the reference's compiled shard loop exactly:
//   kernels.py:178-220 (_coefficient_solve), :38-150 (_solve_rescaled),
//   :153-175 (_take_step), fast-break blocks :35, :246-248, :266-267.
//
// Two kernels:
//  * nnls_ref_kernel<T> (nnls_ref.cu): one thread per problem, every reduction
//    in the reference's sequential index order, no FMA contraction (Exact<T>).
//    With T=double it reproduces the reference bit for bit (fp64 check mode).
//  * nnls_fast_kernel<E, L, B> (nnls_fast.cuh): fp32 production kernel.  A
//    problem is owned by a group of L lanes, each holding E coordinates
//    (k = e*L + l) of y, grad and Q*d in registers; the compact Q (R x S, S odd
//    => conflict-free rows) is staged once per CTA in shared memory;
//    line-search dot products and the greedy-CD argmax (ties -> lowest index,
//    as kernels.py:119 strict >) are group shuffles.  CTA = B fast-break
//    blocks of 32 problems.
//
// Fast-break: see resolve_block_warp in common.cuh.
#include "nnls_common.cuh"

namespace nmfb {

template <typename T, typename TH>
int launch_ref_impl(const NnlsLaunch &p);
int fast_pick_l1(int need);
int fast_pick_l2(int need);
int fast_pick_l4(int need);
int fast_pick_l8(int need);
int fast_launch_l1(const NnlsLaunch &p, int E, bool h64);
int fast_launch_l2(const NnlsLaunch &p, int E, bool h64);
int fast_launch_l4(const NnlsLaunch &p, int E, bool h64);
int fast_launch_l8(const NnlsLaunch &p, int E, bool h64);
int fast_pick_lx(int code, int need);
int fast_launch_lx(const NnlsLaunch &p, int code, int E, bool h64);

static int launch_fast(const NnlsLaunch &p) {
    // with a device-side ra the variant must cover the full rank r
    const int need = p.ra_dev ? p.r : p.ra;
    int L = p.lanes;
    if (L == 0) L = need <= 16 ? 1 : (need <= 56 ? 8 : (need <= 128 ? 8 : 8));
    const bool h64 = p.h_dtype == NMFB_F64;
    int E;
    switch (L) {
        case 1: E = fast_pick_l1(need); return E ? fast_launch_l1(p, E, h64) : NMFB_ERR_ARG;
        case 2: E = fast_pick_l2(need); return E ? fast_launch_l2(p, E, h64) : NMFB_ERR_ARG;
        case 4: E = fast_pick_l4(need); return E ? fast_launch_l4(p, E, h64) : NMFB_ERR_ARG;
        case 8: E = fast_pick_l8(need); return E ? fast_launch_l8(p, E, h64) : NMFB_ERR_ARG;
        default: E = fast_pick_lx(L, need); return E ? fast_launch_lx(p, L, E, h64) : NMFB_ERR_ARG;
    }
}

int nnls_launch(const NnlsLaunch &p) {
    if (p.count <= 0) return NMFB_OK;
    if (p.r <= 0 || p.ra < 0 || p.ra > p.r || p.index_base < 0 || p.max_inner < 1)
        return NMFB_ERR_ARG;
    if (p.nmirror < 0 || p.nmirror > NMFB_MAX_PEERS) return NMFB_ERR_ARG;
    for (int q = 0; q < p.nmirror; ++q)
        if (!p.mirror[q]) return NMFB_ERR_ARG;
    // the fused all-gather lives in the fast kernel only
    if (p.nmirror > 0 && (p.dtype == NMFB_F64 || p.mode == NMFB_MODE_REFERENCE))
        return NMFB_ERR_ARG;
    if (p.dtype == NMFB_F64) {
        if (p.h_dtype != NMFB_F64) return NMFB_ERR_ARG;
        return launch_ref_impl<double, double>(p);
    }
    if (p.mode == NMFB_MODE_REFERENCE)
        return p.h_dtype == NMFB_F64 ? launch_ref_impl<float, double>(p)
                                     : launch_ref_impl<float, float>(p);
    return launch_fast(p);
}

}  // namespace nmfb
