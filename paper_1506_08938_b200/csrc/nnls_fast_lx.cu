// Fast NNLS instantiations for large ranks: wider lane groups (L = 16, 32)
// and L = 8 with two fast-break blocks per CTA, so more problems share the
// CTA's staged Q (at r = 200, Q alone is 160 KB of shared memory: one CTA
// per SM, and the group width sets how many warps the SM can hide latency
// with).
#include "nnls_fast.cuh"

namespace nmfb {

#define NMFB_VARIANTS_LX(X) X(7, 16, 1) X(13, 16, 1) X(4, 32, 1) X(7, 32, 1) \
    X(13, 8, 2) X(25, 8, 2) X(28, 8, 2)

// lanes code: L, or 100 * (B - 1) + L for B > 1 blocks per CTA
int fast_pick_lx(int code, int need) {
    int best = 0;
#define NMFB_PICK(E_, L_, B_) \
    if (100 * (B_ - 1) + L_ == code && E_ * L_ >= need && (best == 0 || E_ < best)) best = E_;
    NMFB_VARIANTS_LX(NMFB_PICK)
#undef NMFB_PICK
    return best;
}

int fast_launch_lx(const NnlsLaunch &p, int code, int E, bool h64) {
#define NMFB_GO(E_, L_, B_)                                                              \
    if (100 * (B_ - 1) + L_ == code && E == E_)                                         \
        return h64 ? launch_fast_variant<double, E_, L_, B_>(p)                         \
                   : launch_fast_variant<float, E_, L_, B_>(p);
    NMFB_VARIANTS_LX(NMFB_GO)
#undef NMFB_GO
    return NMFB_ERR_ARG;
}

}  // namespace nmfb
