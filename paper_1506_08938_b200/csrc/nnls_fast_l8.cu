// Fast NNLS instantiations with L = 8 lanes per problem (split per L so the
// heavy template instantiations compile in parallel).
#include "nnls_fast.cuh"

namespace nmfb {

#define NMFB_VARIANTS_L8(X) X(7, 8, 1) X(8, 8, 1) X(13, 8, 1) X(16, 8, 1) X(25, 8, 1) X(28, 8, 1)

// smallest E with E * 8 >= need; returns E or 0
int fast_pick_l8(int need) {
    int best = 0;
#define NMFB_PICK(E_, L_, B_) \
    if (E_ * L_ >= need && (best == 0 || E_ < best)) best = E_;
    NMFB_VARIANTS_L8(NMFB_PICK)
#undef NMFB_PICK
    return best;
}

int fast_launch_l8(const NnlsLaunch &p, int E, bool h64) {
#define NMFB_GO(E_, L_, B_)                                                              \
    if (E == E_)                                                                        \
        return h64 ? launch_fast_variant<double, E_, L_, B_>(p)                         \
                   : launch_fast_variant<float, E_, L_, B_>(p);
    NMFB_VARIANTS_L8(NMFB_GO)
#undef NMFB_GO
    return NMFB_ERR_ARG;
}

}  // namespace nmfb
