// Fast NNLS instantiations with L = 4 lanes per problem (split per L so the
// heavy template instantiations compile in parallel).
#include "nnls_fast.cuh"

namespace nmfb {

#define NMFB_VARIANTS_L4(X) X(13, 4, 2) X(16, 4, 2) X(25, 4, 2) X(32, 4, 2)

// smallest E with E * 4 >= need; returns E or 0
int fast_pick_l4(int need) {
    int best = 0;
#define NMFB_PICK(E_, L_, B_) \
    if (E_ * L_ >= need && (best == 0 || E_ < best)) best = E_;
    NMFB_VARIANTS_L4(NMFB_PICK)
#undef NMFB_PICK
    return best;
}

int fast_launch_l4(const NnlsLaunch &p, int E, bool h64) {
#define NMFB_GO(E_, L_, B_)                                                              \
    if (E == E_)                                                                        \
        return h64 ? launch_fast_variant<double, E_, L_, B_>(p)                         \
                   : launch_fast_variant<float, E_, L_, B_>(p);
    NMFB_VARIANTS_L4(NMFB_GO)
#undef NMFB_GO
    return NMFB_ERR_ARG;
}

}  // namespace nmfb
