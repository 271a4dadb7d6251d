// Internal launch descriptors shared by the .cu translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/nmfb.h"

namespace nmfb {

struct NnlsLaunch {
    int dtype;         // NMFB_F32 | NMFB_F64 (type of Qa, scale_a, x, final_out)
    int mode;          // NMFB_MODE_FAST | NMFB_MODE_REFERENCE
    const void *Qa;    // (ra, ra) compact, row-major
    const void *scale_a;
    const int32_t *act_idx;
    const uint8_t *active;
    int r, ra;
    const int32_t *ra_dev;  // nullable: device copy of ra (overrides ra)
    const void *h;
    int h_dtype;
    int h_parts;
    int64_t h_ld, h_pstride;
    double h_base;
    void *x;
    int64_t count, index_base;
    double eps;
    int max_inner;
    double max_stop0;
    int32_t *iters_out;
    void *final_out;
    unsigned long long *stats;
    void *hist = nullptr;  // reference kernel: (count, hist_ld, 2) norm/objective history
    int hist_ld = 0;
    bool independent = false;
    bool check_grad = false;  // reference kernel: fresh-gradient check every iteration
    int lanes;  // 0 = auto
    cudaStream_t stream;
    // fused all-gather (multi-GPU): every solution row is also stored at the
    // same offset from each mirror base (peer GPUs' copies of x, NVLink)
    void *mirror[NMFB_MAX_PEERS] = {};
    int nmirror = 0;
};

// Placement of a GEMM's partial slots.  Row i of slot s is written to
//   dst[o] + ((src * parts + s) * chunk + (i - o * chunk)) * N,   o = i / chunk.
// world = 1, chunk = M: the plain [slot][M][N] layout.  world > 1: each owner
// o's 32-aligned row chunk lands directly in o's receive buffer (peer stores
// over NVLink), so the epilogue IS the reduce-scatter's transfer and owner o
// sums its world * parts slots in a fixed order.
struct RowOut {
    float *dst[NMFB_MAX_PEERS];
    int world, src;
    int64_t chunk;
};

int nnls_launch(const NnlsLaunch &p);

// NMFB_OK, or NMFB_ERR_CUDA after recording the launch error for nmfb_last_error()
int launch_status();

}  // namespace nmfb
