// Peer-memory exchange over NVLink / NVSwitch (multi-GPU column-sharded fit).
//
// Every rank maps the other ranks' symmetric buffers (torch symmetric memory
// hands out the peer pointers); producers write their outputs straight into
// the consumer's buffer:
//   * the X F^T tensor-core GEMM stores each owner's rows of its Y^T partial
//     slots into the owner's receive buffer (RowOut, tc_gemm.cu) -- the
//     reduce-scatter's transfer, overlapped with the GEMM tile by tile;
//   * the component-step NNLS stores every solved G row into each peer's G
//     (NnlsLaunch::mirror) -- the all-gather, fused into the solve;
//   * small fp64 vectors (the r x r partial Gram F_g F_g^T, objective
//     pieces) are pushed into a per-source slot of every peer (peer_put).
// Completion is a flag per (receiver, source): after its writes a rank
// stores `epoch` into flag[source] of every peer with release semantics at
// system scope; a consumer waits (acquire, system scope) until all world
// flags reach the epoch.  Epochs grow monotonically and every rank issues
// the same exchange sequence, so flags never need resetting.  The receiver
// sums the per-source slots in source order: deterministic results that do
// not depend on the collective's internal reduction order.
#include "common.cuh"
#include "nmfb_internal.h"

namespace nmfb {

struct PeerPtrs {
    void *p[NMFB_MAX_PEERS];
};

__device__ __forceinline__ void st_release_sys(unsigned long long *a, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *a) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long gtime_ns_peer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// dst.p[q] (q < world) <- src (n8 8-byte words), then, when every CTA is
// done, flag[rank] = epoch on every peer (flags.p[q] = rank q's flag array).
// src == nullptr: signal only (the data was written by a fused producer).
__global__ void peer_put_kernel(const uint2 *__restrict__ src, int64_t n8, PeerPtrs dst,
                                int world, int rank, PeerPtrs flags, unsigned *ticket,
                                unsigned long long epoch, int signal) {
    if (src) {
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8;
             i += (int64_t)gridDim.x * blockDim.x) {
            const uint2 v = src[i];
            for (int q = 0; q < world; ++q) reinterpret_cast<uint2 *>(dst.p[q])[i] = v;
        }
    }
    if (!signal) return;
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned t = atomicAdd(ticket, 1u);
        if (t == gridDim.x - 1) {
            *ticket = 0u;  // every CTA has arrived; reset for the next call
            __threadfence_system();
            for (int q = 0; q < world; ++q)
                st_release_sys(reinterpret_cast<unsigned long long *>(flags.p[q]) + rank, epoch);
        }
    }
}

// Wait until my flag[q] >= epoch for every source q.  Bounded: after
// ~timeout_ms the kernel records an error word (flags[world]) and returns
// instead of hanging the device.
__global__ void peer_wait_kernel(unsigned long long *flags, int world, unsigned long long epoch,
                                 long long timeout_ns) {
    const int q = threadIdx.x;
    if (q < world) {
        const unsigned long long t0 = gtime_ns_peer();
        while (ld_acquire_sys(flags + q) < epoch) {
            __nanosleep(64);
            if ((long long)(gtime_ns_peer() - t0) > timeout_ns) {
                atomicMax(flags + world, epoch);
                break;
            }
        }
    }
    __syncthreads();
}

// out[i] = sum_{s < S} slots[s * stride + i], in slot order (fp64)
__global__ void sum_slots_f64_kernel(const double *__restrict__ slots, int S, int64_t len,
                                     int64_t stride, double *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len;
         i += (int64_t)gridDim.x * blockDim.x) {
        double acc = slots[i];
        for (int s = 1; s < S; ++s) acc += slots[(int64_t)s * stride + i];
        out[i] = acc;
    }
}

int peer_put_launch(const void *src, int64_t bytes, void *const *dst, int world, int rank,
                    void *const *flags, unsigned *ticket, unsigned long long epoch, int signal,
                    cudaStream_t st) {
    if (world < 1 || world > NMFB_MAX_PEERS || rank < 0 || rank >= world || bytes < 0)
        return NMFB_ERR_ARG;
    if (src && (bytes % 8 != 0 || (uintptr_t)src % 8 != 0)) return NMFB_ERR_ARG;
    if (signal && (!ticket || !flags)) return NMFB_ERR_ARG;
    PeerPtrs d{}, f{};
    for (int q = 0; q < world; ++q) {
        if (src) {
            if (!dst || !dst[q] || (uintptr_t)dst[q] % 8 != 0) return NMFB_ERR_ARG;
            d.p[q] = dst[q];
        }
        if (signal) {
            if (!flags[q]) return NMFB_ERR_ARG;
            f.p[q] = flags[q];
        }
    }
    const int64_t n8 = src ? bytes / 8 : 0;
    int blocks = (int)std::min<int64_t>(148, std::max<int64_t>(1, (n8 + 255) / 256));
    peer_put_kernel<<<blocks, 256, 0, st>>>((const uint2 *)(src ? src : nullptr), n8, d, world,
                                            rank, f, ticket, epoch, signal);
    return launch_status();
}

int peer_wait_launch(void *flags, int world, unsigned long long epoch, double timeout_s,
                     cudaStream_t st) {
    if (!flags || world < 1 || world > NMFB_MAX_PEERS) return NMFB_ERR_ARG;
    const long long ns = (long long)((timeout_s > 0 ? timeout_s : 30.0) * 1e9);
    peer_wait_kernel<<<1, 32, 0, st>>>((unsigned long long *)flags, world, epoch, ns);
    return launch_status();
}

int sum_slots_f64_launch(const double *slots, int S, int64_t len, int64_t stride, double *out,
                         cudaStream_t st) {
    if (S < 1 || len < 0 || stride < len) return NMFB_ERR_ARG;
    if (len == 0) return NMFB_OK;
    const int blocks = (int)std::min<int64_t>(148, (len + 255) / 256);
    sum_slots_f64_kernel<<<blocks, 256, 0, st>>>(slots, S, len, stride, out);
    return launch_status();
}

}  // namespace nmfb
