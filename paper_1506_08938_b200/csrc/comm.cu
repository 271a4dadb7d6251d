// C-ABI collectives of the multi-GPU layouts:
// comm_init / allreduce_r2 / reduce_scatter_panel / allgather_panel over NCCL
// (NVLink / NVSwitch inside a box).  NCCL is resolved at run time with
// dlopen("libnccl.so.2"): inside a PyTorch process that is the NCCL torch
// already loaded (one library instance per process); a plain C caller gets
// the system one.  No link-time dependency, so libnmfb.so loads without NCCL.
//
// Used by paper_1506_08938_b200/dist_rows.py (NMFB_COMM=native) for the
// row-sharded layout's per-iteration exchanges:
//   allreduce_r2          Q_g, H_f (r x r fp64) and the objective pieces
//   reduce_scatter_panel  the partial linear terms, m x r fp32 -> column blocks
//   allgather_panel       F^T rows of every column block
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "nmfb_internal.h"

namespace nmfb {
namespace {

struct Nccl {
    ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                               ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*reduce_scatter)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                                   ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*all_gather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    bool ok = false;
};

const Nccl &nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        n.get_unique_id = (decltype(n.get_unique_id))dlsym(h, "ncclGetUniqueId");
        n.comm_init_rank = (decltype(n.comm_init_rank))dlsym(h, "ncclCommInitRank");
        n.comm_destroy = (decltype(n.comm_destroy))dlsym(h, "ncclCommDestroy");
        n.all_reduce = (decltype(n.all_reduce))dlsym(h, "ncclAllReduce");
        n.reduce_scatter = (decltype(n.reduce_scatter))dlsym(h, "ncclReduceScatter");
        n.all_gather = (decltype(n.all_gather))dlsym(h, "ncclAllGather");
        n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.all_reduce &&
               n.reduce_scatter && n.all_gather;
    });
    return n;
}

int status(ncclResult_t r) { return r == ncclSuccess ? NMFB_OK : NMFB_ERR_CUDA; }

bool nccl_type(int dtype, ncclDataType_t *t) {
    if (dtype == NMFB_F32) {
        *t = ncclFloat32;
        return true;
    }
    if (dtype == NMFB_F64) {
        *t = ncclFloat64;
        return true;
    }
    return false;
}

}  // namespace

int comm_available() { return nccl().ok ? 1 : 0; }

int comm_unique_id(void *id) {
    const Nccl &n = nccl();
    if (!n.ok || !id) return NMFB_ERR_ARG;
    return status(n.get_unique_id(reinterpret_cast<ncclUniqueId *>(id)));
}

int comm_init(const void *id, int rank, int nranks, void **comm) {
    const Nccl &n = nccl();
    if (!n.ok || !id || !comm || nranks < 1 || rank < 0 || rank >= nranks) return NMFB_ERR_ARG;
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    ncclComm_t c = nullptr;
    const int s = status(n.comm_init_rank(&c, nranks, uid, rank));
    *comm = c;
    return s;
}

int comm_destroy(void *comm) {
    const Nccl &n = nccl();
    if (!n.ok || !comm) return NMFB_ERR_ARG;
    return status(n.comm_destroy((ncclComm_t)comm));
}

int allreduce_r2(void *comm, double *buf, int64_t count, cudaStream_t st) {
    const Nccl &n = nccl();
    if (!n.ok || !comm || count < 0 || (count > 0 && !buf)) return NMFB_ERR_ARG;
    if (count == 0) return NMFB_OK;
    return status(n.all_reduce(buf, buf, (size_t)count, ncclFloat64, ncclSum, (ncclComm_t)comm, st));
}

int reduce_scatter_panel(void *comm, const void *send, void *recv, int64_t recv_count, int dtype,
                         cudaStream_t st) {
    const Nccl &n = nccl();
    ncclDataType_t t;
    if (!n.ok || !comm || recv_count < 0 || !nccl_type(dtype, &t) ||
        (recv_count > 0 && (!send || !recv)))
        return NMFB_ERR_ARG;
    if (recv_count == 0) return NMFB_OK;
    return status(
        n.reduce_scatter(send, recv, (size_t)recv_count, t, ncclSum, (ncclComm_t)comm, st));
}

int allgather_panel(void *comm, const void *send, void *recv, int64_t send_count, int dtype,
                    cudaStream_t st) {
    const Nccl &n = nccl();
    ncclDataType_t t;
    if (!n.ok || !comm || send_count < 0 || !nccl_type(dtype, &t) ||
        (send_count > 0 && (!send || !recv)))
        return NMFB_ERR_ARG;
    if (send_count == 0) return NMFB_OK;
    return status(n.all_gather(send, recv, (size_t)send_count, t, (ncclComm_t)comm, st));
}

}  // namespace nmfb
