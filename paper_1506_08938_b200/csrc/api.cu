// C ABI (include/nmfb.h).  Thin argument checking + launch composition; all
// numerics live in nnls.cu / gram.cu / dense.cu / sparse.cu / reduce.cu.
#include <cstdio>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "nmfb_internal.h"

namespace nmfb {
int sum_slots_rescale_launch(int dtype, const double *slots, int S, int64_t stride, double *H,
                             int r, double diag_add, void *Qa, void *scale_a, int32_t *act_idx,
                             uint8_t *active, int32_t *ra_dev, cudaStream_t st);
int csc_segments_launch(const int64_t *indptr, const int32_t *rowidx, int64_t m, int64_t blk,
                        int nblk, int64_t *seg, cudaStream_t st);
int chunk_segments_launch(const int64_t *chunks, int64_t nchunks, const int32_t *colidx,
                          int64_t blk, int nblk, int64_t *seg, cudaStream_t st);
int csc_linear_vec_launch(const int64_t *indptr, const int64_t *seg, int nblk,
                          const int32_t *rowidx, const float *vals, int64_t lo, int64_t hi,
                          const float *G, int r, double mu1, float *h, cudaStream_t st);
int csr_yt_chunked_vec_launch(const int64_t *chunks, int64_t nchunks, const int64_t *heavy,
                              int64_t nheavy, const int64_t *seg, int nblk, const int32_t *colidx,
                              const float *vals, const float *FT, int r, int yt_dtype, void *YT,
                              void *part, cudaStream_t st);
int pcg64_factors_launch(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                         int64_t n, int64_t m, int r, double scale, int dtype, void *G, void *FT,
                         cudaStream_t st);
int mur_update_launch(int dtype, const double *Q, int r, const void *h, int h_dtype, int S,
                      int64_t h_ld, int64_t h_pstride, double h_base, void *x, int64_t count,
                      double floor_, uint64_t *stats, cudaStream_t st);
int csc_from_triplets_launch(int64_t rows, int64_t cols, int64_t count, const int64_t *i,
                             const int64_t *j, const double *v, int sum_dup, int64_t *indptr,
                             int32_t *rowidx, void *vals, int vals_dtype, int64_t *nnz_out,
                             int64_t *info, cudaStream_t st);
int csc_to_csr_launch(int64_t rows, int64_t cols, int64_t nnz, const int64_t *indptr,
                      const int32_t *rowidx, const void *vals, int vals_dtype, int64_t *rowptr,
                      int32_t *colidx, void *cvals, cudaStream_t st);
int csc_validate_launch(int64_t rows, int64_t cols, int64_t nnz, const int64_t *indptr,
                        const int32_t *rowidx, const void *vals, int vals_dtype, int64_t *info,
                        cudaStream_t st);
int ingest_release_scratch();
int csr_chunk_plan_launch(const int64_t *rowptr, int64_t rows, int64_t chunk, int64_t *chunks,
                          int64_t *heavy, int64_t *counts_out, cudaStream_t st);
int comm_available();
int comm_unique_id(void *id);
int comm_init(const void *id, int rank, int nranks, void **comm);
int comm_destroy(void *comm);
int allreduce_r2(void *comm, double *buf, int64_t count, cudaStream_t st);
int reduce_scatter_panel(void *comm, const void *send, void *recv, int64_t recv_count, int dtype,
                         cudaStream_t st);
int allgather_panel(void *comm, const void *send, void *recv, int64_t send_count, int dtype,
                    cudaStream_t st);
int nqp_step_launch(int op, const double *Q, int r, const double *x, const double *g,
                    int64_t count, int sweeps, double *xo, double *go, cudaStream_t st);
int narrow_indices_launch(const int64_t *in, int64_t n, int32_t *out, int64_t *info,
                          cudaStream_t st);
size_t gram_workspace_bytes(int64_t rows, int r);
int gram_launch(int dtype, const void *A, int64_t rows, int r, int64_t lda, double *out, void *ws,
                cudaStream_t st);
int gram_rescale_launch(int dtype, const void *A, int64_t rows, int r, int64_t lda, double *out,
                        void *ws, double diag_add, void *Qa, void *scale_a, int32_t *act_idx,
                        uint8_t *active, int32_t *ra_dev, cudaStream_t st);
int rescale_launch(int dtype, const double *G, int r, double diag_add, void *Qa, void *scale_a,
                   int32_t *act_idx, uint8_t *active, int32_t *ra_dev, double *full_scale,
                   cudaStream_t st);
int gemm_tall_launch(const float *A, int a_kmajor, int64_t M, int64_t K, int64_t lda,
                     const float *B, int N, int64_t ldb, float *C, int splits, cudaStream_t st);
int dense_linear_ref_launch(int dtype, const void *VT, int64_t n, int64_t col_lo, int64_t col_hi,
                            const void *G, int r, double mu1, void *h, cudaStream_t st);
int dense_yt_ref_launch(int dtype, const void *VT, int64_t m, int64_t n, const void *FT, int r,
                        const int64_t *bounds, int workers, void *YT, cudaStream_t st);
int hp_ref_launch(int dtype, const void *FT, int64_t m, int r, const int64_t *bounds, int workers,
                  void *HF, cudaStream_t st);
size_t residual_workspace_bytes(int64_t m, int64_t n);
int dense_residual_launch(int dtype, const void *XT, int64_t m, int64_t n, const void *G,
                          const void *FT, int r, double *out, void *ws, cudaStream_t st);
int csc_linear_launch(int dtype, int mode, const int64_t *indptr, const int32_t *rowidx,
                      const void *vals, int64_t lo, int64_t hi, const void *G, int r, double mu1,
                      void *h, cudaStream_t st);
int csr_yt_launch(int dtype, int mode, const int64_t *rowptr, const int32_t *colidx,
                  const void *vals, int64_t n, const void *FT, int r, int yt_dtype,
                  const int64_t *bounds, int workers, void *YT, cudaStream_t st);
size_t dot_workspace_bytes(int64_t len);
int dot_launch(const void *a, int a_dtype, const void *b, int b_dtype, int64_t len, double *out,
               void *ws, cudaStream_t st);
int add_into_launch(int dtype, void *dst, const void *src, int64_t len, int upper_r,
                    cudaStream_t st);
int sum_parts_launch(const float *parts, int S, int64_t len, float *out, cudaStream_t st);
int csr_yt_chunked_launch(int dtype, const int64_t *chunks, int64_t nchunks, const int64_t *heavy,
                          int64_t nheavy, const int32_t *colidx, const void *vals, const void *FT,
                          int r, int yt_dtype, void *YT, void *part, cudaStream_t st);
int dense_residual_kmajor_launch(const float *XT, int64_t m, int64_t n, const float *Gt,
                                 const float *Ft, int r, double *out, void *ws, cudaStream_t st);
int tc_gemm_launch(const float *A, int64_t M, int64_t K, const float *Bt_hi, const float *Bt_lo,
                   int N, float *C, int splits, int stages, cudaStream_t st);
int tc_effective_splits(int64_t K, int splits);
int tc_gemm_rows_launch(const float *A, int64_t M, int64_t K, const float *Bt_hi,
                        const float *Bt_lo, int N, const RowOut &out, int splits, int stages,
                        cudaStream_t st);
int peer_put_launch(const void *src, int64_t bytes, void *const *dst, int world, int rank,
                    void *const *flags, unsigned *ticket, unsigned long long epoch, int signal,
                    cudaStream_t st);
int peer_wait_launch(void *flags, int world, unsigned long long epoch, double timeout_s,
                     cudaStream_t st);
int sum_slots_f64_launch(const double *slots, int S, int64_t len, int64_t stride, double *out,
                         cudaStream_t st);
size_t slice_bytes(int64_t rows, int r);
int slice_u8_launch(const float *A, int64_t rows, int r, int64_t lda, void *out, cudaStream_t st);
size_t residual_i8_workspace_bytes();
int residual_i8_launch(const float *X, int64_t n, int64_t m, const void *Gsl, const void *Fsl,
                       int r, double *out, void *ws, cudaStream_t st);
int tc_parts(int64_t M, int64_t K, int N, int splits);
int data_stats_launch(const void *a, int a_dtype, int64_t len, double *out, void *ws,
                      cudaStream_t st);
int split_transpose_launch(const float *B, int64_t K, int r, float *hi, float *lo,
                           cudaStream_t st);
int transpose_launch(const float *in, int64_t rows, int64_t cols, float *out, cudaStream_t st);
int csc_scatter_yt_launch(int dtype, const int64_t *indptr, const int32_t *rowidx,
                          const void *vals, int64_t lo, int64_t hi, const void *FT, int r,
                          void *YT, cudaStream_t st);
}  // namespace nmfb

using namespace nmfb;

static thread_local char g_err[256] = "";

static int cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return NMFB_OK;
    snprintf(g_err, sizeof(g_err), "%s", cudaGetErrorString(e));
    return NMFB_ERR_CUDA;
}
namespace nmfb {
int launch_status() { return cuda_status(cudaGetLastError()); }
}  // namespace nmfb
static int check(int status) { return status; }
static inline size_t esize(int dtype) { return dtype == NMFB_F64 ? 8 : 4; }

extern "C" {

int nmfb_version(void) { return 100; }
const char *nmfb_last_error(void) { return g_err; }
int nmfb_device_sm_count(void) {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    return v;
}

int nmfb_nnls_batch(int dtype, int mode, const void *Qa, const void *scale_a,
                    const int32_t *act_idx, const uint8_t *active, int32_t r, int32_t ra,
                    const int32_t *ra_dev, const void *h, int h_dtype, int32_t h_parts,
                    int64_t h_ld, int64_t h_pstride, double h_base, void *x, int64_t count,
                    int64_t index_base, double eps, int32_t max_inner, double max_stop0,
                    int32_t *iters_out, void *final_out, uint64_t *stats, int32_t lanes,
                    void *stream) {
    NnlsLaunch p;
    p.dtype = dtype;
    p.mode = mode;
    p.Qa = Qa;
    p.scale_a = scale_a;
    p.act_idx = act_idx;
    p.active = active;
    p.r = r;
    p.ra = ra;
    p.ra_dev = ra_dev;
    p.h = h;
    p.h_dtype = h_dtype;
    p.h_parts = h_parts;
    p.h_ld = h_ld;
    p.h_pstride = h_pstride;
    p.h_base = h_base;
    p.x = x;
    p.count = count;
    p.index_base = index_base;
    p.eps = eps;
    p.max_inner = max_inner;
    p.max_stop0 = max_stop0;
    p.iters_out = iters_out;
    p.final_out = final_out;
    p.stats = (unsigned long long *)stats;
    p.lanes = lanes;
    p.stream = (cudaStream_t)stream;
    if (h_parts < 0 || eps < 0.0 || eps > 1.0 || !stats) return NMFB_ERR_ARG;
    return check(nnls_launch(p));
}

int nmfb_nnls_batch_peers(int dtype, int mode, const void *Qa, const void *scale_a,
                          const int32_t *act_idx, const uint8_t *active, int32_t r, int32_t ra,
                          const int32_t *ra_dev, const void *h, int h_dtype, int32_t h_parts,
                          int64_t h_ld, int64_t h_pstride, double h_base, void *x,
                          int64_t count, int64_t index_base, double eps, int32_t max_inner,
                          double max_stop0, int32_t *iters_out, void *final_out,
                          uint64_t *stats, int32_t lanes, void *const *mirror, int32_t nmirror,
                          void *stream) {
    NnlsLaunch p;
    p.dtype = dtype;
    p.mode = mode;
    p.Qa = Qa;
    p.scale_a = scale_a;
    p.act_idx = act_idx;
    p.active = active;
    p.r = r;
    p.ra = ra;
    p.ra_dev = ra_dev;
    p.h = h;
    p.h_dtype = h_dtype;
    p.h_parts = h_parts;
    p.h_ld = h_ld;
    p.h_pstride = h_pstride;
    p.h_base = h_base;
    p.x = x;
    p.count = count;
    p.index_base = index_base;
    p.eps = eps;
    p.max_inner = max_inner;
    p.max_stop0 = max_stop0;
    p.iters_out = iters_out;
    p.final_out = final_out;
    p.stats = (unsigned long long *)stats;
    p.lanes = lanes;
    p.stream = (cudaStream_t)stream;
    if (h_parts < 0 || eps < 0.0 || eps > 1.0 || !stats) return NMFB_ERR_ARG;
    if (nmirror < 0 || nmirror > NMFB_MAX_PEERS || (nmirror > 0 && !mirror)) return NMFB_ERR_ARG;
    p.nmirror = nmirror;
    for (int q = 0; q < nmirror; ++q) p.mirror[q] = mirror[q];
    return check(nnls_launch(p));
}

int nmfb_nqp_solve(const double *Qa, const double *scale_a, const int32_t *act_idx,
                   const uint8_t *active, int32_t r, const int32_t *ra_dev, const double *h,
                   double *x, int64_t count, double eps, int32_t max_inner, double max_stop,
                   int32_t *iters_out, double *final_out, double *hist, int32_t hist_ld,
                   int32_t check_gradients, uint64_t *stats, void *stream) {
    NnlsLaunch p;
    p.dtype = NMFB_F64;
    p.mode = NMFB_MODE_REFERENCE;
    p.Qa = Qa;
    p.scale_a = scale_a;
    p.act_idx = act_idx;
    p.active = active;
    p.r = r;
    p.ra = r;
    p.ra_dev = ra_dev;
    p.h = h;
    p.h_dtype = NMFB_F64;
    p.h_parts = 0;
    p.h_ld = r;
    p.h_pstride = 0;
    p.h_base = 0.0;
    p.x = x;
    p.count = count;
    p.index_base = 0;
    p.eps = eps;
    p.max_inner = max_inner;
    p.max_stop0 = max_stop;
    p.iters_out = iters_out;
    p.final_out = final_out;
    p.stats = (unsigned long long *)stats;
    p.hist = hist;
    p.hist_ld = hist_ld;
    p.independent = true;
    p.check_grad = check_gradients != 0;
    p.lanes = 0;
    p.stream = (cudaStream_t)stream;
    if (eps < 0.0 || eps > 1.0 || !stats || max_inner < 1) return NMFB_ERR_ARG;
    return check(nnls_launch(p));
}

int nmfb_nqp_step(int32_t op, const double *Q, int32_t r, const double *x, const double *grad,
                  int64_t count, int32_t sweeps, double *x_out, double *grad_out, void *stream) {
    return check(nqp_step_launch(op, Q, r, x, grad, count, sweeps, x_out, grad_out,
                                 (cudaStream_t)stream));
}

size_t nmfb_gram_workspace_bytes(int64_t rows, int32_t r) { return gram_workspace_bytes(rows, r); }

int nmfb_gram_rescale(int dtype, const void *A, int64_t rows, int32_t r, int64_t lda, double *out,
                      void *workspace, double diag_add, void *Qa, void *scale_a, int32_t *act_idx,
                      uint8_t *active, int32_t *ra_dev, void *stream) {
    return check(gram_rescale_launch(dtype, A, rows, r, lda, out, workspace, diag_add, Qa, scale_a,
                                     act_idx, active, ra_dev, (cudaStream_t)stream));
}

int nmfb_gram(int dtype, const void *A, int64_t rows, int32_t r, int64_t lda, double *out,
              void *workspace, void *stream) {
    return check(gram_launch(dtype, A, rows, r, lda, out, workspace, (cudaStream_t)stream));
}

int nmfb_rescale(int dtype, const double *G, int32_t r, double diag_add, void *Qa,
                 void *scale_a, int32_t *act_idx, uint8_t *active, int32_t *ra_dev,
                 double *full_scale, void *stream) {
    return check(rescale_launch(dtype, G, r, diag_add, Qa, scale_a, act_idx, active, ra_dev,
                                full_scale, (cudaStream_t)stream));
}

int nmfb_gemm_tall(const float *A, int a_kmajor, int64_t M, int64_t K, int64_t lda,
                   const float *B, int32_t N, int64_t ldb, float *C, int32_t splits,
                   void *stream) {
    return check(gemm_tall_launch(A, a_kmajor, M, K, lda, B, N, ldb, C, splits,
                                  (cudaStream_t)stream));
}

int nmfb_dense_linear_ref(int dtype, const void *VT, int64_t n, int64_t col_lo, int64_t col_hi,
                          const void *G, int32_t r, double mu1, void *h, void *stream) {
    return check(dense_linear_ref_launch(dtype, VT, n, col_lo, col_hi, G, r, mu1, h,
                                         (cudaStream_t)stream));
}

int nmfb_dense_yt_ref(int dtype, const void *VT, int64_t m, int64_t n, const void *FT,
                      int32_t r, const int64_t *shard_bounds, int32_t workers, void *YT,
                      void *stream) {
    return check(dense_yt_ref_launch(dtype, VT, m, n, FT, r, shard_bounds, workers, YT,
                                     (cudaStream_t)stream));
}

int nmfb_hp_ref(int dtype, const void *FT, int64_t m, int32_t r, const int64_t *shard_bounds,
                int32_t workers, void *HF, void *stream) {
    return check(hp_ref_launch(dtype, FT, m, r, shard_bounds, workers, HF, (cudaStream_t)stream));
}

int nmfb_csc_linear(int dtype, int mode, const int64_t *indptr, const int32_t *rowidx,
                    const void *vals, int64_t col_lo, int64_t col_hi, const void *G, int32_t r,
                    double mu1, void *h, void *stream) {
    return check(csc_linear_launch(dtype, mode, indptr, rowidx, vals, col_lo, col_hi, G, r, mu1,
                                   h, (cudaStream_t)stream));
}

int nmfb_csr_yt(int dtype, int mode, const int64_t *rowptr, const int32_t *colidx,
                const void *vals, int64_t n, const void *FT, int32_t r, int yt_dtype,
                const int64_t *shard_bounds, int32_t workers, void *YT, void *stream) {
    return check(csr_yt_launch(dtype, mode, rowptr, colidx, vals, n, FT, r, yt_dtype,
                               shard_bounds, workers, YT, (cudaStream_t)stream));
}

size_t nmfb_residual_workspace_bytes(int64_t m, int64_t n) {
    return residual_workspace_bytes(m, n);
}

int nmfb_dense_residual(int dtype, const void *XT, int64_t m, int64_t n, const void *G,
                        const void *FT, int32_t r, double *out, void *workspace, void *stream) {
    return check(dense_residual_launch(dtype, XT, m, n, G, FT, r, out, workspace,
                                       (cudaStream_t)stream));
}

int nmfb_csr_yt_chunked(int dtype, const int64_t *chunks, int64_t nchunks, const int64_t *heavy,
                        int64_t nheavy, const int32_t *colidx, const void *vals, const void *FT,
                        int32_t r, int yt_dtype, void *YT, void *part, void *stream) {
    return check(csr_yt_chunked_launch(dtype, chunks, nchunks, heavy, nheavy, colidx, vals, FT, r,
                                       yt_dtype, YT, part, (cudaStream_t)stream));
}

int nmfb_dense_residual_kmajor(const float *XT, int64_t m, int64_t n, const float *Gt,
                               const float *Ft, int32_t r, double *out, void *workspace,
                               void *stream) {
    return check(dense_residual_kmajor_launch(XT, m, n, Gt, Ft, r, out, workspace,
                                              (cudaStream_t)stream));
}

size_t nmfb_slice_bytes(int64_t rows, int32_t r) { return slice_bytes(rows, r); }
int nmfb_slice_u8(const float *A, int64_t rows, int32_t r, int64_t lda, void *out, void *stream) {
    return check(slice_u8_launch(A, rows, r, lda, out, (cudaStream_t)stream));
}
size_t nmfb_residual_i8_workspace_bytes(void) { return residual_i8_workspace_bytes(); }
int nmfb_residual_i8(const float *X, int64_t n, int64_t m, const void *Gsl, const void *Fsl,
                     int32_t r, double *out, void *workspace, void *stream) {
    return check(residual_i8_launch(X, n, m, Gsl, Fsl, r, out, workspace, (cudaStream_t)stream));
}

size_t nmfb_dot_workspace_bytes(int64_t len) { return dot_workspace_bytes(len); }

int nmfb_data_stats(const void *a, int a_dtype, int64_t len, double *out, void *workspace,
                    void *stream) {
    return check(data_stats_launch(a, a_dtype, len, out, workspace, (cudaStream_t)stream));
}

int nmfb_sum_parts(const float *parts, int32_t S, int64_t len, float *out, void *stream) {
    return check(sum_parts_launch(parts, S, len, out, (cudaStream_t)stream));
}

int nmfb_tc_gemm(const float *A, int64_t M, int64_t K, const float *Bt_hi, const float *Bt_lo,
                 int32_t N, float *C, int32_t splits, int32_t stages, void *stream) {
    return check(tc_gemm_launch(A, M, K, Bt_hi, Bt_lo, N, C, splits, stages,
                                (cudaStream_t)stream));
}

int nmfb_tc_gemm_rows(const float *A, int64_t M, int64_t K, const float *Bt_hi,
                      const float *Bt_lo, int32_t N, int32_t splits, float *const *dst,
                      int32_t world, int64_t chunk, int32_t src, void *stream) {
    if (!dst || world < 1 || world > NMFB_MAX_PEERS) return NMFB_ERR_ARG;
    RowOut out{};
    for (int q = 0; q < world; ++q) out.dst[q] = dst[q];
    out.world = world;
    out.src = src;
    out.chunk = chunk;
    return check(tc_gemm_rows_launch(A, M, K, Bt_hi, Bt_lo, N, out, splits, 0,
                                     (cudaStream_t)stream));
}

int nmfb_peer_put(const void *src, int64_t bytes, void *const *dst, int32_t world, int32_t rank,
                  void *const *flags, uint32_t *ticket, uint64_t epoch, int32_t signal,
                  void *stream) {
    return check(peer_put_launch(src, bytes, dst, world, rank, flags, ticket,
                                 (unsigned long long)epoch, signal, (cudaStream_t)stream));
}

int nmfb_peer_wait(uint64_t *flags, int32_t world, uint64_t epoch, double timeout_s,
                   void *stream) {
    return check(peer_wait_launch(flags, world, (unsigned long long)epoch, timeout_s,
                                  (cudaStream_t)stream));
}

int nmfb_sum_slots_f64(const double *slots, int32_t S, int64_t len, int64_t stride,
                       double *out, void *stream) {
    return check(sum_slots_f64_launch(slots, S, len, stride, out, (cudaStream_t)stream));
}

int nmfb_tc_splits(int64_t K, int32_t splits) { return tc_effective_splits(K, splits); }
int nmfb_tc_parts(int64_t M, int64_t K, int32_t N, int32_t splits) {
    return tc_parts(M, K, N, splits);
}

int nmfb_split_transpose(const float *B, int64_t K, int32_t r, float *Bt_hi, float *Bt_lo,
                         void *stream) {
    return check(split_transpose_launch(B, K, r, Bt_hi, Bt_lo, (cudaStream_t)stream));
}

int nmfb_transpose(const float *in, int64_t rows, int64_t cols, float *out, void *stream) {
    return check(transpose_launch(in, rows, cols, out, (cudaStream_t)stream));
}

int nmfb_sum_slots_rescale(int dtype, const double *slots, int32_t S, int64_t stride, double *H,
                           int32_t r, double diag_add, void *Qa, void *scale_a,
                           int32_t *act_idx, uint8_t *active, int32_t *ra_dev, void *stream) {
    return check(sum_slots_rescale_launch(dtype, slots, S, stride, H, r, diag_add, Qa, scale_a,
                                          act_idx, active, ra_dev, (cudaStream_t)stream));
}

int nmfb_csc_segments(const int64_t *indptr, const int32_t *rowidx, int64_t m, int64_t blk,
                      int32_t nblk, int64_t *seg, void *stream) {
    return check(csc_segments_launch(indptr, rowidx, m, blk, nblk, seg, (cudaStream_t)stream));
}

int nmfb_chunk_segments(const int64_t *chunks, int64_t nchunks, const int32_t *colidx,
                        int64_t blk, int32_t nblk, int64_t *seg, void *stream) {
    return check(chunk_segments_launch(chunks, nchunks, colidx, blk, nblk, seg,
                                       (cudaStream_t)stream));
}

int nmfb_csc_linear_blocked(const int64_t *indptr, const int64_t *seg, int32_t nblk,
                            const int32_t *rowidx, const float *vals, int64_t m, const float *G,
                            int32_t r, double mu1, float *h, void *stream) {
    return check(csc_linear_vec_launch(indptr, seg, nblk, rowidx, vals, 0, m, G, r, mu1, h,
                                       (cudaStream_t)stream));
}

int nmfb_csr_yt_chunked_blocked(const int64_t *chunks, int64_t nchunks, const int64_t *heavy,
                                int64_t nheavy, const int64_t *seg, int32_t nblk,
                                const int32_t *colidx, const float *vals, const float *FT,
                                int32_t r, int yt_dtype, void *YT, void *part, void *stream) {
    return check(csr_yt_chunked_vec_launch(chunks, nchunks, heavy, nheavy, seg, nblk, colidx,
                                           vals, FT, r, yt_dtype, YT, part,
                                           (cudaStream_t)stream));
}

int nmfb_init_factors(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                      int64_t n, int64_t m, int32_t r, double scale, int dtype, void *G,
                      void *FT, void *stream) {
    return check(pcg64_factors_launch(state_hi, state_lo, inc_hi, inc_lo, n, m, r, scale, dtype,
                                      G, FT, (cudaStream_t)stream));
}

int nmfb_mur_update(int dtype, const double *Q, int32_t r, const void *h, int h_dtype,
                    int32_t h_parts, int64_t h_ld, int64_t h_pstride, double h_base, void *x,
                    int64_t count, double floor_, uint64_t *stats, void *stream) {
    return check(mur_update_launch(dtype, Q, r, h, h_dtype, h_parts, h_ld, h_pstride, h_base, x,
                                   count, floor_, stats, (cudaStream_t)stream));
}

int nmfb_csc_from_triplets(int64_t rows, int64_t cols, int64_t count, const int64_t *i,
                           const int64_t *j, const double *v, int sum_duplicates,
                           int64_t *indptr, int32_t *rowidx, void *vals, int vals_dtype,
                           int64_t *nnz_out, int64_t *info, void *stream) {
    return check(csc_from_triplets_launch(rows, cols, count, i, j, v, sum_duplicates, indptr,
                                          rowidx, vals, vals_dtype, nnz_out, info,
                                          (cudaStream_t)stream));
}

int nmfb_csc_to_csr(int64_t rows, int64_t cols, int64_t nnz, const int64_t *indptr,
                    const int32_t *rowidx, const void *vals, int vals_dtype, int64_t *rowptr,
                    int32_t *colidx, void *cvals, void *stream) {
    return check(csc_to_csr_launch(rows, cols, nnz, indptr, rowidx, vals, vals_dtype, rowptr,
                                   colidx, cvals, (cudaStream_t)stream));
}

int nmfb_csc_validate(int64_t rows, int64_t cols, int64_t nnz, const int64_t *indptr,
                      const int32_t *rowidx, const void *vals, int vals_dtype, int64_t *info,
                      void *stream) {
    return check(csc_validate_launch(rows, cols, nnz, indptr, rowidx, vals, vals_dtype, info,
                                     (cudaStream_t)stream));
}

int nmfb_ingest_release_scratch(void) { return check(ingest_release_scratch()); }

int nmfb_csr_chunk_plan(const int64_t *rowptr, int64_t rows, int64_t chunk, int64_t *chunks,
                        int64_t *heavy, int64_t *counts_out, void *stream) {
    return check(csr_chunk_plan_launch(rowptr, rows, chunk, chunks, heavy, counts_out,
                                       (cudaStream_t)stream));
}

int nmfb_comm_available(void) { return comm_available(); }
int nmfb_comm_unique_id(void *id_out) { return check(comm_unique_id(id_out)); }
int nmfb_comm_init(const void *id, int32_t rank, int32_t nranks, void **comm_out) {
    return check(comm_init(id, rank, nranks, comm_out));
}
int nmfb_comm_destroy(void *comm) { return check(comm_destroy(comm)); }
int nmfb_allreduce_r2(void *comm, double *buf, int64_t count, void *stream) {
    return check(allreduce_r2(comm, buf, count, (cudaStream_t)stream));
}
int nmfb_reduce_scatter_panel(void *comm, const void *send, void *recv, int64_t recv_count,
                              int dtype, void *stream) {
    return check(reduce_scatter_panel(comm, send, recv, recv_count, dtype, (cudaStream_t)stream));
}
int nmfb_allgather_panel(void *comm, const void *send, void *recv, int64_t send_count, int dtype,
                         void *stream) {
    return check(allgather_panel(comm, send, recv, send_count, dtype, (cudaStream_t)stream));
}

int nmfb_narrow_indices(const int64_t *in, int64_t n, int32_t *out, int64_t *info,
                        void *stream) {
    return check(narrow_indices_launch(in, n, out, info, (cudaStream_t)stream));
}

int nmfb_dot(const void *a, int a_dtype, const void *b, int b_dtype, int64_t len, double *out,
             void *workspace, void *stream) {
    return check(dot_launch(a, a_dtype, b, b_dtype, len, out, workspace, (cudaStream_t)stream));
}

// ---------------------------------------------------------------------------
// Reference drop-in shard entry points (synchronous results).
// ---------------------------------------------------------------------------
struct Scratch {
    cudaStream_t st;
    std::vector<void *> ptrs;
    explicit Scratch(cudaStream_t s) : st(s) {}
    void *get(size_t bytes) {
        void *p = nullptr;
        if (cudaMallocAsync(&p, bytes ? bytes : 16, st) != cudaSuccess) return nullptr;
        ptrs.push_back(p);
        return p;
    }
    ~Scratch() {
        for (void *p : ptrs) cudaFreeAsync(p, st);
    }
};

// Finish a shard call: read stats + the last block's final norms, return the
// reference tuple (kernels.py:281/336/378: inner_total, max_stop, fail).
static int finish_shard(cudaStream_t st, int dtype, uint64_t *stats_dev, const void *finals_dev,
                        int64_t lo, int64_t hi, double max_stop0, int64_t *inner_total,
                        double *max_stop, int64_t *fail) {
    uint64_t stats[2];
    cudaError_t e = cudaMemcpyAsync(stats, stats_dev, sizeof(stats), cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_status(e);
    int64_t last_lo = (hi - 1) / 32 * 32;
    double ms = (last_lo <= lo) ? max_stop0 : 0.0;
    int64_t from = last_lo > lo ? last_lo : lo;
    std::vector<double> fin(hi - from);
    if (hi > from) {
        if (dtype == NMFB_F64) {
            e = cudaMemcpyAsync(fin.data(), (const double *)finals_dev + (from - lo),
                                sizeof(double) * (hi - from), cudaMemcpyDeviceToHost, st);
        } else {
            std::vector<float> tmp(hi - from);
            e = cudaMemcpyAsync(tmp.data(), (const float *)finals_dev + (from - lo),
                                sizeof(float) * (hi - from), cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            for (size_t k = 0; k < tmp.size(); ++k) fin[k] = tmp[k];
        }
        if (e != cudaSuccess) return cuda_status(e);
    }
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_status(e);
    for (double f : fin)
        if (f > ms) ms = f;
    *inner_total = (int64_t)stats[0];
    *max_stop = ms;
    *fail = stats[1] == ~0ull ? NMFB_FAIL_NONE : (int64_t)stats[1];
    return *fail == NMFB_FAIL_NONE ? NMFB_OK : NMFB_ERR_NUMERIC;
}

static int run_shard_nnls(int dtype, int mode, const void *Qa, const void *scale_a,
                          const int32_t *act_idx, int32_t ra, const uint8_t *active, int32_t r,
                          const void *h, int h_parts, double h_base, void *x, int64_t lo,
                          int64_t hi, double eps, int32_t max_inner, double max_stop0,
                          Scratch &s, uint64_t **stats_out, void **finals_out) {
    uint64_t *stats = (uint64_t *)s.get(2 * sizeof(uint64_t));
    void *finals = s.get(esize(dtype) * (hi - lo));
    if (!stats || !finals) return launch_status() == NMFB_OK ? NMFB_ERR_CUDA : NMFB_ERR_CUDA;
    uint64_t init[2] = {0ull, ~0ull};
    cudaMemcpyAsync(stats, init, sizeof(init), cudaMemcpyHostToDevice, s.st);
    int rc = nmfb_nnls_batch(dtype, mode, Qa, scale_a, act_idx, active, r, ra, nullptr, h, dtype,
                             h_parts, r, (hi - lo) * (int64_t)r, h_base,
                             (char *)x + esize(dtype) * lo * r, hi - lo, lo, eps, max_inner,
                             max_stop0, nullptr, finals, stats, 0, s.st);
    *stats_out = stats;
    *finals_out = finals;
    // the host copy of `init` must outlive the async copy
    cudaStreamSynchronize(s.st);
    return rc;
}

int nmfb_estep_dense(int dtype, int mode, const void *VT, int64_t m, int64_t n, int64_t col_lo,
                     int64_t col_hi, const void *G, int32_t r, const void *Qa,
                     const void *scale_a, const int32_t *act_idx, int32_t ra,
                     const uint8_t *active, double mu1, double eps, int32_t max_inner,
                     double max_stop0, void *FT, void *YT, void *HP, int64_t *inner_total,
                     double *max_stop, int64_t *fail, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (col_lo < 0 || col_hi > m || col_lo > col_hi) return NMFB_ERR_ARG;
    if (dtype == NMFB_F64 && mode == NMFB_MODE_FAST) mode = NMFB_MODE_REFERENCE;
    int64_t cols = col_hi - col_lo;
    *inner_total = 0;
    *max_stop = max_stop0;
    *fail = NMFB_FAIL_NONE;
    if (cols == 0) return NMFB_OK;
    Scratch s(st);
    void *h = s.get(esize(dtype) * cols * r);
    if (!h) return cuda_status(cudaGetLastError());
    int rc;
    int h_parts = 0;
    if (mode == NMFB_MODE_REFERENCE) {
        rc = nmfb_dense_linear_ref(dtype, VT, n, col_lo, col_hi, G, r, mu1, h, st);
    } else {
        rc = nmfb_gemm_tall((const float *)VT + col_lo * n, 1, cols, n, n, (const float *)G, r, r,
                            (float *)h, 1, st);
        h_parts = 1;
    }
    if (rc) return rc;
    uint64_t *stats;
    void *finals;
    rc = run_shard_nnls(dtype, mode, Qa, scale_a, act_idx, ra, active, r, h, h_parts, mu1, FT,
                        col_lo, col_hi, eps, max_inner, max_stop0, s, &stats, &finals);
    if (rc) return rc;
    // accumulators: YT += X[:, lo:hi] F[lo:hi]^T, HP += upper(F F^T)
    void *yt = s.get(esize(dtype) * n * r);
    void *hp = s.get(esize(dtype) * r * r);
    int64_t bounds[2] = {col_lo, col_hi};
    if (mode == NMFB_MODE_REFERENCE) {
        rc = nmfb_dense_yt_ref(dtype, VT, m, n, FT, r, bounds, 1, yt, st);
        if (!rc) rc = nmfb_hp_ref(dtype, FT, m, r, bounds, 1, hp, st);
    } else {
        rc = nmfb_gemm_tall((const float *)VT + col_lo * n, 0, n, cols, n,
                            (const float *)FT + col_lo * r, r, r, (float *)yt, 1, st);
        if (!rc) rc = nmfb_hp_ref(dtype, FT, m, r, bounds, 1, hp, st);
    }
    if (!rc) rc = check(add_into_launch(dtype, YT, yt, n * (int64_t)r, 0, st));
    if (!rc) rc = check(add_into_launch(dtype, HP, hp, (int64_t)r * r, r, st));
    if (rc) return rc;
    return finish_shard(st, dtype, stats, finals, col_lo, col_hi, max_stop0, inner_total,
                        max_stop, fail);
}

int nmfb_estep_sparse(int dtype, int mode, const int64_t *indptr, const int32_t *rowidx,
                      const void *vals, int64_t m, int64_t n, int64_t col_lo, int64_t col_hi,
                      const void *G, int32_t r, const void *Qa, const void *scale_a,
                      const int32_t *act_idx, int32_t ra, const uint8_t *active, double mu1,
                      double eps, int32_t max_inner, double max_stop0, void *FT, void *YT,
                      void *HP, int64_t *inner_total, double *max_stop, int64_t *fail,
                      void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (col_lo < 0 || col_hi > m || col_lo > col_hi) return NMFB_ERR_ARG;
    if (dtype == NMFB_F64 && mode == NMFB_MODE_FAST) mode = NMFB_MODE_REFERENCE;
    int64_t cols = col_hi - col_lo;
    *inner_total = 0;
    *max_stop = max_stop0;
    *fail = NMFB_FAIL_NONE;
    if (cols == 0) return NMFB_OK;
    Scratch s(st);
    void *h = s.get(esize(dtype) * cols * r);
    int rc = nmfb_csc_linear(dtype, mode, indptr, rowidx, vals, col_lo, col_hi, G, r, mu1, h, st);
    if (rc) return rc;
    uint64_t *stats;
    void *finals;
    rc = run_shard_nnls(dtype, mode, Qa, scale_a, act_idx, ra, active, r, h, 0, 0.0, FT, col_lo,
                        col_hi, eps, max_inner, max_stop0, s, &stats, &finals);
    if (rc) return rc;
    void *hp = s.get(esize(dtype) * r * r);
    int64_t bounds[2] = {col_lo, col_hi};
    rc = nmfb_hp_ref(dtype, FT, m, r, bounds, 1, hp, st);
    if (!rc) rc = check(add_into_launch(dtype, HP, hp, (int64_t)r * r, r, st));
    if (rc) return rc;
    // YT[row] += x_col * v over the shard's columns in column order
    // (kernels.py:270-274); fit() uses the CSR pass instead
    rc = check(csc_scatter_yt_launch(dtype, indptr, rowidx, vals, col_lo, col_hi, FT, r, YT, st));
    if (rc) return rc;
    return finish_shard(st, dtype, stats, finals, col_lo, col_hi, max_stop0, inner_total,
                        max_stop, fail);
}

int nmfb_mstep_rows(int dtype, int mode, const void *YT, int64_t row_lo, int64_t row_hi,
                    const void *Qa, const void *scale_a, const int32_t *act_idx, int32_t ra,
                    const uint8_t *active, double beta1, double eps, int32_t max_inner,
                    double max_stop0, void *G, int32_t r, int64_t *inner_total,
                    double *max_stop, int64_t *fail, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (row_lo < 0 || row_lo > row_hi) return NMFB_ERR_ARG;
    if (dtype == NMFB_F64 && mode == NMFB_MODE_FAST) mode = NMFB_MODE_REFERENCE;
    *inner_total = 0;
    *max_stop = max_stop0;
    *fail = NMFB_FAIL_NONE;
    if (row_hi == row_lo) return NMFB_OK;
    Scratch s(st);
    uint64_t *stats;
    void *finals;
    const void *h = (const char *)YT + esize(dtype) * row_lo * r;
    int rc = run_shard_nnls(dtype, mode, Qa, scale_a, act_idx, ra, active, r, h, 1, beta1, G,
                            row_lo, row_hi, eps, max_inner, max_stop0, s, &stats, &finals);
    if (rc) return rc;
    return finish_shard(st, dtype, stats, finals, row_lo, row_hi, max_stop0, inner_total,
                        max_stop, fail);
}

}  // extern "C"
