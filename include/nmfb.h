/*
 * nmfb.h -- C ABI of the B200-native alternating-NNLS hot path
 * (arXiv 1506.08938 anti-lopsided + greedy coordinate-descent NMF).
 *
 * Library: paper_1506_08938_b200/libnmfb.so (sm_100a).  Plain pointers,
 * sizes and status codes only; no torch types.  All device pointers are
 * caller-owned; every call is ordered on the given CUDA stream (`stream` is a
 * cudaStream_t passed as void*, NULL = legacy default stream).
 *
 * Reference boundary replaced (paths relative to the reference's
 * pkg/src/nmfkit/):
 *   nmfb_estep_dense   <- kernels.estep_dense   kernels.py:284-336 (called parallel.py:117-121)
 *   nmfb_estep_sparse  <- kernels.estep_sparse  kernels.py:223-281 (called parallel.py:110-114)
 *   nmfb_mstep_rows    <- kernels.mstep_rows    kernels.py:339-378 (called parallel.py:206-209)
 *   nmfb_nnls_batch    <- kernels._coefficient_solve + _solve_rescaled, batched
 *                         (kernels.py:38-220); FAIL_NONE kernels.py:27,
 *                         FASTBREAK_BLOCK kernels.py:35
 *   nmfb_gram          <- matrix.gram           matrix.py:181-197
 *   nmfb_rescale       <- nqp.rescale_arrays + parallel._rescale_for_step
 *                         (nqp.py:116-131, parallel.py:87-91; H = Q + 2*lambda*I at
 *                         parallel.py:104,196)
 *   nmfb_gemm_tall     <- the data products G^T X / X F^T of kernels.py:251-258,
 *                         270-274, 306-313, 325-329 (dense)
 *   nmfb_csc_linear / nmfb_csr_yt <- the same products for CSC data (sparse)
 *   nmfb_dense_residual, nmfb_dot, nmfb_objective
 *                      <- matrix.frobenius_objective / nmf.regularized_objective
 *                         (matrix.py:227-260, nmf.py:152-165)
 *
 * Status codes: NMFB_OK; NMFB_ERR_NUMERIC (a subproblem produced NaN/Inf or
 * has an unbounded frozen dimension; *fail_index = lowest failing global
 * index, the reference's returned fail column/row); NMFB_ERR_ARG;
 * NMFB_ERR_CUDA (see nmfb_last_error()); NMFB_ERR_DEGENERATE (every diagonal
 * frozen; single-problem solve only, nqp.py:137-141).
 */
#ifndef NMFB_H
#define NMFB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NMFB_OK 0
#define NMFB_ERR_NUMERIC 1
#define NMFB_ERR_ARG 2
#define NMFB_ERR_CUDA 3
#define NMFB_ERR_DEGENERATE 4

#define NMFB_F32 0
#define NMFB_F64 1

/* NMFB_MODE_REFERENCE: thread-per-problem kernels in the reference's exact
 * operation order, no FMA contraction -- bit-identical to the reference in
 * fp64.  NMFB_MODE_FAST: register-resident warp-group kernels (fp32). */
#define NMFB_MODE_FAST 0
#define NMFB_MODE_REFERENCE 1

/* largest world size of the peer-memory (NVLink) exchange entry points */
#define NMFB_MAX_PEERS 8

#define NMFB_FAIL_NONE (-1)      /* kernels.py:27 */
#define NMFB_FASTBREAK_BLOCK 32  /* kernels.py:35 */
#define NMFB_MAX_WORKERS 64

int nmfb_version(void);
const char *nmfb_last_error(void);
int nmfb_device_sm_count(void);

/* ---------------- reference drop-in shard entry points -------------------
 * Same arguments and meaning as the numba kernels, on device buffers:
 *   VT (m, n) C-order, G (n, r), FT (m, r), YT (n, r), HP (r, r) upper
 *   triangle accumulated (caller mirrors), Qa (ra, ra), scale_a (ra),
 *   act_idx (ra, int32), active (r, uint8).  dtype of every real array =
 *   `dtype`.  Solutions overwrite FT / G rows [lo, hi); YT/HP accumulate.
 * Synchronous: the stream is synchronized before returning the reference's
 * result tuple (inner_total, max_stop, fail) through host pointers.
 * Returns NMFB_OK or NMFB_ERR_NUMERIC (then *fail = failing column/row). */
int nmfb_estep_dense(int dtype, int mode, const void *VT, int64_t m, int64_t n, int64_t col_lo,
                     int64_t col_hi, const void *G, int32_t r, const void *Qa,
                     const void *scale_a, const int32_t *act_idx, int32_t ra,
                     const uint8_t *active, double mu1, double eps, int32_t max_inner,
                     double max_stop0, void *FT, void *YT, void *HP, int64_t *inner_total,
                     double *max_stop, int64_t *fail, void *stream);

int nmfb_estep_sparse(int dtype, int mode, const int64_t *indptr, const int32_t *rowidx,
                      const void *vals, int64_t m, int64_t n, int64_t col_lo, int64_t col_hi,
                      const void *G, int32_t r, const void *Qa, const void *scale_a,
                      const int32_t *act_idx, int32_t ra, const uint8_t *active, double mu1,
                      double eps, int32_t max_inner, double max_stop0, void *FT, void *YT,
                      void *HP, int64_t *inner_total, double *max_stop, int64_t *fail,
                      void *stream);

int nmfb_mstep_rows(int dtype, int mode, const void *YT, int64_t row_lo, int64_t row_hi,
                    const void *Qa, const void *scale_a, const int32_t *act_idx, int32_t ra,
                    const uint8_t *active, double beta1, double eps, int32_t max_inner,
                    double max_stop0, void *G, int32_t r, int64_t *inner_total,
                    double *max_stop, int64_t *fail, void *stream);

/* ---------------- stream-ordered building blocks (async) ---------------- */

/* Batched NNLS over `count` problems with global indices index_base..+count
 * (fast-break blocks are the 32-aligned runs of global indices; the first
 * partial block starts from max_stop0, kernels.py:245-248).
 * Linear terms: h_parts == 0 -> h (count, h_ld) is h itself; else
 * h = h_base - sum_{s < h_parts} h[s * h_pstride + j * h_ld + i] (the data
 * products as split-K partials; h_parts == 1 is the reference's
 * beta1 - YT[row], kernels.py:365).  h_dtype may be F64 with dtype F32.
 * ra_dev (nullable): device int32 ra written by nmfb_rescale; when given,
 * Qa is read with leading dimension ra and `ra` is ignored.
 * stats (device, 2 x uint64): [0] += total inner iterations,
 * [1] = min(stats[1], lowest failing global index) -- initialise [1] to
 * UINT64_MAX.  iters_out / final_out (device, nullable): per-problem
 * iteration count (-1 = failed) and final squared passive-gradient norm.
 * lanes: lanes per problem for the fast kernel (0 = auto; 1,2,4,8). */
int nmfb_nnls_batch(int dtype, int mode, const void *Qa, const void *scale_a,
                    const int32_t *act_idx, const uint8_t *active, int32_t r, int32_t ra,
                    const int32_t *ra_dev, const void *h, int h_dtype, int32_t h_parts,
                    int64_t h_ld, int64_t h_pstride, double h_base, void *x, int64_t count,
                    int64_t index_base, double eps, int32_t max_inner, double max_stop0,
                    int32_t *iters_out, void *final_out, uint64_t *stats, int32_t lanes,
                    void *stream);

/* Public single-problem NQP solve (nqp.solve, nqp.py:217-320) for `count`
 * problems sharing one rescaled Hessian but each with its OWN stop state
 * (threshold max_stop, no fast-break sharing), fp64, reference order.
 * hist (nullable, count x hist_ld x 2 doubles): per-iteration squared
 * passive-gradient norm and rescaled objective, entry 0 = initial.
 * check_gradients != 0: every iteration compares the incremental gradient
 * with a fresh Q y + q (nqp.py:295-299); a drift beyond 1e-9 max(1, |fresh|)
 * stops that problem with iters_out = -2. */
int nmfb_nqp_solve(const double *Qa, const double *scale_a, const int32_t *act_idx,
                   const uint8_t *active, int32_t r, const int32_t *ra_dev, const double *h,
                   double *x, int64_t count, double eps, int32_t max_inner, double max_stop,
                   int32_t *iters_out, double *final_out, double *hist, int32_t hist_ld,
                   int32_t check_gradients, uint64_t *stats, void *stream);

/* One step of the public NQP building blocks on `count` problems sharing a
 * unit-diagonal Q (r x r fp64, row-major); x, grad (count x r) in, x_out,
 * grad_out out (may alias x / grad).  fp64, one thread per problem.
 *   NMFB_NQP_LINE_SEARCH: nqp.exact_line_search_step (nqp.py:151-183)
 *   NMFB_NQP_GREEDY_CD:   nqp.greedy_cd_pass with `sweeps` updates
 *                         (nqp.py:186-209; sweeps < 0 = r). */
#define NMFB_NQP_LINE_SEARCH 0
#define NMFB_NQP_GREEDY_CD 1
int nmfb_nqp_step(int32_t op, const double *Q, int32_t r, const double *x, const double *grad,
                  int64_t count, int32_t sweeps, double *x_out, double *grad_out, void *stream);

/* Gram A^T A of A (rows, r) row-major (leading dim lda) with a fixed
 * (deterministic) summation order; out = full symmetric r x r fp64.
 *   NMFB_F64: accumulated in fp64 (within 1e-14 of the BLAS Gram, matrix.py:181-197).
 *   NMFB_F32: r % 4 == 0, 16 <= r <= 224, lda % 4 == 0, >= 2048 rows and a 16-byte
 *     aligned A take the tcgen05 path (3xTF32 products, 64-row chunks folded
 *     into round-to-nearest running sums, fp64 partials; within 1e-6 of the
 *     exact Gram of the fp32 values); anything else sums 32-row fp32 slabs into
 *     fp64 on the CUDA cores.  NMFB_GRAM_TC=0 in the environment forces the latter.
 * workspace: nmfb_gram_workspace_bytes(rows, r) bytes of device memory. */
size_t nmfb_gram_workspace_bytes(int64_t rows, int32_t r);
/* Gram with the anti-lopsided rescale fused into its epilogue: out = A^T A
 * (as nmfb_gram), then Qa / scale_a / act_idx / active / ra_dev exactly as
 * nmfb_rescale(dtype, out, r, diag_add, ...) would write them -- one stream-
 * ordered pass, the last reducing CTA runs the rescale. */
int nmfb_gram_rescale(int dtype, const void *A, int64_t rows, int32_t r, int64_t lda, double *out,
                      void *workspace, double diag_add, void *Qa, void *scale_a, int32_t *act_idx,
                      uint8_t *active, int32_t *ra_dev, void *stream);
int nmfb_gram(int dtype, const void *A, int64_t rows, int32_t r, int64_t lda, double *out,
              void *workspace, void *stream);

/* H = G + diag_add * I (G r x r fp64), then the anti-lopsided unit-diagonal
 * rescale: active = diag > 1e-12 * max diag; scale = sqrt(diag);
 * Q = H / outer(scale, scale) over active dims.  Writes the compact Qa
 * (ra x ra, dtype), scale_a (ra, dtype), act_idx (ra), active (r) and the
 * device scalar ra_dev.  Bit-exact against nqp.rescale_arrays in fp64.
 * full_scale (nullable, r doubles): sqrt(diag) for every dim. */
int nmfb_rescale(int dtype, const double *G, int32_t r, double diag_add, void *Qa,
                 void *scale_a, int32_t *act_idx, uint8_t *active, int32_t *ra_dev,
                 double *full_scale, void *stream);

/* Split-K tall-skinny GEMM, fp32: C[s] (M x N, row-major, ld N) =
 * A(M x K) B(K x N) over the s-th K chunk, s < splits.  A(i, k) =
 * A[i*lda + k] if a_kmajor else A[k*lda + i]; B (K x N) row-major, ld ldb.
 * C must hold splits*M*N floats.  Deterministic. */
int nmfb_gemm_tall(const float *A, int a_kmajor, int64_t M, int64_t K, int64_t lda,
                   const float *B, int32_t N, int64_t ldb, float *C, int32_t splits,
                   void *stream);

/* Tensor-core (tcgen05, kind::tf32, 3xTF32 split) split-K GEMM:
 * C[s] (M x N row-major) = A(M x K, K contiguous) * Bt(N x K, K contiguous)^T
 * over the s-th K part, so sum_s C[s] = A Bt^T.  Bt_lo = Bt - tf32(Bt)
 * (nmfb_split_transpose makes both from a K x N row-major B).  K % 4 == 0,
 * N <= 160, 16-byte aligned pointers.  splits > 0: fixed K chunks;
 * splits <= 0: balanced schedule (every SM gets an equal run of 128 x 32
 * k-blocks; a tile's parts are the runs that cover it, unused parts zeroed).
 * C must hold nmfb_tc_parts(M, K, N, splits) * M * N floats.  stages: smem
 * pipeline depth (0 = auto).  Deterministic for a given device. */
int nmfb_tc_gemm(const float *A, int64_t M, int64_t K, const float *Bt_hi, const float *Bt_lo,
                 int32_t N, float *C, int32_t splits, int32_t stages, void *stream);
int nmfb_tc_parts(int64_t M, int64_t K, int32_t N, int32_t splits);
/* fixed-chunk count for splits > 0 (= nmfb_tc_parts for that case) */
int nmfb_tc_splits(int64_t K, int32_t splits);
/* B (K x r row-major) -> Bt_hi = B^T (r x K), Bt_lo = B^T - tf32(B^T). */
int nmfb_split_transpose(const float *B, int64_t K, int32_t r, float *Bt_hi, float *Bt_lo,
                         void *stream);
/* out (cols x rows) = in (rows x cols)^T, fp32. */
int nmfb_transpose(const float *in, int64_t rows, int64_t cols, float *out, void *stream);

/* Reference-order dense products (check mode), dtype F64 or F32:
 * h[col - col_lo][i] = mu1 - sum_{row, v != 0} G[row][i] * v, v = VT[col][row]
 * (kernels.py:306-313).  Cols [col_lo, col_hi). */
int nmfb_dense_linear_ref(int dtype, const void *VT, int64_t n, int64_t col_lo, int64_t col_hi,
                          const void *G, int32_t r, double mu1, void *h, void *stream);
/* YT[row][i] = sum_w ( sum_{col in shard w} x[col][i] * v ) with per-worker
 * partials summed in worker order (kernels.py:325-329 + parallel.py:150-156).
 * shard_bounds: host array of workers+1 ascending column bounds. */
int nmfb_dense_yt_ref(int dtype, const void *VT, int64_t m, int64_t n, const void *FT,
                      int32_t r, const int64_t *shard_bounds, int32_t workers, void *YT,
                      void *stream);
/* H_f[a][b] = sum_w sum_{col in shard w, x_a != 0} x_a x_b, mirrored
 * (kernels.py:276-280 / 331-335 + parallel.py:127-128, 150-156). */
int nmfb_hp_ref(int dtype, const void *FT, int64_t m, int32_t r, const int64_t *shard_bounds,
                int32_t workers, void *HF, void *stream);

/* Sparse products.  CSC (indptr int64 m+1, rowidx int32, vals):
 * h[col - col_lo][i] = mu1 - sum_t G[rowidx[t]][i] * vals[t]  (kernels.py:251-258)
 * mode REFERENCE: exact sequential order.  CSR of the same matrix (rowptr
 * int64 n+1, colidx int32 ascending per row, vals):
 * YT[row][i] = sum over the row's entries x[col][i] * v, accumulated in
 * YT's dtype (yt_dtype F64 for the trace-identity objective); REFERENCE mode
 * emulates the per-worker partial sums of shard_bounds (kernels.py:270-274). */
int nmfb_csc_linear(int dtype, int mode, const int64_t *indptr, const int32_t *rowidx,
                    const void *vals, int64_t col_lo, int64_t col_hi, const void *G, int32_t r,
                    double mu1, void *h, void *stream);
int nmfb_csr_yt(int dtype, int mode, const int64_t *rowptr, const int32_t *colidx,
                const void *vals, int64_t n, const void *FT, int32_t r, int yt_dtype,
                const int64_t *shard_bounds, int32_t workers, void *YT, void *stream);

/* Load-balanced production form of the Y^T pass (fast mode): rows cut into
 * chunks of bounded length (a plan built once per matrix, see
 * paper_1506_08938_b200/device.py csr_chunk_plan).  chunks: int64
 * [nchunks][4] = (row, lo, hi, slot) with slot -1 for single-chunk rows;
 * heavy: int64 [nheavy][3] = (row, first slot, count); part: workspace of
 * (total slots) x r doubles (the fp32 production form accumulates every row
 * in fp64 and rounds Y^T once; yt_dtype is the output type).  Deterministic. */
int nmfb_csr_yt_chunked(int dtype, const int64_t *chunks, int64_t nchunks, const int64_t *heavy,
                        int64_t nheavy, const int32_t *colidx, const void *vals, const void *FT,
                        int32_t r, int yt_dtype, void *YT, void *part, void *stream);

/* Dense residual 0.5 * ||X - G F||^2 with X given as XT (m, n) row-major,
 * G (n, r), FT (m, r); fp64 accumulation; result added to *out (device
 * double) deterministically.  workspace: nmfb_residual_workspace_bytes. */
size_t nmfb_residual_workspace_bytes(int64_t m, int64_t n);
int nmfb_dense_residual(int dtype, const void *XT, int64_t m, int64_t n, const void *G,
                        const void *FT, int32_t r, double *out, void *workspace, void *stream);

/* fp32 production form: the same residual from the k-major operand copies the
 * tensor-core passes keep, Gt = G^T (r x n) and Ft = F (r x m); XT (m x n). */
int nmfb_dense_residual_kmajor(const float *XT, int64_t m, int64_t n, const float *Gt,
                               const float *Ft, int32_t r, double *out, void *workspace,
                               void *stream);

/* Exact-product residual on the int8 tensor cores (G, F >= 0).  Per iteration
 * the factors are cut into three 8-bit slices with a power-of-two scale per
 * row: nmfb_slice_u8(A rows x r, lda) writes nmfb_slice_bytes(rows, r) bytes
 * (3 x rows x KB u8 slices, KB = 64 if r <= 64 else 128, then rows float
 * scales); r <= 128.
 * nmfb_residual_i8 adds 0.5 ||X - G F||^2 to *out (device double) with
 * X (n x m) row-major, m % 4 == 0, Gsl = slices of G (n x r), Fsl = slices of
 * F^T (m x r).  G F is exact up to the 2^-24 slicing; X - G F is formed and
 * squared in fp32 (round-to-nearest), summed in fp64, deterministically. */
size_t nmfb_slice_bytes(int64_t rows, int32_t r);
int nmfb_slice_u8(const float *A, int64_t rows, int32_t r, int64_t lda, void *out, void *stream);
size_t nmfb_residual_i8_workspace_bytes(void);
int nmfb_residual_i8(const float *X, int64_t n, int64_t m, const void *Gsl, const void *Fsl,
                     int32_t r, double *out, void *workspace, void *stream);

/* out[i] = sum_{s < S} parts[s * len + i], fixed order (split-K partials of
 * X F^T summed before the multi-GPU reduce-scatter).  float32. */
int nmfb_sum_parts(const float *parts, int32_t S, int64_t len, float *out, void *stream);

/* ---- multi-GPU exchange over NVLink peer memory -----------------
 * Replaces, for the column-sharded fit, the reference's process-level
 * ordered reduce of the worker accumulators (parallel.reduce,
 * parallel.py:141-159) and the shard fan-out of run_estep / run_mstep
 * (parallel.py:94-133, 189-223): the data-product partials and solved rows
 * move by peer stores issued from inside the producing kernels.  dst / flags
 * / mirror are host arrays of `world` device pointers (peer mappings of
 * symmetric buffers, e.g. torch symmetric memory); world <= NMFB_MAX_PEERS.
 *
 * nmfb_tc_gemm_rows: nmfb_tc_gemm whose partial slot s of row i is stored at
 *   dst[o] + ((src * P + s) * chunk + i - o * chunk) * N, o = i / chunk,
 *   P = nmfb_tc_parts(M, K, N, splits): owner o's receive buffer holds
 *   world * P slots of (chunk x N) -- sum them in order (nmfb_nnls_batch with
 *   h_parts = world * P, h_pstride = chunk * N).  world = 1, chunk = M is
 *   nmfb_tc_gemm.  Requires chunk * world >= M.
 * nmfb_nnls_batch_peers: nmfb_nnls_batch (fast mode) that also stores every
 *   solution row j at mirror[q] + j * r (q < nmirror): the all-gather of the
 *   solved rows fused into the solve.
 * nmfb_peer_put: copy `bytes` (8-byte multiple) from src to dst[q] for every
 *   q < world (src NULL: no copy); if signal, then store epoch into
 *   flags[q][rank] for every q (release, system scope) once all of it is done.
 *   ticket: a zero-initialised device word private to this rank.
 * nmfb_peer_wait: wait until flags[q] >= epoch for all q < world (acquire,
 *   system scope); after timeout_s the wait gives up and records epoch in
 *   flags[world] (the caller checks it) instead of hanging the device.
 * nmfb_sum_slots_f64: out[i] = sum_{s<S} slots[s * stride + i] in order. */
int nmfb_tc_gemm_rows(const float *A, int64_t M, int64_t K, const float *Bt_hi,
                      const float *Bt_lo, int32_t N, int32_t splits, float *const *dst,
                      int32_t world, int64_t chunk, int32_t src, void *stream);
int nmfb_nnls_batch_peers(int dtype, int mode, const void *Qa, const void *scale_a,
                          const int32_t *act_idx, const uint8_t *active, int32_t r, int32_t ra,
                          const int32_t *ra_dev, const void *h, int h_dtype, int32_t h_parts,
                          int64_t h_ld, int64_t h_pstride, double h_base, void *x,
                          int64_t count, int64_t index_base, double eps, int32_t max_inner,
                          double max_stop0, int32_t *iters_out, void *final_out,
                          uint64_t *stats, int32_t lanes, void *const *mirror, int32_t nmirror,
                          void *stream);
int nmfb_peer_put(const void *src, int64_t bytes, void *const *dst, int32_t world, int32_t rank,
                  void *const *flags, uint32_t *ticket, uint64_t epoch, int32_t signal,
                  void *stream);
int nmfb_peer_wait(uint64_t *flags, int32_t world, uint64_t epoch, double timeout_s,
                   void *stream);
int nmfb_sum_slots_f64(const double *slots, int32_t S, int64_t len, int64_t stride,
                       double *out, void *stream);

/* out[0] = sum a_i * b_i, out[1] = sum |a_i|, out[2] = sum a_i^2 (fp64,
 * deterministic).  b may be NULL (then out[0] = 0).  a_dtype / b_dtype. */
size_t nmfb_dot_workspace_bytes(int64_t len);
/* Data-matrix check in one pass: out[0] = number of entries that are negative
 * or not finite, out[1] = sum |a|, out[2] = sum a^2 (fp64, deterministic);
 * workspace: nmfb_dot_workspace_bytes. */
int nmfb_data_stats(const void *a, int a_dtype, int64_t len, double *out, void *workspace,
                    void *stream);
int nmfb_dot(const void *a, int a_dtype, const void *b, int b_dtype, int64_t len, double *out,
             void *workspace, void *stream);

/* ---------------- sparse ingest on the device ----------------------------
 * SparseMatrix.from_triplets (matrix.py:104-125), transpose (matrix.py:149-154)
 * and _validate + require_nonnegative (matrix.py:81-101,169-178) on device
 * buffers.  Stream-ordered; scratch from the stream's memory pool.
 * info (device, NMFB_INGEST_CODES int64): info[c] = lowest offending
 * triplet / column / position of check c, INT64_MAX when the check passed. */
#define NMFB_INGEST_TRIPLET_RANGE 0 /* "triplet index out of range" */
#define NMFB_INGEST_INDPTR_SPAN 1   /* "column pointers must span [0, nnz]" */
#define NMFB_INGEST_INDPTR_ORDER 2  /* "column pointers must be non-decreasing" */
#define NMFB_INGEST_ROW_RANGE 3     /* "row index out of range" */
#define NMFB_INGEST_ROW_ORDER 4     /* "row indices not strictly increasing in column j" */
#define NMFB_INGEST_NONFINITE 5     /* "sparse values must be finite" */
#define NMFB_INGEST_NONPOSITIVE 6   /* "stored sparse values must be > 0" */
#define NMFB_INGEST_CODES 7

/* CSC from `count` triplets (i, j int64, v fp64): stable order by (col, row),
 * duplicates summed in input order when sum_duplicates (fp64, bit-identical
 * to np.add.at), zeros dropped.  Outputs: indptr (cols+1 int64), rowidx /
 * vals (capacity count; vals in vals_dtype), *nnz_out (device int64).
 * Requires rows < 2^31, count < 2^32. */
int nmfb_csc_from_triplets(int64_t rows, int64_t cols, int64_t count, const int64_t *i,
                           const int64_t *j, const double *v, int sum_duplicates,
                           int64_t *indptr, int32_t *rowidx, void *vals, int vals_dtype,
                           int64_t *nnz_out, int64_t *info, void *stream);

/* CSR of a CSC matrix (= CSC of its transpose): rowptr (rows+1 int64),
 * colidx ascending within each row, values permuted alongside. */
int nmfb_csc_to_csr(int64_t rows, int64_t cols, int64_t nnz, const int64_t *indptr,
                    const int32_t *rowidx, const void *vals, int vals_dtype, int64_t *rowptr,
                    int32_t *colidx, void *cvals, void *stream);

/* CSC invariants + finite / strictly positive values -> info. */
int nmfb_csc_validate(int64_t rows, int64_t cols, int64_t nnz, const int64_t *indptr,
                      const int32_t *rowidx, const void *vals, int vals_dtype, int64_t *info,
                      void *stream);

/* Collectives of the multi-GPU layouts (NCCL over
 * NVLink, resolved at run time from libnccl.so.2 -- the NCCL a PyTorch process
 * already holds).  The reference has no transport ("one would slot in",
 * parallel.py:9-12); these are the exchanges of paper_1506_08938_b200/
 * dist_rows.py's row-sharded layout.
 *   nmfb_comm_available      1 if NCCL could be resolved
 *   nmfb_comm_unique_id      128-byte id (rank 0 creates, every rank passes it)
 *   nmfb_comm_init           one communicator per rank (collective)
 *   nmfb_allreduce_r2        in-place fp64 sum (r x r Grams, objective pieces)
 *   nmfb_reduce_scatter_panel   sum of world panels of world*recv_count
 *                               elements, block g -> rank g (fp32 / fp64)
 *   nmfb_allgather_panel     send_count elements per rank -> every rank
 * Stream-ordered on `stream`. */
int nmfb_comm_available(void);
int nmfb_comm_unique_id(void *id_out);
int nmfb_comm_init(const void *id, int32_t rank, int32_t nranks, void **comm_out);
int nmfb_comm_destroy(void *comm);
int nmfb_allreduce_r2(void *comm, double *buf, int64_t count, void *stream);
int nmfb_reduce_scatter_panel(void *comm, const void *send, void *recv, int64_t recv_count,
                              int dtype, void *stream);
int nmfb_allgather_panel(void *comm, const void *send, void *recv, int64_t send_count, int dtype,
                         void *stream);

/* Row-chunk plan of the load-balanced Y^T pass, built on the device from
 * the CSR row pointer: row i with k nonzeros -> max(1, ceil(k / chunk))
 * chunks [4 x int64: row, lo, hi, slot] in row order (slot -1 for single-chunk
 * rows, else the heavy rows' partial slots numbered consecutively); heavy
 * rows [3 x int64: row, first slot, count].  Capacities: chunks rows + nnz /
 * chunk + 1 entries, heavy rows entries.  counts_out (HOST int64[3]): number
 * of chunks, heavy rows, slots (synchronises the stream). */
int nmfb_csr_chunk_plan(const int64_t *rowptr, int64_t rows, int64_t chunk, int64_t *chunks,
                        int64_t *heavy, int64_t *counts_out, void *stream);

/* Return the ingest kernels' cached scratch (a private stream-ordered pool on
 * the current device, kept mapped between ingests) to the driver.  Waits for
 * the device. */
int nmfb_ingest_release_scratch(void);

/* int64 -> int32 index narrowing (info[NMFB_INGEST_ROW_RANGE] = first
 * element that does not fit). */
int nmfb_narrow_indices(const int64_t *in, int64_t n, int32_t *out, int64_t *info,
                        void *stream);

/* ---------------- multiplicative-update baseline (baselines.py:41-85) ----
 * In place, per problem row x (count x r, dtype):
 *   x_i <- x_i * (num_i / (sum_k Q[i][k] x_k + floor)),  num = -h,
 * Q the raw fp64 Gram (r x r) and h in nmfb_nnls_batch's linear-term
 * convention (h_parts partials summed and subtracted from h_base; pass
 * h_base = 0 so num is the data product G^T V or V F^T).
 * stats (nullable, device uint64): [0] += count (one update per subproblem,
 * the reference's k_bar = 1 convention). */
int nmfb_mur_update(int dtype, const double *Q, int32_t r, const void *h, int h_dtype,
                    int32_t h_parts, int64_t h_ld, int64_t h_pstride, double h_base, void *x,
                    int64_t count, double floor_, uint64_t *stats, void *stream);

/* ---------------- seeded initial factors (nmf.py:115-127) ---------------
 * numpy default_rng(seed) PCG64 stream regenerated on the device, bit-identical
 * to the host draw: G (n x r, row-major) = U * scale drawn first, then
 * F (r x m, C-order) = U * scale written transposed into FT (m x r).
 * (state, inc) = np.random.PCG64(seed).state (128-bit, split hi/lo). */
int nmfb_init_factors(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                      int64_t n, int64_t m, int32_t r, double scale, int dtype, void *G,
                      void *FT, void *stream);

/* ---------------- L2-blocked sparse data products (fp32, r % 4 == 0) -----
 * The gathered factor's rows (G for G^T X, F^T for X F^T) are cut into nblk
 * blocks of blk rows; pass b only walks the entries that gather from block b,
 * so the block stays L2-resident.  seg ((outputs) x (nblk + 1) int64) holds
 * each output's sub-range per block, built once per matrix by
 * nmfb_csc_segments (CSC columns, row blocks) / nmfb_chunk_segments (CSR row
 * chunks, column blocks).  Results are bit-identical to the unblocked
 * kernels (the running sums are carried through the output in its own type).
 * The linear term covers all m columns (h = mu1 - G^T X, h (m x r)). */
int nmfb_csc_segments(const int64_t *indptr, const int32_t *rowidx, int64_t m, int64_t blk,
                      int32_t nblk, int64_t *seg, void *stream);
int nmfb_chunk_segments(const int64_t *chunks, int64_t nchunks, const int32_t *colidx,
                        int64_t blk, int32_t nblk, int64_t *seg, void *stream);
int nmfb_csc_linear_blocked(const int64_t *indptr, const int64_t *seg, int32_t nblk,
                            const int32_t *rowidx, const float *vals, int64_t m, const float *G,
                            int32_t r, double mu1, float *h, void *stream);
int nmfb_csr_yt_chunked_blocked(const int64_t *chunks, int64_t nchunks, const int64_t *heavy,
                                int64_t nheavy, const int64_t *seg, int32_t nblk,
                                const int32_t *colidx, const float *vals, const float *FT,
                                int32_t r, int yt_dtype, void *YT, void *part, void *stream);

/* Multi-GPU H_f: out H = sum over S per-source r x r slots (slot order,
 * slot s at slots + s * stride), then nmfb_rescale(H, diag_add, ...) -- one
 * launch (the peer-memory path's replacement for an allreduce + rescale). */
int nmfb_sum_slots_rescale(int dtype, const double *slots, int32_t S, int64_t stride, double *H,
                           int32_t r, double diag_add, void *Qa, void *scale_a,
                           int32_t *act_idx, uint8_t *active, int32_t *ra_dev, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* NMFB_H */
