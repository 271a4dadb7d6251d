// Sparse ingest on the device: CSC construction from coordinate triplets,
// the CSC -> CSR transpose the Y^T pass reads, and the CSC invariant checks.
//
// Reference (host numpy) behaviour restated here:
//   SparseMatrix.from_triplets  matrix.py:104-125  stable lexsort by (col, row),
//       duplicates summed in their input order (np.unique + np.add.at from
//       0.0), explicit zeros dropped after summing, indptr by counting;
//   SparseMatrix.transpose      matrix.py:149-154  (CSR of X = CSC of X^T:
//       rows ascending, columns ascending within a row);
//   SparseMatrix._validate      matrix.py:81-101 and require_nonnegative
//       matrix.py:169-178.
// Integer work is exact; the fp64 duplicate sums are sequential per run in
// the stable order, so the values are bit-identical to np.add.at.
//
// Sorting uses the CUDA toolkit's CUB radix sort (stable LSD) -- a library
// primitive like cuBLAS for a plain GEMM; ingest is not on the per-iteration
// path.  Everything else is hand-written.  Scratch comes from the stream's
// memory pool (cudaMallocAsync), so the entry points need no workspace.
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "nmfb_internal.h"

namespace nmfb {

namespace {

constexpr int TB = 256;

inline unsigned grid_for(int64_t n) {
    int64_t g = (n + TB - 1) / TB;
    return (unsigned)(g < 1 ? 1 : (g > (1 << 30) ? (1 << 30) : g));
}

int key_bits(uint64_t maxval) {
    int b = 1;
    while (b < 64 && (maxval >> b) != 0) ++b;
    return b;
}

// info[c] = min index failing check c (INT64_MAX when none)
__device__ __forceinline__ void flag(int64_t *info, int code, int64_t where) {
    atomicMin((unsigned long long *)&info[code], (unsigned long long)where);
}

__global__ void triplet_keys_kernel(int64_t rows, int64_t cols, int64_t count,
                                    const int64_t *__restrict__ i, const int64_t *__restrict__ j,
                                    uint64_t *__restrict__ key, uint32_t *__restrict__ pos,
                                    int64_t *info) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = i[t], b = j[t];
        if (a < 0 || a >= rows || b < 0 || b >= cols) {
            flag(info, NMFB_INGEST_TRIPLET_RANGE, t);
            key[t] = 0;
        } else {
            key[t] = (uint64_t)b * (uint64_t)rows + (uint64_t)a;
        }
        pos[t] = (uint32_t)t;
    }
}

__global__ void run_heads_kernel(int64_t count, const uint64_t *__restrict__ key, int sum_dup,
                                 uint32_t *__restrict__ head) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
         t += (int64_t)gridDim.x * blockDim.x)
        head[t] = (!sum_dup || t == 0 || key[t] != key[t - 1]) ? 1u : 0u;
}

// one thread per run: the run's values summed from 0.0 in the stable order
// (np.add.at), then the zero test of matrix.py:120
__global__ void run_sums_kernel(int64_t count, const uint64_t *__restrict__ key,
                                const uint32_t *__restrict__ pos, const double *__restrict__ v,
                                const uint32_t *__restrict__ head,
                                const uint32_t *__restrict__ head_at, uint64_t *__restrict__ ukey,
                                double *__restrict__ usum, uint32_t *__restrict__ keep) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
         t += (int64_t)gridDim.x * blockDim.x) {
        if (!head[t]) continue;
        double s = 0.0;
        int64_t e = t;
        do {
            s = __dadd_rn(s, v[pos[e]]);
            ++e;
        } while (e < count && !head[e]);
        const uint32_t u = head_at[t];
        ukey[u] = key[t];
        usum[u] = s;
        keep[u] = (s != 0.0) ? 1u : 0u;
    }
}

template <typename TV>
__global__ void compact_csc_kernel(int64_t nuniq, int64_t rows, const uint64_t *__restrict__ ukey,
                                   const double *__restrict__ usum,
                                   const uint32_t *__restrict__ keep,
                                   const uint32_t *__restrict__ keep_at,
                                   int32_t *__restrict__ rowidx, TV *__restrict__ vals,
                                   int64_t *__restrict__ colcount) {
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nuniq;
         u += (int64_t)gridDim.x * blockDim.x) {
        if (!keep[u]) continue;
        const uint64_t k = ukey[u];
        const int64_t col = (int64_t)(k / (uint64_t)rows);
        const uint32_t o = keep_at[u];
        rowidx[o] = (int32_t)(k - (uint64_t)col * (uint64_t)rows);
        vals[o] = (TV)usum[u];
        atomicAdd((unsigned long long *)&colcount[col + 1], 1ull);
    }
}

__global__ void last_total_kernel(const uint32_t *__restrict__ flag_, const uint32_t *__restrict__ at,
                                  int64_t n, int64_t *__restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0)
        *out = n > 0 ? (int64_t)at[n - 1] + (int64_t)flag_[n - 1] : 0;
}

// column of every CSC position (one warp per column)
__global__ void col_of_kernel(int64_t cols, const int64_t *__restrict__ indptr,
                              uint32_t *__restrict__ col_of) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int64_t c = w; c < cols; c += ((int64_t)gridDim.x * blockDim.x) >> 5)
        for (int64_t p = indptr[c] + lane; p < indptr[c + 1]; p += 32) col_of[p] = (uint32_t)c;
}

__global__ void row_keys_kernel(int64_t nnz, const int32_t *__restrict__ rowidx,
                                uint32_t *__restrict__ key, uint32_t *__restrict__ pos,
                                int64_t *__restrict__ rowcount) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nnz;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t rr = rowidx[t];
        key[t] = (uint32_t)rr;
        pos[t] = (uint32_t)t;
        atomicAdd((unsigned long long *)&rowcount[rr + 1], 1ull);
    }
}

template <typename TV>
__global__ void gather_csr_kernel(int64_t nnz, const uint32_t *__restrict__ perm,
                                  const uint32_t *__restrict__ col_of,
                                  const TV *__restrict__ vals, int32_t *__restrict__ colidx,
                                  TV *__restrict__ cvals) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nnz;
         t += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t p = perm[t];
        colidx[t] = (int32_t)col_of[p];
        cvals[t] = vals[p];
    }
}

// matrix.py:81-101 + require_nonnegative: every failing check records the
// lowest offending column / position
template <typename TV>
__global__ void validate_kernel(int64_t rows, int64_t cols, int64_t nnz,
                                const int64_t *__restrict__ indptr,
                                const int32_t *__restrict__ rowidx, const TV *__restrict__ vals,
                                int64_t *info) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    if (w == 0 && lane == 0 && (indptr[0] != 0 || indptr[cols] != nnz))
        flag(info, NMFB_INGEST_INDPTR_SPAN, 0);
    for (int64_t c = w; c < cols; c += nw) {
        const int64_t lo = indptr[c], hi = indptr[c + 1];
        if (hi < lo) {
            if (lane == 0) flag(info, NMFB_INGEST_INDPTR_ORDER, c);
            continue;
        }
        if (lo < 0 || hi > nnz) continue;  // reported through the span check
        bool bad_range = false, bad_order = false;
        for (int64_t p = lo + lane; p < hi; p += 32) {
            const int32_t rr = rowidx[p];
            if (rr < 0 || rr >= rows) bad_range = true;
            if (p > lo && rowidx[p - 1] >= rr) bad_order = true;
            const double x = (double)vals[p];
            if (!isfinite(x)) flag(info, NMFB_INGEST_NONFINITE, p);
            else if (x <= 0.0) flag(info, NMFB_INGEST_NONPOSITIVE, p);
        }
        if (__any_sync(0xffffffffu, bad_range) && lane == 0) flag(info, NMFB_INGEST_ROW_RANGE, c);
        if (__any_sync(0xffffffffu, bad_order) && lane == 0) flag(info, NMFB_INGEST_ROW_ORDER, c);
    }
}

__global__ void info_init_kernel(int64_t *info) {
    if (threadIdx.x < NMFB_INGEST_CODES) info[threadIdx.x] = INT64_MAX;
}

// Ingest scratch comes from a PRIVATE stream-ordered pool per device (the
// process's default pool and PyTorch's allocator are left alone).  Its
// release threshold keeps freed scratch mapped between ingests (threshold 0
// would re-map GBs of scratch at every synchronisation: 10-400 ms host
// stalls); nmfb_ingest_release_scratch() hands it back to the driver.
constexpr int kMaxDevices = 64;
static cudaMemPool_t g_pool[kMaxDevices];
static bool g_pool_ok[kMaxDevices];

static cudaMemPool_t ingest_pool(int dev) {
    if (dev < 0 || dev >= kMaxDevices) return nullptr;
    if (!g_pool_ok[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        if (cudaMemPoolCreate(&g_pool[dev], &props) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(g_pool[dev], cudaMemPoolAttrReleaseThreshold, &keep);
        g_pool_ok[dev] = true;
    }
    return g_pool[dev];
}

struct Pool {
    cudaStream_t st;
    cudaMemPool_t mp = nullptr;
    std::vector<void *> ptrs;
    explicit Pool(cudaStream_t s) : st(s) {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) mp = ingest_pool(dev);
    }
    template <typename T>
    T *get(size_t n) {
        void *p = nullptr;
        const size_t bytes = n * sizeof(T) + 16;
        cudaError_t e = mp ? cudaMallocFromPoolAsync(&p, bytes, mp, st) : cudaMallocAsync(&p, bytes, st);
        if (e != cudaSuccess) return nullptr;
        ptrs.push_back(p);
        return (T *)p;
    }
    ~Pool() {
        for (void *p : ptrs) cudaFreeAsync(p, st);
    }
};

template <typename T>
int exclusive_sum(Pool &pool, const T *in, T *out, int64_t n) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, pool.st);
    void *tmp = pool.get<char>(bytes);
    if (!tmp) return NMFB_ERR_CUDA;
    if (cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, n, pool.st) != cudaSuccess)
        return NMFB_ERR_CUDA;
    return NMFB_OK;
}

template <typename K>
int sort_pairs(Pool &pool, K *&key, K *&key_alt, uint32_t *&val, uint32_t *&val_alt, int64_t n,
               int end_bit) {
    cub::DoubleBuffer<K> dk(key, key_alt);
    cub::DoubleBuffer<uint32_t> dv(val, val_alt);
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, dk, dv, n, 0, end_bit, pool.st);
    void *tmp = pool.get<char>(bytes);
    if (!tmp) return NMFB_ERR_CUDA;
    if (cub::DeviceRadixSort::SortPairs(tmp, bytes, dk, dv, n, 0, end_bit, pool.st) !=
        cudaSuccess)
        return NMFB_ERR_CUDA;
    key = dk.Current();
    key_alt = dk.Alternate();
    val = dv.Current();
    val_alt = dv.Alternate();
    return NMFB_OK;
}

}  // namespace

int csc_from_triplets_launch(int64_t rows, int64_t cols, int64_t count, const int64_t *i,
                             const int64_t *j, const double *v, int sum_dup, int64_t *indptr,
                             int32_t *rowidx, void *vals, int vals_dtype, int64_t *nnz_out,
                             int64_t *info, cudaStream_t st) {
    if (rows <= 0 || cols <= 0 || count < 0 || rows >= (1ll << 31) || count >= (1ll << 32) ||
        !indptr || !nnz_out || !info || (count > 0 && (!i || !j || !v || !rowidx || !vals)) ||
        (vals_dtype != NMFB_F32 && vals_dtype != NMFB_F64) ||
        (double)rows * (double)cols >= 1.8e19)
        return NMFB_ERR_ARG;
    info_init_kernel<<<1, 32, 0, st>>>(info);
    cudaMemsetAsync(indptr, 0, sizeof(int64_t) * (cols + 1), st);
    if (count == 0) {
        cudaMemsetAsync(nnz_out, 0, sizeof(int64_t), st);
        return launch_status();
    }
    Pool pool(st);
    uint64_t *key = pool.get<uint64_t>(count), *key_alt = pool.get<uint64_t>(count);
    uint32_t *pos = pool.get<uint32_t>(count), *pos_alt = pool.get<uint32_t>(count);
    uint32_t *head = pool.get<uint32_t>(count), *head_at = pool.get<uint32_t>(count);
    if (!key || !key_alt || !pos || !pos_alt || !head || !head_at) return NMFB_ERR_CUDA;
    triplet_keys_kernel<<<grid_for(count), TB, 0, st>>>(rows, cols, count, i, j, key, pos, info);
    int rc = sort_pairs(pool, key, key_alt, pos, pos_alt, count,
                        key_bits((uint64_t)rows * (uint64_t)cols - 1));
    if (rc) return rc;
    run_heads_kernel<<<grid_for(count), TB, 0, st>>>(count, key, sum_dup, head);
    if ((rc = exclusive_sum(pool, head, head_at, count))) return rc;
    // unique runs: at most `count`; reuse the key/pos alternates as storage
    uint64_t *ukey = key_alt;
    double *usum = pool.get<double>(count);
    uint32_t *keep = pos_alt, *keep_at = pool.get<uint32_t>(count);
    int64_t *nuniq_d = pool.get<int64_t>(1);
    if (!usum || !keep_at || !nuniq_d) return NMFB_ERR_CUDA;
    cudaMemsetAsync(keep, 0, sizeof(uint32_t) * count, st);
    run_sums_kernel<<<grid_for(count), TB, 0, st>>>(count, key, pos, v, head, head_at, ukey, usum,
                                                    keep);
    // the scan over all `count` slots: slots past the last run keep 0
    if ((rc = exclusive_sum(pool, keep, keep_at, count))) return rc;
    if (vals_dtype == NMFB_F64)
        compact_csc_kernel<double><<<grid_for(count), TB, 0, st>>>(
            count, rows, ukey, usum, keep, keep_at, rowidx, (double *)vals, indptr);
    else
        compact_csc_kernel<float><<<grid_for(count), TB, 0, st>>>(
            count, rows, ukey, usum, keep, keep_at, rowidx, (float *)vals, indptr);
    last_total_kernel<<<1, 32, 0, st>>>(keep, keep_at, count, nnz_out);
    // indptr[c + 1] holds column c's count: inclusive prefix sum in place
    int64_t *cnt = pool.get<int64_t>(cols + 1);
    if (!cnt) return NMFB_ERR_CUDA;
    cudaMemcpyAsync(cnt, indptr, sizeof(int64_t) * (cols + 1), cudaMemcpyDeviceToDevice, st);
    size_t bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, bytes, cnt, indptr, cols + 1, st);
    void *tmp = pool.get<char>(bytes);
    if (!tmp || cub::DeviceScan::InclusiveSum(tmp, bytes, cnt, indptr, cols + 1, st) !=
                    cudaSuccess)
        return NMFB_ERR_CUDA;
    return launch_status();
}

int csc_to_csr_launch(int64_t rows, int64_t cols, int64_t nnz, const int64_t *indptr,
                      const int32_t *rowidx, const void *vals, int vals_dtype, int64_t *rowptr,
                      int32_t *colidx, void *cvals, cudaStream_t st) {
    if (rows <= 0 || cols <= 0 || nnz < 0 || rows >= (1ll << 31) || cols >= (1ll << 32) ||
        nnz >= (1ll << 32) || !indptr || !rowptr ||
        (nnz > 0 && (!rowidx || !vals || !colidx || !cvals)) ||
        (vals_dtype != NMFB_F32 && vals_dtype != NMFB_F64))
        return NMFB_ERR_ARG;
    cudaMemsetAsync(rowptr, 0, sizeof(int64_t) * (rows + 1), st);
    if (nnz == 0) return launch_status();
    Pool pool(st);
    uint32_t *key = pool.get<uint32_t>(nnz), *key_alt = pool.get<uint32_t>(nnz);
    uint32_t *pos = pool.get<uint32_t>(nnz), *pos_alt = pool.get<uint32_t>(nnz);
    uint32_t *col_of = pool.get<uint32_t>(nnz);
    int64_t *cnt = pool.get<int64_t>(rows + 1);
    if (!key || !key_alt || !pos || !pos_alt || !col_of || !cnt) return NMFB_ERR_CUDA;
    cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (rows + 1), st);
    col_of_kernel<<<grid_for(cols * 32), TB, 0, st>>>(cols, indptr, col_of);
    row_keys_kernel<<<grid_for(nnz), TB, 0, st>>>(nnz, rowidx, key, pos, cnt);
    // stable by row: positions (column-major, rows ascending) keep their
    // column order within a row
    int rc = sort_pairs(pool, key, key_alt, pos, pos_alt, nnz, key_bits((uint64_t)rows - 1));
    if (rc) return rc;
    if (vals_dtype == NMFB_F64)
        gather_csr_kernel<double><<<grid_for(nnz), TB, 0, st>>>(
            nnz, pos, col_of, (const double *)vals, colidx, (double *)cvals);
    else
        gather_csr_kernel<float><<<grid_for(nnz), TB, 0, st>>>(
            nnz, pos, col_of, (const float *)vals, colidx, (float *)cvals);
    size_t bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, bytes, cnt, rowptr, rows + 1, st);
    void *tmp = pool.get<char>(bytes);
    if (!tmp || cub::DeviceScan::InclusiveSum(tmp, bytes, cnt, rowptr, rows + 1, st) !=
                    cudaSuccess)
        return NMFB_ERR_CUDA;
    return launch_status();
}

int csc_validate_launch(int64_t rows, int64_t cols, int64_t nnz, const int64_t *indptr,
                        const int32_t *rowidx, const void *vals, int vals_dtype, int64_t *info,
                        cudaStream_t st) {
    if (rows < 0 || cols < 0 || nnz < 0 || !indptr || !info ||
        (nnz > 0 && (!rowidx || !vals)) || (vals_dtype != NMFB_F32 && vals_dtype != NMFB_F64))
        return NMFB_ERR_ARG;
    info_init_kernel<<<1, 32, 0, st>>>(info);
    const unsigned grid = grid_for((cols > 0 ? cols : 1) * 32);
    if (vals_dtype == NMFB_F64)
        validate_kernel<double><<<grid, TB, 0, st>>>(rows, cols, nnz, indptr, rowidx,
                                                     (const double *)vals, info);
    else
        validate_kernel<float><<<grid, TB, 0, st>>>(rows, cols, nnz, indptr, rowidx,
                                                    (const float *)vals, info);
    return launch_status();
}

__global__ void narrow_kernel(const int64_t *__restrict__ in, int64_t n, int32_t *__restrict__ out,
                              int64_t *info) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = in[t];
        if (x < INT32_MIN || x > INT32_MAX) flag(info, NMFB_INGEST_ROW_RANGE, t);
        out[t] = (int32_t)x;
    }
}

// ---------------------------------------------------------------------------
// Row-chunk plan of the load-balanced Y^T pass (paper_1506_08938_b200/device.py
// csr_chunk_plan, same definition): row i with k nonzeros -> max(1,
// ceil(k / chunk)) chunks (row, lo, hi, slot); rows with more than one chunk
// ("heavy") number their chunks' partial slots consecutively in row order and
// get an entry (row, first slot, count).  counts_out (host int64[3]): total
// chunks, heavy rows, slots.  chunks_out capacity: rows + nnz / chunk + 1;
// heavy_out capacity: rows.
// ---------------------------------------------------------------------------
__global__ void chunk_counts_kernel(const int64_t *__restrict__ rowptr, int64_t rows, int64_t chunk,
                                    int64_t *nch, int64_t *hch, int64_t *hflag) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = rowptr[i + 1] - rowptr[i];
        int64_t c = (k + chunk - 1) / chunk;
        if (c < 1) c = 1;
        nch[i] = c;
        hch[i] = c > 1 ? c : 0;
        hflag[i] = c > 1 ? 1 : 0;
    }
}

__global__ void chunk_fill_kernel(const int64_t *__restrict__ rowptr, int64_t rows, int64_t chunk,
                                  const int64_t *__restrict__ nch, const int64_t *__restrict__ first,
                                  const int64_t *__restrict__ hfirst,
                                  const int64_t *__restrict__ hidx, int64_t *chunks,
                                  int64_t *heavy) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = nch[i], f = first[i], p0 = rowptr[i], p1 = rowptr[i + 1];
        const bool hv = c > 1;
        for (int64_t q = 0; q < c; ++q) {
            const int64_t lo = p0 + q * chunk;
            int64_t *o = chunks + 4 * (f + q);
            o[0] = i;
            o[1] = lo;
            o[2] = lo + chunk < p1 ? lo + chunk : p1;
            o[3] = hv ? hfirst[i] + q : -1;
        }
        if (hv) {
            int64_t *h = heavy + 3 * hidx[i];
            h[0] = i;
            h[1] = hfirst[i];
            h[2] = c;
        }
    }
}

int csr_chunk_plan_launch(const int64_t *rowptr, int64_t rows, int64_t chunk, int64_t *chunks,
                          int64_t *heavy, int64_t *counts_out, cudaStream_t st) {
    if (rows <= 0 || chunk <= 0 || !rowptr || !chunks || !heavy || !counts_out)
        return NMFB_ERR_ARG;
    Pool pool(st);
    int64_t *nch = pool.get<int64_t>(rows), *hch = pool.get<int64_t>(rows);
    int64_t *hflag = pool.get<int64_t>(rows), *first = pool.get<int64_t>(rows);
    int64_t *hfirst = pool.get<int64_t>(rows), *hidx = pool.get<int64_t>(rows);
    int64_t *tail = pool.get<int64_t>(6);
    if (!nch || !hch || !hflag || !first || !hfirst || !hidx || !tail) return NMFB_ERR_CUDA;
    const unsigned grid = grid_for(rows);
    chunk_counts_kernel<<<grid, TB, 0, st>>>(rowptr, rows, chunk, nch, hch, hflag);
    int rc = exclusive_sum(pool, nch, first, rows);
    if (!rc) rc = exclusive_sum(pool, hch, hfirst, rows);
    if (!rc) rc = exclusive_sum(pool, hflag, hidx, rows);
    if (rc) return rc;
    chunk_fill_kernel<<<grid, TB, 0, st>>>(rowptr, rows, chunk, nch, first, hfirst, hidx, chunks,
                                           heavy);
    // totals = last exclusive prefix + last count
    const int64_t *src[6] = {first + rows - 1, nch + rows - 1, hidx + rows - 1,
                             hflag + rows - 1, hfirst + rows - 1, hch + rows - 1};
    for (int k = 0; k < 6; ++k)
        cudaMemcpyAsync(tail + k, src[k], sizeof(int64_t), cudaMemcpyDeviceToDevice, st);
    int64_t h[6];
    if (cudaMemcpyAsync(h, tail, sizeof(h), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return NMFB_ERR_CUDA;
    counts_out[0] = h[0] + h[1];
    counts_out[1] = h[2] + h[3];
    counts_out[2] = h[4] + h[5];
    return launch_status();
}

int ingest_release_scratch() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return NMFB_ERR_CUDA;
    if (dev >= 0 && dev < kMaxDevices && g_pool_ok[dev]) {
        if (cudaDeviceSynchronize() != cudaSuccess) return NMFB_ERR_CUDA;
        if (cudaMemPoolTrimTo(g_pool[dev], 0) != cudaSuccess) return NMFB_ERR_CUDA;
    }
    return NMFB_OK;
}

int narrow_indices_launch(const int64_t *in, int64_t n, int32_t *out, int64_t *info,
                          cudaStream_t st) {
    if (n < 0 || (n > 0 && (!in || !out)) || !info) return NMFB_ERR_ARG;
    info_init_kernel<<<1, 32, 0, st>>>(info);
    if (n > 0) narrow_kernel<<<grid_for(n), TB, 0, st>>>(in, n, out, info);
    return launch_status();
}

}  // namespace nmfb
