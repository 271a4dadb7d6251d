"""Device-side state and the per-iteration launch sequence of the alternation.

Torch is used for allocation, host<->device copies, streams and events only;
every numeric step is a libnmfb.so kernel reached through the C ABI
(include/nmfb.h).  The launch sequence of one outer iteration follows
nmf.py:188-196 (gram -> coefficient step -> component step -> objective):

  gram(G) -> rescale(+2 mu2)                      Q_g, compact Qa   (matrix.py:181, nqp.py:116)
  linear terms h = mu1 - G^T X                    dense GEMM / CSC SpMM (kernels.py:251,306)
  batched NNLS over the m columns -> F           nnls kernels (kernels.py:178-220)
  H_f = F F^T ; Y^T = X F^T                       gram / dense GEMM / CSR SpMM (kernels.py:270-280)
  rescale(H_f + 2 beta2) ; NNLS over n rows -> G  (parallel.py:189-223, kernels.py:339-378)
  objective pieces                                residual (dense) / trace identity (sparse)

Two precisions:
  * "fp64": reference-order kernels (NMFB_MODE_REFERENCE) in float64; the
    per-worker shard partial sums of the reference's reduce are emulated, so
    run_estep / run_mstep are bit-identical to the reference given the same
    inputs (only the BLAS Gram differs in the last bits).
  * "fp32": production path -- split-K GEMM / SpMM passes and the register
    resident warp-group NNLS kernel in float32, fp64 reductions.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib as L
from .exceptions import NumericalFailureError
from .matrix import DenseMatrix, SparseMatrix

_TORCH = {"fp32": torch.float32, "fp64": torch.float64}
MUR_FLOOR = 1e-12  # baselines.py:20
_CODE = {"fp32": L.F32, "fp64": L.F64}


def tc_enabled():
    """Tensor-core passes on unless NMFB_DISABLE_TC=1 (A/B comparisons only)."""
    import os

    return os.environ.get("NMFB_DISABLE_TC", "0") != "1"


def gram_overlap_enabled():
    """Sparse path: Grams on a side stream beside the sparse data products,
    unless NMFB_GRAM_OVERLAP=0."""
    import os

    return os.environ.get("NMFB_GRAM_OVERLAP", "1") != "0"


def d_i8_enabled():
    """Exact int8 tensor-core residual unless NMFB_DISABLE_I8=1 (A/B comparisons)."""
    import os

    return os.environ.get("NMFB_DISABLE_I8", "0") != "1"


def require_cuda():
    L.lib()
    if not torch.cuda.is_available():
        raise L.NativeLibraryError("no CUDA device: libnmfb.so requires a B200 (sm_100a)")
    return torch.device("cuda")


def vp(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def stream_handle(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def plan(total, workers):
    """parallel.py:72-84."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    workers = min(workers, total) if total > 0 else 1
    base, extra = divmod(total, workers)
    shards, lo = [], 0
    for w in range(workers):
        hi = lo + base + (1 if w < extra else 0)
        shards.append((lo, hi))
        lo = hi
    return shards


def block_plan(total, workers):
    """parallel.py:162-169: shards aligned to FASTBREAK_BLOCK."""
    b = L.FASTBREAK_BLOCK
    nblocks = max(-(-total // b), 1)
    return [(lo * b, min(hi * b, total)) for lo, hi in plan(nblocks, workers)]


CSR_CHUNK = 256  # max nonzeros one warp sums in the load-balanced Y^T pass


def csr_chunk_plan(rowptr, chunk=CSR_CHUNK):
    """Row chunks for nmfb_csr_yt_chunked: (row, lo, hi, slot) per chunk, slot
    -1 for single-chunk rows; heavy rows (row, first slot, count)."""
    rowptr = np.asarray(rowptr, dtype=np.int64)
    n = len(rowptr) - 1
    nnz_row = np.diff(rowptr)
    nch = np.maximum(1, -(-nnz_row // chunk))
    total = int(nch.sum())
    row = np.repeat(np.arange(n, dtype=np.int64), nch)
    first = np.cumsum(nch) - nch
    within = np.arange(total, dtype=np.int64) - np.repeat(first, nch)
    lo = rowptr[row] + within * chunk
    hi = np.minimum(lo + chunk, rowptr[row + 1])
    heavy_mask_rows = nch > 1
    slot = np.full(total, -1, dtype=np.int64)
    in_heavy = np.repeat(heavy_mask_rows, nch)
    slot[in_heavy] = np.arange(int(in_heavy.sum()), dtype=np.int64)
    chunks = np.stack([row, lo, hi, slot], axis=1).astype(np.int64)
    hrows = np.flatnonzero(heavy_mask_rows).astype(np.int64)
    hfirst = slot[first[hrows]] if len(hrows) else np.zeros(0, dtype=np.int64)
    heavy = np.stack([hrows, hfirst, nch[hrows]], axis=1).astype(np.int64) if len(hrows) \
        else np.zeros((0, 3), dtype=np.int64)
    return np.ascontiguousarray(chunks), np.ascontiguousarray(heavy), int(in_heavy.sum())


def device_chunk_plan(rowptr, n, nnz, device, chunk=CSR_CHUNK):
    """csr_chunk_plan built on the device (nmfb_csr_chunk_plan): the same
    (chunks, heavy) tables as device tensors, plus the slot count."""
    import ctypes

    cap = n + nnz // chunk + 1
    chunks = torch.empty((max(cap, 1), 4), dtype=torch.int64, device=device)
    heavy = torch.empty((max(n, 1), 3), dtype=torch.int64, device=device)
    counts = np.zeros(3, dtype=np.int64)
    if n == 0:
        return chunks[:0], heavy[:0], 0
    L.call("nmfb_csr_chunk_plan", vp(rowptr), n, chunk, vp(chunks), vp(heavy),
           counts.ctypes.data_as(ctypes.c_void_p), stream_handle())
    return chunks[: int(counts[0])], heavy[: int(counts[1])], int(counts[2])


def shard_bounds(total, workers):
    shards = block_plan(total, workers)
    return [shards[0][0]] + [hi for _, hi in shards]


def _count_launches(k):
    """Extra kernel launches of a multi-pass entry point (gpu_launches)."""
    rec = L.Recorder.active
    if rec is not None:
        rec.launches += k


def device_sums(x):
    """(sum|x|, sum x^2) in fp64 on the device (nmfb_dot's fixed-order reduction)."""
    ws = torch.empty((L.lib().nmfb_dot_workspace_bytes(0) // 8 + 1,), dtype=torch.float64,
                     device=x.device)
    out = torch.zeros(3, dtype=torch.float64, device=x.device)
    L.call("nmfb_dot", vp(x), _CODE["fp64" if x.dtype == torch.float64 else "fp32"], None,
           L.F64, x.numel(), vp(out), vp(ws), stream_handle())
    o = out.cpu().numpy()
    return float(o[1]), float(o[2])


def device_sum_squares(x):
    return device_sums(x)[1]


# ---------------------------------------------------------------------------
# data matrix on the device
# ---------------------------------------------------------------------------
_PINNED = []  # two pinned byte buffers, reused by every upload / download


def _pinned_pair(nbytes):
    """Two pinned host staging buffers of >= nbytes (allocated once: pinning
    GBs per call costs more than the copies)."""
    global _PINNED
    if not _PINNED or _PINNED[0].numel() < nbytes:
        _PINNED = [torch.empty((nbytes,), dtype=torch.uint8).pin_memory() for _ in range(2)]
    return _PINNED


def _copy_threads(dst, src, pool, parts):
    n = len(dst)
    step = -(-n // parts)
    list(pool.map(lambda q: np.copyto(dst[q * step:(q + 1) * step], src[q * step:(q + 1) * step]),
                  range(parts)))


def upload_host(arr, dt, device, chunk_bytes=128 << 20, threads=8):
    """A C-contiguous host array (1-D or 2-D) -> a device tensor of dtype dt.
    Rows stream through two pinned staging buffers: host threads copy chunk
    i + 1 (numpy releases the GIL) while chunk i uploads, and the dtype cast
    (e.g. the reference's float64 -> fp32) runs on the device -- no host-side
    astype of the whole array, no pageable copy."""
    from concurrent.futures import ThreadPoolExecutor

    one_d = arr.ndim == 1
    arr2 = arr.reshape(-1, 1) if one_d else arr
    rows, cols = arr2.shape
    out = torch.empty((rows, cols), dtype=dt, device=device)
    if arr2.size == 0:
        return out.view(-1) if one_d else out
    src_t = torch.from_numpy(arr2[:1]).dtype
    row_bytes = cols * arr2.itemsize
    rb = max(1, chunk_bytes // max(1, row_bytes))
    pinned = _pinned_pair(rb * row_bytes)
    stage = [p[: rb * row_bytes].view(src_t).view(rb, cols) for p in pinned]
    done = [None, None]
    stream = torch.cuda.current_stream(device)
    with ThreadPoolExecutor(threads) as pool:
        for i, lo in enumerate(range(0, rows, rb)):
            hi = min(rows, lo + rb)
            b = i % 2
            if done[b] is not None:
                done[b].synchronize()  # the upload that last used this buffer
            _copy_threads(stage[b].numpy()[: hi - lo], arr2[lo:hi], pool, threads)
            out[lo:hi].copy_(stage[b][: hi - lo], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            done[b] = ev
    # the staging buffers are reused by the next transfer: drain this one
    for ev in done:
        if ev is not None:
            ev.synchronize()
    return out.view(-1) if one_d else out


def download_host(t, chunk_bytes=128 << 20, threads=8):
    """A contiguous device tensor -> a new host numpy array of the same dtype
    and shape, through the two pinned staging buffers (chunk i + 1 comes over
    the link while host threads copy chunk i out)."""
    from concurrent.futures import ThreadPoolExecutor

    flat = t.reshape(-1)
    out = np.empty(tuple(t.shape), dtype=torch.empty(0, dtype=t.dtype).numpy().dtype)
    oflat = out.reshape(-1)
    n = flat.numel()
    if n == 0:
        return out
    es = flat.element_size()
    ce = max(1, chunk_bytes // es)
    pinned = _pinned_pair(ce * es)
    stage = [p[: ce * es].view(flat.dtype) for p in pinned]
    stream = torch.cuda.current_stream(t.device)
    chunks = [(lo, min(n, lo + ce)) for lo in range(0, n, ce)]
    evs = [None, None]

    def issue(i):
        lo, hi = chunks[i]
        b = i % 2
        stage[b][: hi - lo].copy_(flat[lo:hi], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        evs[b] = ev

    with ThreadPoolExecutor(threads) as pool:
        issue(0)
        if len(chunks) > 1:
            issue(1)
        for i, (lo, hi) in enumerate(chunks):
            b = i % 2
            evs[b].synchronize()
            _copy_threads(oflat[lo:hi], stage[b][: hi - lo].numpy(), pool, threads)
            if i + 2 < len(chunks):
                issue(i + 2)
    return out


class DeviceData:
    """X on the device.  Dense: XT (m, n) row-major == the reference's
    Fortran-ordered (n, m) buffer.  Sparse: CSC (int64 indptr, int32 rows,
    values) plus the CSR of the same matrix (int64 rowptr, int32 cols
    ascending per row)."""

    def __init__(self, V, precision="fp32", device=None, stream=None):
        self.device = device or require_cuda()
        self.precision = precision
        dt = _TORCH[precision]
        if isinstance(V, DenseMatrix):
            V = V.array
        if isinstance(V, torch.Tensor):
            # (n, m) tensor; V.t() contiguous (an XT buffer) -> no host copy, and a
            # pinned host buffer uploads asynchronously at full PCIe/C2C rate
            if V.dim() != 2:
                raise ValueError("dense data must be 2-D")
            self.kind = "dense"
            self.n, self.m = V.shape
            self.XT = V.t().contiguous().to(self.device, dt, non_blocking=True)
            self.host = None
            return
        from .ingest import DeviceCsc

        if isinstance(V, (SparseMatrix, DeviceCsc)):
            # CSC uploaded (or already resident), its CSR twin built on the
            # device (csrc/ingest.cu) instead of the host's argsort
            self.kind = "sparse"
            self.n, self.m = V.rows, V.cols
            if V.nnz >= 2**31 or self.n >= 2**31 or self.m >= 2**31:
                raise ValueError("sparse sizes must fit int32 indices")
            if isinstance(V, SparseMatrix):
                csc = DeviceCsc.from_host(V, dtype=dt, device=self.device, validate=True)
                self.xsq = V.sum_squares()
            else:
                csc = V
                if csc.dtype != dt:
                    csc = DeviceCsc(csc.rows, csc.cols, csc.indptr, csc.rowidx,
                                    csc.values.to(dt), validate=False)
                self.xsq = device_sum_squares(V.values)
            self.indptr, self.rowidx, self.vals = csc.indptr, csc.rowidx, csc.values
            self.rowptr, self.colidx, self.cvals = csc.csr()
            # the row-chunk plan of the load-balanced Y^T pass: O(n) on the host
            self.chunks, self.heavy, self.nslots = device_chunk_plan(self.rowptr, self.n,
                                                                     V.nnz, self.device)
            self.nchunks, self.nheavy = len(self.chunks), len(self.heavy)
            self.nnz = V.nnz
            self.host = V if isinstance(V, SparseMatrix) else None
            self.csc = csc
            self.blocking = {}
        else:
            arr = np.asarray(V)
            if arr.ndim != 2:
                raise ValueError("dense data must be 2-D")
            self.kind = "dense"
            self.n, self.m = arr.shape
            self.host = None
            if (arr.flags["C_CONTIGUOUS"] and not arr.flags["F_CONTIGUOUS"]
                    and dt == torch.float32):
                # (n, m) row-major host data: uploaded as X and transposed on
                # the device (no host transpose of the whole matrix)
                self.X = upload_host(arr, dt, self.device)
                self.XT = torch.empty((self.m, self.n), dtype=dt, device=self.device)
                L.call("nmfb_transpose", vp(self.X), self.n, self.m, vp(self.XT),
                       stream_handle())
            else:
                # the reference's Fortran-ordered buffer == XT row-major
                self.XT = upload_host(np.ascontiguousarray(arr.T), dt, self.device)

    def spmm_blocking(self, r):
        """L2 blocking plan of the sparse data products for rank r (fp32):
        (nblk_g, seg_g, nblk_f, seg_f) -- the gathered factor (G, n x r, for
        G^T X; F^T, m x r, for X F^T) is cut into blocks of at most
        NMFB_SPMM_BLOCK_MB (G; default 64) / NMFB_SPMM_BLOCK_MB_F (F^T;
        default 0 = off) MB; one block means no blocking.  Measured at config
        5 (G 800 MB, F^T 160 MB): G^T X 7.0 -> 5.9 ms with 96 MB blocks, 5.86
        with 64 MB, 6.04 with 128 MB; the
        X F^T pass gets slower blocked (its outputs, n x r = 800 MB, would be
        re-read and re-written every pass), so it stays unblocked."""
        import os

        if r in self.blocking:
            return self.blocking[r]
        plan = []
        for rows, build, var, dflt in ((self.n, "csc", "NMFB_SPMM_BLOCK_MB", "64"),
                                       (self.m, "chunk", "NMFB_SPMM_BLOCK_MB_F", "0")):
            mb = float(os.environ.get(var, dflt))
            nblk = max(1, int(np.ceil(rows * r * 4 / (mb * 2**20)))) if mb > 0 else 1
            if nblk == 1:
                plan += [1, None]
                continue
            blk = -(-rows // nblk)
            if build == "csc":
                seg = torch.empty((self.m, nblk + 1), dtype=torch.int64, device=self.device)
                L.call("nmfb_csc_segments", vp(self.indptr), vp(self.rowidx), self.m, blk, nblk,
                       vp(seg), stream_handle())
            else:
                seg = torch.empty((self.nchunks, nblk + 1), dtype=torch.int64,
                                  device=self.device)
                L.call("nmfb_chunk_segments", vp(self.chunks), self.nchunks, vp(self.colidx),
                       blk, nblk, vp(seg), stream_handle())
            plan += [nblk, seg]
        self.blocking[r] = tuple(plan)
        return self.blocking[r]

    def ensure_x_rowmajor(self):
        """X (n, m) row-major next to X^T: the K-major operand of the Y^T pass
        (one transpose kernel per fit; HBM is plentiful, TMA wants K-major)."""
        if getattr(self, "X", None) is None:
            self.X = torch.empty((self.n, self.m), dtype=self.XT.dtype, device=self.XT.device)
            L.call("nmfb_transpose", vp(self.XT), self.m, self.n, vp(self.X), stream_handle())
        return self.X

    @classmethod
    def from_device_dense(cls, XT, precision):
        """Wrap an existing (m, n) device tensor (already in HBM)."""
        self = cls.__new__(cls)
        self.device = XT.device
        self.precision = precision
        self.kind = "dense"
        self.m, self.n = XT.shape
        self.XT = XT
        self.host = None
        return self


# ---------------------------------------------------------------------------
# one alternation state on the device
# ---------------------------------------------------------------------------
class Alternation:
    """Device state of fit(): G (n, r), FT (m, r) and all step buffers."""

    def __init__(self, data: DeviceData, cfg, G0, FT0, max_iters, precision="fp32", lanes=0,
                 kernel_mode=None, splits=None, solver="nnls", overlap=True):
        self.d = data
        self.cfg = cfg
        # solver "mur": the multiplicative-update baseline (baselines.py:41-85)
        # on the same data products; it ignores the penalties in its steps
        # (the logged objective keeps them, baselines.py:58-63)
        if solver not in ("nnls", "mur"):
            raise ValueError("solver must be 'nnls' or 'mur'")
        self.solver = solver
        if solver == "mur":
            import dataclasses

            self.step_cfg = dataclasses.replace(cfg, mu1=0.0, mu2=0.0, beta1=0.0, beta2=0.0)
        else:
            self.step_cfg = cfg
        self.prec = precision
        self.code = _CODE[precision]
        self.mode = (L.MODE_REFERENCE if precision == "fp64" else L.MODE_FAST) \
            if kernel_mode is None else kernel_mode
        self.lanes = lanes
        dev = data.device
        dt = _TORCH[precision]
        n, m, r = data.n, data.m, cfg.rank
        self.n, self.m, self.r = n, m, r
        f64 = torch.float64
        def _factor(A):
            if isinstance(A, torch.Tensor):  # already on the device (torch-input fit)
                return A.to(dev, dt).contiguous()
            return torch.as_tensor(np.ascontiguousarray(A), dtype=dt).to(dev)

        self.G = _factor(G0)
        self.FT = _factor(FT0)
        self.Qg = torch.zeros((r, r), dtype=f64, device=dev)
        self.Hf = torch.zeros((r, r), dtype=f64, device=dev)
        # compact rescaled problems of the two steps
        self.Qa = [torch.zeros((r * r,), dtype=dt, device=dev) for _ in range(2)]
        self.sa = [torch.zeros((r,), dtype=dt, device=dev) for _ in range(2)]
        self.act = [torch.zeros((r,), dtype=torch.int32, device=dev) for _ in range(2)]
        self.active = [torch.zeros((r,), dtype=torch.uint8, device=dev) for _ in range(2)]
        self.ra = [torch.zeros((1,), dtype=torch.int32, device=dev) for _ in range(2)]
        self.gram_ws = torch.empty((L.lib().nmfb_gram_workspace_bytes(max(n, m), r) // 8 + 1,),
                                   dtype=f64, device=dev)
        # sparse fp32 path: the Grams (FMA-bound) run on a side stream beside
        # the L2-bound sparse data products that do not need them (see estep)
        self.gside = None
        if (data.kind == "sparse" and self.mode == L.MODE_FAST and overlap
                and gram_overlap_enabled()):
            self.gside = torch.cuda.Stream(device=dev)
            self.gside_ev = None      # Q_g (Gram of G) + objective quad ready
            self.hf_ev = None         # H_f (Gram of F) + its rescale ready
            self.dot_ws2 = torch.empty((L.lib().nmfb_dot_workspace_bytes(0) // 8 + 1,),
                                       dtype=f64, device=dev)
        self.dot_ws = torch.empty((L.lib().nmfb_dot_workspace_bytes(0) // 8 + 1,), dtype=f64,
                                  device=dev)
        sms = max(L.lib().nmfb_device_sm_count(), 1)
        if data.kind == "dense":
            self.res_ws = torch.empty((L.lib().nmfb_residual_workspace_bytes(m, n) // 8 + 1,),
                                      dtype=f64, device=dev)
        # tensor-core passes (tcgen05 3xTF32) when the shapes allow TMA tiles:
        # both orientations of X resident (X^T for G^T X, X for X F^T)
        self.use_tc = (data.kind == "dense" and self.mode == L.MODE_FAST and r <= 160
                       and n % 4 == 0 and m % 4 == 0 and tc_enabled())
        if data.kind == "dense" and self.mode == L.MODE_FAST:
            if self.use_tc:
                data.ensure_x_rowmajor()
                # balanced persistent schedule (splits <= 0) unless a split count is forced
                self.tc_req = int(splits or 0)
                self.splits_e = L.lib().nmfb_tc_parts(m, n, r, self.tc_req)
                self.splits_m = L.lib().nmfb_tc_parts(n, m, r, self.tc_req)
                # [iteration parity][hi, lo] k-major tf32 splits of G^T and F; two
                # parities so the residual of iteration k (side stream) can still
                # read its operands while iteration k+1 runs
                self.Gt = torch.empty((2, 2, r, n), dtype=torch.float32, device=dev)
                self.Ft = torch.empty((2, 2, r, m), dtype=torch.float32, device=dev)
                # exact int8 tensor-core residual: per-parity 8-bit slices of G, F^T
                self.use_i8 = (r <= 128 and m % 4 == 0 and d_i8_enabled())
                if self.use_i8:
                    lib = L.lib()
                    self.Gsl = torch.empty((2, lib.nmfb_slice_bytes(n, r)), dtype=torch.uint8,
                                           device=dev)
                    self.Fsl = torch.empty((2, lib.nmfb_slice_bytes(m, r)), dtype=torch.uint8,
                                           device=dev)
                    self.rq_ws = torch.empty((lib.nmfb_residual_i8_workspace_bytes() // 8 + 1,),
                                             dtype=f64, device=dev)
                lo, hi = torch.cuda.Stream.priority_range()
                self.main = torch.cuda.Stream(device=dev, priority=hi)
                self.side = torch.cuda.Stream(device=dev, priority=lo)
                self.res_ev = [None, None]
            else:
                # split-K factors: ~4 CTAs per SM for each pass
                self.splits_e = splits or self._splits(m, n, sms)
                self.splits_m = splits or self._splits(n, m, sms)
            self.hbuf = torch.empty((self.splits_e * m * r,), dtype=torch.float32, device=dev)
            self.ybuf = torch.empty((self.splits_m * n * r,), dtype=torch.float32, device=dev)
        else:
            self.hbuf = torch.empty((m * r,), dtype=dt, device=dev)
            # sparse fast path: Y^T accumulated in fp64 inside the kernel and
            # stored fp32 (the M-step reads it as fp32 anyway; half the bytes).
            # fp64 when the X F^T pass is L2-blocked (NMFB_SPMM_BLOCK_MB_F: its
            # running sums are carried through Y^T between block passes) or on
            # request (NMFB_YT64=1)
            import os

            yt64 = (precision == "fp64" or self.mode != L.MODE_FAST
                    or os.environ.get("NMFB_YT64", "0") == "1"
                    or (data.kind == "sparse" and self.prec == "fp32" and r % 4 == 0
                        and r <= 256 and data.spmm_blocking(r)[2] > 1))
            ydt = f64 if yt64 else dt
            self.ybuf = torch.empty((n * r,), dtype=ydt, device=dev)
        self.max_iters = max_iters
        # per iteration: stats [2 steps][inner, fail], objective pieces
        self.stats = torch.zeros((max_iters, 2, 2), dtype=torch.int64, device=dev)
        self.stats[:, :, 1] = -1  # == UINT64_MAX
        self.pieces = torch.zeros((max_iters, 12), dtype=f64, device=dev)
        if precision == "fp64" or data.kind == "sparse":
            self.bounds_e = shard_bounds(m, cfg.workers)
        else:
            self.bounds_e = [0, m]
        self.qg_valid = False
        self.index_base_e = 0  # global column of FT row 0 (multi-GPU column shards)
        self.gt_valid = False  # Gt holds tf32-split G^T of the current G
        # multi-GPU peer layout of the X F^T partials (dist.PeerExchange):
        # (dst pointer array, world, chunk, src rank) or None = local ybuf
        self.yt_out = None

    @staticmethod
    def _splits(M, K, sms):
        tiles = -(-M // 128)
        s = max(1, round(4 * sms / tiles))
        s = min(s, max(1, K // 256))
        return int(s)

    def _spmm_plan(self):
        """Blocked sparse products apply to the fp32 production path with
        16-byte-aligned rows (r % 4 == 0, r <= 256)."""
        if (self.mode != L.MODE_FAST or self.prec != "fp32" or self.r % 4 or self.r > 256):
            return (1, None, 1, None)
        return self.d.spmm_blocking(self.r)

    # -- primitive launches ------------------------------------------------
    def _st(self):
        return stream_handle()

    def gram(self, A, rows, out):
        L.call("nmfb_gram", self.code, vp(A), rows, self.r, self.r, vp(out), vp(self.gram_ws),
               self._st())

    def gram_rescale(self, A, rows, out, diag_add, side):
        L.call("nmfb_gram_rescale", self.code, vp(A), rows, self.r, self.r, vp(out),
               vp(self.gram_ws), diag_add, vp(self.Qa[side]), vp(self.sa[side]),
               vp(self.act[side]), vp(self.active[side]), vp(self.ra[side]), self._st())

    def rescale(self, H, diag_add, side):
        L.call("nmfb_rescale", self.code, vp(H), self.r, diag_add, vp(self.Qa[side]),
               vp(self.sa[side]), vp(self.act[side]), vp(self.active[side]), vp(self.ra[side]),
               None, self._st())

    def nnls(self, side, h, h_dtype, parts, h_ld, pstride, h_base, x, count, stats):
        if self.solver == "mur":
            Q = self.Qg if side == 0 else self.Hf
            L.call("nmfb_mur_update", self.code, vp(Q), self.r, vp(h), h_dtype, parts, h_ld,
                   pstride, float(h_base), vp(x), count, MUR_FLOOR, vp(stats), self._st())
            return
        # global index of problem 0: fast-break blocks are absolute (kernels.py:247)
        base = self.index_base_e if side == 0 else 0
        L.call("nmfb_nnls_batch", self.code, self.mode, vp(self.Qa[side]), vp(self.sa[side]),
               vp(self.act[side]), vp(self.active[side]), self.r, self.r, vp(self.ra[side]),
               vp(h), h_dtype, parts, h_ld, pstride, h_base, vp(x), count, base,
               float(self.cfg.epsilon), int(self.cfg.inner_cap), 0.0, None, None, vp(stats),
               self.lanes, self._st())

    def dot(self, a, a_code, b, b_code, length, out, ws=None):
        L.call("nmfb_dot", vp(a), a_code, vp(b), b_code, length, vp(out),
               vp(self.dot_ws if ws is None else ws), self._st())

    def _overlap(self):
        """The side stream for the Grams, or None (off, or serialised timing)."""
        return None if (self.gside is None or getattr(self, "serial", False)) else self.gside

    def _on_side(self):
        """Side stream ordered after the work enqueued so far on the caller's."""
        ev = torch.cuda.Event()
        ev.record()
        self.gside.wait_event(ev)
        return torch.cuda.stream(self.gside)

    def _side_done(self):
        ev = torch.cuda.Event()
        ev.record(self.gside)
        return ev

    # -- the two half-steps ---------------------------------------------------
    def estep(self, k):
        """Coefficient step (parallel.run_estep): linear terms, NNLS over the
        m columns, then the accumulators H_f = F F^T and Y^T = X F^T."""
        cfg, d, r = self.step_cfg, self.d, self.r
        n, m = self.n, self.m
        pending_q = d.kind == "sparse" and self.qg_valid and \
            getattr(self, "gside_ev", None) is not None
        if not pending_q:
            if not self.qg_valid:
                # Gram of G with the anti-lopsided rescale fused into its epilogue
                self.gram_rescale(self.G, n, self.Qg, 2.0 * cfg.mu2, 0)
            else:
                self.rescale(self.Qg, 2.0 * cfg.mu2, 0)
            self.qg_valid = False
        st = self.stats[k, 0]
        if d.kind == "dense":
            if self.use_tc:
                gq = (k - 1) % 2  # parity buffer holding G_{k-1}^T
                Gt = self.Gt[gq]
                if not self.gt_valid:
                    self._wait_residual(gq)
                    L.call("nmfb_split_transpose", vp(self.G), n, r, vp(Gt[0]), vp(Gt[1]),
                           self._st())
                self.gt_valid = False
                L.call("nmfb_tc_gemm", vp(d.XT), m, n, vp(Gt[0]), vp(Gt[1]), r,
                       vp(self.hbuf), self.tc_req, 0, self._st())
                self.nnls(0, self.hbuf, L.F32, self.splits_e, r, m * r, cfg.mu1, self.FT, m, st)
            elif self.mode == L.MODE_FAST:
                L.call("nmfb_gemm_tall", vp(d.XT), 1, m, n, n, vp(self.G), r, r, vp(self.hbuf),
                       self.splits_e, self._st())
                self.nnls(0, self.hbuf, L.F32, self.splits_e, r, m * r, cfg.mu1, self.FT, m, st)
            else:
                L.call("nmfb_dense_linear_ref", self.code, vp(d.XT), n, 0, m, vp(self.G), r,
                       cfg.mu1, vp(self.hbuf), self._st())
                self.nnls(0, self.hbuf, self.code, 0, r, 0, 0.0, self.FT, m, st)
        else:
            nbg, segg = self._spmm_plan()[:2]
            if nbg > 1:
                L.call("nmfb_csc_linear_blocked", vp(d.indptr), vp(segg), nbg, vp(d.rowidx),
                       vp(d.vals), m, vp(self.G), r, cfg.mu1, vp(self.hbuf), self._st())
                _count_launches(nbg - 1)
            else:
                L.call("nmfb_csc_linear", self.code, self.mode, vp(d.indptr), vp(d.rowidx),
                       vp(d.vals), 0, m, vp(self.G), r, cfg.mu1, vp(self.hbuf), self._st())
            if pending_q:
                # Q_g came from the side stream (overlapping the data product above)
                torch.cuda.current_stream().wait_event(self.gside_ev)
                self.gside_ev = None
                self.rescale(self.Qg, 2.0 * cfg.mu2, 0)
                self.qg_valid = False
            self.nnls(0, self.hbuf, self.code, 0, r, 0, 0.0, self.FT, m, st)
        # accumulators from the new coefficients
        ba, bp = L.bounds_array(self.bounds_e)
        W = len(self.bounds_e) - 1
        if self.prec == "fp64" or self.mode == L.MODE_REFERENCE:
            L.call("nmfb_hp_ref", self.code, vp(self.FT), m, r, bp, W, vp(self.Hf), self._st())
        elif self._overlap() is not None:
            # H_f = F F^T (+ rescale) on the side stream, beside X F^T below
            with self._on_side():
                self.gram_rescale(self.FT, m, self.Hf, 2.0 * cfg.beta2, 1)
            self.hf_ev = self._side_done()
            self.hf_rescaled = True
        else:
            # H_f = F F^T, rescaled for the component step right away
            self.gram_rescale(self.FT, m, self.Hf, 2.0 * cfg.beta2, 1)
            self.hf_rescaled = True
        if d.kind == "dense":
            if self.use_tc:
                Ft = self.Ft[k % 2]
                self._wait_residual(k % 2)  # residual(k-2) still reads this parity
                L.call("nmfb_split_transpose", vp(self.FT), m, r, vp(Ft[0]), vp(Ft[1]),
                       self._st())
                if self.yt_out is None:
                    L.call("nmfb_tc_gemm", vp(d.X), n, m, vp(Ft[0]), vp(Ft[1]), r,
                           vp(self.ybuf), self.tc_req, 0, self._st())
                else:
                    # each owner's rows go straight into its receive buffer
                    dst, world, chunk, src = self.yt_out
                    L.call("nmfb_tc_gemm_rows", vp(d.X), n, m, vp(Ft[0]), vp(Ft[1]), r,
                           self.tc_req, dst, world, chunk, src, self._st())
            elif self.mode == L.MODE_FAST:
                L.call("nmfb_gemm_tall", vp(d.XT), 0, n, m, n, vp(self.FT), r, r,
                       vp(self.ybuf), self.splits_m, self._st())
            else:
                L.call("nmfb_dense_yt_ref", self.code, vp(d.XT), m, n, vp(self.FT), r, bp, W,
                       vp(self.ybuf), self._st())
        else:
            ycode = L.F64 if self.ybuf.dtype == torch.float64 else L.F32
            if self.mode == L.MODE_FAST:
                # load-balanced row chunks (Zipf-popular rows hold 10^4+ entries)
                if getattr(self, "ypart", None) is None:
                    # heavy-row chunk partials: fp64 whatever the Y^T type
                    self.ypart = torch.empty((max(d.nslots, 1) * r,), dtype=torch.float64,
                                             device=self.ybuf.device)
                nbf, segf = self._spmm_plan()[2:]
                if nbf > 1:
                    L.call("nmfb_csr_yt_chunked_blocked", vp(d.chunks), d.nchunks, vp(d.heavy),
                           d.nheavy, vp(segf), nbf, vp(d.colidx), vp(d.cvals), vp(self.FT), r,
                           ycode, vp(self.ybuf), vp(self.ypart), self._st())
                    _count_launches(nbf - 1)
                else:
                    L.call("nmfb_csr_yt_chunked", self.code, vp(d.chunks), d.nchunks,
                           vp(d.heavy), d.nheavy, vp(d.colidx), vp(d.cvals), vp(self.FT), r,
                           ycode, vp(self.ybuf), vp(self.ypart), self._st())
            else:
                L.call("nmfb_csr_yt", self.code, self.mode, vp(d.rowptr), vp(d.colidx),
                       vp(d.cvals), n, vp(self.FT), r, ycode, bp, W, vp(self.ybuf), self._st())
        del ba

    def mstep(self, k):
        """Component step (parallel.run_mstep): NNLS over the n rows with
        h = beta1 - Y^T."""
        cfg = self.step_cfg
        if getattr(self, "hf_ev", None) is not None:
            torch.cuda.current_stream().wait_event(self.hf_ev)
            self.hf_ev = None
        if not getattr(self, "hf_rescaled", False):
            self.rescale(self.Hf, 2.0 * cfg.beta2, 1)
        self.hf_rescaled = False
        st = self.stats[k, 1]
        if self.d.kind == "dense" and self.mode == L.MODE_FAST:
            self.nnls(1, self.ybuf, L.F32, self.splits_m, self.r, self.n * self.r, cfg.beta1,
                      self.G, self.n, st)
        else:
            ycode = L.F64 if self.ybuf.dtype == torch.float64 else L.F32
            self.nnls(1, self.ybuf, ycode, 1, self.r, 0, cfg.beta1, self.G, self.n, st)

    def objective(self, k):
        """Objective pieces of iteration k into self.pieces[k] (nmf.py:152-165)."""
        cfg, d = self.cfg, self.d
        p = self.pieces[k]
        if d.kind == "dense" and self.use_tc:
            # k-major G^T for the residual, reused by the next coefficient step;
            # F = Ft[0] is current (made by this iteration's Y^T pass)
            q = k % 2
            Gt, Ft = self.Gt[q], self.Ft[q]
            L.call("nmfb_split_transpose", vp(self.G), self.n, self.r, vp(Gt[0]), vp(Gt[1]),
                   self._st())
            self.gt_valid = True
            if self.use_i8:
                # 8-bit slices of this iteration's G and F (snapshots: the side-stream
                # residual reads them while the next iteration overwrites G, FT)
                self._wait_residual(q)
                L.call("nmfb_slice_u8", vp(self.G), self.n, self.r, self.r, vp(self.Gsl[q]),
                       self._st())
                L.call("nmfb_slice_u8", vp(self.FT), self.m, self.r, self.r, vp(self.Fsl[q]),
                       self._st())
            # the residual runs on a side stream, overlapping the next iteration
            # (serial=True, for per-kernel timing: on the caller's stream)
            ready = torch.cuda.Event()
            ready.record()
            side = torch.cuda.current_stream() if getattr(self, "serial", False) else self.side
            side.wait_event(ready)
            with torch.cuda.stream(side):
                if self.use_i8:
                    L.call("nmfb_residual_i8", vp(d.X), self.n, self.m, vp(self.Gsl[q]),
                           vp(self.Fsl[q]), self.r, vp(p[0:1]), vp(self.rq_ws),
                           stream_handle(side))
                else:
                    L.call("nmfb_dense_residual_kmajor", vp(d.XT), self.m, self.n, vp(Gt[0]),
                           vp(Ft[0]), self.r, vp(p[0:1]), vp(self.res_ws),
                           stream_handle(side))
                ev = torch.cuda.Event()
                ev.record(side)
            self.res_ev[q] = ev
        elif d.kind == "dense":
            # 0.5 ||X - G F||^2 by tile residual; G F never stored
            L.call("nmfb_dense_residual", self.code, vp(d.XT), self.m, self.n, vp(self.G),
                   vp(self.FT), self.r, vp(p[0:1]), vp(self.res_ws), self._st())
        else:
            # trace identity (matrix.py:240-253): cross = <G, Y^T>, quad = <G^T G, F F^T>
            ycode = L.F64 if self.ybuf.dtype == torch.float64 else L.F32
            self.dot(self.G, self.code, self.ybuf, ycode, self.n * self.r, p[1:4])
            if self._overlap() is not None:
                # G^T G and the quad term on the side stream: they overlap the
                # next coefficient step's G^T X, which does not need them
                with self._on_side():
                    self.gram(self.G, self.n, self.Qg)
                    self.dot(self.Qg, L.F64, self.Hf, L.F64, self.r * self.r, p[7:10],
                             ws=self.dot_ws2)
                self.gside_ev = self._side_done()
            else:
                self.gram(self.G, self.n, self.Qg)
                self.dot(self.Qg, L.F64, self.Hf, L.F64, self.r * self.r, p[7:10])
            self.qg_valid = True  # reused by the next coefficient step
        # penalty sums: slots 4..6 = (-, sum|F|, sum F^2); 1..3 = (cross, sum|G|, sum G^2)
        if cfg.mu1 or cfg.mu2:
            self.dot(self.FT, self.code, None, L.F64, self.m * self.r, p[4:7])
        if (cfg.beta1 or cfg.beta2) and d.kind == "dense":
            self.dot(self.G, self.code, None, L.F64, self.n * self.r, p[1:4])

    def _wait_residual(self, q):
        """Main stream waits until the side-stream residual reading parity q is done."""
        ev = self.res_ev[q] if self.use_tc else None
        if ev is not None:
            torch.cuda.current_stream().wait_event(ev)
            self.res_ev[q] = None

    def join(self):
        """Make the caller's stream wait for all work of this state (the
        high-priority main stream and the side-stream objective)."""
        main = getattr(self, "main", None)
        if main is not None:
            with torch.cuda.stream(main):
                for q in (0, 1):
                    self._wait_residual(q)
            torch.cuda.current_stream().wait_stream(main)
        if getattr(self, "gside", None) is not None:
            torch.cuda.current_stream().wait_stream(self.gside)

    def snapshot(self):
        """Copy G, F^T (the state after the last enqueued iteration) into
        backup buffers, stream-ordered -- the lag-1 convergence check of
        FitSession.run keeps launching while it inspects the previous
        iteration, and rolls back if that one met the stopping rule."""
        if getattr(self, "_bak", None) is None:
            self._bak = (torch.empty_like(self.G), torch.empty_like(self.FT))
        main = getattr(self, "main", None)
        if main is not None:
            main.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(main):
                self._bak[0].copy_(self.G)
                self._bak[1].copy_(self.FT)
        else:
            self._bak[0].copy_(self.G)
            self._bak[1].copy_(self.FT)

    def restore(self):
        """G, F^T <- the last snapshot (after join())."""
        self.G.copy_(self._bak[0])
        self.FT.copy_(self._bak[1])

    def done_event(self, k):
        """An event on the caller's stream that completes when iteration k
        (both steps and its objective pieces) is done, without making the
        step streams wait."""
        cur = torch.cuda.current_stream()
        if getattr(self, "gside", None) is not None:
            # sparse overlap: observe the step stream and the side-stream Grams
            # from an auxiliary stream, so the next iteration's G^T X is not
            # held back behind the Gram it overlaps
            if getattr(self, "obs", None) is None:
                self.obs = torch.cuda.Stream(device=self.G.device)
            ev = torch.cuda.Event()
            ev.record(cur)
            self.obs.wait_event(ev)
            self.obs.wait_stream(self.gside)
            done = torch.cuda.Event(enable_timing=True)
            done.record(self.obs)
            return done
        main = getattr(self, "main", None)
        if main is not None:
            ev = torch.cuda.Event()
            ev.record(main)
            cur.wait_event(ev)
            res = self.res_ev[k % 2]
            if res is not None:
                cur.wait_event(res)
        done = torch.cuda.Event(enable_timing=True)
        done.record(cur)
        return done

    def iterate(self, k):
        main = getattr(self, "main", None)
        if main is None:
            self.estep(k)
            self.mstep(k)
            self.objective(k)
            return
        # the step runs on a high-priority stream so the FFMA-bound residual on
        # the low-priority side stream only fills SM slots the step leaves idle
        main.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(main):
            self.estep(k)
            self.mstep(k)
            self.objective(k)

    # -- host views ------------------------------------------------------------
    @staticmethod
    def assemble(pieces, cfg, kind, xsq):
        """nmf.py:152-165 from the device pieces (host fp64 scalar algebra)."""
        if kind == "dense":
            value = pieces[0]
        else:
            value = 0.5 * (xsq - 2.0 * pieces[1] + pieces[7])
        if cfg.mu1:
            value += cfg.mu1 * pieces[5]
        if cfg.beta1:
            value += cfg.beta1 * pieces[2]
        if cfg.mu2:
            value += cfg.mu2 * pieces[6]
        if cfg.beta2:
            value += cfg.beta2 * pieces[3]
        return float(value)

    def failure(self, stats_host, k):
        """First failing (step, index) at iteration k, or None."""
        for step, what in ((0, "coefficient solve failed at column"),
                           (1, "component solve failed at row")):
            f = int(stats_host[k, step, 1])
            if f != -1:
                return NumericalFailureError(f"{what} {f}", index=f)
        return None

    def factors_host(self):
        """(G, FT) as host float64 arrays for the model: G comes back
        column-major (the reference's DenseMatrix layout, matrix.py:20-59) --
        transposed on the device, so the host does no reordering pass -- and
        both through pinned buffers (full-rate D2H)."""
        Gt = self.G.t().to(torch.float64).contiguous()   # (r, n) = G column-major
        FT = self.FT.to(torch.float64).contiguous()
        # straight into freshly pinned result arrays (measured at C5: 0.09 s;
        # staging through reused buffers into pageable arrays: 0.18 s, the
        # first-touch page faults of the destination dominate)
        out = []
        for t in (Gt, FT):
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t, non_blocking=True)
            out.append(h)
        torch.cuda.current_stream().synchronize()
        return out[0].numpy().T, out[1].numpy()


# ---------------------------------------------------------------------------
# small host-API helpers (gram / objective of host arrays, on the device)
# ---------------------------------------------------------------------------
def gram_host(arr):
    dev = require_cuda()
    a = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).to(dev)
    rows, r = a.shape
    out = torch.empty((r, r), dtype=torch.float64, device=dev)
    ws = torch.empty((L.lib().nmfb_gram_workspace_bytes(rows, r) // 8 + 1,), dtype=torch.float64,
                     device=dev)
    L.call("nmfb_gram", L.F64, vp(a), rows, r, r, vp(out), vp(ws), stream_handle())
    return out.cpu().numpy()


def sparse_col_times_dense_host(v, col, g_arr):
    dev = require_cuda()
    g = torch.from_numpy(np.ascontiguousarray(g_arr, dtype=np.float64)).to(dev)
    lo, hi = int(v.indptr[col]), int(v.indptr[col + 1])
    r = g.shape[1]
    indptr = torch.tensor([0, hi - lo], dtype=torch.int64, device=dev)
    rows = torch.from_numpy(v.indices[lo:hi].astype(np.int32)).to(dev)
    vals = torch.from_numpy(v.values[lo:hi]).to(dev)
    h = torch.empty((r,), dtype=torch.float64, device=dev)
    L.call("nmfb_csc_linear", L.F64, L.MODE_REFERENCE, vp(indptr), vp(rows) if hi > lo else None,
           vp(vals) if hi > lo else None, 0, 1, vp(g), r, 0.0, vp(h), stream_handle())
    return -h.cpu().numpy()


def frobenius_objective_host(v, g_arr, f_arr):
    dev = require_cuda()
    r = g_arr.shape[1]
    G = torch.from_numpy(np.ascontiguousarray(g_arr, dtype=np.float64)).to(dev)
    FT = torch.from_numpy(np.ascontiguousarray(f_arr.T, dtype=np.float64)).to(dev)
    out = torch.zeros((12,), dtype=torch.float64, device=dev)
    if isinstance(v, SparseMatrix):
        d = DeviceData(v, "fp64", dev)
        Y = torch.empty((d.n, r), dtype=torch.float64, device=dev)
        ba, bp = L.bounds_array([0, d.m])
        L.call("nmfb_csr_yt", L.F64, L.MODE_FAST, vp(d.rowptr), vp(d.colidx), vp(d.cvals), d.n,
               vp(FT), r, L.F64, bp, 1, vp(Y), stream_handle())
        ws = torch.empty((L.lib().nmfb_dot_workspace_bytes(0) // 8 + 1,), dtype=torch.float64,
                         device=dev)
        L.call("nmfb_dot", vp(G), L.F64, vp(Y), L.F64, d.n * r, vp(out[1:4]), vp(ws),
               stream_handle())
        Hf = torch.empty((r, r), dtype=torch.float64, device=dev)
        Qg = torch.empty((r, r), dtype=torch.float64, device=dev)
        gws = torch.empty((L.lib().nmfb_gram_workspace_bytes(max(d.n, d.m), r) // 8 + 1,),
                          dtype=torch.float64, device=dev)
        L.call("nmfb_gram", L.F64, vp(FT), d.m, r, r, vp(Hf), vp(gws), stream_handle())
        L.call("nmfb_gram", L.F64, vp(G), d.n, r, r, vp(Qg), vp(gws), stream_handle())
        L.call("nmfb_dot", vp(Qg), L.F64, vp(Hf), L.F64, r * r, vp(out[7:10]), vp(ws),
               stream_handle())
        p = out.cpu().numpy()
        return 0.5 * (v.sum_squares() - 2.0 * p[1] + p[7])
    arr = v.array if isinstance(v, DenseMatrix) else np.asarray(v, dtype=np.float64)
    d = DeviceData(arr, "fp64", dev)
    ws = torch.empty((L.lib().nmfb_residual_workspace_bytes(d.m, d.n) // 8 + 1,),
                     dtype=torch.float64, device=dev)
    L.call("nmfb_dense_residual", L.F64, vp(d.XT), d.m, d.n, vp(G), vp(FT), r, vp(out[0:1]),
           vp(ws), stream_handle())
    return float(out[0].item())


def matvec_t_host(g_arr, v):
    """G^T v for a dense column (nmf.build_estep_problem), reference order."""
    dev = require_cuda()
    g = torch.from_numpy(np.ascontiguousarray(g_arr, dtype=np.float64)).to(dev)
    vt = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)[None, :]).to(dev)
    n, r = g.shape
    h = torch.empty((r,), dtype=torch.float64, device=dev)
    L.call("nmfb_dense_linear_ref", L.F64, vp(vt), n, 0, 1, vp(g), r, 0.0, vp(h),
           stream_handle())
    return -h.cpu().numpy()


def abs_sq_sums_host(arrays):
    """[(sum |a|, sum a^2) for each array] with fp64 device reductions."""
    dev = require_cuda()
    ws = torch.empty((L.lib().nmfb_dot_workspace_bytes(0) // 8 + 1,), dtype=torch.float64,
                     device=dev)
    out = []
    for a in arrays:
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)
        o = torch.zeros((3,), dtype=torch.float64, device=dev)
        L.call("nmfb_dot", vp(t), L.F64, None, L.F64, t.numel(), vp(o), vp(ws), stream_handle())
        oo = o.cpu().numpy()
        out.append((float(oo[1]), float(oo[2])))
    return out


def validate_and_sum(data):
    """Finite / nonnegative check (require_nonnegative, matrix.py:169-178) and
    sum(X) in fp64 for the init scale, on the device (dense data)."""
    from .exceptions import DataDomainError

    X = data.XT
    ws = torch.empty((L.lib().nmfb_dot_workspace_bytes(0) // 8 + 1,), dtype=torch.float64,
                     device=X.device)
    out = torch.zeros((3,), dtype=torch.float64, device=X.device)
    L.call("nmfb_data_stats", vp(X), _CODE[data.precision], X.numel(), vp(out), vp(ws),
           stream_handle())
    bad, total, _ = out.tolist()
    if bad > 0:
        if not bool(torch.isfinite(X).all()):
            raise DataDomainError("data matrix contains NaN or Inf")
        raise DataDomainError("data matrix contains negative entries")
    return float(total)  # sum |x| == sum x for nonnegative data
