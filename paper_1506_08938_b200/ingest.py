"""Sparse data matrices built and checked on the GPU.

The reference ingests on the host with numpy (matrix.py): ``from_triplets``
sorts, sums duplicates and drops zeros (matrix.py:104-125), ``transpose``
re-sorts for row access (matrix.py:149-154), and ``_validate`` checks the CSC
invariants with a per-column Python loop (matrix.py:81-101).  At config 5
(1e8 nonzeros) that host work, not the iterations, dominates a fit's wall
time.  ``DeviceCsc`` does the same on the device (csrc/ingest.cu):

* ``DeviceCsc.from_triplets(rows, cols, i, j, v, sum_duplicates=True)`` --
  identical CSC (indices exact, duplicate sums bit-identical to np.add.at);
* ``DeviceCsc.from_host(SparseMatrix)`` -- upload + on-device checks;
* ``.csr()`` -- the CSR twin the Y^T pass reads (= ``transpose()``'s arrays);
* ``.validate()`` -- the reference's checks, raising the reference's
  exception types and messages; ``.to_host()`` -- back to a SparseMatrix.

``fit`` accepts a ``DeviceCsc`` directly (the data never leaves the GPU).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from .exceptions import DataDomainError, MatrixSizeError

_NO_FAULT = (1 << 63) - 1

_MESSAGES = {
    L.INGEST_TRIPLET_RANGE: (MatrixSizeError, "triplet index out of range"),
    L.INGEST_INDPTR_SPAN: (MatrixSizeError, "column pointers must span [0, nnz]"),
    L.INGEST_INDPTR_ORDER: (MatrixSizeError, "column pointers must be non-decreasing"),
    L.INGEST_ROW_RANGE: (MatrixSizeError, "row index out of range"),
    L.INGEST_ROW_ORDER: (MatrixSizeError, "row indices not strictly increasing in column {}"),
    L.INGEST_NONFINITE: (DataDomainError, "sparse values must be finite"),
    L.INGEST_NONPOSITIVE: (DataDomainError,
                           "stored sparse values must be > 0 (no explicit zeros)"),
}
# the order in which the reference's checks run (matrix.py:81-101)
_ORDER = (L.INGEST_TRIPLET_RANGE, L.INGEST_INDPTR_SPAN, L.INGEST_INDPTR_ORDER,
          L.INGEST_ROW_RANGE, L.INGEST_ROW_ORDER, L.INGEST_NONFINITE, L.INGEST_NONPOSITIVE)


def _vp(t):
    return None if t is None else t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _device():
    from .device import require_cuda

    return require_cuda()


def release_scratch():
    """Hand the ingest kernels' cached scratch (kept mapped between ingests to
    avoid re-mapping GBs per call) back to the driver (nmfb_ingest_release_scratch)."""
    _device()
    L.call("nmfb_ingest_release_scratch")


def raise_for(info, codes=_ORDER):
    """Raise the reference's exception for the first failing check in `info`
    (host int64 array of NMFB_INGEST_CODES entries)."""
    for c in codes:
        if int(info[c]) != _NO_FAULT:
            exc, msg = _MESSAGES[c]
            raise exc(msg.format(int(info[c])))


def _dev_array(a, dtype, device):
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a), dtype=_NP[dtype])).to(device)


_NP = {torch.int64: np.int64, torch.float64: np.float64, torch.float32: np.float32,
       torch.int32: np.int32}
_CODE = {torch.float32: L.F32, torch.float64: L.F64}


class DeviceCsc:
    """CSC matrix on the GPU: indptr (cols+1, int64), rowidx (nnz, int32
    ascending within a column), values (nnz, float64 or float32)."""

    def __init__(self, rows, cols, indptr, rowidx, values, validate=True):
        self.rows, self.cols = int(rows), int(cols)
        self.indptr, self.rowidx, self.values = indptr, rowidx, values
        self._csr = None
        if self.indptr.numel() != self.cols + 1:
            raise MatrixSizeError("column pointer array must have cols+1 entries")
        if self.rowidx.numel() != self.values.numel():
            raise MatrixSizeError("row-index and value arrays must match")
        if validate:
            self.validate()

    @property
    def nnz(self):
        return self.values.numel()

    @property
    def device(self):
        return self.values.device

    @property
    def dtype(self):
        return self.values.dtype

    def __repr__(self):
        return f"DeviceCsc({self.rows}x{self.cols}, nnz={self.nnz}, {self.dtype})"

    # -- construction -----------------------------------------------------
    @classmethod
    def from_triplets(cls, rows, cols, i, j, v, sum_duplicates=True, dtype=torch.float64,
                      device=None):
        """matrix.py:104-125 on the device; i, j, v host arrays or tensors."""
        device = device or _device()
        rows, cols = int(rows), int(cols)
        i = _dev_array(i, torch.int64, device).reshape(-1)
        j = _dev_array(j, torch.int64, device).reshape(-1)
        v = _dev_array(v, torch.float64, device).reshape(-1)
        if not (i.numel() == j.numel() == v.numel()):
            raise MatrixSizeError("triplet arrays must have equal length")
        count = i.numel()
        if rows >= 2**31 or count >= 2**32:
            raise MatrixSizeError("sizes must fit the device index types")
        indptr = torch.empty(cols + 1, dtype=torch.int64, device=device)
        rowidx = torch.empty(max(count, 1), dtype=torch.int32, device=device)
        vals = torch.empty(max(count, 1), dtype=dtype, device=device)
        nnz = torch.zeros(1, dtype=torch.int64, device=device)
        info = torch.empty(L.INGEST_CODES, dtype=torch.int64, device=device)
        L.call("nmfb_csc_from_triplets", rows, cols, count, _vp(i), _vp(j), _vp(v),
               1 if sum_duplicates else 0, _vp(indptr), _vp(rowidx), _vp(vals), _CODE[dtype],
               _vp(nnz), _vp(info), _stream())
        host = info.cpu().numpy()
        raise_for(host, (L.INGEST_TRIPLET_RANGE,))
        k = int(nnz.item())
        # the reference builds through the validating constructor (matrix.py:125)
        return cls(rows, cols, indptr, rowidx[:k], vals[:k], validate=True)

    @classmethod
    def from_host(cls, V, dtype=torch.float64, device=None, validate=True):
        """Upload a host SparseMatrix (int64 indices narrowed on the device)."""
        device = device or _device()
        if V.rows >= 2**31 or V.nnz >= 2**32:
            raise MatrixSizeError("sizes must fit the device index types")
        indptr = torch.from_numpy(np.ascontiguousarray(V.indptr, dtype=np.int64)).to(
            device, non_blocking=True)
        from .device import upload_host

        # the big arrays through pinned staging (threaded host copies, the
        # float64 -> dtype cast on the device)
        idx64 = upload_host(np.ascontiguousarray(V.indices, dtype=np.int64), torch.int64,
                            device)
        rowidx = torch.empty(max(V.nnz, 1), dtype=torch.int32, device=device)[: V.nnz]
        info = torch.empty(L.INGEST_CODES, dtype=torch.int64, device=device)
        L.call("nmfb_narrow_indices", _vp(idx64), V.nnz, _vp(rowidx), _vp(info), _stream())
        vals = upload_host(np.ascontiguousarray(V.values, dtype=np.float64), dtype, device)
        del idx64
        if validate:
            raise_for(info.cpu().numpy(), (L.INGEST_ROW_RANGE,))
        return cls(V.rows, V.cols, indptr, rowidx, vals, validate=validate)

    # -- checks and views -----------------------------------------------------
    def validate(self):
        """matrix.py:81-101 (+ require_nonnegative's finiteness) on the device."""
        info = torch.empty(L.INGEST_CODES, dtype=torch.int64, device=self.device)
        L.call("nmfb_csc_validate", self.rows, self.cols, self.nnz, _vp(self.indptr),
               _vp(self.rowidx), _vp(self.values), _CODE[self.dtype], _vp(info), _stream())
        raise_for(info.cpu().numpy())
        return self

    def csr(self):
        """(rowptr int64, colidx int32, values) of the same matrix, columns
        ascending within a row (the reference's transpose(), cached)."""
        if self._csr is None:
            dev = self.device
            rowptr = torch.empty(self.rows + 1, dtype=torch.int64, device=dev)
            colidx = torch.empty(max(self.nnz, 1), dtype=torch.int32, device=dev)[: self.nnz]
            cvals = torch.empty(max(self.nnz, 1), dtype=self.dtype, device=dev)[: self.nnz]
            L.call("nmfb_csc_to_csr", self.rows, self.cols, self.nnz, _vp(self.indptr),
                   _vp(self.rowidx), _vp(self.values), _CODE[self.dtype], _vp(rowptr),
                   _vp(colidx), _vp(cvals), _stream())
            self._csr = (rowptr, colidx, cvals)
        return self._csr

    def transpose(self):
        """DeviceCsc of X^T (matrix.py:149-154)."""
        rowptr, colidx, cvals = self.csr()
        return DeviceCsc(self.cols, self.rows, rowptr, colidx, cvals, validate=False)

    def to_host(self):
        from .matrix import SparseMatrix

        return SparseMatrix(self.rows, self.cols, self.indptr.cpu().numpy(),
                            self.rowidx.cpu().numpy().astype(np.int64),
                            self.values.double().cpu().numpy(), validate=False)

    def sum_squares(self):
        from .device import device_sum_squares

        return device_sum_squares(self.values)
