"""Drop-in device versions of the reference's compiled shard kernels.

Same names, argument order, meaning and return tuple as nmfkit/kernels.py
(estep_sparse :223-281, estep_dense :284-336, mstep_rows :339-378), executed
by libnmfb.so (nmfb_estep_sparse / nmfb_estep_dense / nmfb_mstep_rows).
Arrays may be numpy (copied to the device and back, in place) or CUDA torch
tensors (used in place).  float64 arrays run the reference-order kernels
(bit-identical results); float32 arrays run the fast kernels.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib as L
from . import device as D

FAIL_NONE = L.FAIL_NONE            # kernels.py:27
FASTBREAK_BLOCK = L.FASTBREAK_BLOCK  # kernels.py:35


class _Args:
    """Uploads numpy arguments once and writes in/out arrays back."""

    def __init__(self):
        self.dev = D.require_cuda()
        self.back = []
        self.keep = []  # device copies must outlive the (async) call

    def dev_t(self, a, dtype=None, inout=False):
        if isinstance(a, torch.Tensor):
            if not a.is_cuda or not a.is_contiguous():
                raise ValueError("torch arguments must be contiguous CUDA tensors")
            return a
        arr = np.asarray(a)
        t = torch.from_numpy(np.ascontiguousarray(arr if dtype is None else arr.astype(dtype)))
        t = t.to(self.dev)
        self.keep.append(t)
        if inout:
            self.back.append((a, t))
        return t

    def finish(self):
        torch.cuda.current_stream().synchronize()
        for host, t in self.back:
            host[...] = t.cpu().numpy()


def _code(a):
    dt = a.dtype if isinstance(a, torch.Tensor) else np.asarray(a).dtype
    if dt in (np.float64, torch.float64):
        return L.F64
    if dt in (np.float32, torch.float32):
        return L.F32
    raise TypeError(f"unsupported dtype {dt}")


def _call(name, *args):
    status = getattr(L.lib(), name)(*args)
    if status not in (L.NMFB_OK, L.NMFB_ERR_NUMERIC):
        L.check(status, name)


def estep_dense(VT, col_lo, col_hi, G, Qa, scale_a, act_idx, active, mu1, eps, max_inner,
                max_stop0, FT, YT, HP):
    """kernels.py:284-336 on the GPU -> (inner_total, max_stop, fail_col)."""
    a = _Args()
    code = _code(FT)
    dt = np.float64 if code == L.F64 else np.float32
    vt = a.dev_t(VT, dt)
    m, n = vt.shape
    inner, ms, fail = ctypes.c_int64(0), ctypes.c_double(0.0), ctypes.c_int64(-1)
    _call("nmfb_estep_dense", code, L.MODE_REFERENCE if code == L.F64 else L.MODE_FAST, D.vp(vt),
          m, n, int(col_lo), int(col_hi), D.vp(a.dev_t(G, dt)), FT.shape[1],
          D.vp(a.dev_t(Qa, dt)), D.vp(a.dev_t(scale_a, dt)), D.vp(a.dev_t(act_idx, np.int32)),
          len(act_idx), D.vp(a.dev_t(active, np.uint8)), float(mu1), float(eps), int(max_inner),
          float(max_stop0), D.vp(a.dev_t(FT, dt, True)), D.vp(a.dev_t(YT, dt, True)),
          D.vp(a.dev_t(HP, dt, True)), ctypes.byref(inner), ctypes.byref(ms), ctypes.byref(fail),
          D.stream_handle())
    a.finish()
    return inner.value, ms.value, fail.value


def estep_sparse(indptr, rowidx, vals, col_lo, col_hi, G, Qa, scale_a, act_idx, active, mu1,
                 eps, max_inner, max_stop0, FT, YT, HP):
    """kernels.py:223-281 on the GPU -> (inner_total, max_stop, fail_col)."""
    a = _Args()
    code = _code(FT)
    dt = np.float64 if code == L.F64 else np.float32
    m = len(indptr) - 1
    n = YT.shape[0]
    inner, ms, fail = ctypes.c_int64(0), ctypes.c_double(0.0), ctypes.c_int64(-1)
    _call("nmfb_estep_sparse", code, L.MODE_REFERENCE if code == L.F64 else L.MODE_FAST,
          D.vp(a.dev_t(indptr, np.int64)), D.vp(a.dev_t(rowidx, np.int32)),
          D.vp(a.dev_t(vals, dt)), m, n, int(col_lo), int(col_hi), D.vp(a.dev_t(G, dt)),
          FT.shape[1], D.vp(a.dev_t(Qa, dt)), D.vp(a.dev_t(scale_a, dt)),
          D.vp(a.dev_t(act_idx, np.int32)), len(act_idx), D.vp(a.dev_t(active, np.uint8)),
          float(mu1), float(eps), int(max_inner), float(max_stop0), D.vp(a.dev_t(FT, dt, True)),
          D.vp(a.dev_t(YT, dt, True)), D.vp(a.dev_t(HP, dt, True)), ctypes.byref(inner),
          ctypes.byref(ms), ctypes.byref(fail), D.stream_handle())
    a.finish()
    return inner.value, ms.value, fail.value


def mstep_rows(YT, row_lo, row_hi, Qa, scale_a, act_idx, active, beta1, eps, max_inner,
               max_stop0, G):
    """kernels.py:339-378 on the GPU -> (inner_total, max_stop, fail_row)."""
    a = _Args()
    code = _code(G)
    dt = np.float64 if code == L.F64 else np.float32
    inner, ms, fail = ctypes.c_int64(0), ctypes.c_double(0.0), ctypes.c_int64(-1)
    _call("nmfb_mstep_rows", code, L.MODE_REFERENCE if code == L.F64 else L.MODE_FAST,
          D.vp(a.dev_t(YT, dt)), int(row_lo), int(row_hi), D.vp(a.dev_t(Qa, dt)),
          D.vp(a.dev_t(scale_a, dt)), D.vp(a.dev_t(act_idx, np.int32)), len(act_idx),
          D.vp(a.dev_t(active, np.uint8)), float(beta1), float(eps), int(max_inner),
          float(max_stop0), D.vp(a.dev_t(G, dt, True)), G.shape[1], ctypes.byref(inner),
          ctypes.byref(ms), ctypes.byref(fail), D.stream_handle())
    a.finish()
    return inner.value, ms.value, fail.value
