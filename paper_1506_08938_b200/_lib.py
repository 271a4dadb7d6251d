"""ctypes binding of libnmfb.so (the C ABI declared in include/nmfb.h).

There is no fallback: if the library is missing, or no CUDA device is
present, every entry point raises.  Torch tensors cross the boundary only as
``data_ptr()`` integers plus the current CUDA stream handle.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .exceptions import NumericalFailureError

PKG = os.path.dirname(os.path.abspath(__file__))
# NMFB_LIB_PATH: an alternative in-tree build (A/B timing of two builds)
LIB_PATH = os.environ.get("NMFB_LIB_PATH") or os.path.join(PKG, "libnmfb.so")

NMFB_OK = 0
NMFB_ERR_NUMERIC = 1
NMFB_ERR_ARG = 2
NMFB_ERR_CUDA = 3
NMFB_ERR_DEGENERATE = 4
F32, F64 = 0, 1
MODE_FAST, MODE_REFERENCE = 0, 1
FAIL_NONE = -1
FASTBREAK_BLOCK = 32
# sparse-ingest check codes (include/nmfb.h NMFB_INGEST_*)
INGEST_TRIPLET_RANGE, INGEST_INDPTR_SPAN, INGEST_INDPTR_ORDER, INGEST_ROW_RANGE, \
    INGEST_ROW_ORDER, INGEST_NONFINITE, INGEST_NONPOSITIVE = range(7)
INGEST_CODES = 7
UINT64_MAX = (1 << 64) - 1

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_int = ctypes.c_int
_f64 = ctypes.c_double
_sz = ctypes.c_size_t
_pi64 = ctypes.POINTER(ctypes.c_int64)
_pf64 = ctypes.POINTER(ctypes.c_double)

# name -> (restype, argtypes); mirrors include/nmfb.h
SIGNATURES = {
    "nmfb_version": (_int, []),
    "nmfb_last_error": (ctypes.c_char_p, []),
    "nmfb_device_sm_count": (_int, []),
    "nmfb_estep_dense": (_int, [_int, _int, _vp, _i64, _i64, _i64, _i64, _vp, _i32, _vp, _vp, _vp,
                                _i32, _vp, _f64, _f64, _i32, _f64, _vp, _vp, _vp, _pi64, _pf64,
                                _pi64, _vp]),
    "nmfb_estep_sparse": (_int, [_int, _int, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _i32,
                                 _vp, _vp, _vp, _i32, _vp, _f64, _f64, _i32, _f64, _vp, _vp, _vp,
                                 _pi64, _pf64, _pi64, _vp]),
    "nmfb_mstep_rows": (_int, [_int, _int, _vp, _i64, _i64, _vp, _vp, _vp, _i32, _vp, _f64, _f64,
                               _i32, _f64, _vp, _i32, _pi64, _pf64, _pi64, _vp]),
    "nmfb_nnls_batch": (_int, [_int, _int, _vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _int, _i32,
                               _i64, _i64, _f64, _vp, _i64, _i64, _f64, _i32, _f64, _vp, _vp, _vp,
                               _i32, _vp]),
    "nmfb_nqp_solve": (_int, [_vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _i64, _f64, _i32, _f64,
                              _vp, _vp, _vp, _i32, _i32, _vp, _vp]),
    "nmfb_nqp_step": (_int, [_i32, _vp, _i32, _vp, _vp, _i64, _i32, _vp, _vp, _vp]),
    "nmfb_gram_workspace_bytes": (_sz, [_i64, _i32]),
    "nmfb_gram": (_int, [_int, _vp, _i64, _i32, _i64, _vp, _vp, _vp]),
    "nmfb_gram_rescale": (_int, [_int, _vp, _i64, _i32, _i64, _vp, _vp, _f64, _vp, _vp, _vp, _vp,
                                 _vp, _vp]),
    "nmfb_rescale": (_int, [_int, _vp, _i32, _f64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "nmfb_gemm_tall": (_int, [_vp, _int, _i64, _i64, _i64, _vp, _i32, _i64, _vp, _i32, _vp]),
    "nmfb_dense_linear_ref": (_int, [_int, _vp, _i64, _i64, _i64, _vp, _i32, _f64, _vp, _vp]),
    "nmfb_dense_yt_ref": (_int, [_int, _vp, _i64, _i64, _vp, _i32, _pi64, _i32, _vp, _vp]),
    "nmfb_hp_ref": (_int, [_int, _vp, _i64, _i32, _pi64, _i32, _vp, _vp]),
    "nmfb_csc_linear": (_int, [_int, _int, _vp, _vp, _vp, _i64, _i64, _vp, _i32, _f64, _vp, _vp]),
    "nmfb_csr_yt": (_int, [_int, _int, _vp, _vp, _vp, _i64, _vp, _i32, _int, _pi64, _i32, _vp,
                           _vp]),
    "nmfb_csr_yt_chunked": (_int, [_int, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _i32, _int, _vp,
                                   _vp, _vp]),
    "nmfb_residual_workspace_bytes": (_sz, [_i64, _i64]),
    "nmfb_dense_residual": (_int, [_int, _vp, _i64, _i64, _vp, _vp, _i32, _vp, _vp, _vp]),
    "nmfb_dense_residual_kmajor": (_int, [_vp, _i64, _i64, _vp, _vp, _i32, _vp, _vp, _vp]),
    "nmfb_dot_workspace_bytes": (_sz, [_i64]),
    "nmfb_data_stats": (_int, [_vp, _int, _i64, _vp, _vp, _vp]),
    "nmfb_sum_parts": (_int, [_vp, _i32, _i64, _vp, _vp]),
    "nmfb_tc_gemm": (_int, [_vp, _i64, _i64, _vp, _vp, _i32, _vp, _i32, _i32, _vp]),
    "nmfb_tc_splits": (_int, [_i64, _i32]),
    "nmfb_tc_parts": (_int, [_i64, _i64, _i32, _i32]),
    "nmfb_slice_bytes": (_sz, [_i64, _i32]),
    "nmfb_slice_u8": (_int, [_vp, _i64, _i32, _i64, _vp, _vp]),
    "nmfb_residual_i8_workspace_bytes": (_sz, []),
    "nmfb_residual_i8": (_int, [_vp, _i64, _i64, _vp, _vp, _i32, _vp, _vp, _vp]),
    "nmfb_split_transpose": (_int, [_vp, _i64, _i32, _vp, _vp, _vp]),
    "nmfb_transpose": (_int, [_vp, _i64, _i64, _vp, _vp]),
    "nmfb_dot": (_int, [_vp, _int, _vp, _int, _i64, _vp, _vp, _vp]),
    "nmfb_tc_gemm_rows": (_int, [_vp, _i64, _i64, _vp, _vp, _i32, _i32, _vp, _i32, _i64, _i32,
                                 _vp]),
    "nmfb_nnls_batch_peers": (_int, [_int, _int, _vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _int,
                                     _i32, _i64, _i64, _f64, _vp, _i64, _i64, _f64, _i32, _f64,
                                     _vp, _vp, _vp, _i32, _vp, _i32, _vp]),
    "nmfb_peer_put": (_int, [_vp, _i64, _vp, _i32, _i32, _vp, _vp, ctypes.c_uint64, _i32, _vp]),
    "nmfb_peer_wait": (_int, [_vp, _i32, ctypes.c_uint64, _f64, _vp]),
    "nmfb_sum_slots_f64": (_int, [_vp, _i32, _i64, _i64, _vp, _vp]),
    "nmfb_csc_from_triplets": (_int, [_i64, _i64, _i64, _vp, _vp, _vp, _int, _vp, _vp, _vp, _int,
                                      _vp, _vp, _vp]),
    "nmfb_csc_to_csr": (_int, [_i64, _i64, _i64, _vp, _vp, _vp, _int, _vp, _vp, _vp, _vp]),
    "nmfb_csc_validate": (_int, [_i64, _i64, _i64, _vp, _vp, _vp, _int, _vp, _vp]),
    "nmfb_ingest_release_scratch": (_int, []),
    "nmfb_csr_chunk_plan": (_int, [_vp, _i64, _i64, _vp, _vp, _vp, _vp]),
    "nmfb_comm_available": (_int, []),
    "nmfb_comm_unique_id": (_int, [_vp]),
    "nmfb_comm_init": (_int, [_vp, _i32, _i32, _vp]),
    "nmfb_comm_destroy": (_int, [_vp]),
    "nmfb_allreduce_r2": (_int, [_vp, _vp, _i64, _vp]),
    "nmfb_reduce_scatter_panel": (_int, [_vp, _vp, _vp, _i64, _int, _vp]),
    "nmfb_allgather_panel": (_int, [_vp, _vp, _vp, _i64, _int, _vp]),
    "nmfb_narrow_indices": (_int, [_vp, _i64, _vp, _vp, _vp]),
    "nmfb_sum_slots_rescale": (_int, [_int, _vp, _i32, _i64, _vp, _i32, _f64, _vp, _vp, _vp, _vp,
                                      _vp, _vp]),
    "nmfb_csc_segments": (_int, [_vp, _vp, _i64, _i64, _i32, _vp, _vp]),
    "nmfb_chunk_segments": (_int, [_vp, _i64, _vp, _i64, _i32, _vp, _vp]),
    "nmfb_csc_linear_blocked": (_int, [_vp, _vp, _i32, _vp, _vp, _i64, _vp, _i32, _f64, _vp,
                                       _vp]),
    "nmfb_csr_yt_chunked_blocked": (_int, [_vp, _i64, _vp, _i64, _vp, _i32, _vp, _vp, _vp, _i32,
                                           _int, _vp, _vp, _vp]),
    "nmfb_init_factors": (_int, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                 ctypes.c_uint64, _i64, _i64, _i32, _f64, _int, _vp, _vp, _vp]),
    "nmfb_mur_update": (_int, [_int, _vp, _i32, _vp, _int, _i32, _i64, _i64, _f64, _vp, _i64,
                               _f64, _vp, _vp]),
}

MAX_PEERS = 8  # NMFB_MAX_PEERS


def ptr_array(ptrs):
    """Host array of device pointers (the `void *const *` arguments)."""
    return (ctypes.c_void_p * max(len(ptrs), 1))(*[ctypes.c_void_p(int(p)) for p in ptrs])

_lib = None


class NativeLibraryError(RuntimeError):
    """libnmfb.so is missing or a CUDA call failed (no CPU fallback exists)."""


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} not found: build it with `python -m paper_1506_08938_b200.build` "
                "(this package has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("NMFB_LIB_PATH") and not hasattr(L, name):
                continue  # an older A/B build may lack newer entry points
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return sorted(SIGNATURES)


def check(status, what):
    if status == NMFB_OK:
        return
    if status == NMFB_ERR_CUDA:
        msg = lib().nmfb_last_error().decode(errors="replace")
        raise NativeLibraryError(f"{what}: CUDA error: {msg}")
    if status == NMFB_ERR_ARG:
        raise ValueError(f"{what}: invalid argument")
    raise NativeLibraryError(f"{what}: status {status}")


# kernels launched by one call of each entry point (gpu_launches accounting)
KERNELS_PER_CALL = {
    "nmfb_nnls_batch": 1, "nmfb_nqp_solve": 1, "nmfb_nqp_step": 1, "nmfb_gram": 2, "nmfb_rescale": 1,
    "nmfb_gemm_tall": 1, "nmfb_dense_linear_ref": 1, "nmfb_dense_yt_ref": 1, "nmfb_hp_ref": 1,
    "nmfb_csc_linear": 1, "nmfb_csr_yt": 1, "nmfb_dense_residual": 2, "nmfb_dot": 2,
    "nmfb_sum_parts": 1, "nmfb_dense_residual_kmajor": 2, "nmfb_csr_yt_chunked": 2, "nmfb_tc_gemm": 1, "nmfb_split_transpose": 1, "nmfb_transpose": 1,
    "nmfb_slice_u8": 1, "nmfb_residual_i8": 2, "nmfb_gram_rescale": 2, "nmfb_data_stats": 2,
    "nmfb_tc_gemm_rows": 1, "nmfb_nnls_batch_peers": 1, "nmfb_peer_put": 1, "nmfb_peer_wait": 1,
    "nmfb_sum_slots_f64": 1, "nmfb_csc_from_triplets": 11, "nmfb_csc_to_csr": 8,
    "nmfb_csc_validate": 2, "nmfb_narrow_indices": 2, "nmfb_mur_update": 1,
    "nmfb_ingest_release_scratch": 0, "nmfb_csr_chunk_plan": 5, "nmfb_comm_available": 0, "nmfb_comm_unique_id": 0,
    "nmfb_comm_init": 0, "nmfb_comm_destroy": 0, "nmfb_allreduce_r2": 1,
    "nmfb_reduce_scatter_panel": 1, "nmfb_allgather_panel": 1,
    "nmfb_init_factors": 1, "nmfb_csc_segments": 1, "nmfb_chunk_segments": 1, "nmfb_sum_slots_rescale": 1,
    "nmfb_csc_linear_blocked": 1, "nmfb_csr_yt_chunked_blocked": 2,
}


class Recorder:
    """Counts kernel launches and (optionally) times every C-ABI call with
    CUDA events on the current stream: ``with Recorder(timing=True) as rec``."""

    active = None

    def __init__(self, timing=False):
        # timing: True (every call), False, or a set of entry-point names
        self.timing = timing
        self.launches = 0
        self.calls = []  # (name, start_event, end_event)

    def __enter__(self):
        Recorder.active = self
        return self

    def __exit__(self, *exc):
        Recorder.active = None

    def summary(self):
        """{name: (calls, total_ms)} (call after synchronizing)."""
        out = {}
        for name, a, b in self.calls:
            c, t = out.get(name, (0, 0.0))
            out[name] = (c + 1, t + a.elapsed_time(b))
        return out


def call(name, *args):
    rec = Recorder.active
    if rec is not None:
        rec.launches += KERNELS_PER_CALL.get(name, 0)
        if rec.timing is True or (rec.timing and name in rec.timing):
            import torch

            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            status = getattr(lib(), name)(*args)
            b.record()
            rec.calls.append((name, a, b))
            check(status, name)
            return status
    status = getattr(lib(), name)(*args)
    check(status, name)
    return status


def bounds_array(bounds):
    arr = np.ascontiguousarray(np.asarray(bounds, dtype=np.int64))
    return arr, arr.ctypes.data_as(_pi64)


def numeric_failure(what, index):
    return NumericalFailureError(f"{what} failed at {index}", index=int(index))
