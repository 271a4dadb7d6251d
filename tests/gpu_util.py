"""Helpers for the GPU parity tests: run the C-ABI kernels on numpy inputs."""

import numpy as np
import torch

from paper_1506_08938_b200 import _lib as L
from paper_1506_08938_b200 import device as D


def dev():
    return D.require_cuda()


def t(a, dtype=None):
    a = np.ascontiguousarray(a if dtype is None else np.asarray(a).astype(dtype))
    return torch.from_numpy(a).to(dev())


def rescale(H, diag_add=0.0, precision="fp64"):
    """nmfb_rescale -> dict of device buffers + host copies."""
    r = H.shape[0]
    dt = torch.float64 if precision == "fp64" else torch.float32
    b = dict(Qa=torch.zeros((r * r,), dtype=dt, device=dev()),
             sa=torch.zeros((r,), dtype=dt, device=dev()),
             act=torch.zeros((r,), dtype=torch.int32, device=dev()),
             active=torch.zeros((r,), dtype=torch.uint8, device=dev()),
             ra=torch.zeros((1,), dtype=torch.int32, device=dev()),
             scale=torch.zeros((r,), dtype=torch.float64, device=dev()))
    Hd = t(H, np.float64)
    L.call("nmfb_rescale", L.F64 if precision == "fp64" else L.F32, D.vp(Hd), r,
           float(diag_add), D.vp(b["Qa"]), D.vp(b["sa"]), D.vp(b["act"]), D.vp(b["active"]),
           D.vp(b["ra"]), D.vp(b["scale"]), D.stream_handle())
    ra = int(b["ra"].item())
    host = dict(ra=ra, Qa=b["Qa"][: ra * ra].double().cpu().numpy().reshape(ra, ra),
                scale_a=b["sa"][:ra].double().cpu().numpy(),
                act_idx=b["act"][:ra].cpu().numpy().astype(np.int64),
                active=b["active"].cpu().numpy().astype(bool))
    return b, host


def nnls(H, h, warm, eps, max_inner, precision="fp64", mode=None, h_base=None, index_base=0,
         max_stop0=0.0, lanes=0, diag_add=0.0):
    """Batched NNLS on the GPU.  If h_base is given the kernel forms
    h = h_base - hp (one partial, the M-step form); else hp is h itself.
    Returns (x, iters, finals, stats)."""
    count, r = h.shape
    b, _ = rescale(H, diag_add, precision)
    dt = np.float64 if precision == "fp64" else np.float32
    if mode is None:
        mode = L.MODE_REFERENCE if precision == "fp64" else L.MODE_FAST
    x = t(warm, dt)
    if h_base is None:
        hp, parts, base = t(h, dt), 0, 0.0
    else:
        hp, parts, base = t(h_base - h, dt), 1, float(h_base)
    iters = torch.zeros((count,), dtype=torch.int32, device=dev())
    finals = torch.zeros((count,), dtype=torch.float64 if precision == "fp64" else torch.float32,
                         device=dev())
    stats = torch.tensor([0, -1], dtype=torch.int64, device=dev())
    code = L.F64 if precision == "fp64" else L.F32
    L.call("nmfb_nnls_batch", code, mode, D.vp(b["Qa"]), D.vp(b["sa"]), D.vp(b["act"]),
           D.vp(b["active"]), r, r, D.vp(b["ra"]), D.vp(hp), code, parts, r, count * r, base,
           D.vp(x), count, index_base, float(eps), int(max_inner), float(max_stop0),
           D.vp(iters), D.vp(finals), D.vp(stats), lanes, D.stream_handle())
    torch.cuda.synchronize()
    return (x.double().cpu().numpy(), iters.cpu().numpy(), finals.double().cpu().numpy(),
            stats.cpu().numpy())


def running_max(finals, count, index_base=0, m0=0.0):
    """max_stop after each problem with 32-block resets (kernels.py:361-375)."""
    out = np.zeros(count)
    ms = m0
    for j in range(count):
        g = index_base + j
        if g % 32 == 0:
            ms = 0.0
        ms = max(ms, finals[j])
        out[j] = ms
    return out


def floored_rel(a, b, floor=1e-3):
    """max |a - b| / max(|b|, floor * max|b|) (SURVEY 7.3 P2 factor metric)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.maximum(np.abs(b), floor * max(np.max(np.abs(b)), 1e-300))
    return float(np.max(np.abs(a - b) / den)) if a.size else 0.0
