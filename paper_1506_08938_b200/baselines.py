"""Comparison solver on the GPU: the multiplicative update rule (reference
baselines.py:41-85), SURVEY.md 8(f) row 4.

``mur_fit(V, cfg)`` runs the classical Lee-Seung updation
    F <- F * (G'V) / (G'G F + floor),  then  G <- G * (V F') / (G (F F') + floor)
with the updated F, from the same seeded start as ``fit`` and with the same
log format: the data products G'V and V F' are the alternating-NNLS path's own
kernels (tcgen05 GEMM / CSC-CSR SpMM / reference-order fp64), the Grams are
``nmfb_gram``, and the elementwise update is ``nmfb_mur_update``
(csrc/mur.cu).  Penalty weights are ignored by the steps and kept in the
logged objective (baselines.py:58-63); k_bar is identically 1.
"""

from __future__ import annotations

import enum

import numpy as np

MUR_FLOOR = 1e-12  # baselines.py:20


class BaselineKind(enum.Enum):
    """baselines.py:23-25 (the plain exact-line-search single-problem solver
    is not on the factorization path and is not provided on the GPU)."""

    MUR = "mur"


def mur_fit(V, cfg, on_iteration=None):
    """baselines.py:55-85 on the device -> (NmfModel, ConvergenceLog)."""
    from .nmf import FitSession

    return FitSession(V, cfg, on_iteration=on_iteration, solver="mur").run()


def mur_step(V, G, F, precision="fp64"):
    """One multiplicative update of both factors (baselines.py:41-52):
    G (n, r), F (r, m) host arrays in, updated copies out."""
    import torch

    from .nmf import FitSession, NmfConfig

    G = np.ascontiguousarray(G, dtype=np.float64)
    FT = np.ascontiguousarray(np.asarray(F, dtype=np.float64).T)
    cfg = NmfConfig(rank=G.shape[1], max_outer=1, rel_change_tol=0.0, precision=precision)
    st = FitSession(V, cfg, init=(G, FT), solver="mur").state
    st.estep(0)
    st.mstep(0)
    torch.cuda.synchronize()
    return st.G.double().cpu().numpy(), st.FT.double().cpu().numpy().T.copy()
