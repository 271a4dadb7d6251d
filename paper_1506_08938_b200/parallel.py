"""Partitioned execution of the alternation steps (reference parallel.py API).

On one B200 the "workers" of the reference are not threads: every column of
the coefficient step and every row of the component step is one subproblem of
a single batched kernel launch.  ``cfg.workers`` is still honoured where it
changes numbers: the reference sums per-worker accumulators in worker order
(parallel.py:141-159), and the fp64 check mode reproduces exactly that order.
Shards stay aligned to FASTBREAK_BLOCK (parallel.py:162-169), so the
subproblem solutions never depend on the partition -- which is also what
makes the multi-GPU column sharding (dist.py) exact.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from . import device as D
from .exceptions import MatrixSizeError
from .matrix import DenseMatrix, SparseMatrix

MSTEP_DISTRIBUTE_FLOPS = 10_000_000  # parallel.py:28 (kept for API parity)
FASTBREAK_BLOCK = L.FASTBREAK_BLOCK


@dataclass
class WorkerPlan:
    """Contiguous shard bounds over [0, total); reduction follows list order."""

    workers: int
    shards: list

    @property
    def sizes(self):
        return [hi - lo for lo, hi in self.shards]


def plan(total, workers):
    """parallel.py:72-84: near-equal contiguous shards."""
    shards = D.plan(total, workers)
    return WorkerPlan(workers=len(shards), shards=shards)


def block_plan(total, workers):
    """parallel.py:162-169: shards aligned to the fast-break block size."""
    shards = D.block_plan(total, workers)
    return WorkerPlan(workers=len(shards), shards=shards)


@dataclass
class StepStats:
    inner_iterations: int = 0
    workers: int = 1
    peak_worker_reals: int = 0


def _vt_as_data(V, precision):
    if isinstance(V, SparseMatrix):
        return D.DeviceData(V, precision)
    vt = V.array.T if isinstance(V, DenseMatrix) else np.asarray(V)
    # run_estep receives V^T (m, n) exactly like the reference (nmf.py:183-191)
    return D.DeviceData(np.asarray(vt).T, precision)


def run_estep(V, G, Q_g, cfg, F):
    """Coefficient step on the GPU (parallel.py:172-186).

    V: SparseMatrix or the (m, n) transposed dense data; G (n, r); Q_g (r, r);
    F: the (m, r) coefficient array, overwritten in place.  Returns
    (Y (r x n), H_f (r x r), StepStats) like the reference.
    """
    data = _vt_as_data(V, cfg.precision)
    G = np.asarray(G)
    Qg = Q_g.array if isinstance(Q_g, DenseMatrix) else np.asarray(Q_g)
    st = D.Alternation(data, cfg, G, F, 1, precision=cfg.precision, lanes=cfg.lanes, overlap=False,
                       splits=1)
    st.Qg.copy_(torch.from_numpy(np.ascontiguousarray(Qg, dtype=np.float64)))
    st.qg_valid = True
    st.estep(0)
    stats = st.stats[0, 0].cpu().numpy()
    if int(stats[1]) != -1:
        from .exceptions import NumericalFailureError
        raise NumericalFailureError(f"coefficient solve failed at column {int(stats[1])}",
                                    index=int(stats[1]))
    F[...] = st.FT.double().cpu().numpy()
    yt = st.ybuf.view(data.n, cfg.rank).double().cpu().numpy()
    Y = DenseMatrix(yt.T)
    H = DenseMatrix(st.Hf.cpu().numpy())
    reals = st.ybuf.numel() + st.Hf.numel() + 12 * cfg.rank
    return Y, H, StepStats(inner_iterations=int(stats[0]), workers=len(st.bounds_e) - 1,
                           peak_worker_reals=int(reals))


def run_mstep(Y, H_f, cfg, G):
    """Component step on the GPU (parallel.py:189-223); G updated in place."""
    n, r = G.shape
    Ya = Y.array if isinstance(Y, DenseMatrix) else np.asarray(Y)
    Ha = H_f.array if isinstance(H_f, DenseMatrix) else np.asarray(H_f)
    if Ya.shape != (r, n) or Ha.shape != (r, r):
        raise MatrixSizeError("Y must be r x n and H_f r x r")
    dev = D.require_cuda()
    dt = D._TORCH[cfg.precision]
    data = D.DeviceData.__new__(D.DeviceData)
    data.device, data.kind, data.n, data.m = dev, "none", n, 0
    st = D.Alternation.__new__(D.Alternation)
    st.d, st.cfg, st.prec, st.code = data, cfg, cfg.precision, D._CODE[cfg.precision]
    st.step_cfg, st.solver = cfg, "nnls"
    st.mode = L.MODE_REFERENCE if cfg.precision == "fp64" else L.MODE_FAST
    st.lanes, st.n, st.m, st.r = cfg.lanes, n, 0, r
    st.G = torch.from_numpy(np.ascontiguousarray(G)).to(dev, dt)
    st.Hf = torch.from_numpy(np.ascontiguousarray(Ha, dtype=np.float64)).to(dev)
    st.Qa = [None, torch.zeros((r * r,), dtype=dt, device=dev)]
    st.sa = [None, torch.zeros((r,), dtype=dt, device=dev)]
    st.act = [None, torch.zeros((r,), dtype=torch.int32, device=dev)]
    st.active = [None, torch.zeros((r,), dtype=torch.uint8, device=dev)]
    st.ra = [None, torch.zeros((1,), dtype=torch.int32, device=dev)]
    ydt = torch.float64 if cfg.precision == "fp64" else torch.float32
    st.ybuf = torch.from_numpy(np.ascontiguousarray(Ya.T)).to(dev, ydt).reshape(-1)
    st.splits_m = 1
    st.stats = torch.zeros((1, 2, 2), dtype=torch.int64, device=dev)
    st.stats[:, :, 1] = -1
    st.mstep(0)
    stats = st.stats[0, 1].cpu().numpy()
    if int(stats[1]) != -1:
        from .exceptions import NumericalFailureError
        raise NumericalFailureError(f"component solve failed at row {int(stats[1])}",
                                    index=int(stats[1]))
    G[...] = st.G.double().cpu().numpy()
    workers = cfg.workers if n * r * r > MSTEP_DISTRIBUTE_FLOPS else 1
    return StepStats(inner_iterations=int(stats[0]), workers=len(D.block_plan(n, workers)),
                     peak_worker_reals=12 * r)
