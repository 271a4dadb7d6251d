"""Alternating factorization driver on the B200 (reference nmf.py API).

``fit(V, cfg, on_iteration=None)`` runs the reference's alternation
(nmf.py:168-211) with every numeric step on the GPU (device.Alternation).
The reference's ``fit`` reads an undefined global ``on_iteration``
(nmf.py:197); here it is the evident intended keyword: a
callback invoked with the ConvergenceLog after every outer iteration.

Host work per fit: seeded factor initialisation (numpy PCG64, exactly
nmf.py:115-127 so both sides start from identical bits), one upload of X and
the factors, one download of the factors and the per-iteration log.  Without
an early-exit tolerance or a callback there is no host synchronisation
inside the loop.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import device as D
from .ingest import DeviceCsc
from .exceptions import NumericalFailureError
from .matrix import (DenseMatrix, SparseMatrix, exact_sum, frobenius_objective, require_nonnegative,
                     sparse_col_times_dense)
from .nqp import DEFAULT_EPSILON, DEFAULT_MAX_INNER, NqpProblem

PRECISIONS = ("fp32", "fp64")


@dataclass
class NmfConfig:
    """Knobs for one factorization run (nmf.py:34-70).

    B200 additions: ``precision`` -- "fp32" (production kernels) or "fp64"
    (reference-order check mode, bit-exact steps); ``lanes`` -- lanes per
    subproblem of the fp32 NNLS kernel (0 = auto).
    """

    rank: int
    max_outer: int = 300
    epsilon: float = DEFAULT_EPSILON
    mu1: float = 0.0
    mu2: float = 0.0
    beta1: float = 0.0
    beta2: float = 0.0
    workers: int = 1
    seed: int = 0
    inner_cap: int = DEFAULT_MAX_INNER
    rel_change_tol: float = 1e-10
    precision: str = "fp32"
    lanes: int = 0

    def __post_init__(self):
        if self.rank < 1:
            raise ValueError("rank must be >= 1")
        if not 0.0 <= self.epsilon <= 1.0:
            raise ValueError("epsilon must lie in [0, 1]")
        for name in ("mu1", "mu2", "beta1", "beta2"):
            if getattr(self, name) < 0.0:
                raise ValueError(f"{name} must be >= 0")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.max_outer < 1:
            raise ValueError("max_outer must be >= 1")
        if self.inner_cap < 1:
            raise ValueError("inner_cap must be >= 1")
        if self.precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {PRECISIONS}")
        if self.rank > 256:
            raise ValueError("rank must be <= 256 on this build")
        if self.precision == "fp32" and self.rank > 224:
            # the fp32 NNLS kernel stages the compact Q in shared memory
            # (224 x 224 fp32 is the largest that fits next to its h rows)
            raise ValueError("rank must be <= 224 with precision='fp32' (use 'fp64' above)")


@dataclass
class NmfModel:
    """Nonnegative factors: components G (n x r) and coefficients F (r x m)."""

    G: DenseMatrix
    F: DenseMatrix


@dataclass
class ConvergenceLog:
    """nmf.py:81-102: objective, cumulative seconds, inner iterations, k_bar."""

    objective: list = field(default_factory=list)
    seconds: list = field(default_factory=list)
    inner_iterations: list = field(default_factory=list)
    k_bar: list = field(default_factory=list)

    def append(self, objective, seconds, inner_iterations, subproblems):
        self.objective.append(float(objective))
        self.seconds.append(float(seconds))
        self.inner_iterations.append(int(inner_iterations))
        self.k_bar.append(inner_iterations / subproblems)

    def __len__(self):
        return len(self.objective)

    @property
    def final_objective(self):
        return self.objective[-1]


def _shape(V):
    return V.rows, V.cols


def _mean(V):
    """nmf.py:109-112."""
    n, m = _shape(V)
    # np.sum's value bit for bit; long sparse value vectors on worker threads
    total = exact_sum(V.values) if isinstance(V, SparseMatrix) else float(np.sum(V.array))
    return total / (n * m)


def initial_factors(V, cfg):
    """nmf.py:115-127: seeded U[0,1) factors, G drawn before F."""
    n, m = _shape(V)
    return initial_factors_from_mean(n, m, _mean(V), cfg)


def initial_draws(n, m, cfg):
    """The seeded U[0,1) draws of nmf.py:115-127 (G before F)."""
    rng = np.random.default_rng(cfg.seed)
    return rng.uniform(size=(n, cfg.rank)), rng.uniform(size=(cfg.rank, m))


def scale_draws(draws, mean, cfg):
    u_g, u_f = draws
    scale = np.sqrt(mean / cfg.rank)
    g = np.ascontiguousarray(u_g * scale)
    ft = np.ascontiguousarray((u_f * scale).T)
    return g, ft


def device_initial_factors(n, m, mean, cfg, device=None):
    """initial_factors on the GPU: numpy's PCG64 stream for cfg.seed
    regenerated in parallel (csrc/init.cu), bit-identical to the host draw,
    scaled by sqrt(mean / r) in fp64 and rounded once to cfg.precision's
    dtype.  Returns device tensors (G (n, r), FT (m, r))."""
    from . import _lib as L

    device = device or D.require_cuda()
    st = np.random.PCG64(cfg.seed).state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    mask = (1 << 64) - 1
    dt = torch.float32 if cfg.precision == "fp32" else torch.float64
    G = torch.empty((n, cfg.rank), dtype=dt, device=device)
    FT = torch.empty((m, cfg.rank), dtype=dt, device=device)
    scale = float(np.sqrt(mean / cfg.rank))
    L.call("nmfb_init_factors", s >> 64, s & mask, inc >> 64, inc & mask, n, m, cfg.rank, scale,
           L.F32 if dt == torch.float32 else L.F64, D.vp(G), D.vp(FT), D.stream_handle())
    return G, FT


def initial_factors_from_mean(n, m, mean, cfg):
    return scale_draws(initial_draws(n, m, cfg), mean, cfg)


def build_estep_problem(Q_g, V, col, G, cfg, warm=None):
    """nmf.py:130-140: H = G^T G + 2 mu2 I, h = -G^T V_col + mu1."""
    r = Q_g.array.shape[0]
    H = Q_g.array + (2.0 * cfg.mu2) * np.eye(r)
    if isinstance(V, SparseMatrix):
        gtv = sparse_col_times_dense(V, col, G)
    else:
        gtv = D.matvec_t_host(G.array, V.array[:, col])
    h = -gtv + cfg.mu1
    return NqpProblem(H, h, warm)


def build_mstep_problem(H_f, Y, row, cfg, warm=None):
    """nmf.py:143-149: H = F F^T + 2 beta2 I, h = -Y_row + beta1."""
    r = H_f.array.shape[0]
    H = H_f.array + (2.0 * cfg.beta2) * np.eye(r)
    h = -Y.array[:, row] + cfg.beta1
    return NqpProblem(H, h, warm)


def regularized_objective(V, model, cfg):
    """nmf.py:152-165, evaluated on the GPU."""
    g = model.G.array
    f = model.F.array
    value = frobenius_objective(V, model.G, model.F)
    if cfg.mu1 or cfg.beta1 or cfg.mu2 or cfg.beta2:
        sums = D.abs_sq_sums_host([f, g])
        if cfg.mu1:
            value += cfg.mu1 * sums[0][0]
        if cfg.beta1:
            value += cfg.beta1 * sums[1][0]
        if cfg.mu2:
            value += cfg.mu2 * sums[0][1]
        if cfg.beta2:
            value += cfg.beta2 * sums[1][1]
    return value


def _as_matrix(V):
    if isinstance(V, (DenseMatrix, SparseMatrix)):
        return V
    if isinstance(V, torch.Tensor):
        V = V.detach().cpu().numpy()
    return DenseMatrix(V)


class FitSession:
    """A prepared fit: data uploaded, factors initialised, loop ready.

    ``run()`` executes the alternation and returns (NmfModel, ConvergenceLog).
    Splitting preparation from the loop lets callers (bench.py) time the
    device-resident loop separately from the end-to-end call.
    """

    def __init__(self, V, cfg, on_iteration=None, init=None, data=None, solver="nnls"):
        self.cfg = cfg
        self.on_iteration = on_iteration
        if data is None and isinstance(V, torch.Tensor):
            # torch input (e.g. a pinned host buffer): upload first, validate
            # and take the mean for the init scale on the device
            data = D.DeviceData(V, cfg.precision)  # asynchronous upload
            n, m = data.n, data.m
            # the init is drawn on the device once the mean is known
            total = D.validate_and_sum(data)
            if init is None:
                init = device_initial_factors(n, m, total / (n * m), cfg, data.device)
        elif data is None and isinstance(V, DeviceCsc):
            # sparse data already on the GPU (ingest.DeviceCsc): checked and
            # averaged there; the init draws are the same host PCG64 stream
            V.validate()
            data = D.DeviceData(V, cfg.precision)
            n, m = V.rows, V.cols
            if init is None:
                init = device_initial_factors(n, m, D.device_sums(V.values)[0] / (n * m), cfg,
                                              data.device)
        elif data is None:
            from concurrent.futures import ThreadPoolExecutor

            V = _as_matrix(V)
            # the host checks (matrix.py:169-178) and the host mean (numpy's
            # summation, as nmf.py:109-112 -- the init must be the reference's
            # bit for bit) run on worker threads while this thread uploads X;
            # the reference's error still wins over any device-side one
            with ThreadPoolExecutor(2) as pool:
                fchk = pool.submit(require_nonnegative, V, "data matrix")
                fmean = pool.submit(_mean, V) if init is None else None
                dev_err = None
                try:
                    data = D.DeviceData(V, cfg.precision)
                except Exception as exc:  # noqa: BLE001 -- re-raised below
                    dev_err = exc
                fchk.result()
                if dev_err is not None:
                    raise dev_err
                mean = fmean.result() if fmean is not None else None
            n, m = _shape(V)
            if init is None:
                # the draws on the device
                init = device_initial_factors(n, m, mean, cfg, data.device)
        else:
            n, m = data.n, data.m
            if init is None:
                raise ValueError("init factors required with preloaded device data")
        self.n, self.m = n, m
        self.data = data
        G0, FT0 = init
        self.state = D.Alternation(data, cfg, G0, FT0, cfg.max_outer, precision=cfg.precision,
                                   lanes=cfg.lanes, solver=solver)

    def run(self):
        cfg, st = self.cfg, self.state
        # the stopping rule / callback need every objective on the host
        sync_each = cfg.rel_change_tol > 0.0 or self.on_iteration is not None
        start = torch.cuda.Event(enable_timing=True)
        log = ConvergenceLog()
        start.record()
        xsq = getattr(self.data, "xsq", 0.0)
        try:
            if sync_each:
                self._run_lagged(st, log, start, xsq)
            else:
                # fixed iteration count: launch everything, read the log once
                events = []
                for k in range(cfg.max_outer):
                    st.iterate(k)
                    events.append(st.done_event(k))
                st.join()
                done = len(events)
                if done:
                    events[-1].synchronize()
                stats = st.stats[:done].cpu().numpy()
                pieces = st.pieces[:done].cpu().numpy()
                for k in range(done):
                    err = st.failure(stats, k)
                    if err is not None:
                        raise err
                    obj = st.assemble(pieces[k], cfg, self.data.kind, xsq)
                    log.append(obj, start.elapsed_time(events[k]) / 1e3,
                               int(stats[k, :, 0].sum()), self.m + self.n)
        except NumericalFailureError as err:
            err.log = log
            raise
        G, FT = st.factors_host()
        model = NmfModel(G=DenseMatrix(G), F=DenseMatrix(np.asfortranarray(FT.T)))
        return model, log

    def _check(self, st, log, k, ev, start, xsq, previous):
        """Host-side bookkeeping of iteration k (nmf.py:193-206) once its
        event is done: failure, log entry, callback, stopping rule.  Returns
        (stop, objective)."""
        cfg = self.cfg
        ev.synchronize()
        stats = st.stats[k].cpu().numpy()
        err = st.failure(stats[None], 0)
        if err is not None:
            raise err
        obj = st.assemble(st.pieces[k].cpu().numpy(), cfg, self.data.kind, xsq)
        log.append(obj, start.elapsed_time(ev) / 1e3, int(stats[:, 0].sum()), self.m + self.n)
        if self.on_iteration is not None:
            self.on_iteration(log)
        stop = (cfg.rel_change_tol > 0.0 and previous is not None
                and abs(previous - obj) <= cfg.rel_change_tol * max(abs(previous), 1e-300))
        return stop, obj

    def _run_lagged(self, st, log, start, xsq):
        """Per-iteration convergence check without a per-iteration stall:
        iteration k+1 is enqueued before the host inspects iteration k (the
        objective needs a device->host read).  A snapshot of (G, F) taken
        before k+1 lets the fit return exactly the state after k when k met
        the stopping rule -- the same result as the synchronous loop."""
        cfg = self.cfg
        pending = None  # (k, event)
        previous = None
        for k in range(cfg.max_outer):
            if pending is not None:
                st.snapshot()  # state after iteration k - 1
            st.iterate(k)
            if pending is not None:
                # inspect k - 1 while k runs; the caller's stream has no wait
                # on iteration k queued yet, so the reads do not stall on it
                stop, previous = self._check(st, log, pending[0], pending[1], start, xsq,
                                             previous)
                if stop:
                    st.join()
                    st.restore()
                    return pending[0] + 1
            pending = (k, st.done_event(k))
        if pending is not None:
            self._check(st, log, pending[0], pending[1], start, xsq, previous)
        st.join()
        return cfg.max_outer


def fit(V, cfg, on_iteration=None):
    """Run the alternation for cfg.max_outer iterations (or until the relative
    objective change falls below cfg.rel_change_tol) -- nmf.py:168-211.

    Deterministic for a fixed seed.  Raises NumericalFailureError (with the
    log up to the failure and the failing column/row index) if a subproblem
    degenerates.
    """
    return FitSession(V, cfg, on_iteration=on_iteration).run()
