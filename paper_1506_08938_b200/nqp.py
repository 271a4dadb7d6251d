"""Nonnegative quadratic programming: minimize 0.5 x'Hx + h'x subject to x >= 0.

Reference API (nqp.py): ``NqpProblem``, ``StopState``, ``rescale``,
``rescale_arrays``, ``passive_mask``, ``solve``.  The solve itself runs on the
GPU through libnmfb.so's reference-order kernel (``nmfb_nqp_solve``): the
anti-lopsided unit-diagonal rescaling (nmfb_rescale, bit-exact against
nqp.rescale_arrays), then exact line search + greedy coordinate descent with
the dual stopping rule, recording the per-iteration passive-gradient norm and
objective histories.  Validation, the two closed-form short-circuits
(h >= 0, KKT warm start; nqp.py:233-253) and the final unscaled gradient are
O(r^2) host arithmetic on the single problem.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .exceptions import DegenerateProblemError, NumericalFailureError

DIAG_FREEZE_REL = 1e-12  # nqp.py:33
DEFAULT_EPSILON = 0.1    # nqp.py:35
DEFAULT_MAX_INNER = 500  # nqp.py:36


@dataclass
class NqpProblem:
    """Quadratic form (H, h) with an optional nonnegative warm start (nqp.py:39-69)."""

    H: np.ndarray
    h: np.ndarray
    x0: np.ndarray | None = None

    def __post_init__(self):
        self.H = np.asarray(self.H, dtype=np.float64)
        self.h = np.asarray(self.h, dtype=np.float64)
        r = self.h.shape[0]
        if self.H.shape != (r, r):
            raise ValueError(f"H must be {r}x{r}, got {self.H.shape}")
        scale = max(1.0, float(np.max(np.abs(self.H))) if self.H.size else 1.0)
        if np.max(np.abs(self.H - self.H.T)) > 1e-12 * scale:
            raise ValueError("H must be symmetric within 1e-12")
        if np.any(np.diag(self.H) < 0):
            raise ValueError("diag(H) must be nonnegative")
        if self.x0 is None:
            self.x0 = np.zeros(r)
        else:
            self.x0 = np.asarray(self.x0, dtype=np.float64)
            if self.x0.shape != (r,):
                raise ValueError(f"x0 must have length {r}")
            if np.any(self.x0 < 0):
                raise ValueError("x0 must be nonnegative")

    @property
    def size(self):
        return self.h.shape[0]


@dataclass
class RescaledProblem:
    """Unit-diagonal form of an NqpProblem over its active dimensions (nqp.py:72-85)."""

    Q: np.ndarray
    q: np.ndarray
    scale: np.ndarray
    active_dims: np.ndarray


@dataclass
class NqpSolution:
    x: np.ndarray
    grad: np.ndarray
    inner_iterations: int
    initial_passive_grad_norm_sq: float
    final_passive_grad_norm_sq: float
    passive_grad_norm_history: np.ndarray
    objective_history: np.ndarray


@dataclass
class StopState:
    """Per-worker stopping state (nqp.py:98-113)."""

    epsilon: float = DEFAULT_EPSILON
    max_stop: float = 0.0

    def __post_init__(self):
        if not 0.0 <= self.epsilon <= 1.0:
            raise ValueError("epsilon must lie in [0, 1]")
        if self.max_stop < 0.0:
            raise ValueError("max_stop must be >= 0")

    def update(self, final_norm_sq):
        self.max_stop = max(self.max_stop, float(final_norm_sq))


def _device_rescale(H, diag_add=0.0):
    """nmfb_rescale on the GPU -> (scale, active, Qa compact, device buffers)."""
    import torch

    from . import _lib as L
    from . import device as D

    dev = D.require_cuda()
    r = H.shape[0]
    Hd = torch.from_numpy(np.ascontiguousarray(H, dtype=np.float64)).to(dev)
    bufs = dict(Qa=torch.zeros((max(r * r, 1),), dtype=torch.float64, device=dev),
                sa=torch.zeros((r,), dtype=torch.float64, device=dev),
                act=torch.zeros((r,), dtype=torch.int32, device=dev),
                active=torch.zeros((r,), dtype=torch.uint8, device=dev),
                ra=torch.zeros((1,), dtype=torch.int32, device=dev),
                scale=torch.zeros((r,), dtype=torch.float64, device=dev))
    L.call("nmfb_rescale", L.F64, D.vp(Hd), r, float(diag_add), D.vp(bufs["Qa"]),
           D.vp(bufs["sa"]), D.vp(bufs["act"]), D.vp(bufs["active"]), D.vp(bufs["ra"]),
           D.vp(bufs["scale"]), D.stream_handle())
    ra = int(bufs["ra"].item())
    active = bufs["active"].cpu().numpy().astype(bool)
    Qa = bufs["Qa"][: ra * ra].cpu().numpy().reshape(ra, ra)
    return bufs["scale"].cpu().numpy(), active, Qa, bufs


def rescale_arrays(H):
    """(scale, active mask, unit-diagonal Q) for a raw H (nqp.py:116-131).
    Computed by the GPU rescale kernel (bit-exact with the reference)."""
    H = np.asarray(H, dtype=np.float64)
    r = H.shape[0]
    if r == 0:
        return np.zeros(0), np.zeros(0, dtype=bool), np.zeros((0, 0))
    scale, active, Qa, _ = _device_rescale(H)
    Q = np.zeros((r, r))
    idx = np.flatnonzero(active)
    Q[np.ix_(idx, idx)] = Qa
    return scale, active, Q


def rescale(p: NqpProblem) -> RescaledProblem:
    """nqp.py:134-143; raises DegenerateProblemError if every dim is frozen."""
    scale, active, Q = rescale_arrays(p.H)
    if not active.any():
        raise DegenerateProblemError(
            "all diagonal entries are numerically zero; objective is linear in every variable")
    q = np.where(active, p.h / np.where(active, scale, 1.0), 0.0)
    return RescaledProblem(Q=Q, q=q, scale=scale, active_dims=active)


def passive_mask(x, grad):
    """Coordinates free to move: positive value or negative gradient (nqp.py:146-148)."""
    return (x > 0) | (grad < 0)


def _passive_norm_sq(x, grad):
    d = np.where(passive_mask(x, grad), grad, 0.0)
    return float(d @ d)


def _device_step(op, Q, x, grad, sweeps=-1):
    """nmfb_nqp_step on the GPU for one problem (1-D x, grad) or a batch of
    problems sharing Q (rows of 2-D x, grad)."""
    import torch

    from . import _lib as L
    from . import device as D

    dev = D.require_cuda()
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    grad = np.asarray(grad, dtype=np.float64)
    r = Q.shape[0]
    if Q.shape != (r, r) or x.shape[-1] != r or grad.shape != x.shape or x.ndim > 2:
        raise ValueError("Q must be r x r and x, grad (r,) or (count, r) alike")
    if r == 0:
        return x.copy(), grad.copy()
    xs, gs = np.atleast_2d(x), np.atleast_2d(grad)
    Qd = torch.from_numpy(Q).to(dev)
    xd = torch.from_numpy(np.ascontiguousarray(xs)).to(dev)
    gd = torch.from_numpy(np.ascontiguousarray(gs)).to(dev)
    L.call("nmfb_nqp_step", op, D.vp(Qd), r, D.vp(xd), D.vp(gd), xs.shape[0], int(sweeps),
           D.vp(xd), D.vp(gd), D.stream_handle())
    xo, go = xd.cpu().numpy(), gd.cpu().numpy()
    return (xo[0], go[0]) if x.ndim == 1 else (xo, go)


def exact_line_search_step(Q, q, x, grad):
    """One projected exact-line-search step along the passive-set gradient
    (nqp.py:151-183), on the GPU: alpha = |d|^2 / d'Qd (1 if the curvature is
    not positive), the projected point, the gradient updated over the changed
    coordinates, and the shortened step at the first breakpoint when the
    projection would increase the objective.  ``q`` is implicit in ``grad``
    (kept for the reference's signature).  x, grad may also be (count, r)
    batches sharing Q."""
    return _device_step(0, Q, x, grad)


def greedy_cd_pass(Q, q, x, grad, sweeps=None):
    """``sweeps`` (default r) greedy coordinate-descent updates (nqp.py:186-209)
    on the GPU: the clamped minimiser of the coordinate with the largest
    decrease (ties to the lowest index), unit-diagonal Q.  Batched like
    ``exact_line_search_step``."""
    if sweeps is not None and sweeps < 0:
        raise ValueError("sweeps must be >= 0")
    return _device_step(1, Q, x, grad, -1 if sweeps is None else int(sweeps))


def solve(p: NqpProblem, stop: StopState | None = None, max_inner: int = DEFAULT_MAX_INNER,
          check_gradients: bool = False) -> NqpSolution:
    """Solve an NQP problem to the accuracy governed by ``stop`` (nqp.py:217-320).

    The iterative solve runs on the GPU (reference-order fp64 kernel).
    ``check_gradients`` compares the incremental gradient with a fresh
    Q y + q after every inner iteration inside the kernel (nqp.py:295-299)
    and raises AssertionError at the first drift beyond 1e-9.
    """
    import torch

    from . import _lib as L
    from . import device as D

    if stop is None:
        stop = StopState()
    if max_inner < 1:
        raise ValueError("max_inner must be >= 1")
    r = p.size
    if np.all(p.h >= 0.0):
        stop.update(0.0)
        return NqpSolution(x=np.zeros(r), grad=p.h.copy(), inner_iterations=0,
                           initial_passive_grad_norm_sq=0.0, final_passive_grad_norm_sq=0.0,
                           passive_grad_norm_history=np.zeros(1), objective_history=np.zeros(1))
    grad0 = p.H @ p.x0 + p.h
    if _passive_norm_sq(p.x0, grad0) == 0.0:
        stop.update(0.0)
        f0 = float(0.5 * p.x0 @ grad0 + 0.5 * p.h @ p.x0)
        return NqpSolution(x=p.x0.copy(), grad=grad0, inner_iterations=0,
                           initial_passive_grad_norm_sq=0.0, final_passive_grad_norm_sq=0.0,
                           passive_grad_norm_history=np.zeros(1),
                           objective_history=np.asarray([f0]))
    scale, active, Qa, bufs = _device_rescale(p.H)
    if not active.any():
        raise DegenerateProblemError(
            "all diagonal entries are numerically zero; objective is linear in every variable")
    if np.any(p.h[~active] < 0.0):
        frozen = int(np.flatnonzero(~active & (p.h < 0.0))[0])
        raise NumericalFailureError(
            f"objective is unbounded along degenerate dimension {frozen} "
            f"(zero curvature, negative slope)", last_x=p.x0.copy())
    dev = bufs["Qa"].device
    h = torch.from_numpy(p.h.copy()).to(dev)
    x = torch.from_numpy(p.x0.copy()).to(dev)
    iters = torch.zeros((1,), dtype=torch.int32, device=dev)
    final = torch.zeros((1,), dtype=torch.float64, device=dev)
    hist = torch.zeros((max_inner + 1, 2), dtype=torch.float64, device=dev)
    stats = torch.tensor([0, -1], dtype=torch.int64, device=dev)
    L.call("nmfb_nqp_solve", D.vp(bufs["Qa"]), D.vp(bufs["sa"]), D.vp(bufs["act"]),
           D.vp(bufs["active"]), r, D.vp(bufs["ra"]), D.vp(h), D.vp(x), 1,
           float(stop.epsilon), int(max_inner), float(stop.max_stop), D.vp(iters), D.vp(final),
           D.vp(hist), max_inner + 1, 1 if check_gradients else 0, D.vp(stats),
           D.stream_handle())
    it = int(iters.item())
    if it == -2:
        raise AssertionError("incremental gradient drifted from Qx + q")
    if it < 0:
        raise NumericalFailureError(f"NaN/Inf after inner iterations (max {max_inner})",
                                    last_x=p.x0.copy())
    xs = x.cpu().numpy()
    hh = hist.cpu().numpy()[: it + 1]
    norm0 = float(hh[0, 0])
    norm_k = float(final.item())
    stop.update(norm_k)
    return NqpSolution(x=xs, grad=p.H @ xs + p.h, inner_iterations=it,
                       initial_passive_grad_norm_sq=norm0, final_passive_grad_norm_sq=norm_k,
                       passive_grad_norm_history=hh[:, 0].copy(),
                       objective_history=hh[:, 1].copy())


@dataclass
class NqpBatchSolution:
    """Solutions of a batch of NQP problems sharing one Hessian (row k of each
    array belongs to problem k; histories only when requested)."""

    x: np.ndarray                     # (count, r)
    grad: np.ndarray                  # (count, r) = H x + h
    inner_iterations: np.ndarray      # (count,) int
    initial_passive_grad_norm_sq: np.ndarray
    final_passive_grad_norm_sq: np.ndarray
    passive_grad_norm_history: np.ndarray | None = None  # (count, max_inner + 1), 0-padded
    objective_history: np.ndarray | None = None

    def __len__(self):
        return self.x.shape[0]

    def solution(self, k):
        """Problem k as the single-problem NqpSolution that ``solve`` returns."""
        it = int(self.inner_iterations[k])
        nh = self.passive_grad_norm_history
        oh = self.objective_history
        return NqpSolution(
            x=self.x[k].copy(), grad=self.grad[k].copy(), inner_iterations=it,
            initial_passive_grad_norm_sq=float(self.initial_passive_grad_norm_sq[k]),
            final_passive_grad_norm_sq=float(self.final_passive_grad_norm_sq[k]),
            passive_grad_norm_history=None if nh is None else nh[k, : it + 1].copy(),
            objective_history=None if oh is None else oh[k, : it + 1].copy())


def solve_batch(H, h, x0=None, epsilon=DEFAULT_EPSILON, max_inner=DEFAULT_MAX_INNER,
                max_stop=0.0, histories=True) -> NqpBatchSolution:
    """``solve`` (nqp.py:217-320) for many problems sharing H: problem k is
    NqpProblem(H, h[k], x0[k]) solved with its own StopState(epsilon,
    max_stop).  One rescale of H and ONE kernel launch for the whole batch
    (nmfb_nqp_solve, reference order, fp64); every problem's result is
    bit-identical to ``solve`` on it alone.  The closed-form short-circuits
    (h >= 0; a KKT warm start) are taken per problem as ``solve`` does.
    Errors: DegenerateProblemError when every diagonal of H is frozen and a
    problem needs the iterative solve; NumericalFailureError naming the
    lowest failing problem (``index``) otherwise."""
    import torch

    from . import _lib as L
    from . import device as D

    H = np.asarray(H, dtype=np.float64)
    h = np.atleast_2d(np.asarray(h, dtype=np.float64))
    count, r = h.shape
    NqpProblem(H, h[0] if count else np.zeros(H.shape[0]))  # H validation (nqp.py:52-61)
    if x0 is None:
        x0 = np.zeros((count, r))
    x0 = np.atleast_2d(np.asarray(x0, dtype=np.float64))
    if x0.shape != (count, r):
        raise ValueError(f"x0 must be {count}x{r}")
    if np.any(x0 < 0):
        raise ValueError("x0 must be nonnegative")
    StopState(epsilon, max_stop)  # argument validation
    if max_inner < 1:
        raise ValueError("max_inner must be >= 1")
    # the KKT short-circuit (nqp.py:241-253) is an exact-zero test: every row
    # with a nonzero warm start gets the same matrix-vector product ``solve``
    # computes (H @ x0 + h), so its decision is bit-identical; a zero warm
    # start has grad0 = h exactly
    grad0 = h.copy()
    for k in np.flatnonzero(np.any(x0 != 0.0, axis=1)):
        grad0[k] = H @ x0[k] + h[k]
    pas = (x0 > 0) | (grad0 < 0)
    norm0 = np.einsum("ij,ij->i", np.where(pas, grad0, 0.0), np.where(pas, grad0, 0.0))
    zero_h = np.all(h >= 0.0, axis=1)
    kkt = ~zero_h & (norm0 == 0.0)
    run = np.flatnonzero(~zero_h & ~kkt)
    x = np.where(zero_h[:, None], 0.0, x0)
    iters = np.zeros(count, dtype=np.int64)
    init = np.zeros(count)
    final = np.zeros(count)
    nh = np.zeros((count, max_inner + 1)) if histories else None
    oh = np.zeros((count, max_inner + 1)) if histories else None
    if histories:  # closed forms: a single history entry (nqp.py:233-253)
        for k in np.flatnonzero(kkt):
            oh[k, 0] = float(0.5 * x0[k] @ grad0[k] + 0.5 * h[k] @ x0[k])
    if run.size:
        scale, active, Qa, bufs = _device_rescale(H)
        if not active.any():
            raise DegenerateProblemError(
                "all diagonal entries are numerically zero; objective is linear in every "
                "variable")
        bad = np.any(h[run][:, ~active] < 0.0, axis=1)
        if bad.any():
            k = int(run[np.flatnonzero(bad)[0]])
            frozen = int(np.flatnonzero(~active & (h[k] < 0.0))[0])
            raise NumericalFailureError(
                f"objective is unbounded along degenerate dimension {frozen} "
                f"(zero curvature, negative slope) in problem {k}", index=k,
                last_x=x0[k].copy())
        dev = bufs["Qa"].device
        hd = torch.from_numpy(np.ascontiguousarray(h[run])).to(dev)
        xd = torch.from_numpy(np.ascontiguousarray(x0[run])).to(dev)
        it_d = torch.zeros((run.size,), dtype=torch.int32, device=dev)
        fin_d = torch.zeros((run.size,), dtype=torch.float64, device=dev)
        # without histories the kernel still records entry 0 (the initial
        # rescaled passive-gradient norm that ``solve`` reports)
        hl = max_inner + 1 if histories else 1
        hist = torch.zeros((run.size, hl, 2), dtype=torch.float64, device=dev)
        stats = torch.tensor([0, -1], dtype=torch.int64, device=dev)
        L.call("nmfb_nqp_solve", D.vp(bufs["Qa"]), D.vp(bufs["sa"]), D.vp(bufs["act"]),
               D.vp(bufs["active"]), r, D.vp(bufs["ra"]), D.vp(hd), D.vp(xd), int(run.size),
               float(epsilon), int(max_inner), float(max_stop), D.vp(it_d), D.vp(fin_d),
               D.vp(hist), hl, 0, D.vp(stats), D.stream_handle())
        it = it_d.cpu().numpy().astype(np.int64)
        if np.any(it < 0):
            k = int(run[np.flatnonzero(it < 0)[0]])
            raise NumericalFailureError(
                f"NaN/Inf after inner iterations (max {max_inner}) in problem {k}", index=k,
                last_x=x0[k].copy())
        x[run] = xd.cpu().numpy()
        iters[run] = it
        final[run] = fin_d.cpu().numpy()
        hh = hist.cpu().numpy()
        init[run] = hh[:, 0, 0]
        if histories:
            for t, k in enumerate(run):
                nh[k, : it[t] + 1] = hh[t, : it[t] + 1, 0]
                oh[k, : it[t] + 1] = hh[t, : it[t] + 1, 1]
    # final gradient per problem as ``solve`` forms it (H @ x + h)
    grad = h.copy()
    for k in np.flatnonzero(np.any(x != 0.0, axis=1)):
        grad[k] = H @ x[k] + h[k]
    return NqpBatchSolution(x=x, grad=grad, inner_iterations=iters,
                            initial_passive_grad_norm_sq=init,
                            final_passive_grad_norm_sq=final,
                            passive_grad_norm_history=nh, objective_history=oh)
