"""numpy + C restatement of the reference's alternating-NNLS loop.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Every function cites the
reference file:line it restates (paths relative to the reference's
``pkg/src/nmfkit/``).  Expressions, array memory orders and summation orders
are kept identical to the reference so the results are bit-identical on the
same machine (checked against committed golden vectors).

The one intentional deviation: ``fit`` takes ``on_iteration=None``.  The
reference reads an undefined global ``on_iteration`` at nmf.py:197 and raises
NameError on every call; the evident intent is a per-iteration callback
(SURVEY.md 0.3), which is what this restatement implements.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

FAIL_NONE = -1            # kernels.py:27
FASTBREAK_BLOCK = 32      # kernels.py:35
DIAG_FREEZE_REL = 1e-12   # nqp.py:33
DEFAULT_EPSILON = 0.1     # nqp.py:35
DEFAULT_MAX_INNER = 500   # nqp.py:36
MSTEP_DISTRIBUTE_FLOPS = 10_000_000  # parallel.py:28


class OracleNumericalFailure(RuntimeError):
    """Mirror of exceptions.py:26-39 NumericalFailureError (index, log)."""

    def __init__(self, message, index=None, log=None):
        super().__init__(message)
        self.index = index
        self.log = log


# --------------------------------------------------------------------------
# C kernels (nnls_oracle.c) via ctypes; ctypes releases the GIL, so shard
# workers run in parallel exactly like the reference's nogil numba kernels.
# --------------------------------------------------------------------------
_lib = None
_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int64)
_B = ctypes.POINTER(ctypes.c_uint8)
_i64 = ctypes.c_int64
_f64 = ctypes.c_double


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.oracle_estep_dense.restype = _i64
        L.oracle_estep_dense.argtypes = [_D, _i64, _i64, _i64, _D, _i64, _D, _D, _I, _i64, _B,
                                         _f64, _f64, _i64, _f64, _D, _D, _D, _I, _D]
        L.oracle_estep_sparse.restype = _i64
        L.oracle_estep_sparse.argtypes = [_I, _I, _D, _i64, _i64, _D, _i64, _D, _D, _I, _i64, _B,
                                          _f64, _f64, _i64, _f64, _D, _D, _D, _I, _D]
        L.oracle_mstep_rows.restype = _i64
        L.oracle_mstep_rows.argtypes = [_D, _i64, _i64, _D, _D, _I, _i64, _B, _f64, _f64, _i64,
                                        _f64, _D, _i64, _I, _D]
        L.oracle_coefficient_solve.restype = _i64
        L.oracle_coefficient_solve.argtypes = [_D, _i64, _I, _i64, _B, _D, _D, _D, _f64, _f64,
                                               _i64, _D, _D, _D]
        L.oracle_sparse_cross.restype = _f64
        L.oracle_sparse_cross.argtypes = [_I, _I, _D, _i64, _i64, _D, _D, _i64]
        _lib = L
    return _lib


def _p(a, kind=_D):
    return a.ctypes.data_as(kind)


def _check(a, dtype, name):
    if a.dtype != dtype or not a.flags["C_CONTIGUOUS"]:
        raise TypeError(f"{name} must be C-contiguous {dtype}")


def estep_dense(VT, col_lo, col_hi, G, Qa, scale_a, act_idx, active, mu1, eps, max_inner,
                max_stop0, FT, YT, HP):
    """kernels.py:284-336 -> (inner_total, max_stop, fail_col)."""
    for a, nm in ((VT, "VT"), (G, "G"), (Qa, "Qa"), (scale_a, "scale_a"), (FT, "FT"),
                  (YT, "YT"), (HP, "HP")):
        _check(a, np.float64, nm)
    act_idx = np.ascontiguousarray(act_idx, dtype=np.int64)
    active = np.ascontiguousarray(active, dtype=np.uint8)
    inner = ctypes.c_int64(0)
    ms = ctypes.c_double(0.0)
    fail = lib().oracle_estep_dense(
        _p(VT), VT.shape[1], col_lo, col_hi, _p(G), FT.shape[1], _p(Qa), _p(scale_a),
        _p(act_idx, _I), act_idx.shape[0], _p(active, _B), mu1, eps, max_inner, max_stop0,
        _p(FT), _p(YT), _p(HP), ctypes.byref(inner), ctypes.byref(ms))
    return inner.value, ms.value, fail


def estep_sparse(indptr, rowidx, vals, col_lo, col_hi, G, Qa, scale_a, act_idx, active, mu1,
                 eps, max_inner, max_stop0, FT, YT, HP):
    """kernels.py:223-281 -> (inner_total, max_stop, fail_col)."""
    for a, nm in ((vals, "vals"), (G, "G"), (Qa, "Qa"), (scale_a, "scale_a"), (FT, "FT"),
                  (YT, "YT"), (HP, "HP")):
        _check(a, np.float64, nm)
    _check(indptr, np.int64, "indptr")
    _check(rowidx, np.int64, "rowidx")
    act_idx = np.ascontiguousarray(act_idx, dtype=np.int64)
    active = np.ascontiguousarray(active, dtype=np.uint8)
    inner = ctypes.c_int64(0)
    ms = ctypes.c_double(0.0)
    fail = lib().oracle_estep_sparse(
        _p(indptr, _I), _p(rowidx, _I), _p(vals), col_lo, col_hi, _p(G), FT.shape[1], _p(Qa),
        _p(scale_a), _p(act_idx, _I), act_idx.shape[0], _p(active, _B), mu1, eps, max_inner,
        max_stop0, _p(FT), _p(YT), _p(HP), ctypes.byref(inner), ctypes.byref(ms))
    return inner.value, ms.value, fail


def mstep_rows(YT, row_lo, row_hi, Qa, scale_a, act_idx, active, beta1, eps, max_inner,
               max_stop0, G):
    """kernels.py:339-378 -> (inner_total, max_stop, fail_row)."""
    for a, nm in ((YT, "YT"), (Qa, "Qa"), (scale_a, "scale_a"), (G, "G")):
        _check(a, np.float64, nm)
    act_idx = np.ascontiguousarray(act_idx, dtype=np.int64)
    active = np.ascontiguousarray(active, dtype=np.uint8)
    inner = ctypes.c_int64(0)
    ms = ctypes.c_double(0.0)
    fail = lib().oracle_mstep_rows(
        _p(YT), row_lo, row_hi, _p(Qa), _p(scale_a), _p(act_idx, _I), act_idx.shape[0],
        _p(active, _B), beta1, eps, max_inner, max_stop0, _p(G), G.shape[1],
        ctypes.byref(inner), ctypes.byref(ms))
    return inner.value, ms.value, fail


def coefficient_solve(h, act_idx, active, scale_a, Qa, warm, eps, max_stop, max_inner):
    """kernels.py:178-220 for one problem -> (iterations, final_norm_sq, x)."""
    h = np.ascontiguousarray(h, dtype=np.float64)
    warm = np.ascontiguousarray(warm, dtype=np.float64)
    act_idx = np.ascontiguousarray(act_idx, dtype=np.int64)
    active = np.ascontiguousarray(active, dtype=np.uint8)
    ra = act_idx.shape[0]
    x = np.zeros(h.shape[0])
    nk = ctypes.c_double(0.0)
    work = np.zeros(7 * max(ra, 1))
    it = lib().oracle_coefficient_solve(
        _p(h), h.shape[0], _p(act_idx, _I), ra, _p(active, _B), _p(scale_a), _p(Qa), _p(warm),
        eps, max_stop, max_inner, _p(x), ctypes.byref(nk), _p(work))
    return it, nk.value, x


# --------------------------------------------------------------------------
# nqp.py pieces on the fit path
# --------------------------------------------------------------------------
def rescale_arrays(H):
    """nqp.py:116-131: (scale, active mask, unit-diagonal Q) for a raw H."""
    diag = np.diag(H).copy()
    delta = DIAG_FREEZE_REL * (float(diag.max()) if diag.size else 0.0)
    active = diag > delta
    scale = np.sqrt(diag)
    q_scale = np.where(active, scale, 1.0)
    Q = H / np.outer(q_scale, q_scale)
    Q[~active, :] = 0.0
    Q[:, ~active] = 0.0
    Q[np.diag_indices_from(Q)] = np.where(active, 1.0, 0.0)
    return scale, active, Q


def rescale_for_step(H):
    """parallel.py:87-91 -> (scale_a, active, act_idx, Qa)."""
    scale, active, Q = rescale_arrays(H)
    idx = np.flatnonzero(active)
    Qa = np.ascontiguousarray(Q[np.ix_(idx, idx)])
    return scale[idx].copy(), active, idx.astype(np.int64), Qa


# --------------------------------------------------------------------------
# matrix.py pieces
# --------------------------------------------------------------------------
class Csc:
    """matrix.py:62-166 SparseMatrix layout: CSC, int64 indices, values > 0."""

    __slots__ = ("rows", "cols", "indptr", "indices", "values")

    def __init__(self, rows, cols, indptr, indices, values):
        self.rows = int(rows)
        self.cols = int(cols)
        self.indptr = np.asarray(indptr, dtype=np.int64)
        self.indices = np.asarray(indices, dtype=np.int64)
        self.values = np.asarray(values, dtype=np.float64)

    @property
    def nnz(self):
        return len(self.values)

    @classmethod
    def from_triplets(cls, rows, cols, i, j, v, sum_duplicates=True):
        """matrix.py:104-128: lexsort by (col, row), sum duplicates, drop zeros."""
        i = np.asarray(i, dtype=np.int64)
        j = np.asarray(j, dtype=np.int64)
        v = np.asarray(v, dtype=np.float64)
        order = np.lexsort((i, j))
        i, j, v = i[order], j[order], v[order]
        if sum_duplicates and len(i):
            keys = j * rows + i
            uniq, inverse = np.unique(keys, return_inverse=True)
            summed = np.zeros(len(uniq))
            np.add.at(summed, inverse, v)
            i = (uniq % rows).astype(np.int64)
            j = (uniq // rows).astype(np.int64)
            v = summed
        keep = v != 0.0
        i, j, v = i[keep], j[keep], v[keep]
        indptr = np.zeros(cols + 1, dtype=np.int64)
        np.add.at(indptr, j + 1, 1)
        np.cumsum(indptr, out=indptr)
        return cls(rows, cols, indptr, i, v)

    @classmethod
    def from_dense(cls, arr):
        """matrix.py:131-136."""
        arr = np.asarray(arr, dtype=np.float64)
        i, j = np.nonzero(arr)
        order = np.lexsort((i, j))
        i, j = i[order], j[order]
        return cls.from_triplets(arr.shape[0], arr.shape[1], i, j, arr[i, j],
                                 sum_duplicates=False)

    def transpose(self):
        """matrix.py:149-154: CSC of the transpose (= CSR of self)."""
        col_of = np.repeat(np.arange(self.cols, dtype=np.int64), np.diff(self.indptr))
        return Csc.from_triplets(self.cols, self.rows, col_of, self.indices, self.values,
                                 sum_duplicates=False)

    def to_dense(self):
        out = np.zeros((self.rows, self.cols), order="F")
        col_of = np.repeat(np.arange(self.cols, dtype=np.int64), np.diff(self.indptr))
        out[self.indices, col_of] = self.values
        return out

    def sum_squares(self):
        return float(self.values @ self.values)


def gram(arr):
    """matrix.py:181-197: A^T A via BLAS, upper triangle mirrored."""
    arr = np.asfortranarray(arr, dtype=np.float64)
    if not np.all(np.isfinite(arr)):
        raise ValueError("gram input contains NaN or Inf")
    r = arr.shape[1]
    prod = arr.T @ arr
    upper = np.triu(prod)
    out = upper + upper.T
    out[np.diag_indices(r)] = np.diag(prod)
    return np.asfortranarray(out)


def frobenius_objective(v, g_arr, f_arr, chunked=False, threads=1):
    """matrix.py:227-260.  g_arr (n, r) and f_arr (r, m) as the reference's
    DenseMatrix arrays (Fortran order).  ``chunked=True`` evaluates the sparse
    cross term as an nnz loop in C (same formula, different summation order)
    for sizes where the reference's nnz x r gathers cannot be allocated."""
    if isinstance(v, Csc):
        q = gram(g_arr)
        if chunked:
            gc = np.ascontiguousarray(g_arr)
            ftc = np.ascontiguousarray(f_arr.T)
            bounds = np.linspace(0, v.cols, max(threads, 1) * 4 + 1).astype(np.int64)

            def part(k):
                return lib().oracle_sparse_cross(
                    _p(v.indptr, _I), _p(v.indices, _I), _p(v.values), int(bounds[k]),
                    int(bounds[k + 1]), _p(gc), _p(ftc), gc.shape[1])

            with ThreadPoolExecutor(max_workers=max(threads, 1)) as pool:
                cross = float(sum(pool.map(part, range(len(bounds) - 1))))
        else:
            col_of = np.repeat(np.arange(v.cols, dtype=np.int64), np.diff(v.indptr))
            gf_at_nnz = np.einsum(
                "ij,ij->i", g_arr[v.indices, :], f_arr[:, col_of].T
            ) if v.nnz else np.zeros(0)
            cross = float(gf_at_nnz @ v.values)
        quad = float(np.sum((q @ f_arr) * f_arr))
        return 0.5 * (v.sum_squares() - 2.0 * cross + quad)
    resid = v - g_arr @ f_arr
    return 0.5 * float(np.sum(resid * resid))


# --------------------------------------------------------------------------
# parallel.py: shard plan, map, reduce
# --------------------------------------------------------------------------
def plan(total, workers):
    """parallel.py:72-84: near-equal contiguous shards."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    workers = min(workers, total) if total > 0 else 1
    base, extra = divmod(total, workers)
    shards = []
    lo = 0
    for w in range(workers):
        hi = lo + base + (1 if w < extra else 0)
        shards.append((lo, hi))
        lo = hi
    return shards


def block_plan(total, workers):
    """parallel.py:162-169: shards aligned to FASTBREAK_BLOCK."""
    nblocks = max(-(-total // FASTBREAK_BLOCK), 1)
    return [(lo * FASTBREAK_BLOCK, min(hi * FASTBREAK_BLOCK, total))
            for lo, hi in plan(nblocks, workers)]


def map_estep(shard, V, G, Q_g, cfg, FT):
    """parallel.py:94-131 -> (Y_part (r, n) Fortran, H_part (r, r), inner)."""
    lo, hi = shard
    n, r = G.shape
    Y_part = np.zeros((r, n), order="F")
    H_part = np.zeros((r, r))
    H = Q_g + (2.0 * cfg.mu2) * np.eye(r)
    scale_a, active, act_idx, Qa = rescale_for_step(H)
    yt = Y_part.T
    if isinstance(V, Csc):
        inner, _, fail = estep_sparse(V.indptr, V.indices, V.values, lo, hi, G, Qa, scale_a,
                                      act_idx, active, cfg.mu1, cfg.epsilon, cfg.inner_cap, 0.0,
                                      FT, yt, H_part)
    else:
        inner, _, fail = estep_dense(V, lo, hi, G, Qa, scale_a, act_idx, active, cfg.mu1,
                                     cfg.epsilon, cfg.inner_cap, 0.0, FT, yt, H_part)
    if fail != FAIL_NONE:
        raise OracleNumericalFailure(f"coefficient solve failed at column {fail}",
                                     index=int(fail))
    upper = np.triu(H_part)
    H_part[:] = upper + upper.T - np.diag(np.diag(upper))
    return Y_part, H_part, int(inner)


def reduce(parts):
    """parallel.py:141-159: ordered sum of worker accumulators."""
    y = np.zeros(parts[0][0].shape, order="F")
    h = np.zeros(parts[0][1].shape)
    inner = 0
    for yp, hp, it in parts:
        y += yp
        h += hp
        inner += it
    return np.asfortranarray(y), np.asfortranarray(h), inner


def run_estep(V, G, Q_g, cfg, FT):
    """parallel.py:172-186 -> (Y (r, n), H_f (r, r), inner_iterations)."""
    m = FT.shape[0]
    shards = block_plan(m, cfg.workers)
    if len(shards) == 1:
        parts = [map_estep(shards[0], V, G, Q_g, cfg, FT)]
    else:
        with ThreadPoolExecutor(max_workers=len(shards)) as pool:
            parts = list(pool.map(lambda s: map_estep(s, V, G, Q_g, cfg, FT), shards))
    return reduce(parts)


def run_mstep(Y, H_f, cfg, G):
    """parallel.py:189-223 -> inner_iterations; G updated in place."""
    n, r = G.shape
    H = H_f + (2.0 * cfg.beta2) * np.eye(r)
    scale_a, active, act_idx, Qa = rescale_for_step(H)
    yt = Y.T
    if not yt.flags["C_CONTIGUOUS"]:
        yt = np.ascontiguousarray(yt)
    workers = cfg.workers if n * r * r > MSTEP_DISTRIBUTE_FLOPS else 1
    shards = block_plan(n, workers)

    def work(shard):
        lo, hi = shard
        inner, _, fail = mstep_rows(yt, lo, hi, Qa, scale_a, act_idx, active, cfg.beta1,
                                    cfg.epsilon, cfg.inner_cap, 0.0, G)
        if fail != FAIL_NONE:
            raise OracleNumericalFailure(f"component solve failed at row {fail}",
                                         index=int(fail))
        return int(inner)

    if len(shards) == 1:
        return work(shards[0])
    with ThreadPoolExecutor(max_workers=len(shards)) as pool:
        return sum(pool.map(work, shards))


# --------------------------------------------------------------------------
# nmf.py: config, init, objective, driver
# --------------------------------------------------------------------------
@dataclass
class Config:
    """nmf.py:34-70 NmfConfig knobs (validation omitted: checker only)."""

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


@dataclass
class Log:
    """nmf.py:81-102 ConvergenceLog."""

    objective: list = field(default_factory=list)
    seconds: list = field(default_factory=list)
    inner_iterations: list = field(default_factory=list)
    k_bar: list = field(default_factory=list)

    def append(self, objective, seconds, inner, subproblems):
        self.objective.append(float(objective))
        self.seconds.append(float(seconds))
        self.inner_iterations.append(int(inner))
        self.k_bar.append(inner / subproblems)

    def __len__(self):
        return len(self.objective)


def _mean(V):
    """nmf.py:109-112."""
    n, m = (V.rows, V.cols) if isinstance(V, Csc) else V.shape
    total = float(np.sum(V.values)) if isinstance(V, Csc) else float(np.sum(V))
    return total / (n * m)


def initial_factors(V, cfg):
    """nmf.py:115-127: G (n, r) then F (r, m) from default_rng(seed)."""
    n, m = (V.rows, V.cols) if isinstance(V, Csc) else V.shape
    rng = np.random.default_rng(cfg.seed)
    scale = np.sqrt(_mean(V) / cfg.rank)
    g = np.ascontiguousarray(rng.uniform(size=(n, cfg.rank)) * scale)
    f = rng.uniform(size=(cfg.rank, m)) * scale
    ft = np.ascontiguousarray(f.T)
    return g, ft


def regularized_objective(V, G, FT, cfg, chunked=False, threads=1):
    """nmf.py:152-165 with model = NmfModel(DenseMatrix(G), DenseMatrix(FT.T))."""
    g = np.asfortranarray(G)
    f = np.asfortranarray(FT.T)
    value = frobenius_objective(V, g, f, chunked=chunked, threads=threads)
    if cfg.mu1:
        value += cfg.mu1 * float(np.sum(np.abs(f)))
    if cfg.beta1:
        value += cfg.beta1 * float(np.sum(np.abs(g)))
    if cfg.mu2:
        value += cfg.mu2 * float(np.sum(f * f))
    if cfg.beta2:
        value += cfg.beta2 * float(np.sum(g * g))
    return value


def fit(V, cfg, on_iteration=None, init=None, chunked_objective=False, step_timer=None):
    """nmf.py:168-211.  V: dense ndarray (n, m) or Csc.  Returns (G, FT, log).

    ``init`` overrides ``initial_factors`` (teacher forcing in tests);
    ``step_timer`` (dict) accumulates E+M-only seconds for the CPU baseline.
    """
    if not isinstance(V, Csc):
        V = np.asfortranarray(V, dtype=np.float64)
        if not np.all(np.isfinite(V)) or (V.size and V.min() < 0):
            raise ValueError("data matrix must be finite and nonnegative")
    n, m = (V.rows, V.cols) if isinstance(V, Csc) else V.shape
    if init is None:
        G, FT = initial_factors(V, cfg)
    else:
        G, FT = (np.ascontiguousarray(a, dtype=np.float64).copy() for a in init)
    log = Log()
    vt_dense = None if isinstance(V, Csc) else np.ascontiguousarray(V.T)
    started = time.perf_counter()
    previous = None
    try:
        for _ in range(cfg.max_outer):
            t0 = time.perf_counter()
            Q_g = gram(G)
            data = V if isinstance(V, Csc) else vt_dense
            Y, H_f, e_inner = run_estep(data, G, Q_g, cfg, FT)
            m_inner = run_mstep(Y, H_f, cfg, G)
            if step_timer is not None:
                step_timer["em_seconds"] = step_timer.get("em_seconds", 0.0) + (
                    time.perf_counter() - t0)
            objective = regularized_objective(V, G, FT, cfg, chunked=chunked_objective,
                                              threads=cfg.workers)
            log.append(objective, time.perf_counter() - started, e_inner + m_inner, m + n)
            if on_iteration is not None:
                on_iteration(log)
            if (cfg.rel_change_tol > 0.0 and previous is not None
                    and abs(previous - objective)
                    <= cfg.rel_change_tol * max(abs(previous), 1e-300)):
                break
            previous = objective
    except OracleNumericalFailure as err:
        err.log = log
        raise
    return G, FT, log


def one_iteration(V, G, FT, cfg):
    """One outer iteration of nmf.py:189-196 from the given state (teacher
    forcing): returns (G', FT', objective, inner, Y, H_f)."""
    G = np.ascontiguousarray(G, dtype=np.float64).copy()
    FT = np.ascontiguousarray(FT, dtype=np.float64).copy()
    data = V if isinstance(V, Csc) else np.ascontiguousarray(np.asarray(V).T)
    Q_g = gram(G)
    Y, H_f, e_inner = run_estep(data, G, Q_g, cfg, FT)
    m_inner = run_mstep(Y, H_f, cfg, G)
    obj = regularized_objective(V if isinstance(V, Csc) else np.asfortranarray(V), G, FT, cfg)
    return G, FT, obj, e_inner + m_inner, Y, H_f
