"""Parity at the BASELINE.json configs' FULL sizes (C2-C5), fp32 production path.

The oracle cannot run the full trajectories at these sizes in test time
(C2 is ~2.4 s per iteration with 16 threads, C5 ~70 s), so each
config is checked through properties that do not depend on size:

* teacher-forced subproblems on sampled fast-break blocks: G and F are read
  back before and after one GPU outer iteration; for 8 seeded 32-aligned
  blocks of columns (E-step) and rows (M-step) the oracle (the bit-exact C
  restatement of kernels.py) rebuilds the problems in float64 from the same
  G_k / F_{k+1} -- Q = Gram + 2 lambda I (parallel.py:104,196), h = mu1 - G^T x_j
  (kernels.py:251-258,306-313) / beta1 - (X F^T)_i (kernels.py:361) -- and
  solves them with the reference's stopping rule and fast-break blocks.
  Blocks are 32-aligned, so the reference's per-block threshold resets
  (kernels.py:246-248) make a sampled block exactly the reference's problem
  sequence.  fp32 tolerance: 1e-5 on the summed subproblem objective, and the
  factors within 10x of the oracle's own movement when only its inputs are
  rounded to float32 (the problems' conditioning, not the kernels, sets the
  factor-level agreement an fp32 path can reach at these sizes);
* the device objective equals a host float64 evaluation of the same factors
  (dense: chunked 0.5 ||X - GF||^2 plus the penalties, nmf.py:152-165; sparse:
  matrix.py:240-253, the cross term as a threaded C nnz loop);
* the objective is non-increasing (block coordinate descent), the factors are
  finite and nonnegative, and at C4 the L1 penalty leaves exact zeros in H.
"""

import os

import numpy as np
import pytest

from oracle import generators
from oracle import nmf_oracle as orc

pytestmark = pytest.mark.gpu

ITERS = {2: 3, 3: 3, 4: 3, 5: 2}
BLOCKS = 8


def _sample_blocks(total, rng):
    nb = total // 32
    return np.sort(rng.choice(nb, size=min(BLOCKS, nb), replace=False))


def _solve_blocks(H, h, warm, cfg):
    """Oracle solves of stacked 32-problem blocks: h (s, r) -> x (s, r)."""
    scale_a, active, act_idx, Qa = orc.rescale_for_step(H)
    YT = np.ascontiguousarray(-h)  # mstep_rows forms h = beta1 - YT with beta1 = 0
    X = np.ascontiguousarray(warm, dtype=np.float64)
    inner, _, fail = orc.mstep_rows(YT, 0, h.shape[0], Qa, scale_a, act_idx, active, 0.0,
                                    cfg["epsilon"], cfg["inner_cap"], 0.0, X)
    assert fail == -1
    return X


def _phi(H, h, x):
    """Per-problem objective 0.5 x'Hx + h'x (rows of x)."""
    return 0.5 * np.einsum("ij,jk,ik->i", x, H, x) + np.einsum("ij,ij->i", h, x)


def _compare(tag, H, h, warm, x_gpu, cfg):
    """GPU solutions vs the oracle's on the same float64 problems.

    The summed subproblem objective must agree to 1e-5 (north star: 1e-4 on
    the objective).  Factor-level agreement is bounded by the problems'
    conditioning: the oracle's own solutions move when only its inputs are
    rounded to float32 (Q and h, as the GPU holds them), so the GPU's factor
    error must lie within 10x of that float32-input sensitivity."""
    from gpu_util import floored_rel

    def per(a, b):
        return np.array([floored_rel(u[None], v[None]) for u, v in zip(a, b)])

    xo = _solve_blocks(H, h, warm, cfg)
    H32 = H.astype(np.float32).astype(np.float64)
    h32 = h.astype(np.float32).astype(np.float64)
    xo32 = _solve_blocks(H32, h32, warm.astype(np.float32).astype(np.float64), cfg)
    e_gpu, e_sens = per(x_gpu, xo), per(xo32, xo)
    pg, po = _phi(H, h, x_gpu), _phi(H, h, xo)
    gap = abs(pg.sum() - po.sum()) / abs(po.sum())
    q = lambda e, p: float(np.percentile(e, p))  # noqa: E731
    print(f"{tag}: factor rel GPU vs oracle median {q(e_gpu, 50):.2e} p90 {q(e_gpu, 90):.2e}; "
          f"oracle fp32-input sensitivity median {q(e_sens, 50):.2e} p90 {q(e_sens, 90):.2e}; "
          f"within 1e-3 {float((e_gpu < 1e-3).mean()):.3f}; summed objective gap {gap:.2e}")
    assert gap < 1e-5, (tag, gap)
    assert q(e_gpu, 50) <= max(10 * q(e_sens, 50), 1e-5), tag
    assert q(e_gpu, 90) <= max(10 * q(e_sens, 90), 1e-4), tag


def _dense_objective(x, G, F):
    n = x.shape[0]
    acc = 0.0
    for lo in range(0, n, 1000):
        d = x[lo:lo + 1000] - G[lo:lo + 1000] @ F
        acc += float(np.einsum("ij,ij->", d, d))
    return 0.5 * acc


@pytest.mark.parametrize("cid", [2, 3, 4, 5])
def test_full_size_config(cid):
    import torch

    from paper_1506_08938_b200 import NmfConfig
    from paper_1506_08938_b200.matrix import SparseMatrix
    from paper_1506_08938_b200.nmf import FitSession

    x, ocfg = generators.make(cid)
    sparse = not isinstance(x, np.ndarray)
    K = ITERS[cid]
    kw = dict(ocfg.__dict__)
    kw.pop("workers")
    kw["max_outer"] = K
    cfg = NmfConfig(precision="fp32", **kw)
    V = SparseMatrix(x.rows, x.cols, x.indptr, x.indices, x.values, validate=False) \
        if sparse else x
    st = FitSession(V, cfg).state
    n, m, r = st.n, st.m, st.r
    objs = []
    G_prev = FT_prev = None
    for k in range(K):
        if k == K - 1:
            st.join()
            G_prev = st.G.double().cpu().numpy()
            FT_prev = st.FT.double().cpu().numpy()
        st.iterate(k)
    st.join()
    torch.cuda.synchronize()
    xsq = x.sum_squares() if sparse else 0.0
    objs = [st.assemble(p, cfg, "sparse" if sparse else "dense", xsq)
            for p in st.pieces[:K].cpu().numpy()]
    G = st.G.double().cpu().numpy()
    FT = st.FT.double().cpu().numpy()
    print(f"C{cid}: objectives {objs}")
    assert np.isfinite(G).all() and np.isfinite(FT).all()
    assert (G >= 0).all() and (FT >= 0).all()
    assert all(b <= a * (1 + 1e-6) for a, b in zip(objs, objs[1:])), objs

    # host float64 objective of the returned factors (nmf.py:152-165)
    if sparse:
        base = orc.frobenius_objective(x, G, FT.T, chunked=True,
                                       threads=os.cpu_count() or 1)
    else:
        base = _dense_objective(x, G, FT.T)
    want = base + cfg.mu1 * FT.sum() + cfg.beta1 * G.sum() + cfg.mu2 * (FT ** 2).sum() \
        + cfg.beta2 * (G ** 2).sum()
    rel = abs(objs[-1] - want) / want
    print(f"C{cid}: device objective rel err vs host fp64 {rel:.2e}")
    assert rel < 1e-6, rel

    # teacher-forced sampled subproblems of the last iteration
    rng = np.random.default_rng(100 + cid)
    c = dict(epsilon=cfg.epsilon, inner_cap=cfg.inner_cap)
    # E-step: columns j, from G_prev and warm F_prev
    cols = (_sample_blocks(m, rng)[:, None] * 32 + np.arange(32)).ravel()
    Hq = G_prev.T @ G_prev + 2.0 * cfg.mu2 * np.eye(r)
    if sparse:
        h = np.empty((len(cols), r))
        for t, j in enumerate(cols):
            lo, hi = x.indptr[j], x.indptr[j + 1]
            h[t] = cfg.mu1 - G_prev[x.indices[lo:hi]].T @ x.values[lo:hi]
    else:
        h = cfg.mu1 - (G_prev.T @ x[:, cols]).T
    _compare(f"C{cid} E-step", Hq, h, FT_prev[cols], FT[cols], c)
    # M-step: rows i, from F_{k+1} (= FT) and warm G_prev
    rows = (_sample_blocks(n, rng)[:, None] * 32 + np.arange(32)).ravel()
    Hf = FT.T @ FT + 2.0 * cfg.beta2 * np.eye(r)
    if sparse:
        sel = np.full(n, -1, dtype=np.int64)
        sel[rows] = np.arange(len(rows))
        pos = sel[x.indices]
        hit = np.flatnonzero(pos >= 0)
        col_of = np.searchsorted(x.indptr, hit, side="right") - 1
        Y = np.zeros((len(rows), r))
        np.add.at(Y, pos[hit], x.values[hit, None] * FT[col_of])
    else:
        Y = x[rows] @ FT
    h = cfg.beta1 - Y
    _compare(f"C{cid} M-step", Hf, h, G_prev[rows], G[rows], c)
    if cid == 4:
        zeros = float((FT == 0).mean())
        print(f"C4: exact-zero fraction of H {zeros:.4f}")
        assert zeros > 0.0
