"""Parity at the BASELINE.json configs' FULL sizes (C2-C5), fp32 production path.

Per config (SURVEY.md 7.3 P2/P3 at full size):

* free-running trajectory: the fp32 GPU fit and the fp64 oracle (the
  bit-exact port of the reference) run K outer iterations from the same
  seeded init; the oracle also runs on the fp32-ROUNDED input -- the
  storage-rounding envelope every fp32 implementation starts from (the
  reference itself moves that much).  Asserted per iteration:
  objective within the north-star 1e-4, or within 10x of that envelope where
  the envelope itself exceeds 1e-4 (the dense configs' early iterations);
* the device objective equals a host float64 evaluation of the returned
  factors (dense: chunked 0.5 ||X - GF||^2 plus penalties, nmf.py:152-165;
  sparse: matrix.py:240-253 with a threaded C nnz loop for the cross term);
* sampled subproblems of the last iteration (8 seeded 32-aligned blocks of
  columns and of rows, rebuilt in float64 from the GPU's own G_k / F_{k+1}):
  the fp32 production NNLS kernel against the fp64 check-mode kernel (== the
  reference's solver, bit for bit) on IDENTICAL fp32-rounded inputs -- the
  arithmetic-only error.  Reported: decision flips (a problem whose inner
  iteration count or zero pattern differs), the factor error of the
  problems without a flip, the summed subproblem objective gap;
* the objective is non-increasing, factors finite and nonnegative, and at C4
  the L1 penalty leaves exact zeros in H.
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
    """Sampled subproblems: (1) the production output against the oracle on
    the float64 problems (summed subproblem objective); (2) the fp32
    production kernel against the fp64 check-mode kernel on identical
    fp32-rounded inputs: decision flips and the factor error without one."""
    from gpu_util import floored_rel, nnls

    def per(a, b):
        return np.array([floored_rel(u[None], v[None]) for u, v in zip(a, b)])

    xo = _solve_blocks(H, h, warm, cfg)
    pg, po = _phi(H, h, x_gpu), _phi(H, h, xo)
    gap = abs(pg.sum() - po.sum()) / abs(po.sum())
    r32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    H32, h32, w32 = r32(H), r32(h), r32(warm)
    x64, it64, _, _ = nnls(H32, h32, w32, cfg["epsilon"], cfg["inner_cap"], precision="fp64")
    x32, it32, _, _ = nnls(H32, h32, w32, cfg["epsilon"], cfg["inner_cap"], precision="fp32")
    flip = (it64 != it32) | np.any((x64 == 0) != (x32 == 0), axis=1)
    e = per(x32, x64)
    keep = ~flip
    q = lambda v, p: float(np.percentile(v, p)) if len(v) else 0.0  # noqa: E731
    g32 = abs(_phi(H32, h32, x32).sum() - _phi(H32, h32, x64).sum()) / abs(_phi(H32, h32, x64).sum())
    print(f"{tag}: {len(e)} problems, decision flips {int(flip.sum())} "
          f"({float(flip.mean()):.3f}); factor err without a flip median {q(e[keep], 50):.1e} "
          f"p90 {q(e[keep], 90):.1e} max {q(e[keep], 100):.1e}; with flips median "
          f"{q(e[flip], 50):.1e}; kernel objective gap {g32:.1e}; production vs oracle "
          f"summed objective gap {gap:.2e}")
    assert gap < 1e-5, (tag, gap)
    assert g32 < 1e-5, (tag, g32)
    # arithmetic-only error where the solver takes the reference's decisions:
    # the typical problem within the north-star 1e-3 (measured medians: C2
    # 4e-5 / 1.4e-4, C3 2e-6 / 4e-6, C4 7e-5 / 3.7e-4 for E / M; the tail, p90
    # up to 4e-2 at C4's M-step, is greedy-CD selections that differ without
    # changing the iteration count or zero pattern); decisions flip on <= 5%
    assert q(e[keep], 50) < 1e-3, tag
    assert q(e[keep], 90) < 0.1, tag
    assert flip.mean() < 0.1, tag
    return dict(problems=len(e), flips=int(flip.sum()), err_noflip_median=q(e[keep], 50),
                err_noflip_p90=q(e[keep], 90), kernel_gap=g32, gap=gap)


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
    # free-running trajectory vs the oracle and its fp32-input envelope
    oc = orc.Config(workers=os.cpu_count() or 1, **kw)
    G0, FT0 = orc.initial_factors(x, oc)
    _, _, olog = orc.fit(x, oc, chunked_objective=sparse)
    xr = orc.Csc(x.rows, x.cols, x.indptr, x.indices, x.values.astype(np.float32).astype(
        np.float64)) if sparse else x.astype(np.float32).astype(np.float64)
    _, _, rlog = orc.fit(xr, oc, chunked_objective=sparse)
    o, fl = np.asarray(olog.objective), np.asarray(rlog.objective)
    rel = np.abs(np.asarray(objs) - o) / o
    env = np.abs(fl - o) / o
    print(f"C{cid}: trajectory rel err {['%.1e' % v for v in rel]}, fp32-input envelope "
          f"{['%.1e' % v for v in env]}")
    assert np.all(rel <= np.maximum(1e-4, 10.0 * env.max())), (rel, env)
    if sparse:
        assert rel.max() < 1e-4, rel
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
