"""End-to-end fit() on the GPU against the reference's trajectories.

Protocol: full fp32 trajectories are chaotic at the 1e-3
level even for the reference itself under 1-ulp perturbations, so
  P1  fp64 check mode: trajectory vs the reference's at 1e-8 (only the BLAS
      Gram differs in the last bits; the reference's own worker-count
      criterion);
  P2  fp32 teacher-forced: one GPU outer iteration from the oracle state at
      iteration k must land within 1e-4 (relative) of the oracle objective at
      k+1 -- the north-star objective tolerance;
  P3  fp32 full trajectory: reported against the envelope (test bounds 1e-2).
"""

import os

import numpy as np
import pytest

from oracle import generators
from oracle import nmf_oracle as orc

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FITS = np.load(os.path.join(GOLD, "fits.npz"))

pytestmark = pytest.mark.gpu


def _fit(X, precision="fp64", **kw):
    from paper_1506_08938_b200 import NmfConfig, fit

    cfg = NmfConfig(precision=precision, **kw)
    return fit(X, cfg)


@pytest.mark.parametrize("name,kw", [
    ("planted", dict(rank=4, max_outer=40, seed=1, rel_change_tol=0.0)),
    ("planted_w4", dict(rank=4, max_outer=40, seed=1, rel_change_tol=0.0, workers=4)),
    ("planted_reg", dict(rank=4, max_outer=40, seed=1, rel_change_tol=0.0, mu1=0.01, mu2=0.02,
                         beta1=0.01, beta2=0.01)),
])
def test_fit_fp64_trajectory_planted(name, kw):
    model, log = _fit(FITS["planted/X"], **kw)
    np.testing.assert_allclose(log.objective, FITS[f"{name}/objective"], rtol=1e-8)
    np.testing.assert_allclose(model.G.array, FITS[f"{name}/G"], rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(model.F.array, FITS[f"{name}/F"], rtol=1e-6, atol=1e-9)


def test_fit_fp64_sparse_and_dense():
    from paper_1506_08938_b200 import SparseMatrix

    X = FITS["sparse/X"]
    kw = dict(rank=5, max_outer=30, seed=2, rel_change_tol=0.0)
    _, log_s = _fit(SparseMatrix.from_dense(X), **kw)
    _, log_d = _fit(X, **kw)
    np.testing.assert_allclose(log_s.objective, FITS["sparse/objective"], rtol=1e-8)
    np.testing.assert_allclose(log_d.objective, FITS["sparse_dense/objective"], rtol=1e-8)
    np.testing.assert_allclose(log_s.objective, log_d.objective, rtol=1e-9)


def test_fit_zero_matrix():
    model, log = _fit(np.zeros((4, 6)), rank=2, max_outer=5, seed=0, rel_change_tol=0.0)
    assert log.objective[0] == 0.0
    assert not model.G.array.any() or not model.F.array.any()


def test_fit_default_early_exit_matches_reference():
    model, log = _fit(FITS["planted/X"], rank=4, max_outer=300, seed=1)
    want = FITS["early_exit/objective"]
    assert len(log) == len(want)
    np.testing.assert_allclose(log.objective, want, rtol=1e-7)


def test_fit_config1_fp64_bit_exact_with_reference_gram():
    """P1, full config-1 run (50 outer iterations): with the reference's own
    BLAS Gram fed in each iteration (the one product whose summation order
    OpenBLAS owns), every other step runs on the GPU and the factors stay
    BIT-IDENTICAL to the reference's for all 50 iterations."""
    import torch

    from paper_1506_08938_b200 import NmfConfig
    from paper_1506_08938_b200 import device as D
    from paper_1506_08938_b200.nmf import initial_factors
    from paper_1506_08938_b200.matrix import DenseMatrix

    x, _ = generators.make(1)
    cfg = NmfConfig(rank=10, max_outer=50, seed=0, rel_change_tol=0.0, precision="fp64")
    V = DenseMatrix(x)
    G0, FT0 = initial_factors(V, cfg)
    st = D.Alternation(D.DeviceData(V, "fp64"), cfg, G0, FT0, 50, precision="fp64")
    objs = []
    for k in range(50):
        Gh = st.G.cpu().numpy()
        st.Qg.copy_(torch.from_numpy(orc.gram(Gh)))
        st.qg_valid = True
        st.iterate(k)
        objs.append(st.assemble(st.pieces[k].cpu().numpy(), cfg, "dense", 0.0))
    # the oracle (bit-exact to the reference, test_oracle_golden.py) run on this
    # host with this host's BLAS Gram -- the same Gram the GPU was fed
    oG, oFT, olog = orc.fit(x, orc.Config(rank=10, max_outer=50, seed=0, rel_change_tol=0.0))
    inner = st.stats[:, :, 0].sum(1).cpu().numpy()
    assert np.array_equal(inner, np.asarray(olog.inner_iterations))
    assert np.array_equal(st.G.cpu().numpy(), oG)
    assert np.array_equal(st.FT.cpu().numpy(), oFT)
    np.testing.assert_allclose(objs, olog.objective, rtol=1e-12)
    # and the reference's committed trajectory (same BLAS build -> identical)
    np.testing.assert_allclose(objs, FITS["c1/objective"], rtol=5e-3)


def test_fit_config1_fp64_free_running_envelope():
    """P3: free-running fp64 (GPU Gram) vs the reference: within the
    reference's own 1-ulp sensitivity envelope (1.4e-3 measured)."""
    x, _ = generators.make(1)
    model, log = _fit(x, rank=10, max_outer=50, seed=0, rel_change_tol=0.0)
    want = FITS["c1/objective"]
    rel = np.abs(np.asarray(log.objective) - want) / want
    assert rel.max() < 5e-3, rel.max()
    assert abs(log.objective[-1] - want[-1]) / want[-1] < 1e-3


def _teacher_forced(x, ocfg, gcfg, ks):
    """Relative objective error of one fp32 GPU outer iteration started from
    the oracle state at each k (P2), plus the factor errors."""
    from gpu_util import floored_rel

    from paper_1506_08938_b200.nmf import FitSession

    out = []
    state = orc.initial_factors(x, ocfg)
    G, FT = state
    for k in range(max(ks) + 1):
        nG, nFT, obj, _, _, _ = orc.one_iteration(x, G, FT, ocfg)
        if k in ks:
            model, log = FitSession(x, gcfg, init=(G, FT)).run()
            out.append((k, abs(log.objective[0] - obj) / obj,
                        floored_rel(model.G.array, nG), floored_rel(model.F.array, nFT.T),
                        (model.F.array == 0) == (nFT.T == 0)))
        G, FT = nG, nFT
    return out


def test_fit_config1_fp32_teacher_forced():
    """P2 on config 1: one fp32 step from the oracle state.  Objective within
    the north-star 1e-4 at (almost) every k; the first step from the random
    start is the most decision-sensitive (approximate eps=0.1 solves: a
    different stop index in one column changes its block's fast-break
    threshold), bounded at 1e-3."""
    from paper_1506_08938_b200 import NmfConfig

    x, ocfg = generators.make(1)
    gcfg = NmfConfig(rank=10, max_outer=1, seed=0, rel_change_tol=0.0, precision="fp32")
    res = _teacher_forced(x, ocfg, gcfg, ks=[0, 1, 2, 5, 10, 20, 30, 45])
    rels = np.array([r[1] for r in res])
    print("teacher-forced objective rel err:", {r[0]: f"{r[1]:.1e}" for r in res})
    assert rels.max() < 1e-3
    assert np.median(rels) < 1e-4
    assert (rels[1:] < 1e-4).mean() >= 0.8


def test_fit_config1_fp32_trajectory_envelope():
    """P3 free-running fp32 on config 1.  The early iterations are chaotic: the
    first step from the random start differs by ~8e-4 (decision-sensitive
    eps=0.1 solves, bounded per step by the teacher-forced test above) and the
    next steps amplify any such difference -- every fp32 product kernel we
    measured (SIMT, 3 tensor-core variants) peaks between 4e-3 and 1.2e-2
    around iteration 1-3.  After the transient the trajectory must settle
    onto the reference's: the tail is held to 1e-3."""
    x, _ = generators.make(1)
    _, log = _fit(x, precision="fp32", rank=10, max_outer=50, seed=0, rel_change_tol=0.0)
    want = FITS["c1/objective"]
    rel = np.abs(np.asarray(log.objective) - want) / want
    print("fp32 C1 trajectory rel:", " ".join(f"{v:.1e}" for v in rel))
    assert rel[:10].max() < 2.5e-2, rel.max()
    assert rel[-10:].max() < 1e-3, rel[-10:].max()


def test_fit_fp32_deterministic():
    x, _ = generators.make(1)
    kw = dict(rank=10, max_outer=10, seed=0, rel_change_tol=0.0)
    m1, l1 = _fit(x, precision="fp32", **kw)
    m2, l2 = _fit(x, precision="fp32", **kw)
    assert l1.objective == l2.objective
    assert np.array_equal(m1.G.array, m2.G.array)
    assert np.array_equal(m1.F.array, m2.F.array)


def _reg_data():
    rng = np.random.default_rng(3)
    X = rng.exponential(size=(200, 8)) @ rng.exponential(size=(8, 300))
    X += np.abs(rng.normal(0, 0.05, size=X.shape))
    return X


def test_fit_regularized_fp32_monotone_and_final():
    """Config-4 variant (L1 0.1 on H, L2 0.01 on W) at small size: the fp32
    trajectory decreases monotonically and ends near the reference's."""
    X = _reg_data()
    kw = dict(rank=8, max_outer=40, seed=3, rel_change_tol=0.0, mu1=0.1, beta2=0.01)
    model, log = _fit(X, precision="fp32", **kw)
    obj = np.array(log.objective)
    assert np.all(np.diff(obj) <= 1e-5 * np.abs(obj[:-1]))
    # the fp64 check mode follows the reference trajectory itself
    _, log64 = _fit(X, precision="fp64", **kw)
    G, FT, olog = orc.fit(X, orc.Config(**kw))
    np.testing.assert_allclose(log64.objective, olog.objective, rtol=1e-8)
    # fp32: a non-convex problem may settle in a different local minimum
    # (SURVEY 0.6); both runs must at least reach the same order of magnitude
    assert obj[-1] < 2.0 * olog.objective[-1]


def test_fit_regularized_fp32_teacher_forced_sparsity():
    """P2 with L1/L2 penalties: objective per step and the exact-zero pattern
    of H (the L1 sparsity) against the oracle."""
    from paper_1506_08938_b200 import NmfConfig

    X = _reg_data()
    kw = dict(rank=8, seed=3, rel_change_tol=0.0, mu1=0.1, beta2=0.01)
    ocfg = orc.Config(max_outer=1, **kw)
    gcfg = NmfConfig(max_outer=1, precision="fp32", **kw)
    res = _teacher_forced(X, ocfg, gcfg, ks=[3, 10, 25])
    for k, rel, eg, ef, zeq in res:
        assert rel < 1e-3, (k, rel)
        assert zeq.mean() > 0.97, (k, zeq.mean())


def _product_sparse(csc):
    from paper_1506_08938_b200 import SparseMatrix

    return SparseMatrix(csc.rows, csc.cols, csc.indptr, csc.indices, csc.values, validate=False)


def test_sparse_zipf_fp32_teacher_forced():
    """Config-3 structure at small size (Zipf rows: popular rows exceed the
    256-entry chunk, so the load-balanced Y^T pass splits and folds them)."""
    from paper_1506_08938_b200 import NmfConfig
    from paper_1506_08938_b200.nmf import FitSession

    X = generators.sparse_zipf(3000, 2000, 0.01, 7)
    assert np.diff(X.transpose().indptr).max() > 256
    ocfg = orc.Config(rank=20, seed=7, rel_change_tol=0.0, max_outer=1)
    gcfg = NmfConfig(rank=20, seed=7, rel_change_tol=0.0, max_outer=1, precision="fp32")
    G, FT = orc.initial_factors(X, ocfg)
    for k in range(6):
        nG, nFT, obj, _, _, _ = orc.one_iteration(X, G, FT, ocfg)
        if k in (0, 2, 5):
            model, log = FitSession(_product_sparse(X), gcfg, init=(G, FT)).run()
            assert abs(log.objective[0] - obj) / obj < 1e-4, (k, log.objective[0], obj)
        G, FT = nG, nFT


def test_sparse_zipf_fp64_bit_exact_with_reference_gram():
    """fp64 check mode on Zipf sparse data, 10 iterations, with the oracle's
    BLAS Gram fed in (the only op whose summation order OpenBLAS owns):
    factors and inner-iteration counts bit-identical to the oracle.  (Free
    running, the Gram's last-bit difference flips a few near-tie CD decisions
    in the first component step on this data -- the SURVEY 0.6 sensitivity.)"""
    import torch

    from paper_1506_08938_b200 import NmfConfig
    from paper_1506_08938_b200 import device as D
    from paper_1506_08938_b200.nmf import initial_factors

    X = generators.sparse_zipf(1500, 1000, 0.01, 8)
    V = _product_sparse(X)
    kw = dict(rank=12, seed=8, rel_change_tol=0.0, max_outer=10)
    cfg = NmfConfig(precision="fp64", **kw)
    G0, FT0 = initial_factors(V, cfg)
    st = D.Alternation(D.DeviceData(V, "fp64"), cfg, G0, FT0, 10, precision="fp64")
    objs = []
    for k in range(10):
        st.Qg.copy_(torch.from_numpy(orc.gram(st.G.cpu().numpy())))
        st.qg_valid = True
        st.iterate(k)
        objs.append(st.assemble(st.pieces[k].cpu().numpy(), cfg, "sparse", X.sum_squares()))
    oG, oFT, olog = orc.fit(X, orc.Config(**kw))
    assert np.array_equal(st.stats[:, :, 0].sum(1).cpu().numpy(), olog.inner_iterations)
    assert np.array_equal(st.G.cpu().numpy(), oG)
    assert np.array_equal(st.FT.cpu().numpy(), oFT)
    np.testing.assert_allclose(objs, olog.objective, rtol=1e-10)


@pytest.mark.parametrize("n,m,r", [
    (640, 960, 8),      # tcgen05 v3 GEMM, int8 residual (1 k-step)
    (600, 1000, 50),    # v3 GEMM, int8 residual (2 k-steps)
    (500, 700, 100),    # v2 GEMM (BN=112), int8 residual (KB=128, 4 k-steps)
    (400, 560, 130),    # v2 GEMM (BN=144), FFMA residual (r > 128)
    (333, 501, 20),     # m % 4 != 0: SIMT split-K GEMM + tile residual
])
def test_fp32_kernel_paths_teacher_forced(n, m, r):
    """Every dense fp32 kernel path (chosen by r and alignment) reproduces the
    oracle's outer iteration from the same state: objective to the north-star
    1e-4 once past the decision-sensitive first iterations."""
    from paper_1506_08938_b200 import NmfConfig

    rng = np.random.default_rng(n + m + r)
    W0 = rng.exponential(size=(n, r))
    H0 = rng.exponential(size=(r, m))
    x = W0 @ H0 + np.abs(rng.normal(0, 0.05, size=(n, m)))
    ocfg = orc.Config(rank=r, seed=1, rel_change_tol=0.0, max_outer=1)
    gcfg = NmfConfig(rank=r, seed=1, rel_change_tol=0.0, max_outer=1, precision="fp32")
    res = _teacher_forced(x, ocfg, gcfg, ks=[0, 1, 2, 3, 4, 6, 8, 12, 16])
    print(n, m, r, "teacher-forced rel:", " ".join(f"{k}:{rel:.1e}" for k, rel, *_ in res))
    rels = np.array([rel for _, rel, *_ in res])
    # the first iterations are decision-sensitive (eps = 0.1 approximate solves,
    # as for config 1 above); once the factors settle every step is within 1e-4
    assert rels.max() < 1e-3, rels
    assert np.median(rels) < 1e-4, rels
    assert (rels[-3:] < 1e-4).all(), rels


@pytest.mark.parametrize("bad", [np.nan, np.inf, -1.0])
@pytest.mark.parametrize("as_torch", [False, True])
def test_fit_rejects_bad_data(bad, as_torch):
    """require_nonnegative (matrix.py:169-178): NaN / Inf / negative entries
    raise DataDomainError before any factor update, numpy or torch input."""
    import torch

    from paper_1506_08938_b200 import NmfConfig, fit
    from paper_1506_08938_b200.exceptions import DataDomainError

    x = np.random.default_rng(0).uniform(size=(64, 96)).astype(np.float32)
    x[5, 7] = bad
    V = torch.from_numpy(x) if as_torch else x
    with pytest.raises(DataDomainError):
        fit(V, NmfConfig(rank=4, max_outer=2, precision="fp32"))


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_lagged_convergence_check_returns_the_stopping_iterate(precision):
    """The per-iteration stopping rule is checked one iteration behind the
    launches (no per-iteration stall); the model must still be the state after
    the iteration that met the rule: identical to a fixed-count fit of that
    many iterations, and the log identical too."""
    X = FITS["planted/X"]
    model, log = _fit(X, precision, rank=4, max_outer=300, seed=1, rel_change_tol=0.05)
    K = len(log)
    assert 2 < K < 300
    ref_model, ref_log = _fit(X, precision, rank=4, max_outer=K, seed=1, rel_change_tol=0.0)
    assert np.array_equal(model.G.array, ref_model.G.array)
    assert np.array_equal(model.F.array, ref_model.F.array)
    assert log.objective == ref_log.objective
    assert log.inner_iterations == ref_log.inner_iterations


def test_on_iteration_callback_sees_every_iteration():
    from paper_1506_08938_b200 import NmfConfig, fit

    seen = []
    X = FITS["planted/X"]
    cfg = NmfConfig(precision="fp32", rank=4, max_outer=7, seed=1, rel_change_tol=0.0)
    model, log = fit(X, cfg, on_iteration=lambda lg: seen.append(len(lg)))
    assert seen == list(range(1, 8))
    ref_model, ref_log = _fit(X, "fp32", rank=4, max_outer=7, seed=1, rel_change_tol=0.0)
    assert np.array_equal(model.G.array, ref_model.G.array)
    assert log.objective == ref_log.objective
