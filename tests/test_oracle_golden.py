"""Pin the CPU oracle (oracle/) to the reference's own outputs.

The golden vectors were produced by running the reference (nmfkit, numba
kernels) itself -- see tests/golden/make_golden.py.  Kernel-level outputs must
match BIT FOR BIT; fit trajectories go through numpy/OpenBLAS and are compared
exactly too (same BLAS build), with a 1e-9 fallback for a different host.
"""

import hashlib
import os

import numpy as np
import pytest

from oracle import generators
from oracle import nmf_oracle as orc

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _cases(npz):
    return sorted({k.split("/")[0] for k in npz.files})


NNLS = np.load(os.path.join(GOLD, "nnls_batches.npz"))
STEPS = np.load(os.path.join(GOLD, "steps.npz"))
FITS = np.load(os.path.join(GOLD, "fits.npz"))


@pytest.mark.parametrize("case", _cases(NNLS))
def test_rescale_matches_reference(case):
    g = lambda k: NNLS[f"{case}/{k}"]  # noqa: E731
    scale_a, active, act_idx, Qa = orc.rescale_for_step(g("H"))
    assert np.array_equal(active, g("active"))
    assert np.array_equal(act_idx, g("act_idx"))
    assert np.array_equal(scale_a, g("scale_a"))
    assert np.array_equal(Qa, g("Qa"))


@pytest.mark.parametrize("case", _cases(NNLS))
def test_mstep_rows_bit_exact(case):
    g = lambda k: NNLS[f"{case}/{k}"]  # noqa: E731
    h, warm = g("h"), g("warm")
    beta1 = float(g("beta1"))
    YT = np.ascontiguousarray(beta1 - h)
    G = np.ascontiguousarray(warm.copy())
    count = h.shape[0]
    iters = np.zeros(count, dtype=np.int64)
    running = np.zeros(count)
    ms = 0.0
    fail = -1
    for row in range(count):
        it, ms, f = orc.mstep_rows(YT, row, row + 1, g("Qa"), g("scale_a"), g("act_idx"),
                                   g("active"), beta1, float(g("eps")), int(g("max_inner")), ms, G)
        if f != -1:
            fail = f
            break
        iters[row] = it
        running[row] = ms
    assert fail == int(g("fail"))
    stop = count if fail < 0 else fail
    assert np.array_equal(iters[:stop], g("iters")[:stop])
    assert np.array_equal(running[:stop], g("running_max_stop")[:stop])
    assert np.array_equal(G[:stop], g("x")[:stop])
    # one shard call == row-by-row replay
    G2 = np.ascontiguousarray(warm.copy())
    tot, _, f2 = orc.mstep_rows(YT, 0, count, g("Qa"), g("scale_a"), g("act_idx"), g("active"),
                                beta1, float(g("eps")), int(g("max_inner")), 0.0, G2)
    assert f2 == fail
    if fail < 0:
        assert tot == iters.sum()
        assert np.array_equal(G2, G)


@pytest.mark.parametrize("kind", ["dense", "sparse"])
@pytest.mark.parametrize("variant", ["plain_w1", "plain_w3", "reg_w1", "reg_w3"])
def test_run_estep_mstep_bit_exact(kind, variant):
    arr, g0, ft0 = STEPS["data/arr"], STEPS["data/g"], STEPS["data/ft"]
    kw = dict(workers=int(variant[-1]))
    if variant.startswith("reg"):
        kw.update(mu1=0.05, mu2=0.02, beta1=0.03, beta2=0.01)
    cfg = orc.Config(rank=g0.shape[1], seed=0, **kw)
    V = orc.Csc.from_dense(arr) if kind == "sparse" else np.ascontiguousarray(arr.T)
    G, FT = g0.copy(), ft0.copy()
    Q_g = orc.gram(G)
    p = f"{kind}/{variant}"
    assert np.array_equal(Q_g, STEPS[p + "/Q_g"])
    Y, H_f, e = orc.run_estep(V, G, Q_g, cfg, FT)
    m = orc.run_mstep(Y, H_f, cfg, G)
    assert np.array_equal(FT, STEPS[p + "/FT"])
    assert np.array_equal(Y, STEPS[p + "/Y"])
    assert np.array_equal(H_f, STEPS[p + "/H_f"])
    assert np.array_equal(G, STEPS[p + "/G"])
    assert e == int(STEPS[p + "/e_inner"]) and m == int(STEPS[p + "/m_inner"])


def _fit_check(name, V, cfg):
    G, FT, log = orc.fit(V, cfg)
    want = FITS[f"{name}/objective"]
    got = np.asarray(log.objective)
    assert got.shape == want.shape
    if not np.array_equal(got, want):  # different BLAS build: reference's own 1e-9 bar
        np.testing.assert_allclose(got, want, rtol=1e-9)
    else:
        assert np.array_equal(np.asarray(log.inner_iterations), FITS[f"{name}/inner"])
        if f"{name}/G" in FITS.files:
            assert np.array_equal(G, FITS[f"{name}/G"])
            assert np.array_equal(FT.T, FITS[f"{name}/F"])


def test_fit_planted():
    _fit_check("planted", FITS["planted/X"], orc.Config(rank=4, max_outer=40, seed=1,
                                                        rel_change_tol=0.0))


def test_fit_planted_workers4():
    _fit_check("planted_w4", FITS["planted/X"],
               orc.Config(rank=4, max_outer=40, seed=1, rel_change_tol=0.0, workers=4))


def test_fit_planted_regularized():
    _fit_check("planted_reg", FITS["planted/X"],
               orc.Config(rank=4, max_outer=40, seed=1, rel_change_tol=0.0, mu1=0.01, mu2=0.02,
                          beta1=0.01, beta2=0.01))


def test_fit_sparse_and_dense():
    X = FITS["sparse/X"]
    cfg = orc.Config(rank=5, max_outer=30, seed=2, rel_change_tol=0.0)
    _fit_check("sparse", orc.Csc.from_dense(X), cfg)
    _fit_check("sparse_dense", X, cfg)


def test_fit_zero_matrix():
    _fit_check("zero", np.zeros((4, 6)), orc.Config(rank=2, max_outer=5, seed=0,
                                                    rel_change_tol=0.0))


def test_fit_default_tolerance():
    _fit_check("early_exit", FITS["planted/X"], orc.Config(rank=4, max_outer=300, seed=1))


def test_c1_generator_pinned():
    x = generators.c1()
    digest = hashlib.sha256(np.ascontiguousarray(x).tobytes()).digest()
    assert np.array_equal(np.frombuffer(digest, dtype=np.uint8), FITS["c1/x_sha256"])


@pytest.mark.slow
def test_fit_config1_full():
    x, cfg = generators.make(1)
    _fit_check("c1", x, cfg)
