"""Multiplicative-update baseline on the GPU (baselines.py:41-85) against the
reference's own trajectories (tests/golden/mur.npz, make_golden_mur.py)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "mur.npz"))


def _cfg(name, precision):
    from paper_1506_08938_b200 import NmfConfig

    kw = {"dense": dict(rank=6, max_outer=40, seed=5),
          "dense_reg": dict(rank=6, max_outer=25, seed=6, mu1=0.05, beta2=0.1),
          "sparse": dict(rank=4, max_outer=30, seed=7)}[name]
    return NmfConfig(rel_change_tol=0.0, precision=precision, **kw)


def _data(name):
    from paper_1506_08938_b200 import SparseMatrix

    if name == "sparse":
        return SparseMatrix.from_dense(GOLD["sparse/X"])
    return np.asfortranarray(GOLD["dense/X"])


@pytest.mark.parametrize("name", ["dense", "dense_reg", "sparse"])
def test_mur_fit_fp64_matches_reference(name):
    from paper_1506_08938_b200.baselines import mur_fit

    model, log = mur_fit(_data(name), _cfg(name, "fp64"))
    np.testing.assert_allclose(log.objective, GOLD[f"{name}/objective"], rtol=1e-10)
    assert list(log.inner_iterations) == list(GOLD[f"{name}/inner"])
    assert all(kb == 1.0 for kb in log.k_bar)
    np.testing.assert_allclose(model.G.array, GOLD[f"{name}/G"], rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(model.F.array, GOLD[f"{name}/F"], rtol=1e-8, atol=1e-12)


@pytest.mark.parametrize("name", ["dense", "sparse"])
def test_mur_fit_fp32_close_to_reference(name):
    """fp32 production data products (tcgen05 GEMM / SpMM): MUR is a
    contraction, so the trajectory stays within fp32 accuracy."""
    from paper_1506_08938_b200.baselines import mur_fit

    _, log = mur_fit(_data(name), _cfg(name, "fp32"))
    np.testing.assert_allclose(log.objective, GOLD[f"{name}/objective"], rtol=2e-5)


def test_mur_step_matches_reference():
    from paper_1506_08938_b200.baselines import mur_step

    G1, F1 = mur_step(np.asfortranarray(GOLD["dense/X"]), GOLD["step/G0"], GOLD["step/F0"])
    np.testing.assert_allclose(G1, GOLD["step/G1"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(F1, GOLD["step/F1"], rtol=1e-12, atol=1e-15)


def test_mur_objective_non_increasing_config1():
    from oracle import generators
    from paper_1506_08938_b200 import NmfConfig
    from paper_1506_08938_b200.baselines import mur_fit

    x, _ = generators.make(1)
    _, log = mur_fit(x, NmfConfig(rank=10, max_outer=50, seed=0, rel_change_tol=0.0,
                                  precision="fp64"))
    obj = np.asarray(log.objective)
    assert np.all(np.diff(obj) <= 1e-12 * obj[:-1])
