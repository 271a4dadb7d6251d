"""Golden trajectories of the reference's multiplicative-update baseline
(baselines.mur_fit / mur_step) on a dense and a sparse problem.

    python tests/golden/make_golden_mur.py      # writes tests/golden/mur.npz
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import import_reference  # noqa: E402


def main():
    nmfkit = import_reference()
    from nmfkit.baselines import mur_fit, mur_step
    from nmfkit.matrix import DenseMatrix, SparseMatrix
    from nmfkit.nmf import NmfConfig, initial_factors

    rng = np.random.default_rng(77)
    W0 = rng.uniform(size=(120, 6))
    H0 = rng.uniform(size=(6, 90))
    X = W0 @ H0 + np.abs(rng.normal(0, 0.01, size=(120, 90)))
    S = np.where(rng.random((150, 110)) < 0.08, rng.uniform(0.5, 3.0, (150, 110)), 0.0)
    out = {"dense/X": X, "sparse/X": S}
    for name, V, cfg in (
            ("dense", DenseMatrix(np.asfortranarray(X)),
             NmfConfig(rank=6, max_outer=40, seed=5, rel_change_tol=0.0)),
            ("dense_reg", DenseMatrix(np.asfortranarray(X)),
             NmfConfig(rank=6, max_outer=25, seed=6, rel_change_tol=0.0, mu1=0.05, beta2=0.1)),
            ("sparse", SparseMatrix.from_dense(DenseMatrix(np.asfortranarray(S))),
             NmfConfig(rank=4, max_outer=30, seed=7, rel_change_tol=0.0))):
        model, log = mur_fit(V, cfg)
        out[f"{name}/objective"] = np.asarray(log.objective)
        out[f"{name}/inner"] = np.asarray(log.inner_iterations)
        out[f"{name}/G"] = model.G.array
        out[f"{name}/F"] = model.F.array
    V = DenseMatrix(np.asfortranarray(X))
    G, FT = initial_factors(V, NmfConfig(rank=6, seed=5))
    G1, F1 = mur_step(X, G, np.ascontiguousarray(FT.T))
    out.update({"step/G0": G, "step/F0": FT.T, "step/G1": G1, "step/F1": F1})
    np.savez_compressed(os.path.join(HERE, "mur.npz"), **out)
    print("wrote mur.npz", len(out))


if __name__ == "__main__":
    main()
