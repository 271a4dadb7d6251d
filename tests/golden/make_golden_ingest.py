"""Golden vectors for the sparse ingest path (SparseMatrix.from_triplets,
transpose, the constructor's validation), produced by the reference itself.

    python tests/golden/make_golden_ingest.py     # writes tests/golden/ingest.npz

Imports the reference from a /tmp copy exactly as make_golden.py does.
Nothing on the GPU box reads /root/reference: the output is committed.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import import_reference  # noqa: E402


def cases(rng):
    out = {}
    # duplicates (summed in input order: 0.1 + 0.2 + 0.3 style rounding),
    # explicit zeros, exact cancellations (dropped), untouched singletons
    rows, cols = 50, 40
    n = 600
    i = rng.integers(0, 12, size=n)
    j = rng.integers(0, 9, size=n)
    v = rng.choice([0.1, 0.2, 0.3, 0.7, 1e-3, 1.0 / 3.0], size=n) * rng.uniform(0.5, 2.0, size=n)
    zi = rng.integers(20, 50, size=30)
    zj = rng.integers(10, 40, size=30)
    ci = np.arange(20, 30)
    cj = np.arange(20, 30)
    cv = rng.uniform(0.5, 1.5, size=10)
    out["dups"] = (rows, cols, np.concatenate([i, zi, ci, ci]), np.concatenate([j, zj, cj, cj]),
                   np.concatenate([v, np.zeros(30), cv, -cv]), True)
    # no duplicates, sum_duplicates=False (triplets in scrambled order)
    keys = rng.choice(rows * cols, size=300, replace=False)
    out["nodup"] = (rows, cols, keys % rows, keys // rows, rng.uniform(0.1, 3.0, size=300), False)
    # a larger Zipf-ish case with heavy duplication
    rows2, cols2 = 3000, 2000
    n2 = 200000
    i2 = np.minimum(rng.zipf(1.3, size=n2) - 1, rows2 - 1)
    j2 = rng.integers(0, cols2, size=n2)
    v2 = np.log1p(rng.poisson(2.0, size=n2) + 1.0)
    out["zipf"] = (rows2, cols2, i2, j2, v2, True)
    # one empty column at each end, single row matrix
    out["edges"] = (1, 5, np.array([0, 0, 0]), np.array([1, 3, 1]), np.array([2.0, 3.0, 4.0]),
                    True)
    out["empty"] = (4, 3, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0), True)
    return out


ERRORS = {
    # name: (rows, cols, i, j, v, sum_duplicates)
    "range_row": (5, 5, [0, 5], [0, 1], [1.0, 1.0], True),
    "range_col": (5, 5, [0, 1], [0, -1], [1.0, 1.0], True),
    "dup_nosum": (5, 5, [1, 1, 2], [3, 3, 0], [1.0, 2.0, 1.0], False),
    "negative": (5, 5, [1, 2], [3, 3], [-1.0, 2.0], True),
    "nan": (5, 5, [1, 2], [3, 3], [np.nan, 2.0], True),
    "inf": (5, 5, [1, 2], [0, 4], [1.0, np.inf], True),
}


def main():
    nmfkit = import_reference()
    from nmfkit.matrix import SparseMatrix

    rng = np.random.default_rng(20261020)
    out = {}
    for name, (rows, cols, i, j, v, sd) in cases(rng).items():
        m = SparseMatrix.from_triplets(rows, cols, i, j, v, sum_duplicates=sd)
        t = m.transpose()
        out.update({f"{name}/rows": rows, f"{name}/cols": cols, f"{name}/i": np.asarray(i),
                    f"{name}/j": np.asarray(j), f"{name}/v": np.asarray(v, dtype=np.float64),
                    f"{name}/sum_duplicates": sd, f"{name}/indptr": m.indptr,
                    f"{name}/indices": m.indices, f"{name}/values": m.values,
                    f"{name}/t_indptr": t.indptr, f"{name}/t_indices": t.indices,
                    f"{name}/t_values": t.values})
    for name, (rows, cols, i, j, v, sd) in ERRORS.items():
        try:
            SparseMatrix.from_triplets(rows, cols, i, j, v, sum_duplicates=sd)
            raise SystemExit(f"{name}: expected the reference to raise")
        except (ValueError, ArithmeticError) as exc:
            out.update({f"err_{name}/args": np.array(
                [rows, cols, sd] + list(i) + list(j) + list(v), dtype=np.float64),
                f"err_{name}/n": len(i), f"err_{name}/type": type(exc).__name__,
                f"err_{name}/message": str(exc)})
    np.savez_compressed(os.path.join(HERE, "ingest.npz"), **out)
    print("wrote", os.path.join(HERE, "ingest.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
