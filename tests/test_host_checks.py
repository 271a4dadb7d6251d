"""Host-side input checks and the init mean (no GPU): the threaded versions in
paper_1506_08938_b200/matrix.py against the reference's plain numpy statements
(matrix.py:169-178 `require_nonnegative`, nmf.py:109-112 the data mean)."""
import numpy as np
import pytest

from paper_1506_08938_b200 import matrix as M
from paper_1506_08938_b200.exceptions import DataDomainError
from paper_1506_08938_b200.matrix import DenseMatrix, SparseMatrix, exact_sum, require_nonnegative


@pytest.mark.parametrize("n", [0, 1, 7, 129, 4096, M._PAR_MIN_SIZE - 3, M._PAR_MIN_SIZE,
                               M._PAR_MIN_SIZE + 1, 17_000_003, 19_437_189])
def test_exact_sum_is_numpy_sum_bit_for_bit(n):
    """exact_sum evaluates np.sum's own pairwise tree on worker threads: the
    seeded init scale (nmf.py:115-127) must be the reference's number exactly."""
    rng = np.random.default_rng(n)
    a = rng.random(n) * rng.choice([1e-6, 1.0, 1e5], size=n)
    assert exact_sum(a) == float(np.sum(a))
    # non-contiguous / other dtypes take the plain path
    assert exact_sum(a[::2]) == float(np.sum(a[::2]))
    assert exact_sum(a.astype(np.float32)) == float(np.sum(a.astype(np.float32)))


def _sparse_with(values):
    n = len(values)
    return SparseMatrix(n, 1, np.array([0, n], dtype=np.int64), np.arange(n, dtype=np.int64),
                        values, validate=False)


@pytest.mark.parametrize("size", [1000, M._PAR_MIN_SIZE + 5])
@pytest.mark.parametrize("bad,msg", [(np.nan, "NaN or Inf"), (np.inf, "NaN or Inf"),
                                     (-np.inf, "NaN or Inf"), (-1e-300, "negative entries"),
                                     (None, None)])
def test_require_nonnegative_matches_reference(size, bad, msg):
    """Same outcome and message as the reference's isfinite().all() / min() < 0
    pair on both the plain and the threaded (large input) path, wherever the
    offending entry sits; NaN / Inf wins over a negative entry."""
    rng = np.random.default_rng(size)
    for pos in (0, size // 2, size - 1):
        v = rng.random(size)
        if bad is not None:
            v[pos] = bad
            if msg == "NaN or Inf":
                v[(pos + 1) % size] = -2.0  # also negative: the NaN / Inf message wins
        for mat in (_sparse_with(v), DenseMatrix(v.reshape(-1, 1 if size % 2 else 2))):
            if bad is None:
                require_nonnegative(mat, "data matrix")
            else:
                with pytest.raises(DataDomainError, match=f"data matrix contains {msg}"):
                    require_nonnegative(mat, "data matrix")


def test_require_nonnegative_fortran_ordered_dense():
    rng = np.random.default_rng(5)
    a = np.asfortranarray(rng.random((4100, 4100)))
    require_nonnegative(DenseMatrix(a), "data matrix")
    a[4099, 17] = -1.0
    with pytest.raises(DataDomainError, match="negative entries"):
        require_nonnegative(DenseMatrix(a), "data matrix")


def test_exact_sum_falls_back_when_the_tree_does_not_match(monkeypatch):
    """The one-time self-check: if this numpy's reduction were not the restated
    pairwise tree, exact_sum must return np.sum's number anyway."""
    a = np.random.default_rng(3).random(M._PAR_MIN_SIZE + 10_000)
    monkeypatch.setattr(M, "_EXACT_SUM_OK", None)
    monkeypatch.setattr(M, "_tree_sum", lambda v: float(np.sum(v)) + 1.0)  # a wrong tree
    assert exact_sum(a) == float(np.sum(a))
    assert M._EXACT_SUM_OK is False
