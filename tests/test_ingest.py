"""Sparse ingest: SparseMatrix.from_triplets /
transpose / validation (matrix.py:81-154) against the reference's own outputs
(tests/golden/ingest.npz, made by tests/golden/make_golden_ingest.py).

CPU: the oracle restatement and the host mirror reproduce the goldens.
GPU: DeviceCsc (csrc/ingest.cu) reproduces them bit for bit -- indices
exactly, duplicate sums bit-identical to np.add.at -- raises the reference's
exception types and messages, builds the CSR twin exactly, and a fit from a
DeviceCsc equals the fit from the host SparseMatrix.
"""

import os

import numpy as np
import pytest

from oracle import nmf_oracle as orc

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "ingest.npz"))
CASES = sorted({k.split("/")[0] for k in GOLD.files if not k.startswith("err_")})
ERRS = sorted({k.split("/")[0][4:] for k in GOLD.files if k.startswith("err_")})


def _case(name):
    g = lambda k: GOLD[f"{name}/{k}"]  # noqa: E731
    return (int(g("rows")), int(g("cols")), g("i"), g("j"), g("v"), bool(g("sum_duplicates")))


def _err(name):
    a = GOLD[f"err_{name}/args"]
    n = int(GOLD[f"err_{name}/n"])
    rows, cols, sd = int(a[0]), int(a[1]), bool(a[2])
    i = a[3:3 + n].astype(np.int64)
    j = a[3 + n:3 + 2 * n].astype(np.int64)
    v = a[3 + 2 * n:3 + 3 * n]
    return (rows, cols, i, j, v, sd), str(GOLD[f"err_{name}/type"]), \
        str(GOLD[f"err_{name}/message"])


@pytest.mark.parametrize("name", CASES)
def test_oracle_from_triplets_matches_reference(name):
    m = orc.Csc.from_triplets(*_case(name))
    assert np.array_equal(m.indptr, GOLD[f"{name}/indptr"])
    assert np.array_equal(m.indices, GOLD[f"{name}/indices"])
    assert np.array_equal(m.values, GOLD[f"{name}/values"])


@pytest.mark.parametrize("name", CASES)
def test_host_mirror_from_triplets_and_csr_match_reference(name):
    from paper_1506_08938_b200 import SparseMatrix

    m = SparseMatrix.from_triplets(*_case(name))
    assert np.array_equal(m.indptr, GOLD[f"{name}/indptr"])
    assert np.array_equal(m.indices, GOLD[f"{name}/indices"])
    assert np.array_equal(m.values, GOLD[f"{name}/values"])
    rowptr, colidx, vals = m.csr()
    assert np.array_equal(rowptr, GOLD[f"{name}/t_indptr"])
    assert np.array_equal(colidx, GOLD[f"{name}/t_indices"])
    assert np.array_equal(vals, GOLD[f"{name}/t_values"])


@pytest.mark.parametrize("name", ERRS)
def test_host_mirror_errors_match_reference(name):
    from paper_1506_08938_b200 import SparseMatrix

    args, typ, msg = _err(name)
    with pytest.raises(ValueError) as ei:
        SparseMatrix.from_triplets(*args)
    assert type(ei.value).__name__ == typ and str(ei.value) == msg


def test_host_validate_catches_each_invariant():
    """The host constructor's checks on hand-broken CSC arrays, with the
    reference's exception types and messages (matrix.py:81-101), in its order."""
    from paper_1506_08938_b200 import SparseMatrix
    from paper_1506_08938_b200.exceptions import DataDomainError, MatrixSizeError

    def mk(indptr, rowidx, vals, rows=4, cols=3):
        return SparseMatrix(rows, cols, indptr, rowidx, vals)

    mk([0, 1, 2, 3], [0, 1, 3], [1.0, 2.0, 3.0])  # valid
    mk([0, 0, 0, 0], [], [])  # empty is valid
    cases = [
        (MatrixSizeError, "column pointer array must have cols+1 entries",
         ([0, 1, 3], [0, 1, 3], [1.0, 2.0, 3.0])),
        (MatrixSizeError, "column pointers must span [0, nnz]",
         ([1, 1, 2, 3], [0, 1, 3], [1.0, 2.0, 3.0])),
        (MatrixSizeError, "column pointers must be non-decreasing",
         ([0, 2, 1, 3], [0, 1, 3], [1.0, 2.0, 3.0])),
        (MatrixSizeError, "row-index and value arrays must match",
         ([0, 1, 2, 3], [0, 1], [1.0, 2.0, 3.0])),
        (MatrixSizeError, "row index out of range", ([0, 1, 2, 3], [0, 4, 3], [1.0, 2.0, 3.0])),
        (MatrixSizeError, "row index out of range", ([0, 1, 2, 3], [0, -1, 3], [1.0, 2.0, 3.0])),
        (MatrixSizeError, "row indices not strictly increasing in column 1",
         ([0, 1, 3, 3], [0, 2, 2], [1.0, 2.0, 3.0])),
        (MatrixSizeError, "row indices not strictly increasing in column 2",
         ([0, 1, 1, 3], [3, 3, 1], [1.0, 2.0, 3.0])),
        (DataDomainError, "sparse values must be finite",
         ([0, 1, 2, 3], [0, 1, 3], [1.0, float("nan"), 3.0])),
        (DataDomainError, "stored sparse values must be > 0 (no explicit zeros)",
         ([0, 1, 2, 3], [0, 1, 3], [1.0, 0.0, 3.0])),
    ]
    for typ, msg, args in cases:
        with pytest.raises(typ) as ei:
            mk(*args)
        assert type(ei.value) is typ and str(ei.value) == msg, (msg, str(ei.value))
    # a decreasing row across a column boundary is fine (column 0 ends at row 3)
    mk([0, 2, 3, 3], [1, 3, 0], [1.0, 2.0, 3.0])


@pytest.mark.parametrize("seed", range(6))
def test_host_containers_match_oracle_restatement(seed):
    """Randomised triplets with duplicates, explicit zeros and cancelling
    pairs: from_triplets / transpose / from_dense / to_dense agree bit for bit
    with the oracle's restatement of matrix.py (pinned to the reference by
    test_oracle_from_triplets_matches_reference)."""
    from paper_1506_08938_b200 import DenseMatrix, SparseMatrix

    rng = np.random.default_rng(seed)
    rows, cols = int(rng.integers(1, 40)), int(rng.integers(1, 40))
    t = int(rng.integers(0, 300))
    i = rng.integers(0, rows, t)
    j = rng.integers(0, cols, t)
    v = rng.choice([0.0, 1.0, 2.5, -2.5, 0.1, 0.2, 0.3], size=t) * rng.uniform(0.5, 2.0)
    if seed % 2:
        v = np.abs(v)  # nonnegative data: only cancellation-free sums
    for sd in (True, False):
        try:
            want = orc.Csc.from_triplets(rows, cols, i, j, v, sum_duplicates=sd)
            want_err = None
        except ValueError as e:
            want_err = (type(e).__name__, str(e))
        try:
            got = SparseMatrix.from_triplets(rows, cols, i, j, v, sum_duplicates=sd)
            got_err = None
        except ValueError as e:
            got_err = (type(e).__name__, str(e))
        if want_err is not None:
            # argument errors: same message as the restatement
            assert got_err is not None and got_err[1] == want_err[1]
            continue
        if got_err is not None:
            # the restatement skips the constructor's validation; the product
            # rejects exactly the outputs that break an invariant
            dup = any((np.diff(want.indices[a:b]) <= 0).any()
                      for a, b in zip(want.indptr[:-1], want.indptr[1:]))
            if dup:
                assert got_err[1].startswith("row indices not strictly increasing")
            else:
                assert (want.values <= 0).any()
                assert got_err == ("DataDomainError",
                                   "stored sparse values must be > 0 (no explicit zeros)")
            continue
        assert np.array_equal(got.indptr, want.indptr)
        assert np.array_equal(got.indices, want.indices)
        assert np.array_equal(got.values, want.values)
        if not (got.values > 0).all():
            continue
        tw, tg = want.transpose(), got.transpose()
        assert np.array_equal(tg.indptr, tw.indptr)
        assert np.array_equal(tg.indices, tw.indices)
        assert np.array_equal(tg.values, tw.values)
        d = got.to_dense()
        assert isinstance(d, DenseMatrix) and d.array.flags.f_contiguous
        assert np.array_equal(d.array, want.to_dense())
        back = SparseMatrix.from_dense(d)
        assert np.array_equal(back.indptr, got.indptr)
        assert np.array_equal(back.indices, got.indices)
        assert np.array_equal(back.values, got.values)


def test_dense_container_layout():
    from paper_1506_08938_b200 import DenseMatrix
    from paper_1506_08938_b200.exceptions import MatrixSizeError

    a = np.arange(12.0).reshape(3, 4)
    d = DenseMatrix(a)
    assert d.array.flags.f_contiguous and (d.rows, d.cols) == (3, 4)
    assert np.array_equal(d.data, a.reshape(-1, order="F"))
    assert np.array_equal(d.column(2), a[:, 2])
    f = np.asfortranarray(a)
    assert DenseMatrix(f).array is f  # no copy for Fortran float64 input
    c = d.copy()
    c.array[0, 0] = -1.0
    assert d.array[0, 0] == 0.0
    z = DenseMatrix.zeros(2, 5)
    assert z.array.shape == (2, 5) and z.array.flags.f_contiguous and not z.array.any()
    with pytest.raises(MatrixSizeError, match="expected 2-D array, got ndim=1"):
        DenseMatrix(np.ones(3))


# ---------------------------------------------------------------------------
# GPU
# ---------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_device_from_triplets_and_csr_bit_exact(name, dtype):
    import torch

    from paper_1506_08938_b200.ingest import DeviceCsc

    dt = torch.float64 if dtype == "f64" else torch.float32
    m = DeviceCsc.from_triplets(*_case(name)[:5], sum_duplicates=_case(name)[5], dtype=dt)
    want_v = GOLD[f"{name}/values"]
    if dtype == "f32":
        want_v = want_v.astype(np.float32)
    assert np.array_equal(m.indptr.cpu().numpy(), GOLD[f"{name}/indptr"])
    assert np.array_equal(m.rowidx.cpu().numpy().astype(np.int64), GOLD[f"{name}/indices"])
    assert np.array_equal(m.values.cpu().numpy(), want_v)
    rowptr, colidx, vals = m.csr()
    want_t = GOLD[f"{name}/t_values"]
    if dtype == "f32":
        want_t = want_t.astype(np.float32)
    assert np.array_equal(rowptr.cpu().numpy(), GOLD[f"{name}/t_indptr"])
    assert np.array_equal(colidx.cpu().numpy().astype(np.int64), GOLD[f"{name}/t_indices"])
    assert np.array_equal(vals.cpu().numpy(), want_t)
    back = m.to_host()
    assert np.array_equal(back.indices, GOLD[f"{name}/indices"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ERRS)
def test_device_errors_match_reference(name):
    from paper_1506_08938_b200.ingest import DeviceCsc

    args, typ, msg = _err(name)
    with pytest.raises(ValueError) as ei:
        DeviceCsc.from_triplets(*args[:5], sum_duplicates=args[5])
    assert type(ei.value).__name__ == typ and str(ei.value) == msg


@pytest.mark.gpu
def test_device_validate_catches_each_invariant():
    """The constructor's checks on hand-broken CSC arrays (matrix.py:81-101)."""
    import torch

    from paper_1506_08938_b200.exceptions import DataDomainError, MatrixSizeError
    from paper_1506_08938_b200.ingest import DeviceCsc

    def mk(indptr, rowidx, vals, rows=4, cols=3):
        dev = torch.device("cuda")
        return DeviceCsc(rows, cols, torch.tensor(indptr, dtype=torch.int64, device=dev),
                         torch.tensor(rowidx, dtype=torch.int32, device=dev),
                         torch.tensor(vals, dtype=torch.float64, device=dev))

    mk([0, 1, 2, 3], [0, 1, 3], [1.0, 2.0, 3.0])  # valid
    with pytest.raises(MatrixSizeError, match=r"span \[0, nnz\]"):
        mk([1, 1, 2, 3], [0, 1, 3], [1.0, 2.0, 3.0])
    with pytest.raises(MatrixSizeError, match="non-decreasing"):
        mk([0, 2, 1, 3], [0, 1, 3], [1.0, 2.0, 3.0])
    with pytest.raises(MatrixSizeError, match="row index out of range"):
        mk([0, 1, 2, 3], [0, 4, 3], [1.0, 2.0, 3.0])
    with pytest.raises(MatrixSizeError, match="strictly increasing in column 1"):
        mk([0, 1, 3, 3], [0, 2, 2], [1.0, 2.0, 3.0])
    with pytest.raises(DataDomainError, match="finite"):
        mk([0, 1, 2, 3], [0, 1, 3], [1.0, float("inf"), 3.0])
    with pytest.raises(DataDomainError, match="> 0"):
        mk([0, 1, 2, 3], [0, 1, 3], [1.0, 0.0, 3.0])
    with pytest.raises(MatrixSizeError, match="cols\\+1"):
        mk([0, 1, 3], [0, 1, 3], [1.0, 2.0, 3.0])


@pytest.mark.gpu
def test_device_csr_of_config3_matches_host():
    """Full BASELINE config-3 matrix (5e6 nonzeros): device upload + narrowing
    + validation + CSR equal the host mirror's arrays exactly."""
    import torch

    from oracle import generators
    from paper_1506_08938_b200 import SparseMatrix
    from paper_1506_08938_b200.ingest import DeviceCsc

    x, _ = generators.make(3)
    V = SparseMatrix(x.rows, x.cols, x.indptr, x.indices, x.values, validate=False)
    d = DeviceCsc.from_host(V, dtype=torch.float32)
    rowptr, colidx, vals = d.csr()
    hr, hc, hv = V.csr()
    assert np.array_equal(rowptr.cpu().numpy(), hr)
    assert np.array_equal(colidx.cpu().numpy().astype(np.int64), hc)
    assert np.array_equal(vals.cpu().numpy(), hv.astype(np.float32))
    # and from the triplets of the same matrix (shuffled) the CSC comes back
    col_of = np.repeat(np.arange(x.cols), np.diff(x.indptr))
    perm = np.random.default_rng(3).permutation(x.indices.size)
    d2 = DeviceCsc.from_triplets(x.rows, x.cols, x.indices[perm], col_of[perm],
                                 x.values[perm])
    assert np.array_equal(d2.indptr.cpu().numpy(), x.indptr)
    assert np.array_equal(d2.rowidx.cpu().numpy().astype(np.int64), x.indices)
    assert np.array_equal(d2.values.cpu().numpy(), x.values)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_fit_from_device_csc_equals_host_input(precision):
    """The same fit from a host SparseMatrix and from a DeviceCsc: identical
    bits given the same starting factors; fit() from a DeviceCsc (mean taken
    on the device) within 1e-9 of the host-input fit."""
    import torch

    from oracle import generators
    from paper_1506_08938_b200 import NmfConfig, SparseMatrix, fit
    from paper_1506_08938_b200.ingest import DeviceCsc
    from paper_1506_08938_b200.nmf import FitSession, initial_factors

    x = generators.sparse_zipf(1500, 1000, 0.01, 8)
    V = SparseMatrix(x.rows, x.cols, x.indptr, x.indices, x.values)
    dt = torch.float64 if precision == "fp64" else torch.float32
    cfg = NmfConfig(rank=8, max_outer=6, seed=3, rel_change_tol=0.0, precision=precision)
    init = initial_factors(V, cfg)
    m1, l1 = FitSession(V, cfg, init=init).run()
    m2, l2 = FitSession(DeviceCsc.from_host(V, dtype=dt), cfg, init=init).run()
    if precision == "fp64":
        assert l1.objective == l2.objective
    else:  # ||X||^2 of the float32 device values vs of the host float64 values
        np.testing.assert_allclose(l2.objective, l1.objective, rtol=1e-7)
    assert np.array_equal(m1.G.array, m2.G.array)
    assert np.array_equal(m1.F.array, m2.F.array)
    _, l3 = fit(DeviceCsc.from_host(V, dtype=dt), cfg)
    # fp32: the init scale is the mean of the float32 values (the fp32
    # trajectory then moves at the 1e-4 level, as under any 1-ulp change)
    np.testing.assert_allclose(l3.objective, l1.objective, rtol=1e-9 if precision == "fp64"
                               else 1e-3)
