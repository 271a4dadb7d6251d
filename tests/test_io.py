"""Dataset loaders / writers (reference io.py) against the reference's own
outputs on good and malformed files (tests/golden/io.npz, io/*.txt, made by
tests/golden/make_golden_io.py): arrays equal, and errors with the
reference's exception type, line and message."""

import os
import warnings

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "io.npz"))
KEYS = sorted({k.rsplit("/", 1)[0] for k in GOLD.files})


def _fmt(name):
    return ("uci-bow" if name.startswith("bow") else
            "matrix-market" if name.startswith("mm") else "csv-dense")


@pytest.mark.parametrize("key", KEYS)
def test_loader_matches_reference(key, monkeypatch):
    from paper_1506_08938_b200 import io

    monkeypatch.chdir(HERE)  # the goldens carry paths relative to tests/
    name, mode = key.split("/")
    spec = io.DatasetSpec(os.path.join("golden", "io", name + ".txt"), _fmt(name),
                          tfidf=(mode == "tfidf"))
    want_err = str(GOLD[f"{key}/error"])
    with warnings.catch_warnings(record=True) as caught:
        warnings.simplefilter("always")
        if want_err:
            with pytest.raises(ValueError) as ei:
                io.load(spec)
            assert f"{type(ei.value).__name__}: {ei.value}" == want_err
            return
        m = io.load(spec)
    assert "|".join(str(w.message) for w in caught) == str(GOLD[f"{key}/warnings"])
    if f"{key}/array" in GOLD.files:
        assert np.array_equal(m.array, GOLD[f"{key}/array"])
    else:
        assert [m.rows, m.cols] == list(GOLD[f"{key}/shape"])
        assert np.array_equal(m.indptr, GOLD[f"{key}/indptr"])
        assert np.array_equal(m.indices, GOLD[f"{key}/indices"])
        assert np.array_equal(m.values, GOLD[f"{key}/values"])


def test_writers_round_trip(tmp_path):
    from paper_1506_08938_b200 import DenseMatrix, SparseMatrix, io
    from paper_1506_08938_b200.nmf import ConvergenceLog

    rng = np.random.default_rng(0)
    a = np.where(rng.random((7, 5)) < 0.4, rng.uniform(0.1, 3, (7, 5)), 0.0)
    io.write_matrix_market(SparseMatrix.from_dense(a), tmp_path / "a.mtx")
    back = io.load(io.DatasetSpec(tmp_path / "a.mtx", "matrix-market"))
    assert np.array_equal(back.to_dense().array, a)
    io.write_dense_csv(DenseMatrix(a), tmp_path / "a.csv")
    assert np.array_equal(io.load(io.DatasetSpec(tmp_path / "a.csv", "csv-dense")).array, a)
    log = ConvergenceLog()
    for k in range(3):
        log.append(1.0 / (k + 1), 0.1 * k, 10 + k, 7)
    io.write_log(log, tmp_path / "log.csv")
    assert (tmp_path / "log.csv").read_text().splitlines()[0] == io.LOG_HEADER
    r = io.read_log(tmp_path / "log.csv")
    assert r.objective == log.objective and r.inner_iterations == log.inner_iterations
    assert r.k_bar == log.k_bar
    with pytest.raises(ValueError):
        io.write_log(ConvergenceLog(), tmp_path / "empty.csv")
    with pytest.raises(ValueError):
        io.DatasetSpec("x", "parquet")


@pytest.mark.gpu
def test_load_to_device_matches_host(monkeypatch):
    """load(spec, device=True): the triplets go to DeviceCsc.from_triplets."""
    from paper_1506_08938_b200 import io

    monkeypatch.chdir(HERE)
    for name, tfidf in (("bow_dups", True), ("bow_good", False), ("mm_good", False)):
        spec = io.DatasetSpec(os.path.join("golden", "io", name + ".txt"), _fmt(name),
                              tfidf=tfidf)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            host = io.load(spec)
            dev = io.load(spec, device=True)
        assert np.array_equal(dev.indptr.cpu().numpy(), host.indptr)
        assert np.array_equal(dev.rowidx.cpu().numpy().astype(np.int64), host.indices)
        assert np.array_equal(dev.values.cpu().numpy(), host.values)
