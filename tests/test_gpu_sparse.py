"""Sparse data products (the fast-path gathers) against fp64 numpy on
Zipf-skewed CSC/CSR data: h = mu1 - G^T X (csc_linear) and Y^T = X F^T
(csr_yt_chunked, heavy rows split into chunks and folded).  r % 4 == 0 takes
the 16-byte vector-load kernels, other r the scalar ones; both must agree
with fp64 to fp32 accumulation accuracy."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _csc(n, m, density, seed):
    rng = np.random.default_rng(seed)
    # Zipf-popular rows, skewed column counts, a few very heavy rows / columns
    counts = np.minimum(rng.zipf(1.3, size=m), 3 * n // 4)
    counts = np.maximum(1, (counts * density * n * m / counts.sum()).astype(np.int64))
    counts[:3] = n // 2
    pop = 1.0 / np.arange(1, n + 1)
    pop /= pop.sum()
    indptr = np.zeros(m + 1, dtype=np.int64)
    rows, vals = [], []
    for j in range(m):
        rr = np.sort(rng.choice(n, size=min(int(counts[j]), n), replace=False, p=pop))
        rows.append(rr)
        vals.append(rng.exponential(size=len(rr)))
        indptr[j + 1] = indptr[j] + len(rr)
    return indptr, np.concatenate(rows).astype(np.int32), np.concatenate(vals)


@pytest.mark.parametrize("r", [4, 50, 100, 128])
def test_sparse_products_match_fp64(r):
    import scipy.sparse as sp

    from paper_1506_08938_b200 import _lib as L
    from paper_1506_08938_b200 import device as D

    dev = D.require_cuda()
    n, m = 3000, 1200
    indptr, rows, vals = _csc(n, m, 0.01, r)
    X = sp.csc_matrix((vals, rows, indptr), shape=(n, m))
    rng = np.random.default_rng(r)
    G = rng.uniform(size=(n, r)).astype(np.float32)
    FT = rng.uniform(size=(m, r)).astype(np.float32)
    mu1 = 0.25
    # csc_linear: h[col] = mu1 - sum_row G[row] v
    h = torch.zeros((m, r), dtype=torch.float32, device=dev)
    keep = []  # device inputs must outlive the asynchronous kernels

    def t(a):
        x = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        keep.append(x)
        return x

    ip, rw, vv = t(indptr), t(rows), t(vals.astype(np.float32))
    L.call("nmfb_csc_linear", L.F32, L.MODE_FAST, D.vp(ip), D.vp(rw), D.vp(vv), 0, m, D.vp(t(G)),
           r, mu1, D.vp(h), D.stream_handle())
    Xf = X.astype(np.float32).astype(np.float64)
    want_h = mu1 - (Xf.T @ G.astype(np.float64))
    got_h = h.double().cpu().numpy()
    scale = np.abs(Xf.T) @ np.abs(G.astype(np.float64)) + 1.0
    assert np.max(np.abs(got_h - want_h) / scale) < 2e-6
    # csr_yt_chunked: Y^T[row] = sum_col FT[col] v, fp64 accumulation
    Xr = X.tocsr()
    Xr.sort_indices()
    rowptr = Xr.indptr.astype(np.int64)
    chunks, heavy, nslots = D.csr_chunk_plan(rowptr, chunk=64)
    assert len(heavy) > 0  # the heavy-row fold is exercised
    yt = torch.zeros((n, r), dtype=torch.float64, device=dev)
    part = torch.zeros((max(nslots, 1), r), dtype=torch.float64, device=dev)
    L.call("nmfb_csr_yt_chunked", L.F32, D.vp(t(chunks)), len(chunks), D.vp(t(heavy)), len(heavy),
           D.vp(t(Xr.indices.astype(np.int32))), D.vp(t(Xr.data.astype(np.float32))), D.vp(t(FT)),
           r, L.F64, D.vp(yt), D.vp(part), D.stream_handle())
    want_y = Xf @ FT.astype(np.float64)
    got_y = yt.cpu().numpy()
    assert np.max(np.abs(got_y - want_y) / (want_y + 1e-30)) < 1e-12


@pytest.mark.parametrize("r", [100, 200, 52])
def test_blocked_spmm_bit_identical(r, monkeypatch):
    """L2-blocked G^T X / X F^T passes (csrc/sparse_blocked.cu): a fit with
    the gathered factors cut into ~1 MB blocks equals the unblocked fit bit
    for bit (running sums carried exactly through the outputs)."""
    from oracle import generators
    from paper_1506_08938_b200 import NmfConfig, SparseMatrix
    from paper_1506_08938_b200.nmf import FitSession

    x = generators.sparse_zipf(20000, 8000, 2e-3, 9)
    V = SparseMatrix(x.rows, x.cols, x.indptr, x.indices, x.values, validate=False)
    cfg = NmfConfig(rank=r, max_outer=3, seed=2, rel_change_tol=0.0, precision="fp32")
    # a blocked X F^T carries its running sums through an fp64 Y^T: compare
    # with the unblocked pass writing fp64 Y^T too
    monkeypatch.setenv("NMFB_YT64", "1")
    monkeypatch.setenv("NMFB_SPMM_BLOCK_MB", "0")
    monkeypatch.setenv("NMFB_SPMM_BLOCK_MB_F", "0")
    m0, l0 = FitSession(V, cfg).run()
    monkeypatch.setenv("NMFB_SPMM_BLOCK_MB", "1")
    monkeypatch.setenv("NMFB_SPMM_BLOCK_MB_F", "1")
    s1 = FitSession(V, cfg)
    assert s1.state._spmm_plan()[0] > 1 and s1.state._spmm_plan()[2] > 1
    m1, l1 = s1.run()
    assert np.array_equal(m0.G.array, m1.G.array)
    assert np.array_equal(m0.F.array, m1.F.array)
    assert l0.objective == l1.objective


def test_gram_side_stream_overlap_bit_identical(monkeypatch):
    """The sparse path's Grams on a side stream (beside G^T X / X F^T) give the
    same bits as the serial order, and the lagged log sees the side-stream
    objective pieces."""
    from oracle import generators
    from paper_1506_08938_b200 import NmfConfig, SparseMatrix
    from paper_1506_08938_b200.nmf import FitSession

    x = generators.sparse_zipf(20000, 8000, 2e-3, 4)
    V = SparseMatrix(x.rows, x.cols, x.indptr, x.indices, x.values, validate=False)
    cfg = NmfConfig(rank=64, max_outer=5, seed=3, rel_change_tol=1e-12, precision="fp32")
    monkeypatch.setenv("NMFB_GRAM_OVERLAP", "0")
    s0 = FitSession(V, cfg)
    assert s0.state.gside is None
    m0, l0 = s0.run()
    monkeypatch.setenv("NMFB_GRAM_OVERLAP", "1")
    s1 = FitSession(V, cfg)
    assert s1.state.gside is not None
    m1, l1 = s1.run()
    assert np.array_equal(m0.G.array, m1.G.array)
    assert np.array_equal(m0.F.array, m1.F.array)
    assert l0.objective == l1.objective


def test_device_chunk_plan_equals_host_plan():
    """nmfb_csr_chunk_plan builds exactly device.csr_chunk_plan's tables."""
    import torch

    from paper_1506_08938_b200 import device as D

    dev = D.require_cuda()
    rng = np.random.default_rng(12)
    for n, chunk in ((1, 256), (5000, 256), (3000, 7), (20000, 64)):
        k = np.minimum(rng.zipf(1.3, size=n) - 1, 3000)
        k[rng.random(n) < 0.1] = 0  # empty rows
        rowptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(k, out=rowptr[1:])
        hc, hh, hs = D.csr_chunk_plan(rowptr, chunk=chunk)
        dc, dh, ds = D.device_chunk_plan(torch.from_numpy(rowptr).to(dev), n, int(rowptr[-1]),
                                         dev, chunk=chunk)
        assert ds == hs
        assert np.array_equal(dc.cpu().numpy(), hc)
        assert np.array_equal(dh.cpu().numpy().reshape(-1, 3), hh.reshape(-1, 3))
