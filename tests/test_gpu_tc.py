"""Tensor-core (tcgen05 3xTF32) data-product GEMM vs an fp64 reference of the
same op (the dense passes G^T X and X F^T).  Tolerance: 3xTF32 carries ~21
mantissa bits per product, accumulation in fp32 -> 2e-5 relative to the
magnitude scale of the output (|A||B|).  The tensor core's fp32 accumulate
truncates, so the kernel folds every few k-blocks into a round-to-nearest
running sum; the error must not grow with K.  splits <= 0 selects the balanced
(stream-K style) schedule: its unused partial slots must come back zeroed
(the output buffer starts as NaN)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _tc(A, B, splits=1, stages=0):
    """C = A (M x K) @ B (K x N) through nmfb_split_transpose + nmfb_tc_gemm."""
    from paper_1506_08938_b200 import _lib as L
    from paper_1506_08938_b200 import device as D

    dev = D.require_cuda()
    M, K = A.shape
    N = B.shape[1]
    a = torch.from_numpy(np.ascontiguousarray(A, dtype=np.float32)).to(dev)
    b = torch.from_numpy(np.ascontiguousarray(B, dtype=np.float32)).to(dev)
    bt_hi = torch.empty((N, K), dtype=torch.float32, device=dev)
    bt_lo = torch.empty((N, K), dtype=torch.float32, device=dev)
    L.call("nmfb_split_transpose", D.vp(b), K, N, D.vp(bt_hi), D.vp(bt_lo), D.stream_handle())
    S = L.lib().nmfb_tc_parts(M, K, N, splits)
    C = torch.full((S, M, N), float("nan"), dtype=torch.float32, device=dev)
    L.call("nmfb_tc_gemm", D.vp(a), M, K, D.vp(bt_hi), D.vp(bt_lo), N, D.vp(C), splits, stages,
           D.stream_handle())
    torch.cuda.synchronize()
    return C.double().sum(0).cpu().numpy(), S


@pytest.mark.parametrize("M,K,N,splits", [
    (128, 32, 16, 1), (256, 64, 50, 1), (300, 1000, 50, 3), (1000, 4096, 64, 4),
    (20000, 1024, 50, 2), (77, 96, 10, 1), (513, 2000, 100, 5), (256, 512, 160, 2), (300, 10000, 50, 1),
    (128, 32, 16, 0), (300, 1000, 50, 0), (20000, 1024, 50, 0), (10000, 4000, 50, 0),
    (513, 2000, 100, 0), (256, 512, 160, 0), (77, 96, 10, 0), (40000, 64, 33, 0), (1000, 20000, 64, 0),
])
def test_tc_gemm_matches_fp64(M, K, N, splits):
    rng = np.random.default_rng(M + K + N)
    A = rng.exponential(size=(M, K)).astype(np.float32).astype(np.float64)
    B = rng.uniform(size=(K, N)).astype(np.float32).astype(np.float64)
    C, S = _tc(A, B, splits)
    want = A @ B
    scale = np.abs(A) @ np.abs(B)
    err = np.abs(C - want) / scale
    assert np.isfinite(C).all()
    assert err.max() < 5e-6, err.max()


@pytest.mark.parametrize("stages", [2, 3, 4])
def test_tc_gemm_stage_depths_agree(stages):
    rng = np.random.default_rng(5)
    A = rng.uniform(size=(512, 2048))
    B = rng.uniform(size=(2048, 50))
    C0, _ = _tc(A, B, 2, stages=4)
    C1, _ = _tc(A, B, 2, stages=stages)
    assert np.array_equal(C0, C1)  # same tiles, same order -> bit-identical


def test_tc_gemm_balanced_deterministic():
    rng = np.random.default_rng(9)
    A = rng.uniform(size=(3000, 5000))
    B = rng.uniform(size=(5000, 50))
    C0, S0 = _tc(A, B, 0)
    C1, S1 = _tc(A, B, 0)
    assert S0 == S1 and np.array_equal(C0, C1)
    C2, _ = _tc(A, B, 4)
    assert np.abs(C2 - C0).max() / np.abs(C0).max() < 1e-6


@pytest.mark.parametrize("m,n,r", [(130, 77, 5), (256, 384, 50), (1000, 500, 64), (300, 1030, 37)])
def test_dense_residual_kmajor_matches_fp64(m, n, r):
    """0.5 ||X - G F||^2 from the k-major operands, fp32 FFMA + fp64 sums."""
    from paper_1506_08938_b200 import _lib as L
    from paper_1506_08938_b200 import device as D

    dev = D.require_cuda()
    rng = np.random.default_rng(m + n + r)
    G = rng.uniform(size=(n, r)).astype(np.float32)
    F = rng.uniform(size=(r, m)).astype(np.float32)
    X = (G.astype(np.float64) @ F + rng.normal(0, 0.1, size=(n, m))).astype(np.float32)
    XT = torch.from_numpy(np.ascontiguousarray(X.T)).to(dev)
    Gt = torch.from_numpy(np.ascontiguousarray(G.T)).to(dev)
    Ft = torch.from_numpy(np.ascontiguousarray(F)).to(dev)
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    ws = torch.empty((L.lib().nmfb_residual_workspace_bytes(m, n) // 8 + 1,),
                     dtype=torch.float64, device=dev)
    L.call("nmfb_dense_residual_kmajor", D.vp(XT), m, n, D.vp(Gt), D.vp(Ft), r, D.vp(out),
           D.vp(ws), D.stream_handle())
    want = 0.5 * np.sum((X.astype(np.float64) - G.astype(np.float64) @ F.astype(np.float64)) ** 2)
    assert abs(float(out.item()) - want) / want < 1e-5


def _slices(A):
    from paper_1506_08938_b200 import _lib as L
    from paper_1506_08938_b200 import device as D

    dev = D.require_cuda()
    rows, r = A.shape
    a = torch.from_numpy(np.ascontiguousarray(A, dtype=np.float32)).to(dev)
    out = torch.zeros((L.lib().nmfb_slice_bytes(rows, r),), dtype=torch.uint8, device=dev)
    L.call("nmfb_slice_u8", D.vp(a), rows, r, r, D.vp(out), D.stream_handle())
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("rows,r", [(1, 1), (100, 50), (1000, 64), (333, 128), (77, 7)])
def test_slice_u8_reconstructs(rows, r):
    """Three 8-bit slices + a power-of-two row scale represent each row to
    2^-24 of its max (the last slice rounded to nearest)."""
    rng = np.random.default_rng(rows + r)
    A = rng.exponential(size=(rows, r)).astype(np.float32)
    A[rng.uniform(size=A.shape) < 0.3] = 0.0  # NNLS outputs are sparse
    if rows > 2:
        A[1] = 0.0  # an all-zero row
        A[2] *= 1e-30  # tiny magnitudes
    out = _slices(A).cpu().numpy()
    kb = 64 if r <= 64 else 128
    S = out[: 3 * rows * kb].reshape(3, rows, kb).astype(np.float64)
    scale = out[3 * rows * kb: 3 * rows * kb + 4 * rows].view(np.float32).astype(np.float64)
    assert (S[:, :, r:] == 0).all()
    rec = (S[0] / 2.0**8 + S[1] / 2.0**16 + S[2] / 2.0**24)[:, :r] * scale[:, None]
    mx = A.max(axis=1, keepdims=True).astype(np.float64)
    err = np.abs(rec - A) / np.where(mx > 0, mx, 1.0)
    assert err.max() <= 2.0**-24, err.max()
    assert np.all(rec[A == 0] == 0)


@pytest.mark.parametrize("n,m,r", [(130, 84, 5), (256, 400, 50), (1000, 500, 64), (300, 1032, 37),
                                   (777, 2000, 128), (128, 80, 1)])
def test_residual_i8_matches_fp64(n, m, r):
    """0.5 ||X - G F||^2 with G F on the int8 tensor cores from 8-bit slices:
    exact products, so the result tracks fp64 at a near-exact fit too."""
    from paper_1506_08938_b200 import _lib as L
    from paper_1506_08938_b200 import device as D

    dev = D.require_cuda()
    rng = np.random.default_rng(n + m + r)
    G = rng.exponential(size=(n, r)).astype(np.float32)
    F = rng.exponential(size=(r, m)).astype(np.float32)
    G[rng.uniform(size=G.shape) < 0.2] = 0.0
    GF = G.astype(np.float64) @ F.astype(np.float64)
    # a near-exact fit: |X - G F| ~ 1e-3 |X|, the regime where a biased G F fails
    X = (GF * (1.0 + 1e-3 * rng.normal(size=GF.shape))).astype(np.float32)
    Gsl = _slices(G)
    Fsl = _slices(np.ascontiguousarray(F.T))
    x = torch.from_numpy(X).to(dev)
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    ws = torch.empty((L.lib().nmfb_residual_i8_workspace_bytes() // 8 + 1,), dtype=torch.float64,
                     device=dev)
    L.call("nmfb_residual_i8", D.vp(x), n, m, D.vp(Gsl), D.vp(Fsl), r, D.vp(out), D.vp(ws),
           D.stream_handle())
    want = 0.5 * np.sum((X.astype(np.float64) - GF) ** 2)
    got = float(out.item())
    assert abs(got - want) / want < 2e-5, (got, want)
