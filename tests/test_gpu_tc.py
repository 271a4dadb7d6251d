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
