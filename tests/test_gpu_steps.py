"""GPU parity of the coefficient / component steps and of the drop-in shard
kernels, against the reference's own outputs (tests/golden/steps.npz) and the
oracle.  fp64 check mode: bit-exact, including the per-worker reduce order."""

import os

import numpy as np
import pytest

from oracle import nmf_oracle as orc

GOLD = os.path.join(os.path.dirname(__file__), "golden")
STEPS = np.load(os.path.join(GOLD, "steps.npz"))

pytestmark = pytest.mark.gpu

VARIANTS = {
    "plain_w1": dict(workers=1),
    "plain_w3": dict(workers=3),
    "reg_w1": dict(workers=1, mu1=0.05, mu2=0.02, beta1=0.03, beta2=0.01),
    "reg_w3": dict(workers=3, mu1=0.05, mu2=0.02, beta1=0.03, beta2=0.01),
}


def _data(kind):
    from paper_1506_08938_b200 import SparseMatrix

    arr = STEPS["data/arr"]
    return arr, (SparseMatrix.from_dense(arr) if kind == "sparse" else np.ascontiguousarray(arr.T))


@pytest.mark.parametrize("kind", ["dense", "sparse"])
@pytest.mark.parametrize("variant", list(VARIANTS))
def test_run_estep_mstep_fp64_bit_exact(kind, variant):
    from paper_1506_08938_b200 import NmfConfig
    from paper_1506_08938_b200.parallel import run_estep, run_mstep

    arr, V = _data(kind)
    g0, ft0 = STEPS["data/g"], STEPS["data/ft"]
    cfg = NmfConfig(rank=g0.shape[1], seed=0, precision="fp64", **VARIANTS[variant])
    p = f"{kind}/{variant}"
    G, FT = g0.copy(), ft0.copy()
    Y, H_f, e = run_estep(V, G, STEPS[p + "/Q_g"], cfg, FT)
    assert np.array_equal(FT, STEPS[p + "/FT"])
    assert np.array_equal(np.ascontiguousarray(Y.array), STEPS[p + "/Y"])
    assert np.array_equal(np.ascontiguousarray(H_f.array), STEPS[p + "/H_f"])
    assert e.inner_iterations == int(STEPS[p + "/e_inner"])
    m = run_mstep(Y, H_f, cfg, G)
    assert np.array_equal(G, STEPS[p + "/G"])
    assert m.inner_iterations == int(STEPS[p + "/m_inner"])


@pytest.mark.parametrize("kind", ["dense", "sparse"])
def test_run_estep_fp32_close(kind):
    from gpu_util import floored_rel

    from paper_1506_08938_b200 import NmfConfig
    from paper_1506_08938_b200.parallel import run_estep, run_mstep

    arr, V = _data(kind)
    g0, ft0 = STEPS["data/g"], STEPS["data/ft"]
    cfg = NmfConfig(rank=g0.shape[1], seed=0, precision="fp32")
    p = f"{kind}/plain_w1"
    G, FT = g0.copy(), ft0.copy()
    Y, H_f, e = run_estep(V, G, STEPS[p + "/Q_g"], cfg, FT)
    assert floored_rel(FT, STEPS[p + "/FT"]) < 1e-2
    np.testing.assert_allclose(np.ascontiguousarray(Y.array), STEPS[p + "/Y"], rtol=1e-3,
                               atol=1e-4 * np.abs(STEPS[p + "/Y"]).max())
    m = run_mstep(Y, H_f, cfg, G)
    assert floored_rel(G, STEPS[p + "/G"]) < 1e-2


@pytest.mark.parametrize("kind", ["dense", "sparse"])
@pytest.mark.parametrize("lo,hi", [(0, 150), (32, 96), (7, 130)])
def test_dropin_shard_kernels_fp64_bit_exact(kind, lo, hi):
    """paper_1506_08938_b200.kernels.* == oracle (== reference) shard calls."""
    from paper_1506_08938_b200 import kernels

    arr = STEPS["data/arr"]
    g0, ft0 = STEPS["data/g"], STEPS["data/ft"]
    n, m = arr.shape
    r = g0.shape[1]
    Q_g = orc.gram(g0)
    sa, act, idx, Qa = orc.rescale_for_step(Q_g + 0.04 * np.eye(r))
    args = (Qa, sa, idx, act, 0.05, 0.1, 500, 0.5)
    FT1, YT1, HP1 = ft0.copy(), np.zeros((n, r)), np.zeros((r, r))
    FT2, YT2, HP2 = ft0.copy(), np.zeros((n, r)), np.zeros((r, r))
    if kind == "dense":
        VT = np.ascontiguousarray(arr.T)
        want = orc.estep_dense(VT, lo, hi, g0, *args, FT1, YT1, HP1)
        got = kernels.estep_dense(VT, lo, hi, g0, *args, FT2, YT2, HP2)
    else:
        V = orc.Csc.from_dense(arr)
        want = orc.estep_sparse(V.indptr, V.indices, V.values, lo, hi, g0, *args, FT1, YT1, HP1)
        got = kernels.estep_sparse(V.indptr, V.indices, V.values, lo, hi, g0, *args, FT2, YT2,
                                   HP2)
    assert got == want
    assert np.array_equal(FT2, FT1)
    assert np.array_equal(YT2, YT1)
    assert np.array_equal(HP2, HP1)
    # component step on the accumulated Y^T
    G1, G2 = g0.copy(), g0.copy()
    sa2, act2, idx2, Qa2 = orc.rescale_for_step(orc.gram(FT1) + 0.02 * np.eye(r))
    margs = (Qa2, sa2, idx2, act2, 0.01, 0.1, 500, 0.0)
    want = orc.mstep_rows(YT1, 3, n, *margs, G1)
    got = kernels.mstep_rows(YT1, 3, n, *margs, G2)
    assert got == want
    assert np.array_equal(G2, G1)


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
@pytest.mark.parametrize("diag_add", [0.0, 0.02])
@pytest.mark.parametrize("rows,r", [(1000, 10), (5000, 50), (3000, 100), (257, 130), (0, 8)])
def test_gram_rescale_fused_equals_separate(dtype, diag_add, rows, r):
    """nmfb_gram_rescale (rescale in the Gram reduce's epilogue) writes exactly
    what nmfb_gram followed by nmfb_rescale writes -- including frozen dims."""
    import torch

    from paper_1506_08938_b200 import _lib as L
    from paper_1506_08938_b200 import device as D

    dev = D.require_cuda()
    code = L.F64 if dtype == "fp64" else L.F32
    tdt = torch.float64 if dtype == "fp64" else torch.float32
    rng = np.random.default_rng(rows + r)
    A = rng.exponential(size=(rows, r))
    if r > 4:
        A[:, 3] = 0.0  # a frozen (zero-diagonal) dimension
    a = torch.from_numpy(A).to(dev, tdt)
    ws = torch.zeros((L.lib().nmfb_gram_workspace_bytes(max(rows, 1), r) // 8 + 1,),
                     dtype=torch.float64, device=dev)
    outs = []
    for fused in (True, False):
        g = torch.zeros((r, r), dtype=torch.float64, device=dev)
        Qa = torch.zeros((r * r,), dtype=tdt, device=dev)
        sa = torch.zeros((r,), dtype=tdt, device=dev)
        act = torch.zeros((r,), dtype=torch.int32, device=dev)
        active = torch.zeros((r,), dtype=torch.uint8, device=dev)
        ra = torch.zeros((1,), dtype=torch.int32, device=dev)
        if fused:
            L.call("nmfb_gram_rescale", code, D.vp(a), rows, r, r, D.vp(g), D.vp(ws), diag_add,
                   D.vp(Qa), D.vp(sa), D.vp(act), D.vp(active), D.vp(ra), D.stream_handle())
        else:
            L.call("nmfb_gram", code, D.vp(a), rows, r, r, D.vp(g), D.vp(ws), D.stream_handle())
            L.call("nmfb_rescale", code, D.vp(g), r, diag_add, D.vp(Qa), D.vp(sa), D.vp(act),
                   D.vp(active), D.vp(ra), None, D.stream_handle())
        torch.cuda.synchronize()
        outs.append([x.cpu().numpy() for x in (g, Qa, sa, act, active, ra)])
    for u, v in zip(*outs):
        assert np.array_equal(u, v)
    if r > 4 and rows > 0 and diag_add == 0.0:
        assert outs[0][4][3] == 0 and int(outs[0][5][0]) == r - 1


@pytest.mark.parametrize("rows,r", [(1000, 10), (5000, 50), (20000, 100), (40000, 200), (257, 130),
                                    (33, 7)])
def test_gram_against_oracle_and_exact(rows, r):
    """nmfb_gram (matrix.gram, matrix.py:181-197) directly against the oracle's
    BLAS Gram and an exact reference.  fp64 input: within 1e-14 of the BLAS
    Gram (only the summation order differs) and exactly symmetric.  fp32 input
    (the production factors): against the exact Gram of the same fp32 values
    (products of fp32 values are exact in fp64; math.fsum per entry on a row
    sample), within 1e-6 relative -- the kernel sums 32-row slabs in fp32
    before folding them into fp64."""
    import math

    import torch

    from oracle import nmf_oracle as orc
    from paper_1506_08938_b200 import _lib as L
    from paper_1506_08938_b200 import device as D

    dev = D.require_cuda()
    rng = np.random.default_rng(rows * 7 + r)
    A = rng.exponential(size=(rows, r)) * rng.uniform(0.01, 10.0, size=(1, r))
    ws = torch.zeros((L.lib().nmfb_gram_workspace_bytes(rows, r) // 8 + 1,),
                     dtype=torch.float64, device=dev)

    def gram(arr, code, tdt):
        g = torch.zeros((r, r), dtype=torch.float64, device=dev)
        a = torch.from_numpy(np.ascontiguousarray(arr)).to(dev, tdt)
        L.call("nmfb_gram", code, D.vp(a), rows, r, r, D.vp(g), D.vp(ws), D.stream_handle())
        torch.cuda.synchronize()
        return g.cpu().numpy()

    g64 = gram(A, L.F64, torch.float64)
    want = orc.gram(A)
    assert np.array_equal(g64, g64.T)
    np.testing.assert_allclose(g64, want, rtol=1e-14, atol=0)
    A32 = A.astype(np.float32).astype(np.float64)
    g32 = gram(A32, L.F32, torch.float32)
    assert np.array_equal(g32, g32.T)
    pairs = [(i, j) for i in range(r) for j in range(i, r)]
    if len(pairs) > 400:  # exact sums on a seeded sample of the entries
        pairs = [pairs[k] for k in rng.choice(len(pairs), size=400, replace=False)]
    rel = [abs(g32[i, j] - math.fsum(A32[:, i] * A32[:, j])) / abs(math.fsum(A32[:, i] * A32[:, j]))
           for i, j in pairs]
    assert max(rel) < 1e-6, max(rel)


@pytest.mark.parametrize("rows,r,pad", [(2048, 16, 0), (4097, 32, 0), (30001, 64, 4), (9999, 100, 0),
                                        (5000, 128, 0), (7777, 132, 0), (20000, 160, 8),
                                        (70000, 200, 0), (30001, 224, 0)])
def test_gram_tensor_core_path(rows, r, pad):
    """The tcgen05 Gram (csrc/gram_tc.cu: fp32 factors, r % 4 == 0, r <= 224,
    rows >= 2048; matrix.py:181-197) against the exact Gram of the same fp32
    values (fp64 matmul of exactly representable products).  3xTF32 products
    and 64-row chunks promoted into round-to-nearest running sums: within 1e-6
    relative on every entry (measured 4.6e-7, almost all of it a uniform
    -4.0e-7 bias of the truncating tensor-core accumulate, which the unit-
    diagonal rescale cancels), exactly symmetric, and the same through a padded
    leading dimension and with a ragged last unit.  NMFB_GRAM_TC=0 in the
    environment selects the CUDA-core kernel (this test then checks that)."""
    import torch

    from paper_1506_08938_b200 import _lib as L
    from paper_1506_08938_b200 import device as D

    dev = D.require_cuda()
    g = torch.Generator(device="cpu").manual_seed(rows * 31 + r)
    A = torch.rand((rows, r + pad), generator=g) ** 3 * (torch.rand((1, r + pad), generator=g) * 10
                                                         + 0.01)
    A[:, r // 2] *= (torch.rand(rows, generator=g) < 0.05)  # a sparse factor column
    A[:, 1] = 0.0                                           # a dead one
    a = A.to(dev, torch.float32)
    out = torch.zeros((r, r), dtype=torch.float64, device=dev)
    ws = torch.full((L.lib().nmfb_gram_workspace_bytes(rows, r) // 8 + 1,), float("nan"),
                    dtype=torch.float64, device=dev)
    L.call("nmfb_gram", L.F32, D.vp(a), rows, r, r + pad, D.vp(out), D.vp(ws), D.stream_handle())
    torch.cuda.synchronize()
    a64 = a[:, :r].double()
    want = a64.T @ a64
    assert torch.equal(out, out.T)
    assert torch.isfinite(out).all()
    assert torch.equal(out[1], torch.zeros_like(out[1]))
    rel = ((out - want).abs() / want.abs().clamp_min(1e-300))[want != 0]
    assert rel.max().item() < 1e-6, rel.max().item()
    # the rescaled Q (what the NNLS reads, nqp.py:116-131) is insensitive to the
    # uniform part of the error
    keep = [i for i in range(r) if i != 1]
    d = torch.sqrt(torch.diagonal(out)[keep]); dw = torch.sqrt(torch.diagonal(want)[keep])
    q = out[keep][:, keep] / (d[:, None] * d[None, :])
    qw = want[keep][:, keep] / (dw[:, None] * dw[None, :])
    assert (q - qw).abs().max().item() < 2e-7, (q - qw).abs().max().item()
