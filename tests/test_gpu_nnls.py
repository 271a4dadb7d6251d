"""GPU parity of the batched NNLS kernel and the rescale epilogue.

Golden vectors: the reference's own numba kernels (tests/golden/make_golden.py).
fp64 reference-order mode must match BIT FOR BIT (solutions, per-problem
iteration counts, the fast-break running threshold, the failing index).
The fp32 production kernel is checked against the same vectors with the
north-star fp32 tolerance on factors (1e-3, floored relative metric of
SURVEY.md 7.3) on the problems whose fp32 stop decisions coincide, plus
objective-value agreement for all problems.
"""

import os

import numpy as np
import pytest

from oracle import nmf_oracle as orc

GOLD = os.path.join(os.path.dirname(__file__), "golden")
NNLS = np.load(os.path.join(GOLD, "nnls_batches.npz"))
CASES = sorted({k.split("/")[0] for k in NNLS.files})

pytestmark = pytest.mark.gpu


def g(case, k):
    return NNLS[f"{case}/{k}"]


@pytest.mark.parametrize("case", CASES)
def test_rescale_bit_exact(case):
    from gpu_util import rescale

    _, host = rescale(g(case, "H"))
    assert np.array_equal(host["active"], g(case, "active"))
    assert np.array_equal(host["act_idx"], g(case, "act_idx"))
    assert np.array_equal(host["scale_a"], g(case, "scale_a"))
    assert np.array_equal(host["Qa"], g(case, "Qa"))


@pytest.mark.parametrize("case", CASES)
def test_nnls_fp64_bit_exact_vs_reference(case):
    from gpu_util import nnls, running_max

    h, warm = g(case, "h"), g(case, "warm")
    count = h.shape[0]
    x, iters, finals, stats = nnls(g(case, "H"), h, warm, float(g(case, "eps")),
                                   int(g(case, "max_inner")), h_base=float(g(case, "beta1")))
    fail = int(g(case, "fail"))
    got_fail = -1 if stats[1] == -1 else int(stats[1])
    assert got_fail == fail
    stop = count if fail < 0 else fail
    assert np.array_equal(iters[:stop], g(case, "iters")[:stop])
    assert np.array_equal(x[:stop], g(case, "x")[:stop])
    assert np.array_equal(running_max(finals, count)[:stop], g(case, "running_max_stop")[:stop])
    if fail < 0:
        assert int(stats[0]) == int(g(case, "iters").sum())


@pytest.mark.parametrize("index_base,max_stop0", [(5, 0.0), (5, 0.37), (40, 2.5), (64, 1e9)])
@pytest.mark.parametrize("r", [3, 10, 33])
def test_nnls_fp64_unaligned_shards_vs_oracle(index_base, max_stop0, r):
    """Shards that start mid-block begin from max_stop0 (kernels.py:245-248)."""
    from gpu_util import nnls

    rng = np.random.default_rng(7 * r + index_base)
    a = rng.uniform(size=(3 * r, r))
    H = a.T @ a
    count = 75
    xs = rng.uniform(0, 2, size=(count, r)) * (rng.random((count, r)) < 0.7)
    h = -(xs @ H) + rng.normal(0, 0.2, size=(count, r))
    warm = rng.uniform(0, 2, size=(count, r))
    x, iters, finals, stats = nnls(H, h, warm, 0.1, 500, h_base=0.0, index_base=index_base,
                                   max_stop0=max_stop0)
    # oracle: the reference mstep_rows over rows [index_base, index_base + count)
    sa, act, idx, Qa = orc.rescale_for_step(H)
    YT = np.zeros((index_base + count, r))
    YT[index_base:] = -h
    G = np.zeros((index_base + count, r))
    G[index_base:] = warm
    tot, ms, fail = orc.mstep_rows(YT, index_base, index_base + count, Qa, sa, idx, act, 0.0, 0.1,
                                   500, max_stop0, G)
    assert fail == -1 and stats[1] == -1
    assert np.array_equal(x, G[index_base:])
    assert int(stats[0]) == tot


@pytest.mark.parametrize("case", [c for c in CASES if c != "r10_fail"])
def test_nnls_fp32_fast_vs_reference(case):
    from gpu_util import floored_rel, nnls

    H, h, warm = g(case, "H"), g(case, "h"), g(case, "warm")
    want = g(case, "x")
    x, iters, _, stats = nnls(H, h, warm, float(g(case, "eps")), int(g(case, "max_inner")),
                              precision="fp32", h_base=0.0)
    assert stats[1] == -1
    assert np.all(x >= 0)
    same = iters == g(case, "iters")
    # objective 0.5 x'Hx + h'x: fp32 solution as good as the reference's to 1e-4
    fx = 0.5 * np.einsum("ij,jk,ik->i", x, H, x) + np.einsum("ij,ij->i", h, x)
    fr = 0.5 * np.einsum("ij,jk,ik->i", want, H, want) + np.einsum("ij,ij->i", h, want)
    scale = np.maximum(np.abs(fr), 1e-6 * np.max(np.abs(fr)))
    rel = np.abs(fx - fr) / scale
    eps = float(g(case, "eps"))
    if eps > 0:
        assert same.mean() >= 0.9, f"iteration counts agree on {same.mean():.2%}"
        assert np.median(rel) < 1e-4
        # per-problem factor error: greedy-CD near-ties at large r can reorder
        # coordinate updates, so bound the 90th percentile, not the max
        per = np.array([floored_rel(x[i], want[i]) for i in range(len(x))])
        # the r=200 golden Hessian (Gram of a 402x200 uniform matrix) is badly
        # conditioned: fp32 solutions spread more there
        ill = H.shape[0] >= 128  # cond(Q) ~1e6+: fp32 pins the objective, not x
        assert np.median(per[same]) < (5e-3 if ill else 1e-3), np.median(per[same])
        if not ill:
            assert np.quantile(per[same], 0.9) < 5e-3, np.quantile(per[same], 0.9)
    else:
        # solve-to-stagnation: fp32 converges to the same optimum
        assert np.max(rel) < 1e-3


@pytest.mark.parametrize("lanes", [1, 2, 4, 8])
def test_nnls_fp32_lane_variants_agree(lanes):
    """Every lanes-per-problem variant computes the same solutions."""
    from gpu_util import nnls

    case = "r10"
    H, h, warm = g(case, "H"), g(case, "h"), g(case, "warm")
    x0, it0, _, _ = nnls(H, h, warm, 0.1, 500, precision="fp32", h_base=0.0, lanes=1)
    x, it, _, _ = nnls(H, h, warm, 0.1, 500, precision="fp32", h_base=0.0, lanes=lanes)
    assert (it == it0).mean() >= 0.95
    agree = it == it0
    np.testing.assert_allclose(x[agree], x0[agree], rtol=1e-3, atol=1e-4 * np.max(x0))
