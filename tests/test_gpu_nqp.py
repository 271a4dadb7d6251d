"""Public NQP API on the GPU: nqp.solve against
the reference's known answers (tests/golden/kats.npz, from test_nqp.py's
problems run through the reference), and the batched solve_batch against
solve problem by problem."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KATS = np.load(os.path.join(os.path.dirname(__file__), "golden", "kats.npz"))


def test_solve_toy_kat():
    """test_nqp.py:17-21 / cli.py:34-35 toy problem: x* ~ [79.0791, 9.2092]."""
    from paper_1506_08938_b200 import NqpProblem, StopState, solve

    sol = solve(NqpProblem(KATS["toy/H"], KATS["toy/h"], KATS["toy/x0"]),
                StopState(epsilon=1e-12))
    np.testing.assert_allclose(sol.x, KATS["toy/x"], rtol=1e-12)
    assert sol.inner_iterations == int(KATS["toy/iters"])
    # the last norm (1e-12, sixteen orders below the first) carries cancellation
    np.testing.assert_allclose(sol.passive_grad_norm_history, KATS["toy/norm_hist"], rtol=1e-7)
    np.testing.assert_allclose(sol.objective_history, KATS["toy/obj_hist"], rtol=1e-12)


@pytest.mark.parametrize("r", [2, 3, 4, 5, 6])
def test_solve_enumeration_kats(r):
    from paper_1506_08938_b200 import NqpProblem, StopState, solve

    for k in range(KATS[f"enum{r}/H"].shape[0]):
        p = NqpProblem(KATS[f"enum{r}/H"][k], KATS[f"enum{r}/h"][k], KATS[f"enum{r}/x0"][k])
        s = solve(p, StopState(epsilon=1e-14), max_inner=2000)
        np.testing.assert_allclose(s.x, KATS[f"enum{r}/x"][k], rtol=1e-9, atol=1e-12)
        assert s.inner_iterations == int(KATS[f"enum{r}/iters"][k])


def _shared_h_batch(r, count, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((2 * r + 2, r))
    H = a.T @ a
    h = rng.standard_normal((count, r)) * rng.uniform(0.5, 3.0, size=(count, 1))
    x0 = rng.uniform(0.0, 2.0, size=(count, r)) * (rng.random((count, r)) < 0.6)
    h[::7] = np.abs(h[::7])          # short-circuit x = 0 (nqp.py:233-240)
    return H, h, x0


@pytest.mark.parametrize("r,count,eps", [(4, 50, 1e-14), (20, 300, 0.1), (64, 129, 1e-3)])
@pytest.mark.parametrize("histories", [True, False])
def test_solve_batch_equals_solve(r, count, eps, histories):
    from paper_1506_08938_b200 import NqpProblem, StopState, solve, solve_batch

    H, h, x0 = _shared_h_batch(r, count, 1000 + r)
    # a KKT warm start: x0 already optimal for problem 3
    s3 = solve(NqpProblem(H, h[3], x0[3]), StopState(epsilon=1e-14), max_inner=5000)
    x0[3] = s3.x
    h[3] = -(H @ s3.x) + np.where(s3.x > 0, 0.0, np.abs(h[3]))  # zero passive gradient
    b = solve_batch(H, h, x0, epsilon=eps, max_inner=500, histories=histories)
    assert len(b) == count
    for k in range(count):
        s = solve(NqpProblem(H, h[k], x0[k]), StopState(epsilon=eps), max_inner=500)
        assert np.array_equal(b.x[k], s.x), k
        assert int(b.inner_iterations[k]) == s.inner_iterations, k
        assert float(b.final_passive_grad_norm_sq[k]) == s.final_passive_grad_norm_sq, k
        assert float(b.initial_passive_grad_norm_sq[k]) == s.initial_passive_grad_norm_sq, k
        if histories:
            one = b.solution(k)
            assert np.array_equal(one.passive_grad_norm_history, s.passive_grad_norm_history)
            assert np.array_equal(one.objective_history, s.objective_history)


def test_solve_batch_errors():
    from paper_1506_08938_b200 import solve_batch
    from paper_1506_08938_b200.exceptions import DegenerateProblemError, NumericalFailureError

    H = np.zeros((3, 3))
    with pytest.raises(DegenerateProblemError):
        solve_batch(H, -np.ones((2, 3)))
    # all-nonnegative h never needs the iterative solve, even with a degenerate H
    b = solve_batch(H, np.ones((2, 3)))
    assert np.array_equal(b.x, np.zeros((2, 3)))
    H = np.diag([1.0, 0.0, 2.0])
    h = np.array([[1.0, 1.0, -1.0], [-1.0, -2.0, 1.0], [-1.0, -1.0, -1.0]])
    with pytest.raises(NumericalFailureError) as ei:
        solve_batch(H, h)
    assert ei.value.index == 1
    with pytest.raises(ValueError):
        solve_batch(H, h, x0=-np.ones((3, 3)))
