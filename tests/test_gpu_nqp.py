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
        assert np.array_equal(b.grad[k], s.grad), k
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


STEPS = np.load(os.path.join(os.path.dirname(__file__), "golden", "nqp_steps.npz"))


@pytest.mark.parametrize("c", range(int(STEPS["count"])))
def test_line_search_and_greedy_cd_against_reference(c):
    """nqp.exact_line_search_step / greedy_cd_pass (nqp.py:151-209) on the GPU
    against the reference's own outputs (tests/golden/make_golden_nqp_steps.py):
    the same projected step, breakpoint fallback, argmax choices and clamps;
    values to 1e-12 (numpy's BLAS products sum in a different order)."""
    from paper_1506_08938_b200.nqp import exact_line_search_step, greedy_cd_pass

    g = {k: STEPS[f"c{c}/{k}"] for k in ("Q", "q", "x", "grad", "x_ls", "g_ls", "x_cd", "g_cd")}
    sweeps = int(STEPS[f"c{c}/sweeps"])
    xl, gl = exact_line_search_step(g["Q"], g["q"], g["x"], g["grad"])
    np.testing.assert_allclose(xl, g["x_ls"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(gl, g["g_ls"], rtol=1e-12, atol=1e-12)
    assert np.array_equal(xl == 0.0, g["x_ls"] == 0.0)
    # the CD pass from the reference's own line-search output (no compounding)
    xc, gc = greedy_cd_pass(g["Q"], g["q"], g["x_ls"], g["g_ls"],
                            sweeps=None if sweeps < 0 else sweeps)
    np.testing.assert_allclose(xc, g["x_cd"], rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(gc, g["g_cd"], rtol=1e-11, atol=1e-11)


def test_step_helpers_batched():
    """Rows of a (count, r) batch sharing Q give the single-problem results."""
    from paper_1506_08938_b200.nqp import exact_line_search_step, greedy_cd_pass

    Q = STEPS["c10/Q"]
    r = Q.shape[0]
    rng = np.random.default_rng(5)
    x = rng.exponential(size=(9, r)) * (rng.random((9, r)) < 0.5)
    q = rng.normal(size=(9, r))
    grad = x @ Q.T + q
    xb, gb = exact_line_search_step(Q, q, x, grad)
    cb, hb = greedy_cd_pass(Q, q, xb, gb, sweeps=3)
    for k in range(9):
        x1, g1 = exact_line_search_step(Q, q[k], x[k], grad[k])
        assert np.array_equal(x1, xb[k]) and np.array_equal(g1, gb[k])
        c1, h1 = greedy_cd_pass(Q, q[k], x1, g1, sweeps=3)
        assert np.array_equal(c1, cb[k]) and np.array_equal(h1, hb[k])


@pytest.mark.parametrize("t", range(4))
def test_solve_check_gradients_every_iteration(t):
    """solve(check_gradients=True) checks the incremental gradient inside the
    kernel after every inner iteration (nqp.py:295-299); on well-posed
    problems it never fires and the solution is the reference's."""
    from paper_1506_08938_b200 import NqpProblem, StopState, solve

    p = NqpProblem(STEPS[f"s{t}/H"], STEPS[f"s{t}/h"])
    s = solve(p, StopState(epsilon=1e-6), check_gradients=True)
    np.testing.assert_allclose(s.x, STEPS[f"s{t}/x"], rtol=1e-9, atol=1e-12)
    assert s.inner_iterations == int(STEPS[f"s{t}/iters"])
    s2 = solve(NqpProblem(STEPS[f"s{t}/H"], STEPS[f"s{t}/h"]), StopState(epsilon=1e-6))
    assert np.array_equal(s.x, s2.x)
