"""Golden vectors for the public NQP building blocks, produced by the reference
itself: ``nqp.exact_line_search_step`` (nqp.py:151-183) and
``nqp.greedy_cd_pass`` (nqp.py:186-209) on rescaled (unit-diagonal) random
problems, plus ``nqp.solve(..., check_gradients=True)`` outcomes.

    python tests/golden/make_golden_nqp_steps.py   # writes tests/golden/nqp_steps.npz

Imports the reference from a /tmp copy (make_golden.import_reference)."""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import import_reference, random_h_problem  # noqa: E402


def main():
    nmfkit = import_reference()
    from nmfkit import nqp

    rng = np.random.default_rng(2024)
    out = {}
    cases = [(1, 3), (4, 5), (10, 6), (37, 4), (64, 3), (130, 2)]
    c = 0
    for r, reps in cases:
        for t in range(reps):
            H = random_h_problem(rng, r, ridge=1e-3)
            _, _, Q = nqp.rescale_arrays(H)
            q = rng.normal(size=r) * rng.uniform(0.1, 10.0)
            x = np.where(rng.uniform(size=r) < 0.4, 0.0, rng.exponential(size=r))
            if t == 1:
                x[:] = 0.0  # cold start
            grad = Q @ x + q
            xl, gl = nqp.exact_line_search_step(Q, q, x, grad)
            sweeps = None if t % 2 == 0 else max(1, r // 3)
            xc, gc = nqp.greedy_cd_pass(Q, q, xl, gl, sweeps=sweeps)
            pre = f"c{c}/"
            out[pre + "Q"] = Q
            out[pre + "q"] = q
            out[pre + "x"] = x
            out[pre + "grad"] = grad
            out[pre + "x_ls"] = xl
            out[pre + "g_ls"] = gl
            out[pre + "sweeps"] = np.int64(-1 if sweeps is None else sweeps)
            out[pre + "x_cd"] = xc
            out[pre + "g_cd"] = gc
            c += 1
    out["count"] = np.int64(c)
    # solve(check_gradients=True) on well-posed problems: the same solutions as
    # without the check (the check never fires)
    for t in range(4):
        r = [3, 8, 20, 50][t]
        H = random_h_problem(rng, r, ridge=1e-2)
        h = -rng.exponential(size=r)
        p = nqp.NqpProblem(H, h)
        s = nqp.solve(p, nqp.StopState(epsilon=1e-6), check_gradients=True)
        out[f"s{t}/H"] = H
        out[f"s{t}/h"] = h
        out[f"s{t}/x"] = s.x
        out[f"s{t}/iters"] = np.int64(s.inner_iterations)
    np.savez_compressed(os.path.join(HERE, "nqp_steps.npz"), **out)
    print("wrote nqp_steps.npz:", c, "step cases")


if __name__ == "__main__":
    main()
