"""Generate the golden vectors that pin the CPU oracle (and the GPU path) to the
reference implementation itself.

Run in the build container, where the reference is mounted read-only:

    python tests/golden/make_golden.py            # writes tests/golden/*.npz

The reference package (``/root/reference/pkg/src/nmfkit``) is imported from a
scratch COPY under /tmp with NUMBA_CACHE_DIR under /tmp, because importing it in
place makes numba write its cache next to kernels.py.  The
one-line shim ``nmfkit.nmf.on_iteration = None`` is applied because the
reference's ``fit`` reads that undefined global (nmf.py:197).

Nothing on the GPU box reads /root/reference: the outputs below are committed.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = os.environ.get("NMFKIT_REF_SRC", "/root/reference/pkg/src")
SCRATCH = "/tmp/nmfkit_ref_copy"


def import_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
    if os.path.exists(SCRATCH):
        shutil.rmtree(SCRATCH)
    shutil.copytree(REF_SRC, SCRATCH)
    sys.path.insert(0, SCRATCH)
    import nmfkit  # noqa: F401
    import nmfkit.nmf

    nmfkit.nmf.on_iteration = None  # shim for nmf.py:197
    return nmfkit


def random_h_problem(rng, r, frozen=0, ridge=0.0, scale=1.0):
    """A PSD H (r x r) with `frozen` zero-curvature dims, Gram-like."""
    a = rng.uniform(size=(3 * r + 2, r)) * scale
    H = a.T @ a + ridge * np.eye(r)
    if frozen:
        dims = rng.choice(r, size=frozen, replace=False)
        H[dims, :] = 0.0
        H[:, dims] = 0.0
    return H


def nnls_batch_case(nmfkit, rng, r, count, eps, max_inner, frozen=0, fail_at=None,
                    ridge=0.0, warm_zero_frac=0.3, beta1=0.0):
    """Run the reference's mstep_rows row by row (threading max_stop through,
    which is exactly what one call does internally) to record per-problem
    iteration counts and the fast-break running threshold."""
    from nmfkit import kernels, parallel

    H = random_h_problem(rng, r, frozen=frozen, ridge=ridge)
    scale_a, active, act_idx, Qa = parallel._rescale_for_step(H)
    # linear terms: mostly negative (interesting problems), some all >= 0
    x_star = rng.uniform(0.0, 2.0, size=(count, r)) * (rng.random((count, r)) < 0.7)
    h = -(x_star @ H) + rng.normal(0.0, 0.3, size=(count, r))
    nonneg_rows = rng.random(count) < 0.05
    h[nonneg_rows] = np.abs(h[nonneg_rows])
    if frozen:
        # frozen dims must have h >= 0 unless we plant a failure
        h[:, ~active] = np.abs(h[:, ~active])
    if fail_at is not None and frozen:
        h[fail_at, np.flatnonzero(~active)[0]] = -1.0
    warm = rng.uniform(0.0, 2.0, size=(count, r))
    warm[rng.random((count, r)) < warm_zero_frac] = 0.0
    YT = np.ascontiguousarray(beta1 - h)  # mstep_rows forms h = beta1 - YT
    G = np.ascontiguousarray(warm.copy())
    iters = np.zeros(count, dtype=np.int64)
    running = np.zeros(count)
    max_stop = 0.0
    fail = -1
    for row in range(count):
        inner, max_stop, f = kernels.mstep_rows(YT, row, row + 1, Qa, scale_a, act_idx, active,
                                                beta1, eps, max_inner, max_stop, G)
        if f != kernels.FAIL_NONE:
            fail = int(f)
            break
        iters[row] = inner
        running[row] = max_stop
    # one shard call over everything must agree with the row-by-row replay
    G2 = np.ascontiguousarray(warm.copy())
    tot, _, f2 = kernels.mstep_rows(YT, 0, count, Qa, scale_a, act_idx, active, beta1, eps,
                                    max_inner, 0.0, G2)
    assert f2 == fail, (f2, fail)
    if fail < 0:
        assert tot == iters.sum()
        assert np.array_equal(G, G2)
    return dict(H=H, h=h, warm=warm, beta1=np.float64(beta1), eps=np.float64(eps),
                max_inner=np.int64(max_inner), x=G, iters=iters, running_max_stop=running,
                fail=np.int64(fail), scale_a=scale_a, active=active, act_idx=act_idx, Qa=Qa)


NNLS_CASES = [
    # (name, r, count, eps, max_inner, frozen, fail_at, ridge)
    ("r1", 1, 40, 0.1, 500, 0, None, 0.0),
    ("r2", 2, 70, 0.1, 500, 0, None, 0.0),
    ("r3_eps0", 3, 70, 0.0, 60, 0, None, 0.0),
    ("r5", 5, 96, 0.1, 500, 0, None, 0.0),
    ("r10", 10, 100, 0.1, 500, 0, None, 0.0),
    ("r10_eps1e-3", 10, 64, 1e-3, 500, 0, None, 0.0),
    ("r10_frozen", 10, 64, 0.1, 500, 2, None, 0.0),
    ("r10_fail", 10, 64, 0.1, 500, 1, 37, 0.0),
    ("r16_ridge", 16, 96, 0.1, 500, 0, None, 0.5),
    ("r31", 31, 70, 0.1, 500, 0, None, 0.0),
    ("r50", 50, 96, 0.1, 500, 0, None, 0.0),
    ("r64_eps0", 64, 40, 0.0, 20, 0, None, 0.0),
    ("r64", 64, 96, 0.1, 500, 0, None, 0.0),
    ("r100", 100, 70, 0.1, 500, 0, None, 0.0),
    ("r200", 200, 40, 0.1, 500, 0, None, 0.0),
]


def make_nnls(nmfkit):
    out = {}
    for k, (name, r, count, eps, mi, frozen, fail_at, ridge) in enumerate(NNLS_CASES):
        rng = np.random.default_rng(1000 + k)
        case = nnls_batch_case(nmfkit, rng, r, count, eps, mi, frozen=frozen, fail_at=fail_at,
                               ridge=ridge)
        for key, val in case.items():
            out[f"{name}/{key}"] = val
    np.savez_compressed(os.path.join(HERE, "nnls_batches.npz"), **out)
    print("nnls_batches:", len(NNLS_CASES), "cases")


def make_steps(nmfkit):
    """run_estep / run_mstep (reference parallel.py) on small dense and sparse
    data, worker counts 1 and 3, with and without regularisation."""
    from nmfkit.matrix import DenseMatrix, SparseMatrix, gram
    from nmfkit.nmf import NmfConfig
    from nmfkit.parallel import run_estep, run_mstep

    out = {}
    rng = np.random.default_rng(77)
    n, m, r = 45, 150, 6
    arr = rng.uniform(size=(n, m))
    arr[arr < 0.45] = 0.0
    g = np.ascontiguousarray(rng.uniform(size=(n, r)))
    ft = np.ascontiguousarray(rng.uniform(size=(m, r)))
    out["data/arr"] = arr
    out["data/g"] = g
    out["data/ft"] = ft
    variants = {
        "plain_w1": dict(workers=1),
        "plain_w3": dict(workers=3),
        "reg_w1": dict(workers=1, mu1=0.05, mu2=0.02, beta1=0.03, beta2=0.01),
        "reg_w3": dict(workers=3, mu1=0.05, mu2=0.02, beta1=0.03, beta2=0.01),
    }
    for kind in ("dense", "sparse"):
        V = SparseMatrix.from_dense(arr) if kind == "sparse" else np.ascontiguousarray(arr.T)
        for vname, kw in variants.items():
            cfg = NmfConfig(rank=r, seed=0, **kw)
            G = g.copy()
            FT = ft.copy()
            Q_g = gram(DenseMatrix(G)).array
            Y, H_f, e = run_estep(V, G, Q_g, cfg, FT)
            mstats = run_mstep(Y, H_f, cfg, G)
            p = f"{kind}/{vname}"
            out[p + "/Q_g"] = Q_g
            out[p + "/FT"] = FT
            out[p + "/Y"] = np.ascontiguousarray(Y.array)
            out[p + "/H_f"] = np.ascontiguousarray(H_f.array)
            out[p + "/G"] = G
            out[p + "/e_inner"] = np.int64(e.inner_iterations)
            out[p + "/m_inner"] = np.int64(mstats.inner_iterations)
    np.savez_compressed(os.path.join(HERE, "steps.npz"), **out)
    print("steps: done")


def make_fits(nmfkit):
    from nmfkit.matrix import DenseMatrix, SparseMatrix
    from nmfkit.nmf import NmfConfig, fit

    sys.path.insert(0, REPO)
    from oracle import generators

    out = {}

    def record(name, V, cfg, store_factors=True):
        model, log = fit(V, cfg)
        out[f"{name}/objective"] = np.asarray(log.objective)
        out[f"{name}/inner"] = np.asarray(log.inner_iterations, dtype=np.int64)
        if store_factors:
            out[f"{name}/G"] = np.ascontiguousarray(model.G.array)
            out[f"{name}/F"] = np.ascontiguousarray(model.F.array)

    rng = np.random.default_rng(5)
    planted = rng.uniform(size=(30, 4)) @ rng.uniform(size=(4, 50))
    out["planted/X"] = planted
    record("planted", planted, NmfConfig(rank=4, max_outer=40, seed=1, rel_change_tol=0.0))
    record("planted_w4", planted,
           NmfConfig(rank=4, max_outer=40, seed=1, rel_change_tol=0.0, workers=4))
    reg = dict(mu1=0.01, mu2=0.02, beta1=0.01, beta2=0.01)
    record("planted_reg", planted,
           NmfConfig(rank=4, max_outer=40, seed=1, rel_change_tol=0.0, **reg))
    sp = rng.uniform(size=(40, 70))
    sp[sp < 0.6] = 0.0
    out["sparse/X"] = sp
    record("sparse", SparseMatrix.from_dense(sp),
           NmfConfig(rank=5, max_outer=30, seed=2, rel_change_tol=0.0))
    record("sparse_dense", DenseMatrix(sp),
           NmfConfig(rank=5, max_outer=30, seed=2, rel_change_tol=0.0))
    record("zero", np.zeros((4, 6)), NmfConfig(rank=2, max_outer=5, seed=0, rel_change_tol=0.0))
    # BASELINE config 1 (CPU-runnable oracle run), full size, 50 iterations
    x1 = generators.c1()
    out["c1/x_sha256"] = np.frombuffer(hashlib.sha256(np.ascontiguousarray(x1).tobytes())
                                       .digest(), dtype=np.uint8)
    record("c1", x1, NmfConfig(rank=10, max_outer=50, seed=0, rel_change_tol=0.0))
    # default rel_change_tol early exit (nmf.py:199-205)
    record("early_exit", planted, NmfConfig(rank=4, max_outer=300, seed=1))
    np.savez_compressed(os.path.join(HERE, "fits.npz"), **out)
    print("fits: done")


def make_kats(nmfkit):
    """Known-answer problems from the reference's own tests (test_nqp.py)."""
    from nmfkit.nqp import NqpProblem, StopState, rescale, solve

    out = {}
    H = np.array([[1.0, 0.1], [0.1, 10.0]])
    h = np.array([-80.0, -100.0])
    x0 = np.array([200.0, 20.0])
    sol = solve(NqpProblem(H, h, x0), StopState(epsilon=1e-12))
    out["toy/H"], out["toy/h"], out["toy/x0"] = H, h, x0
    out["toy/x"] = sol.x
    out["toy/iters"] = np.int64(sol.inner_iterations)
    out["toy/norm_hist"] = sol.passive_grad_norm_history
    out["toy/obj_hist"] = sol.objective_history
    rs = rescale(NqpProblem(H, h))
    out["toy/Q"], out["toy/q"], out["toy/scale"] = rs.Q, rs.q, rs.scale
    # enumeration-oracle style random problems (test_nqp.py:224-233 generator)
    for r in (2, 3, 4, 5, 6):
        rng = np.random.default_rng(100 + r)
        Hs, hs, x0s, xs, its = [], [], [], [], []
        for _ in range(20):
            a = rng.standard_normal((2 * r + 2, r))
            Hr = a.T @ a
            hr = rng.standard_normal(r) * rng.uniform(0.5, 3.0)
            x0r = rng.uniform(0.0, 2.0, size=r)
            s = solve(NqpProblem(Hr, hr, x0r), StopState(epsilon=1e-14), max_inner=2000)
            Hs.append(Hr), hs.append(hr), x0s.append(x0r), xs.append(s.x)
            its.append(s.inner_iterations)
        out[f"enum{r}/H"] = np.array(Hs)
        out[f"enum{r}/h"] = np.array(hs)
        out[f"enum{r}/x0"] = np.array(x0s)
        out[f"enum{r}/x"] = np.array(xs)
        out[f"enum{r}/iters"] = np.array(its, dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "kats.npz"), **out)
    print("kats: done")


if __name__ == "__main__":
    ref = import_reference()
    make_nnls(ref)
    make_steps(ref)
    make_fits(ref)
    make_kats(ref)
