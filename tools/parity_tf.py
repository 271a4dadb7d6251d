"""Teacher-forced parity table: one fp32 GPU outer iteration
from the oracle state at iteration k, against
  (a) the fp64 oracle step from the same state, and
  (b) the fp64 oracle step from the state rounded to fp32 (X, G, F^T) --
      the storage-rounding floor every fp32 implementation starts from.
Usage: python tools/parity_tf.py [case ...]   (cases: c1 d8 d50 d100 zipf reg)
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import generators  # noqa: E402
from oracle import nmf_oracle as orc  # noqa: E402


def f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def cases():
    out = {}
    x, cfg = generators.make(1)
    out["c1"] = (x, dict(rank=10, seed=0), [0, 1, 2, 3, 5, 10, 20, 30, 45])
    for n, m, r in [(640, 960, 8), (600, 1000, 50), (500, 700, 100)]:
        rng = np.random.default_rng(n + m + r)
        x = rng.exponential(size=(n, r)) @ rng.exponential(size=(r, m))
        x += np.abs(rng.normal(0, 0.05, size=(n, m)))
        out[f"d{r}"] = (x, dict(rank=r, seed=1), [0, 1, 2, 3, 4, 6, 8, 12, 16])
    out["zipf"] = (generators.sparse_zipf(3000, 2000, 0.01, 7), dict(rank=20, seed=7),
                   [0, 1, 2, 3, 5])
    rng = np.random.default_rng(3)
    x = rng.exponential(size=(200, 8)) @ rng.exponential(size=(8, 300))
    x += np.abs(rng.normal(0, 0.05, size=x.shape))
    out["reg"] = (x, dict(rank=8, seed=3, mu1=0.1, beta2=0.01), [0, 1, 3, 10, 25])
    return out


def rounded(x):
    if isinstance(x, np.ndarray):
        return f32(x)
    return orc.Csc(x.rows, x.cols, x.indptr, x.indices, f32(x.values))


def gpu_step(V, gcfg, G, FT, mode):
    """One fp32 outer iteration on the GPU from (G, FT): the production path
    (mode None) or every kernel in reference order (NMFB_MODE_REFERENCE:
    thread per problem, sequential sums, fp32 arithmetic)."""
    from paper_1506_08938_b200 import _lib as L
    from paper_1506_08938_b200 import device as D
    from paper_1506_08938_b200.nmf import FitSession

    if mode is None:
        _, log = FitSession(V, gcfg, init=(G, FT)).run()
        return log.objective[0]
    d = D.DeviceData(V, "fp32")
    st = D.Alternation(d, gcfg, G, FT, 1, precision="fp32", kernel_mode=L.MODE_REFERENCE)
    st.iterate(0)
    st.join()
    import torch

    torch.cuda.synchronize()
    xsq = 0.0 if isinstance(V, np.ndarray) else float(np.asarray(V.values, np.float32).astype(np.float64) @ np.asarray(V.values, np.float32).astype(np.float64))
    return st.assemble(st.pieces[0].cpu().numpy(), gcfg, d.kind, xsq)


MODE = None


def run(name, x, kw, ks):
    from paper_1506_08938_b200 import NmfConfig, SparseMatrix

    ocfg = orc.Config(max_outer=1, rel_change_tol=0.0, **kw)
    gcfg = NmfConfig(max_outer=1, rel_change_tol=0.0, precision="fp32", **kw)
    V = x if isinstance(x, np.ndarray) else SparseMatrix(x.rows, x.cols, x.indptr, x.indices,
                                                         x.values, validate=False)
    xr = rounded(x)
    G, FT = orc.initial_factors(x, ocfg)
    rows = []
    for k in range(max(ks) + 1):
        nG, nFT, obj, *_ = orc.one_iteration(x, G, FT, ocfg)
        if k in ks:
            _, _, obj_r, *_ = orc.one_iteration(xr, f32(G), f32(FT), ocfg)
            g = gpu_step(V, gcfg, G, FT, MODE)
            rows.append((k, abs(g - obj) / obj, abs(obj_r - obj) / obj, abs(g - obj_r) / obj_r))
        G, FT = nG, nFT
    print(f"{name}: k | gpu vs fp64 oracle | fp32-rounded oracle vs fp64 oracle | gpu vs rounded")
    for k, a, b, c in rows:
        print(f"  {k:3d} | {a:.1e} | {b:.1e} | {c:.1e}")
    arr = np.array([r[1:] for r in rows])
    print(f"  max  | {arr[:, 0].max():.1e} | {arr[:, 1].max():.1e} | {arr[:, 2].max():.1e}", flush=True)
    return rows


if __name__ == "__main__":
    allc = cases()
    args = sys.argv[1:]
    if args and args[0] == "--ref32":
        from paper_1506_08938_b200 import _lib as _L

        MODE = _L.MODE_REFERENCE
        args = args[1:]
    for name in (args or list(allc)):
        run(name, *allc[name])
