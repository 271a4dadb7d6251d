"""Repeat the public fit() on a sparse config; per repetition: wall time and
the host functions with the largest own time (cProfile)."""
import cProfile, io, pstats, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from oracle import generators
from paper_1506_08938_b200 import NmfConfig, SparseMatrix, fit
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
x, c = generators.make(cid)
V = SparseMatrix(x.rows, x.cols, x.indptr, x.indices, x.values, validate=False)
kw = dict(c.__dict__); kw.pop("workers")
cfg = NmfConfig(precision="fp32", **kw)
fit(V, NmfConfig(precision="fp32", **dict(kw, max_outer=2)))
for i in range(6):
    pr = cProfile.Profile()
    torch.cuda.synchronize(); t = time.perf_counter()
    pr.enable(); m, log = fit(V, cfg); torch.cuda.synchronize(); pr.disable()
    dt = time.perf_counter() - t
    del m
    s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(4)
    top = [l for l in s.getvalue().split("\n") if l.strip() and l.strip()[0].isdigit()][:4]
    print(f"fit {i}: {dt:.3f} s", flush=True)
    for l in top: print("    ", l.strip()[:150])
