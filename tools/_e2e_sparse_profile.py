"""Host-side phase profile of the public fit() on a sparse config (cProfile)."""
import cProfile, pstats, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from oracle import generators
from paper_1506_08938_b200 import NmfConfig, SparseMatrix, fit
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
x, c = generators.make(cid)
V = SparseMatrix(x.rows, x.cols, x.indptr, x.indices, x.values, validate=False)
kw = dict(c.__dict__); kw.pop("workers"); kw["max_outer"] = 3
cfg = NmfConfig(precision="fp32", **kw)
fit(V, NmfConfig(precision="fp32", **dict(kw, max_outer=1)))
torch.cuda.synchronize()
pr = cProfile.Profile()
t = time.perf_counter()
pr.enable()
model, log = fit(V, cfg)
torch.cuda.synchronize()
pr.disable()
print("fit (3 iterations) s", time.perf_counter() - t)
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
