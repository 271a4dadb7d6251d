import os, sys, numpy as np
sys.path.insert(0, ".")
from oracle import generators
from paper_1506_08938_b200 import NmfConfig, SparseMatrix
from paper_1506_08938_b200.nmf import FitSession
x = generators.sparse_zipf(20000, 8000, 2e-3, 4)
V = SparseMatrix(x.rows, x.cols, x.indptr, x.indices, x.values, validate=False)
cfg = NmfConfig(rank=64, max_outer=5, seed=3, rel_change_tol=0.0, precision="fp32")
res = []
for ov in ("0", "1", "1", "0"):
    os.environ["NMFB_GRAM_OVERLAP"] = ov
    m, l = FitSession(V, cfg).run()
    res.append((ov, m.G.array, m.F.array, l.objective))
for ov, G, F, o in res:
    print(ov, np.abs(G - res[0][1]).max(), np.abs(F - res[0][2]).max(), [f"{a:.10e}" for a in o])
