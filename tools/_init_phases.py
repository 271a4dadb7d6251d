"""Wall-clock phases of FitSession.__init__ / run / factors download on a sparse config."""
import sys, time, functools
import numpy as np, torch
sys.path.insert(0, '.')
from oracle import generators
import paper_1506_08938_b200 as P
from paper_1506_08938_b200 import NmfConfig, SparseMatrix, fit, nmf, device as D, ingest, matrix
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
x, c = generators.make(cid)
V = SparseMatrix(x.rows, x.cols, x.indptr, x.indices, x.values, validate=False)
kw = dict(c.__dict__); kw.pop("workers")
import os
if os.environ.get("PLAIN"):
    matrix._PAR_MIN_SIZE = 1 << 62  # the plain numpy checks / np.sum
T = {}
def wrap(obj, name, label=None, sync=False):
    f = getattr(obj, name)
    @functools.wraps(f)
    def g(*a, **k):
        t = time.perf_counter()
        r = f(*a, **k)
        if sync: torch.cuda.synchronize()
        T.setdefault(label or name, []).append(time.perf_counter() - t)
        return r
    setattr(obj, name, g)
wrap(ingest.DeviceCsc, "from_host"); wrap(SparseMatrix, "sum_squares"); wrap(ingest.DeviceCsc, "csr")
wrap(D, "device_chunk_plan"); wrap(nmf, "require_nonnegative"); wrap(nmf, "_mean")
wrap(nmf, "device_initial_factors"); wrap(D, "Alternation"); wrap(D.DeviceData, "__init__", "DeviceData.__init__")
wrap(nmf.FitSession, "__init__", "FitSession.__init__"); wrap(nmf.FitSession, "run", "FitSession.run")
for it in [int(v) for v in os.environ.get("SEQ", "2,30,30,30").split(",")]:
    T.clear()
    cfg = NmfConfig(precision="fp32", **dict(kw, max_outer=it, rel_change_tol=0.0))
    torch.cuda.synchronize(); t = time.perf_counter()
    fit(V, cfg); torch.cuda.synchronize()
    print(f"fit({it} it) {time.perf_counter() - t:.4f} s")
    for k, v in T.items(): print(f"   {k:28s} {sum(v):.4f}")
