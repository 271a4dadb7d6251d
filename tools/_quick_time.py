import time, sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import generators
from paper_1506_08938_b200 import NmfConfig, _lib
from paper_1506_08938_b200.nmf import FitSession
from paper_1506_08938_b200.matrix import DenseMatrix, SparseMatrix
cfgid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
t0=time.time(); x, cfg = generators.make(cfgid); print("gen", time.time()-t0, flush=True)
V = DenseMatrix(x) if isinstance(x, np.ndarray) else SparseMatrix(x.rows, x.cols, x.indptr, x.indices, x.values, validate=False)
kw = dict(cfg.__dict__); kw.pop('workers'); kw['max_outer'] = 6
g = NmfConfig(precision="fp32", **kw)
s = FitSession(V, g)
torch.cuda.synchronize()
t0 = time.time(); model, log = s.run(); torch.cuda.synchronize(); dt = time.time()-t0
print("6 iters", dt, "s  per iter ms", dt/6*1e3, "obj", log.objective, "kbar", log.k_bar, flush=True)
st = s.state
with _lib.Recorder(timing=True) as rec:
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(3):
        st.iterate(k)
    st.join(); b.record()
torch.cuda.synchronize()
print("steady per-iter ms", a.elapsed_time(b) / 3)
for name, (c, tms) in sorted(rec.summary().items(), key=lambda kv: -kv[1][1]):
    print(f"{name:28s} calls {c:3d} total {tms:9.3f} ms  per call {tms/c:8.3f} ms")
print("launches", rec.launches)
