import time, sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import generators
from paper_1506_08938_b200 import NmfConfig
from paper_1506_08938_b200.nmf import FitSession, initial_factors
from paper_1506_08938_b200.matrix import DenseMatrix
t0=time.time(); x, cfg = generators.make(2); print("gen", time.time()-t0, flush=True)
V = DenseMatrix(x)
g = NmfConfig(rank=50, max_outer=5, seed=1, rel_change_tol=0.0, precision="fp32")
s = FitSession(V, g)
torch.cuda.synchronize()
for rep in range(2):
    s.state.qg_valid = False
    t0 = time.time(); model, log = s.run(); torch.cuda.synchronize(); dt = time.time()-t0
    print("5 iters", dt, "s  per iter ms", dt/5*1e3, "obj", log.objective, "kbar", log.k_bar, flush=True)
# per-phase timing
st = s.state
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
ev[0].record(); st.estep(0); ev[1].record(); st.mstep(0); ev[2].record(); st.objective(0); ev[3].record()
torch.cuda.synchronize()
print("estep ms", ev[0].elapsed_time(ev[1]), "mstep ms", ev[1].elapsed_time(ev[2]), "obj ms", ev[2].elapsed_time(ev[3]))
