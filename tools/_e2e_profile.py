"""Phase timing of the public fit() from a pinned host tensor (C2 shape)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from oracle import generators
from paper_1506_08938_b200 import NmfConfig, fit
from paper_1506_08938_b200 import device as D
from paper_1506_08938_b200.nmf import FitSession
x, _ = generators.make(2)
XT = torch.from_numpy(np.ascontiguousarray(x.T, dtype=np.float32)).pin_memory()
V = XT.t()
cfg = NmfConfig(rank=50, max_outer=20, seed=0, rel_change_tol=0.0, precision="fp32")
fit(V, NmfConfig(rank=50, max_outer=2, seed=0, rel_change_tol=0.0, precision="fp32"))
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    data = D.DeviceData(V, "fp32"); torch.cuda.synchronize(); t1 = time.perf_counter()
    total = D.validate_and_sum(data); torch.cuda.synchronize(); t2 = time.perf_counter()
    s = FitSession(V, cfg); torch.cuda.synchronize(); t3 = time.perf_counter()
    model, log = s.run(); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.1f} ms  validate {1e3*(t2-t1):.1f}  session(all setup incl upload) {1e3*(t3-t2):.1f}  run {1e3*(t4-t3):.1f}")
    t0 = time.perf_counter(); model, log = fit(V, cfg); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"fit total {1e3*(t1-t0):.1f} ms")
