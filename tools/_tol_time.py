"""Time fit() at C2 with the per-iteration stopping rule on vs off."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import generators  # noqa: E402
from paper_1506_08938_b200 import NmfConfig, fit  # noqa: E402

X, cfg0 = generators.make(2)
Xt = torch.from_numpy(np.ascontiguousarray(X.T, dtype=np.float32)).pin_memory().t()
for tol in (0.0, 1e-10, 0.0, 1e-10):
    cfg = NmfConfig(rank=50, max_outer=30, seed=1, rel_change_tol=tol, precision="fp32")
    torch.cuda.synchronize()
    t = time.perf_counter()
    model, log = fit(Xt, cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"tol={tol:g}: {len(log)} iterations, {dt * 1e3:.1f} ms, last-iteration "
          f"{(log.seconds[-1] - log.seconds[-11]) / 10 * 1e3:.3f} ms/iter "
          f"obj {log.final_objective:.6e}", flush=True)
