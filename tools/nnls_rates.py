"""NNLS-only solve rates per rank ("Report NNLS-only solves/s via
kernels.mstep_rows at each r"): planted component-step problems (the survey's
recipe: F ~ U^{r x 2000}, G* ~ U, Y^T = (G* F) F^T, warm start G* . U[0.5, 1.5],
epsilon = 0.1), solved by
  * the GPU fast kernel (nmfb_nnls_batch, fp32), `count_gpu` problems, best of 5;
  * the CPU reference path: the oracle's bit-exact C restatement of
    kernels.mstep_rows on `count_cpu` problems, one 32-aligned shard per host
    core (the reference's thread-pool sharding).
Writes one JSON object per rank.  python tools/nnls_rates.py [out.json]
"""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import nmf_oracle as orc  # noqa: E402


def problems(r, count, seed):
    rng = np.random.default_rng(seed)
    F = rng.uniform(size=(r, 2000))
    Gs = rng.uniform(size=(count, r))
    YT = (Gs @ F) @ F.T
    H = F @ F.T
    warm = Gs * rng.uniform(0.5, 1.5, size=Gs.shape)
    return H, YT, warm


def gpu_rate(r, count):
    import torch
    from gpu_util import rescale

    from paper_1506_08938_b200 import _lib as L
    from paper_1506_08938_b200 import device as D

    H, YT, warm = problems(r, count, 100 + r)
    b, _ = rescale(H, 0.0, "fp32")
    dev = D.require_cuda()
    hp = torch.from_numpy(YT.astype(np.float32)).to(dev)
    x0 = torch.from_numpy(warm.astype(np.float32)).to(dev)
    x = x0.clone()
    stats = torch.zeros(2, dtype=torch.int64, device=dev)
    best = 1e30
    for _ in range(6):
        x.copy_(x0)
        stats.zero_()
        stats[1] = -1
        a = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        a.record()
        L.call("nmfb_nnls_batch", L.F32, L.MODE_FAST, D.vp(b["Qa"]), D.vp(b["sa"]),
               D.vp(b["act"]), D.vp(b["active"]), r, r, D.vp(b["ra"]), D.vp(hp), L.F32, 1, r,
               0, 0.0, D.vp(x), count, 0, 0.1, 500, 0.0, None, None, D.vp(stats), 0,
               D.stream_handle())
        e.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(e))
    kbar = int(stats[0].item()) / count
    return count / (best / 1e3), kbar, best


def cpu_rate(r, count):
    H, YT, warm = problems(r, count, 100 + r)
    sa, act, idx, Qa = orc.rescale_for_step(H)
    cores = os.cpu_count() or 1
    shards = orc.block_plan(count, cores)
    G = np.ascontiguousarray(warm)
    YT = np.ascontiguousarray(YT)
    orc.mstep_rows(YT, 0, min(32, count), Qa, sa, idx, act, 0.0, 0.1, 500, 0.0, G.copy())

    def work(s):
        return orc.mstep_rows(YT, s[0], s[1], Qa, sa, idx, act, 0.0, 0.1, 500, 0.0, G)[0]

    t = time.perf_counter()
    with ThreadPoolExecutor(len(shards)) as pool:
        inner = sum(pool.map(work, shards))
    dt = time.perf_counter() - t
    return count / dt, inner / count, cores


def main(out=None):
    res = []
    for r, ng, nc in ((10, 200000, 65536), (50, 200000, 32768), (64, 200000, 32768),
                      (100, 100000, 16384), (200, 100000, 8192)):
        g, kg, ms = gpu_rate(r, ng)
        c, kc, cores = cpu_rate(r, nc)
        row = {"r": r, "gpu_solves_per_s": g, "gpu_k_bar": kg, "gpu_problems": ng,
               "gpu_ms": ms, "cpu_solves_per_s": c, "cpu_k_bar": kc, "cpu_problems": nc,
               "cpu_threads": cores, "ratio": g / c}
        print(json.dumps(row), flush=True)
        res.append(row)
    if out:
        with open(out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
