"""Full-size parity table (SURVEY 7.3 P2/P3 at the BASELINE configs' sizes).

For each config: the fp32 GPU fit and the fp64 oracle (the bit-exact port of
the reference) run K free outer iterations from the same seeded init; the
oracle is also run on the fp32-rounded input (X rounded once, fp64
arithmetic) -- the storage-rounding floor any fp32 implementation starts
from.  Reported per iteration: relative objective error GPU vs oracle and
floor vs oracle; after the last iteration the floored factor error
(max|a-b| / max(|b|, 1e-3 max|b|), per row), the fraction of factor rows
within 1e-3, and the exact-zero pattern agreement of H.

    python tools/parity_full.py [cid ...] [--json out.json]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import generators  # noqa: E402
from oracle import nmf_oracle as orc  # noqa: E402

ITERS = {1: 10, 2: 3, 3: 3, 4: 3, 5: 2}


def rowwise_floored(a, b):
    scale = np.maximum(np.abs(b).max(axis=1), 1e-300)
    den = np.maximum(np.abs(b), 1e-3 * scale[:, None])
    return (np.abs(a - b) / den).max(axis=1)


def run(cid):
    import torch

    from paper_1506_08938_b200 import NmfConfig, fit
    from paper_1506_08938_b200.matrix import SparseMatrix

    x, ocfg = generators.make(cid)
    sparse = not isinstance(x, np.ndarray)
    K = ITERS[cid]
    kw = dict(ocfg.__dict__)
    kw.pop("workers")
    kw["max_outer"] = K
    cores = os.cpu_count() or 1
    t = time.time()
    V = SparseMatrix(x.rows, x.cols, x.indptr, x.indices, x.values, validate=False) \
        if sparse else x
    prec = "fp64" if cid == 1 else "fp32"
    model, log = fit(V, NmfConfig(precision="fp32", **kw))
    torch.cuda.synchronize()
    t_gpu = time.time() - t
    oc = orc.Config(workers=cores, **kw)
    t = time.time()
    oG, oFT, olog = orc.fit(x, oc, chunked_objective=sparse)
    t_orc = time.time() - t
    if sparse:
        xr = orc.Csc(x.rows, x.cols, x.indptr, x.indices,
                     x.values.astype(np.float32).astype(np.float64))
    else:
        xr = x.astype(np.float32).astype(np.float64)
    rG, rFT, rlog = orc.fit(xr, oc, chunked_objective=sparse)
    g = np.asarray(log.objective)
    o = np.asarray(olog.objective)
    fl = np.asarray(rlog.objective)
    G = model.G.array
    F = model.F.array
    eG = rowwise_floored(G, oG)
    eF = rowwise_floored(F.T, oFT)
    zero = float(((F == 0) == (oFT.T == 0)).mean())
    fG, fF = rowwise_floored(rG, oG), rowwise_floored(rFT, oFT)
    nrm = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
    res = {
        "config": cid, "iterations": K, "precision_gpu": prec if cid == 1 else "fp32",
        "objective_gpu": g.tolist(), "objective_oracle": o.tolist(),
        "rel_err_gpu": (np.abs(g - o) / o).tolist(),
        "rel_err_fp32_input_floor": (np.abs(fl - o) / o).tolist(),
        "factor_rows_within_1e-3": {"G": float((eG < 1e-3).mean()), "F": float((eF < 1e-3).mean())},
        "factor_err_median": {"G": float(np.median(eG)), "F": float(np.median(eF))},
        "factor_err_p90": {"G": float(np.percentile(eG, 90)), "F": float(np.percentile(eF, 90))},
        "H_zero_pattern_agreement": zero,
        "factor_normwise": {"G": nrm(G, oG), "F": nrm(F.T, oFT)},
        "floor_factor_normwise": {"G": nrm(rG, oG), "F": nrm(rFT, oFT)},
        "floor_factor_err_median": {"G": float(np.median(fG)), "F": float(np.median(fF))},
        "floor_H_zero_pattern_agreement": float(((rFT == 0) == (oFT == 0)).mean()),
        "inner_iterations_gpu_vs_oracle": [list(map(int, log.inner_iterations)),
                                           list(map(int, olog.inner_iterations))],
        "seconds": {"gpu_fit": t_gpu, "oracle_fit": t_orc, "oracle_threads": cores},
    }
    print(json.dumps(res), flush=True)
    return res


if __name__ == "__main__":
    args = sys.argv[1:]
    out = None
    if "--json" in args:
        i = args.index("--json")
        out = args[i + 1]
        args = args[:i] + args[i + 2:]
    cids = [int(a) for a in args] or [2, 3, 4, 5]
    allres = [run(c) for c in cids]
    if out:
        with open(out, "w") as f:
            json.dump(allres, f, indent=1)
