"""torchrun helper for tests/test_gpu_peer.py: one rank runs the column-
sharded fit (peer-memory or NCCL path, per NMFB_DIST_PEER) and the
single-GPU fit from the same start, and writes whether they agree bit for bit.

    python -m torch.distributed.run --nproc-per-node=1 tests/_dist_fit_check.py out.json
"""

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1506_08938_b200 import NmfConfig  # noqa: E402
from paper_1506_08938_b200 import dist as PD  # noqa: E402
from paper_1506_08938_b200.nmf import FitSession, initial_factors_from_mean  # noqa: E402


def main(out_path):
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rng = np.random.default_rng(3)
    K = 6
    if os.environ.get("NMFB_CHECK_SPARSE") == "1" or os.environ.get("NMFB_CHECK_ROWS") == "1":
        # sparse column block through DistFit(m_total=...) (the config 3/5
        # strong-scaling path of bench.py)
        from oracle import generators
        from paper_1506_08938_b200.matrix import SparseMatrix

        x = generators.sparse_zipf(6000, 3000, 4e-3, 5)
        n, m, r = x.rows, x.cols, 40
        X = SparseMatrix(x.rows, x.cols, x.indptr, x.indices, x.values, validate=False)
        mean = float(x.values.sum()) / (n * m)
        block = PD.csc_column_block(x, *PD.ShardPlan(n, m, 1).col_range(0))
    else:
        n, m, r = 1000, 2048, 50
        X = (rng.exponential(size=(n, r)) @ rng.exponential(size=(r, m))
             + np.abs(rng.normal(0, 0.05, size=(n, m)))).astype(np.float32)
        mean = float(X.astype(np.float64).mean())
        block = X
    cfg = NmfConfig(rank=r, max_outer=K, seed=0, rel_change_tol=0.0, precision="fp32")
    G0, FT0 = initial_factors_from_mean(n, m, mean, cfg)

    single = FitSession(X, cfg, init=(G0, FT0)).state
    for k in range(K):
        single.iterate(k)
    single.join()

    if os.environ.get("NMFB_CHECK_ROWS") == "1":
        # the row-sharded layout for tall sparse data (dist_rows.py)
        from paper_1506_08938_b200.dist_rows import RowShardedFit

        sess = RowShardedFit(X, cfg, init=(G0, FT0))
    else:
        sess = PD.DistFit(block, cfg, init=(G0, FT0), m_total=m)
    st = sess.state
    for k in range(K):
        st.iterate(k)
    st.join()
    torch.cuda.synchronize()
    if getattr(sess, "peer", False):
        sess.engine.px.check()
    res = {
        "peer": bool(getattr(sess, "peer", False)),
        "peer_error": getattr(sess, "peer_error", None),
        "G_equal": bool(torch.equal(st.st.G, single.G)),
        "FT_equal": bool(torch.equal(st.st.FT, single.FT)),
        "obj_equal": bool(torch.equal(st.pieces[:K], single.pieces[:K])),
        "G_maxdiff": float((st.st.G - single.G).abs().max()),
        "obj": st.pieces[:K, 0].tolist(),
        "obj_single": single.pieces[:K, 0].tolist(),
    }
    with open(out_path, "w") as f:
        json.dump(res, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
