"""Micro-benchmark of the batched NNLS kernel on the real C2 E/M-step problems."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from oracle import generators
from paper_1506_08938_b200 import NmfConfig, _lib as L
from paper_1506_08938_b200 import device as D
from paper_1506_08938_b200.nmf import FitSession
from paper_1506_08938_b200.matrix import DenseMatrix
cfgid = sys.argv[1] if len(sys.argv) > 1 else "2"
if ":" in cfgid:  # custom sparse shape n:m:density:rank
    n_, m_, dens_, r_ = cfgid.split(":")
    x = generators.sparse_zipf(int(n_), int(m_), float(dens_), 5)
    from oracle.nmf_oracle import Config
    cfg = Config(rank=int(r_), seed=5, max_outer=8, rel_change_tol=0.0)
else:
    x, cfg = generators.make(int(cfgid))
from paper_1506_08938_b200.matrix import SparseMatrix
V = DenseMatrix(x) if isinstance(x, np.ndarray) else SparseMatrix(x.rows, x.cols, x.indptr, x.indices, x.values, validate=False)
kw = dict(cfg.__dict__); kw.pop('workers'); kw['max_outer'] = 8
s = FitSession(V, NmfConfig(precision="fp32", **kw))
st = s.state
for k in range(3):
    st.iterate(k)
torch.cuda.synchronize()
# E-step problem setup of iteration 3 (h from the data pass), then time only NNLS
st.gram(st.G, st.n, st.Qg); st.rescale(st.Qg, 0.0, 0)
d = st.d
FT0 = st.FT.clone()
if d.kind == "dense":
    L.call("nmfb_split_transpose", D.vp(st.G), st.n, st.r, D.vp(st.Gt[0]), D.vp(st.Gt[1]), D.stream_handle())
    L.call("nmfb_tc_gemm", D.vp(d.XT), st.m, st.n, D.vp(st.Gt[0]), D.vp(st.Gt[1]), st.r, D.vp(st.hbuf), st.tc_req, 0, D.stream_handle())
    args = (st.hbuf, L.F32, st.splits_e, st.r, st.m * st.r, 0.0)
else:
    L.call("nmfb_csc_linear", st.code, st.mode, D.vp(d.indptr), D.vp(d.rowidx), D.vp(d.vals), 0, st.m, D.vp(st.G), st.r, 0.0, D.vp(st.hbuf), D.stream_handle())
    args = (st.hbuf, st.code, 0, st.r, 0, 0.0)
stats = torch.zeros(2, dtype=torch.int64, device='cuda')
iters = torch.zeros(st.m, dtype=torch.int32, device='cuda')
LANES = [int(a) for a in sys.argv[2].split(',')] if len(sys.argv) > 2 else [1, 2, 4, 8]
for lanes in LANES:
    try:
        times = []
        for rep in range(5):
            st.FT.copy_(FT0); stats.zero_(); stats[1] = -1
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record()
            L.call("nmfb_nnls_batch", st.code, st.mode, D.vp(st.Qa[0]), D.vp(st.sa[0]), D.vp(st.act[0]), D.vp(st.active[0]), st.r, st.r, D.vp(st.ra[0]),
                   D.vp(args[0]), args[1], args[2], args[3], args[4], args[5], D.vp(st.FT), st.m, 0, 0.1, 500, 0.0, D.vp(iters), None, D.vp(stats), lanes, D.stream_handle())
            b.record(); torch.cuda.synchronize(); times.append(a.elapsed_time(b))
        it = iters.cpu().numpy()
        blk = it[: (len(it)//32)*32].reshape(-1, 32)
        print(f"lanes={lanes}: {min(times):.3f} ms  inner total {int(stats[0])}  mean {it.mean():.3f} max {it.max()}  mean-of-block-max {blk.max(1).mean():.2f}", flush=True)
    except Exception as e:
        print("lanes", lanes, "failed", e)
