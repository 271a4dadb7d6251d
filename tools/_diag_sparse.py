import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import generators, nmf_oracle as orc
from paper_1506_08938_b200 import SparseMatrix, NmfConfig
from paper_1506_08938_b200.matrix import frobenius_objective
from paper_1506_08938_b200 import device as D
X = generators.sparse_zipf(1500, 1000, 0.01, 8)
V = SparseMatrix(X.rows, X.cols, X.indptr, X.indices, X.values, validate=False)
cfg = orc.Config(rank=12, seed=8, rel_change_tol=0.0, max_outer=1)
G, FT = orc.initial_factors(X, cfg)
want = orc.regularized_objective(X, G, FT, cfg)
got = frobenius_objective(V, np.asfortranarray(G), np.asfortranarray(FT.T))
print("objective of init state: oracle", want, "gpu", got, "rel", abs(got-want)/want)
# dense check of the same state
Xd = X.to_dense()
wd = 0.5*np.sum((Xd - G @ FT.T)**2)
print("dense", wd, "rel vs oracle", abs(wd-want)/want)
# one iteration
G1, FT1, obj1, _, Y, Hf = orc.one_iteration(X, G, FT, cfg)
from paper_1506_08938_b200.nmf import FitSession
s = FitSession(V, NmfConfig(rank=12, seed=8, rel_change_tol=0.0, max_outer=1, precision="fp64"), init=(G, FT))
m, log = s.run()
print("iter obj oracle", obj1, "gpu", log.objective[0])
print("G diff", np.abs(m.G.array - G1).max(), "F diff", np.abs(m.F.array - FT1.T).max())
st = s.state
p = st.pieces[0].cpu().numpy()
print("pieces cross", p[1], "quad", p[7], "xsq", s.data.xsq)
g = np.asfortranarray(G1); f = np.asfortranarray(FT1.T)
col_of = np.repeat(np.arange(X.cols), np.diff(X.indptr))
cross = float(np.einsum("ij,ij->i", g[X.indices, :], f[:, col_of].T) @ X.values)
q = orc.gram(g); quad = float(np.sum((q @ f) * f))
print("oracle cross", cross, "quad", quad, "xsq", X.sum_squares())
yt = st.ybuf.view(st.n, st.r).cpu().numpy()
print("YT diff vs oracle Y.T", np.abs(yt - Y.T).max(), np.abs(Y).max())
hf = st.Hf.cpu().numpy()
print("Hf diff", np.abs(hf - Hf).max(), "diag min", np.diag(Hf).min(), "n frozen", (np.diag(Hf) <= 1e-12*np.diag(Hf).max()).sum())
sa, act, idx, Qa = orc.rescale_for_step(Hf)
print("active", act.sum(), "ra dev", int(st.ra[1].item()))
Gm = np.ascontiguousarray(G.copy())
it, ms, fail = orc.mstep_rows(np.ascontiguousarray(yt), 0, st.n, Qa, sa, idx, act, 0.0, 0.1, 500, 0.0, Gm)
print("oracle mstep from gpu inputs: diff to gpu G", np.abs(Gm - m.G.array).max(), "diff to oracle G1", np.abs(Gm - G1).max())
bad = np.argwhere(np.abs(m.G.array - G1) > 1e-6)
print("bad rows", np.unique(bad[:,0])[:20], len(np.unique(bad[:,0])))
