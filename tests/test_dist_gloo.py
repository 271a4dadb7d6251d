"""Multi-rank (world_size 2, gloo, CPU) test of the column-sharded driver.

The product's DistAlternation (paper_1506_08938_b200/dist.py) -- shard plan,
allreduce of H_f and of the row-block Grams, reduce-scatter of Y^T, allgather
of G, objective pieces -- runs unchanged; only the per-rank math is supplied
by an oracle engine (numpy + the C restatement of the reference kernels), so
the sharding/collective logic is checked on CPU against the single-process
reference run with the same 32-aligned shards (workers=2).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import nmf_oracle as orc


class OracleEngine:
    """Per-rank math in float64 through the oracle (test infrastructure)."""

    def __init__(self, X, cfg, G0, FT0):
        self.X = np.asfortranarray(X)
        self.VT = np.ascontiguousarray(X.T)
        self.cfg = cfg
        self.G = np.ascontiguousarray(G0).copy()
        self.FT = np.ascontiguousarray(FT0).copy()
        self.r = cfg.rank
        self.pieces = {}

    def gram_rows(self, lo, hi):
        return torch.from_numpy(orc.gram(self.G[lo:hi]) if hi > lo else np.zeros((self.r,) * 2))

    def set_gram(self, Q):
        self.Qg = Q.numpy().copy()

    def estep(self, k, col_offset):
        n, r = self.G.shape
        lo, hi = self.cols
        H = self.Qg + (2.0 * self.cfg.mu2) * np.eye(r)
        sa, act, idx, Qa = orc.rescale_for_step(H)
        YT = np.zeros((n, r))
        HP = np.zeros((r, r))
        _, _, fail = orc.estep_dense(self.VT, lo, hi, self.G, Qa, sa, idx, act, self.cfg.mu1,
                                     self.cfg.epsilon, self.cfg.inner_cap, 0.0, self.FT, YT, HP)
        assert fail == -1
        up = np.triu(HP)
        HP = up + up.T - np.diag(np.diag(up))
        return torch.from_numpy(HP), torch.from_numpy(YT)

    def mstep(self, k, Hf, yt_rows, lo, hi):
        n, r = self.G.shape
        H = Hf.numpy() + (2.0 * self.cfg.beta2) * np.eye(r)
        sa, act, idx, Qa = orc.rescale_for_step(H)
        YT = np.zeros((n, r))
        YT[lo:hi] = yt_rows.numpy()
        _, _, fail = orc.mstep_rows(YT, lo, hi, Qa, sa, idx, act, self.cfg.beta1,
                                    self.cfg.epsilon, self.cfg.inner_cap, 0.0, self.G)
        assert fail == -1

    def g_padded(self, plan):
        Gp = np.zeros((plan.padded_rows, self.r))
        Gp[: self.G.shape[0]] = self.G
        return torch.from_numpy(Gp)

    def set_g(self, G):
        self.G = np.ascontiguousarray(G.numpy()[: self.G.shape[0]])

    def objective_pieces(self, k, yt_rows, lo, hi):
        clo, chi = self.cols
        p = np.zeros(12)
        resid = self.X[:, clo:chi] - self.G @ self.FT[clo:chi].T
        p[0] = 0.5 * float(np.sum(resid * resid))
        p[5] = float(np.sum(np.abs(self.FT[clo:chi])))
        p[6] = float(np.sum(self.FT[clo:chi] ** 2))
        p[2] = float(np.sum(np.abs(self.G[lo:hi])))
        p[3] = float(np.sum(self.G[lo:hi] ** 2))
        return torch.from_numpy(p)

    def store_pieces(self, k, pieces):
        self.pieces[k] = pieces.numpy().copy()


def _assemble(p, cfg):
    value = p[0]
    if cfg.mu1:
        value += cfg.mu1 * p[5]
    if cfg.beta1:
        value += cfg.beta1 * p[2]
    if cfg.mu2:
        value += cfg.mu2 * p[6]
    if cfg.beta2:
        value += cfg.beta2 * p[3]
    return value


def _worker(rank, world, port, X, kw, iters, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1506_08938_b200.dist import DistAlternation, ShardPlan

    cfg = orc.Config(**kw)
    n, m = X.shape
    G0, FT0 = orc.initial_factors(X, cfg)
    plan = ShardPlan(n, m, world)
    eng = OracleEngine(X, cfg, G0, FT0)
    eng.cols = plan.col_range(rank)
    da = DistAlternation(eng, plan, rank)
    for k in range(iters):
        da.iterate(k)
    if rank == 0:
        out["obj"] = [_assemble(eng.pieces[k], cfg) for k in range(iters)]
        out["G"] = eng.G.copy()
    clo, chi = plan.col_range(rank)
    out[f"FT{rank}"] = eng.FT[clo:chi].copy()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("reg", [False, True])
def test_two_rank_column_sharding_matches_reference(reg):
    rng = np.random.default_rng(11)
    n, m, r = 70, 150, 5
    X = rng.uniform(size=(n, r)) @ rng.uniform(size=(r, m)) + 0.01 * rng.random((n, m))
    kw = dict(rank=r, seed=4, rel_change_tol=0.0, max_outer=12)
    if reg:
        kw.update(mu1=0.02, mu2=0.01, beta1=0.01, beta2=0.02)
    iters = kw["max_outer"]
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(_worker, args=(2, _free_port(), X, kw, iters, out), nprocs=2,
                           join=True, start_method="fork")
        res = dict(out)
    # single-process reference run with the same 32-aligned shards
    G, FT, log = orc.fit(X, orc.Config(workers=2, **kw))
    np.testing.assert_allclose(res["obj"], log.objective, rtol=1e-9)
    np.testing.assert_allclose(res["G"], G, rtol=1e-7, atol=1e-12)
    FTd = np.concatenate([res["FT0"], res["FT1"]], 0)
    np.testing.assert_allclose(FTd, FT, rtol=1e-7, atol=1e-12)


def test_shard_plan_alignment():
    from paper_1506_08938_b200.dist import ShardPlan

    for n, m, w in [(10000, 20000, 8), (70, 150, 2), (33, 31, 4), (1000, 200000, 8)]:
        p = ShardPlan(n, m, w)
        assert len(p.cols) == w and len(p.rows) == w
        # non-empty shards start on a fast-break block boundary
        assert all(lo % 32 == 0 for lo, hi in p.cols if hi > lo)
        assert all(lo % 32 == 0 for lo, hi in p.rows if hi > lo)
        assert p.cols[-1][1] == m and p.rows[-1][1] == n
        assert sum(hi - lo for lo, hi in p.cols) == m
        assert p.row_chunk >= max(hi - lo for lo, hi in p.rows)


def test_csc_column_block_slices():
    from oracle import generators
    from paper_1506_08938_b200.dist import ShardPlan, csc_column_block

    x = generators.sparse_zipf(300, 257, 0.05, 3)
    dense = np.zeros((x.rows, x.cols))
    col_of = np.repeat(np.arange(x.cols), np.diff(x.indptr))
    dense[x.indices, col_of] = x.values
    for world in (1, 2, 3, 8):
        plan = ShardPlan(x.rows, x.cols, world)
        parts = []
        for g in range(world):
            lo, hi = plan.col_range(g)
            b = csc_column_block(x, lo, hi)
            assert b.cols == hi - lo and b.indptr[0] == 0 and b.indptr[-1] == b.nnz
            parts.append(b.to_dense().array)
        assert np.array_equal(np.concatenate(parts, 1), dense)
