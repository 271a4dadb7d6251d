"""Multi-rank (world_size 2 and 3, gloo, CPU) test of the ROW-sharded driver
for tall sparse data (paper_1506_08938_b200/dist_rows.py).

The product's RowShardedAlternation -- Gram allreduce, reduce-scatter of the
partial linear terms onto the column-block owners, H_f allreduce, allgather
of F, objective pieces -- runs unchanged; the per-rank math comes from an
oracle engine (numpy + the C restatement of the reference kernels), so the
layout and collectives are checked on CPU against the single-process
reference fit (the per-column / per-row problems are the reference's:
blocks are 32-aligned; only the fp64 summation order of h across row blocks
differs).  The solves run to a tight tolerance (epsilon = 1e-10): with the
default epsilon = 0.1 a 1e-16 change in a linear term can flip an approximate
solve's stop decision, which is the algorithm's sensitivity, not
the layout's."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import generators
from oracle import nmf_oracle as orc


class RowOracleEngine:
    def __init__(self, X, cfg, G0, FT0, plan, rank):
        from paper_1506_08938_b200.dist_rows import csc_row_block

        self.cfg, self.plan, self.rank = cfg, plan, rank
        self.r = cfg.rank
        self.rlo, self.rhi = plan.row_range(rank)
        self.clo, self.chi = plan.col_range(rank)
        rows, cols, indptr, idx, vals = csc_row_block(X, self.rlo, self.rhi)
        dense = np.zeros((rows, cols))
        col_of = np.repeat(np.arange(cols), np.diff(indptr))
        dense[idx, col_of] = vals
        self.Xl = dense                      # my row block (n_loc x m)
        self.blk = (idx, col_of, vals)
        self.G = np.array(G0, dtype=np.float64)   # full-size; rows R_g are mine
        self.FTpad = np.zeros((plan.padded_cols, self.r))
        self.FTpad[: plan.m] = FT0
        self.pieces = {}

    def gram_local(self):
        Gl = self.G[self.rlo:self.rhi]
        return torch.from_numpy(orc.gram(Gl) if len(Gl) else np.zeros((self.r,) * 2))

    def set_gram(self, Q):
        self.Qg = Q.numpy().copy()

    def hcol_buffer(self):
        return torch.zeros((self.plan.col_chunk, self.r), dtype=torch.float64)

    def linear_partial(self, first):
        hp = np.zeros((self.plan.padded_cols, self.r))
        mu1 = self.cfg.mu1 if first else 0.0
        hp[: self.plan.m] = mu1 - self.Xl.T @ self.G[self.rlo:self.rhi]
        return torch.from_numpy(hp)

    def estep_solve(self, k, hcol):
        m, r = self.plan.m, self.r
        H = self.Qg + (2.0 * self.cfg.mu2) * np.eye(r)
        sa, act, idx, Qa = orc.rescale_for_step(H)
        YT = np.zeros((m, r))
        cnt = self.chi - self.clo
        YT[self.clo:self.chi] = -hcol.numpy()[:cnt]
        FT = np.ascontiguousarray(self.FTpad[:m])
        _, _, fail = orc.mstep_rows(YT, self.clo, self.chi, Qa, sa, idx, act, 0.0,
                                    self.cfg.epsilon, self.cfg.inner_cap, 0.0, FT)
        assert fail == -1
        self.FTpad[:m] = FT
        F = FT[self.clo:self.chi]
        return torch.from_numpy(F.T @ F if cnt else np.zeros((r, r)))

    def set_hf(self, Hf):
        self.Hf = Hf.numpy().copy()

    def ft_padded(self):
        return torch.from_numpy(self.FTpad)

    def set_ft(self, ft):
        self.FTpad = ft.numpy().copy()

    def mstep(self, k):
        n, r = self.G.shape
        FT = self.FTpad[: self.plan.m]
        H = self.Hf + (2.0 * self.cfg.beta2) * np.eye(r)
        sa, act, idx, Qa = orc.rescale_for_step(H)
        YT = np.zeros((n, r))
        # Y^T rows in the reference's accumulation order (kernels.py:270-274:
        # columns ascending, x * v added per nonzero)
        rows_l, col_of, vals = self.blk
        Yl = np.zeros((self.rhi - self.rlo, r))
        np.add.at(Yl, rows_l, FT[col_of] * vals[:, None])
        YT[self.rlo:self.rhi] = Yl
        self.YTl = YT[self.rlo:self.rhi].copy()
        G = np.ascontiguousarray(self.G)
        _, _, fail = orc.mstep_rows(YT, self.rlo, self.rhi, Qa, sa, idx, act, self.cfg.beta1,
                                    self.cfg.epsilon, self.cfg.inner_cap, 0.0, G)
        assert fail == -1
        self.G = G

    def objective_pieces(self, k, first):
        p = np.zeros(12)
        Gl = self.G[self.rlo:self.rhi]
        p[1] = float(np.sum(Gl * self.YTl))
        p[2] = float(np.sum(np.abs(Gl)))
        p[3] = float(np.sum(Gl ** 2))
        if first:
            p[7] = float(np.sum(self.Qg * self.Hf))
        F = self.FTpad[self.clo:self.chi]
        p[5] = float(np.sum(np.abs(F)))
        p[6] = float(np.sum(F ** 2))
        return torch.from_numpy(p)

    def store_pieces(self, k, pieces):
        self.pieces[k] = pieces.numpy().copy()


def _assemble(p, cfg, xsq):
    v = 0.5 * (xsq - 2.0 * p[1] + p[7])
    return v + cfg.mu1 * p[5] + cfg.beta1 * p[2] + cfg.mu2 * p[6] + cfg.beta2 * p[3]


def _worker(rank, world, port, X, kw, iters, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1506_08938_b200.dist_rows import RowPlan, RowShardedAlternation

    cfg = orc.Config(**kw)
    G0, FT0 = orc.initial_factors(X, cfg)
    plan = RowPlan(X.rows, X.cols, world)
    eng = RowOracleEngine(X, cfg, G0, FT0, plan, rank)
    da = RowShardedAlternation(eng, plan, rank)
    for k in range(iters):
        da.iterate(k)
    xsq = float(X.values @ X.values)
    if rank == 0:
        out["obj"] = [_assemble(eng.pieces[k], cfg, xsq) for k in range(iters)]
        out["FT"] = eng.FTpad[: X.cols].copy()
    lo, hi = plan.row_range(rank)
    out[f"G{rank}"] = eng.G[lo:hi].copy()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world,reg", [(2, False), (3, True)])
def test_row_sharding_matches_reference(world, reg):
    X = generators.sparse_zipf(300, 200, 0.05, 9)
    kw = dict(rank=6, seed=5, rel_change_tol=0.0, max_outer=8, epsilon=1e-10)
    if reg:
        kw.update(mu1=0.02, mu2=0.01, beta1=0.01, beta2=0.02)
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(_worker, args=(world, _free_port(), X, kw, kw["max_outer"], out),
                           nprocs=world, join=True, start_method="fork")
        res = dict(out)
    G, FT, log = orc.fit(X, orc.Config(**kw))
    # (near-converged solves at epsilon = 1e-10: the cross-rank summation
    # order moves the objective by ~5e-9; a layout or collective error would
    # show at 1e-3 or more)
    np.testing.assert_allclose(res["obj"], log.objective, rtol=1e-7)
    Gd = np.concatenate([res[f"G{g}"] for g in range(world)], 0)
    np.testing.assert_allclose(Gd, G, rtol=1e-5, atol=1e-9)
    np.testing.assert_allclose(res["FT"], FT, rtol=1e-5, atol=1e-9)


def test_row_plan_and_blocks():
    from paper_1506_08938_b200.dist_rows import RowPlan, csc_row_block

    x = generators.sparse_zipf(301, 257, 0.05, 3)
    dense = np.zeros((x.rows, x.cols))
    col_of = np.repeat(np.arange(x.cols), np.diff(x.indptr))
    dense[x.indices, col_of] = x.values
    for world in (1, 2, 3, 8):
        p = RowPlan(x.rows, x.cols, world)
        assert all(lo % 32 == 0 for lo, hi in p.rows if hi > lo)
        assert all(lo % 32 == 0 for lo, hi in p.cols if hi > lo)
        assert p.rows[-1][1] == x.rows and p.cols[-1][1] == x.cols
        assert p.padded_cols >= x.cols and p.padded_cols == p.col_chunk * world
        parts = []
        for g in range(world):
            lo, hi = p.row_range(g)
            rows, cols, indptr, idx, vals = csc_row_block(x, lo, hi)
            assert rows == hi - lo and indptr[-1] == len(idx)
            d = np.zeros((rows, cols))
            d[idx, np.repeat(np.arange(cols), np.diff(indptr))] = vals
            parts.append(d)
        assert np.array_equal(np.concatenate(parts, 0), dense)
    b = RowPlan(1_000_000, 200_000, 8).exchange_bytes(200)
    assert b["reduce_scatter_h"] < 2e8 and b["allgather_F"] < 2e8
