"""Multi-GPU alternation for tall sparse data (n > m, BASELINE config 5):
ROW-sharded layout, SURVEY.md 8(e) "Row-sharded ... best when n > m".

Rank g owns a 32-aligned block R_g of the ROWS of X (its CSC and CSR) and of
G, plus a 32-aligned block C_g of the columns for the coefficient solves; F
is replicated.  G's rows never leave their rank.  Per outer iteration
(torch.distributed: NCCL over NVLink on GPUs, gloo in the CPU tests):

  allreduce       Q_g = sum_g G[R_g]^T G[R_g]                  r x r   fp64
  reduce-scatter  P = sum_g (mu1 [g = 0] - G[R_g]^T X[R_g, :])  m x r   fp32
                  -> the linear terms h of my columns C_g (kernels.py:251-258)
  (coefficient NNLS on C_g; F F^T partial over C_g)
  allreduce       H_f = sum_g F[:, C_g] F[:, C_g]^T             r x r   fp64
  allgather       F^T rows C_g -> every rank                    m x r   fp32
  (Y^T[R_g] = X[R_g, :] F^T locally; component NNLS on R_g)
  allreduce       Q_g of the new G (objective quad term, next coefficient step)
  allreduce       objective pieces                              12 fp64

At config 5 (m = 200 000, r = 200) the two panel collectives move 2 x 160 MB
per iteration, against 1.6 GB (fp64 Y^T) + 800 MB (G) for the column-sharded
layout of dist.py, and no rank ever holds all of G (800 MB).  Column and row
blocks are 32-aligned, so every fast-break block (kernels.py:35, 247-248)
lives on one rank and the per-problem results do not depend on the rank
count; only the fp32 summation order of h across ranks does.

The per-rank math comes from an engine (RowCudaEngine below; the CPU tests
plug in an oracle engine), the driver itself does no arithmetic.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L
from . import device as D

BLOCK = L.FASTBREAK_BLOCK


def _chunk(total, world):
    c = -(-total // world // BLOCK) * BLOCK if total else BLOCK
    c = max(c, BLOCK)
    while c * world < total:
        c += BLOCK
    return c


class RowPlan:
    """Uniform 32-aligned chunks: rows [g c_r, (g+1) c_r) and columns
    [g c_c, (g+1) c_c) of rank g (clipped), so the panel collectives work on
    the natural (rows, r) layouts padded to world * chunk rows."""

    def __init__(self, n, m, world):
        self.n, self.m, self.world = n, m, world
        self.row_chunk = _chunk(n, world)
        self.col_chunk = _chunk(m, world)
        self.rows = [(min(n, g * self.row_chunk), min(n, (g + 1) * self.row_chunk))
                     for g in range(world)]
        self.cols = [(min(m, g * self.col_chunk), min(m, (g + 1) * self.col_chunk))
                     for g in range(world)]
        self.padded_cols = self.col_chunk * world

    def row_range(self, rank):
        return self.rows[rank]

    def col_range(self, rank):
        return self.cols[rank]

    def exchange_bytes(self, r, fp_bytes=4):
        """Bytes each rank sends per outer iteration in the panel collectives
        (ring algorithms: (world - 1) / world of the buffer, twice)."""
        w = self.world
        panel = self.padded_cols * r * fp_bytes
        return {"reduce_scatter_h": panel * (w - 1) / w, "allgather_F": panel * (w - 1) / w,
                "allreduce_r2": 3 * 2 * r * r * 8 * (w - 1) / w}


def csc_row_block(X, lo, hi):
    """Rows [lo, hi) of a host CSC matrix (SparseMatrix or the oracle's Csc),
    all columns, row indices renumbered from 0: (rows, cols, indptr, indices,
    values) arrays."""
    idx = np.asarray(X.indices)
    keep = (idx >= lo) & (idx < hi)
    col_of = np.repeat(np.arange(X.cols, dtype=np.int64), np.diff(np.asarray(X.indptr)))
    counts = np.bincount(col_of[keep], minlength=X.cols)
    indptr = np.zeros(X.cols + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    return hi - lo, X.cols, indptr, idx[keep] - lo, np.asarray(X.values)[keep]


class NativeComm:
    """The C-ABI collectives (nmfb_comm_init / allreduce_r2 /
    reduce_scatter_panel / allgather_panel, csrc/comm.cu): one NCCL
    communicator per rank, its unique id handed out through the
    torch.distributed group; stream-ordered on the current stream."""

    def __init__(self, group=None):
        import ctypes

        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if not L.lib().nmfb_comm_available():
            raise RuntimeError("libnccl.so.2 could not be resolved")
        uid = np.zeros(128, dtype=np.uint8)
        if self.rank == 0:
            L.call("nmfb_comm_unique_id", uid.ctypes.data_as(ctypes.c_void_p))
        t = torch.from_numpy(uid)
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        dist.broadcast(t, 0, group=group)
        uid = t.cpu().numpy()
        self.handle = ctypes.c_void_p()
        L.call("nmfb_comm_init", uid.ctypes.data_as(ctypes.c_void_p), self.rank, self.world,
               ctypes.byref(self.handle))

    def allreduce(self, t):
        assert t.dtype == torch.float64 and t.is_contiguous()
        L.call("nmfb_allreduce_r2", self.handle, D.vp(t), t.numel(), D.stream_handle())
        return t

    def reduce_scatter(self, full, out):
        code = L.F32 if out.dtype == torch.float32 else L.F64
        L.call("nmfb_reduce_scatter_panel", self.handle, D.vp(full), D.vp(out), out.numel(),
               code, D.stream_handle())
        return out

    def allgather(self, full, mine):
        code = L.F32 if full.dtype == torch.float32 else L.F64
        L.call("nmfb_allgather_panel", self.handle, D.vp(mine), D.vp(full), mine.numel(), code,
               D.stream_handle())
        return full

    def close(self):
        if getattr(self, "handle", None):
            L.call("nmfb_comm_destroy", self.handle)
            self.handle = None


class RowShardedAlternation:
    """One rank's share of the alternation in the row layout.  Collectives:
    the C-ABI NCCL ones (NativeComm) when given, else torch.distributed."""

    def __init__(self, engine, plan: RowPlan, rank, group=None, native=None):
        self.e = engine
        self.plan = plan
        self.rank = rank
        self.group = group
        self.native = native
        self.comm = dist.is_available() and dist.is_initialized()
        if not self.comm and plan.world != 1:
            raise RuntimeError("world > 1 needs an initialised torch.distributed group")
        self.qg_valid = False

    def _allreduce(self, t):
        if self.native is not None:
            return self.native.allreduce(t)
        if self.comm:
            dist.all_reduce(t, group=self.group)
        return t

    def _reduce_scatter(self, full, out):
        if self.native is not None:
            return self.native.reduce_scatter(full, out)
        if self.comm:
            dist.reduce_scatter_tensor(out, full, group=self.group)
        else:
            out.copy_(full[: out.shape[0]])
        return out

    def _allgather(self, full):
        c = self.plan.col_chunk
        mine = full[self.rank * c: (self.rank + 1) * c]
        if self.native is not None:
            # in place: my block already sits at full + rank * chunk
            return self.native.allgather(full, mine)
        if self.comm:
            dist.all_gather_into_tensor(full, mine, group=self.group)
        return full

    def iterate(self, k):
        e = self.e
        if not self.qg_valid:
            e.set_gram(self._allreduce(e.gram_local()))
        # coefficient step: partial linear terms of all columns, summed onto
        # each column block's owner, then the owner's solves
        hpad = e.linear_partial(first=(self.rank == 0))
        hcol = self._reduce_scatter(hpad, e.hcol_buffer())
        e.set_hf(self._allreduce(e.estep_solve(k, hcol)))
        e.set_ft(self._allgather(e.ft_padded()))
        # component step on my rows with the replicated F
        e.mstep(k)
        e.set_gram(self._allreduce(e.gram_local()))
        self.qg_valid = True
        e.store_pieces(k, self._allreduce(e.objective_pieces(k, self.rank == 0)))


class RowCudaEngine:
    """Local math of one rank on its GPU (C-ABI kernels only)."""

    def __init__(self, X_rows, cfg, G0_rows, FT0, plan: RowPlan, rank, max_iters):
        from .matrix import SparseMatrix

        self.cfg = cfg
        self.r = r = cfg.rank
        self.plan = plan
        self.rank = rank
        self.rlo, self.rhi = plan.row_range(rank)
        self.clo, self.chi = plan.col_range(rank)
        if not isinstance(X_rows, SparseMatrix) or X_rows.rows != self.rhi - self.rlo:
            raise ValueError("X_rows must be this rank's row block as a SparseMatrix")
        if cfg.precision != "fp32":
            raise ValueError("the row-sharded multi-GPU path runs the fp32 production kernels")
        self.data = D.DeviceData(X_rows, "fp32")
        dev = self.data.device
        m = plan.m
        # F^T replicated in the padded (world * col_chunk, r) allgather layout
        self.ft_pad = torch.zeros((plan.padded_cols, r), dtype=torch.float32, device=dev)
        self.ft_pad[:m].copy_(torch.as_tensor(np.asarray(FT0, dtype=np.float32)))
        # the Alternation supplies the buffers and primitive launches (its G is
        # my row block, its F^T the replicated one)
        self.st = D.Alternation(self.data, cfg, G0_rows, FT0, max_iters, precision="fp32",
                                lanes=cfg.lanes, overlap=False)
        self.st.FT = self.ft_pad[:m]
        self.hpad = torch.zeros((plan.padded_cols, r), dtype=torch.float32, device=dev)
        self.hcol = torch.zeros((plan.col_chunk, r), dtype=torch.float32, device=dev)
        self.Qtmp = torch.zeros((r, r), dtype=torch.float64, device=dev)
        self.pieces = torch.zeros((12,), dtype=torch.float64, device=dev)

    # -- Grams ------------------------------------------------------------------
    def gram_local(self):
        st = self.st
        n_loc = self.rhi - self.rlo
        if n_loc > 0:
            L.call("nmfb_gram", st.code, D.vp(st.G), n_loc, self.r, self.r, D.vp(self.Qtmp),
                   D.vp(st.gram_ws), D.stream_handle())
        else:
            self.Qtmp.zero_()
        return self.Qtmp

    def set_gram(self, Q):
        if Q.data_ptr() != self.st.Qg.data_ptr():
            self.st.Qg.copy_(Q)

    def set_hf(self, Hf):
        st = self.st
        if Hf.data_ptr() != st.Hf.data_ptr():
            st.Hf.copy_(Hf)
        st.rescale(st.Hf, 2.0 * self.cfg.beta2, 1)

    # -- coefficient step ---------------------------------------------------------
    def hcol_buffer(self):
        return self.hcol

    def linear_partial(self, first):
        """hpad[:m] = (mu1 if first else 0) - G[R_g]^T X[R_g, :] (all columns)."""
        st, d = self.st, self.data
        m, r = self.plan.m, self.r
        mu1 = self.cfg.mu1 if first else 0.0
        nbg, segg = st._spmm_plan()[:2]
        if nbg > 1:
            L.call("nmfb_csc_linear_blocked", D.vp(d.indptr), D.vp(segg), nbg, D.vp(d.rowidx),
                   D.vp(d.vals), m, D.vp(st.G), r, mu1, D.vp(self.hpad), D.stream_handle())
        else:
            L.call("nmfb_csc_linear", st.code, st.mode, D.vp(d.indptr), D.vp(d.rowidx),
                   D.vp(d.vals), 0, m, D.vp(st.G), r, mu1, D.vp(self.hpad), D.stream_handle())
        return self.hpad

    def estep_solve(self, k, hcol):
        """NNLS of my columns with h = hcol, then the partial F F^T of them."""
        st, cfg, r = self.st, self.cfg, self.r
        st.rescale(st.Qg, 2.0 * cfg.mu2, 0)
        cnt = self.chi - self.clo
        FTc = self.ft_pad[self.clo:self.chi]
        if cnt > 0:
            L.call("nmfb_nnls_batch", st.code, st.mode, D.vp(st.Qa[0]), D.vp(st.sa[0]),
                   D.vp(st.act[0]), D.vp(st.active[0]), r, r, D.vp(st.ra[0]), D.vp(hcol),
                   L.F32, 0, r, 0, 0.0, D.vp(FTc), cnt, self.clo, float(cfg.epsilon),
                   int(cfg.inner_cap), 0.0, None, None, D.vp(st.stats[k, 0]), st.lanes,
                   D.stream_handle())
            L.call("nmfb_gram", st.code, D.vp(FTc), cnt, r, r, D.vp(self.Qtmp),
                   D.vp(st.gram_ws), D.stream_handle())
        else:
            self.Qtmp.zero_()
        return self.Qtmp

    def ft_padded(self):
        return self.ft_pad

    def set_ft(self, ft_pad):
        pass  # the allgather filled ft_pad in place

    # -- component step ------------------------------------------------------------
    def mstep(self, k):
        """Y^T[R_g] = X[R_g, :] F^T (load-balanced CSR chunks), then the NNLS
        of my rows with h = beta1 - Y^T."""
        st, d, cfg, r = self.st, self.data, self.cfg, self.r
        n_loc = self.rhi - self.rlo
        if n_loc == 0:
            return
        ycode = L.F64 if st.ybuf.dtype == torch.float64 else L.F32
        if getattr(st, "ypart", None) is None:
            st.ypart = torch.empty((max(d.nslots, 1) * r,), dtype=torch.float64,
                                   device=st.ybuf.device)
        L.call("nmfb_csr_yt_chunked", st.code, D.vp(d.chunks), d.nchunks, D.vp(d.heavy),
               d.nheavy, D.vp(d.colidx), D.vp(d.cvals), D.vp(st.FT), r, ycode, D.vp(st.ybuf),
               D.vp(st.ypart), D.stream_handle())
        L.call("nmfb_nnls_batch", st.code, st.mode, D.vp(st.Qa[1]), D.vp(st.sa[1]),
               D.vp(st.act[1]), D.vp(st.active[1]), r, r, D.vp(st.ra[1]), D.vp(st.ybuf), ycode,
               1, r, 0, cfg.beta1, D.vp(st.G), n_loc, self.rlo, float(cfg.epsilon),
               int(cfg.inner_cap), 0.0, None, None, D.vp(st.stats[k, 1]), st.lanes,
               D.stream_handle())

    # -- objective -------------------------------------------------------------------
    def objective_pieces(self, k, first):
        """Additive pieces (device.Alternation slot layout): cross <G, Y^T>
        over my rows; quad <G^T G, H_f> (global, counted by rank 0 only);
        penalty sums over my F columns and G rows."""
        st, cfg, r = self.st, self.cfg, self.r
        p = self.pieces
        p.zero_()
        n_loc = self.rhi - self.rlo
        ycode = L.F64 if st.ybuf.dtype == torch.float64 else L.F32
        if n_loc > 0:
            st.dot(st.G, st.code, st.ybuf, ycode, n_loc * r, p[1:4])
        if first:
            st.dot(st.Qg, L.F64, st.Hf, L.F64, r * r, p[7:10])
        if (cfg.mu1 or cfg.mu2) and self.chi > self.clo:
            st.dot(self.ft_pad[self.clo:self.chi], st.code, None, L.F64,
                   (self.chi - self.clo) * r, p[4:7])
        return p

    def store_pieces(self, k, pieces):
        self.st.pieces[k].copy_(pieces)


class RowShardedFit:
    """bench.py / users: the row-sharded fit state on this rank's GPU."""

    def __init__(self, X, cfg, init, group=None):
        """X: the FULL host CSC matrix (SparseMatrix) -- each rank keeps its
        row block; init = (G0, FT0) full host factors (seeded, identical on
        every rank)."""
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        from .matrix import SparseMatrix

        self.plan = RowPlan(X.rows, X.cols, world)
        lo, hi = self.plan.row_range(rank)
        rows, cols, indptr, indices, values = csc_row_block(X, lo, hi)
        Xr = SparseMatrix(rows, cols, indptr, indices, values, validate=False)
        G0, FT0 = init
        self.engine = RowCudaEngine(Xr, cfg, np.asarray(G0)[lo:hi], FT0, self.plan, rank,
                                    cfg.max_outer)
        # collectives: the C-ABI NCCL ones by default on an NCCL group
        # (NMFB_COMM=torch: torch.distributed's)
        import os

        self.native = None
        if (dist.is_initialized() and dist.get_backend(group) == "nccl"
                and os.environ.get("NMFB_COMM", "native") == "native"):
            self.native = NativeComm(group)
        self.state = _RowStateView(RowShardedAlternation(self.engine, self.plan, rank, group,
                                                         native=self.native), self.engine.st)
        self.peer = False


class _RowStateView:
    def __init__(self, da, st):
        self.da = da
        self.st = st
        self.pieces = st.pieces
        self.stats = st.stats

    def iterate(self, k):
        self.da.iterate(k)

    def join(self):
        self.st.join()

    def assemble(self, *a, **kw):
        return self.st.assemble(*a, **kw)
