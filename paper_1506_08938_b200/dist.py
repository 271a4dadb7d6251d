"""Multi-GPU alternation: one process per GPU, columns of X / F sharded.

Layout (column-sharded; north star "sharding the columns of X
and H (and the rows of X and W for the W-update)"):

* rank g owns data columns C_g (32-aligned, parallel.block_plan over
  ranks, so fast-break blocks never straddle ranks and the per-column
  solutions are identical to a single-GPU run) and the matching rows of F^T;
* every rank holds all of G (n x r) for its G^T X_g pass, and solves the
  component rows R_g (32-aligned row blocks) in the M-step.

Collectives per outer iteration (torch.distributed; NCCL over NVLink on
GPUs, gloo in the CPU tests):
  allreduce   H_f = sum_g F_g F_g^T                 r x r fp64
  reduce-scatter  Y^T = sum_g X_g F_g^T -> rows R_g  n x r (padded to P blocks)
  allreduce   Q_g = sum_g G[R_g]^T G[R_g]            r x r fp64 (north-star Gram allreduce)
  allgather   G rows R_g -> full G                   n x r
  allreduce   objective pieces                       a few fp64 scalars
The allgather is required by the column layout (the next coefficient step
needs all of G); the north star lists only the first two.

The per-rank numerics come from an *engine* (the CUDA engine below for the
product; tests/ plug an oracle engine in to check the sharding logic on CPU
with gloo).  The driver itself does no arithmetic beyond summing scalars.

Peer-memory path (dense fp32 on GPUs with peer access; the default when
torch symmetric memory is available, NMFB_DIST_PEER=0 forces NCCL).  The
exchanges above become stores issued by the producing kernels into the
consumers' symmetric buffers over NVLink (PeerExchange, csrc/peer.cu):
  X F^T GEMM epilogue  -> owner rank's Y^T receive slots    (reduce-scatter)
  M-step NNLS epilogue -> every rank's copy of G            (all-gather)
  F_g F_g^T, objective pieces -> per-source slots            (allreduce)
with one epoch flag barrier after each producer and a fixed-order slot sum
at the consumer, so every rank computes the same bits independent of any
collective's reduction order.  G is then replicated exactly, so the Gram of
G is computed locally (fused with its rescale) instead of allreduced.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L
from . import device as D

BLOCK = L.FASTBREAK_BLOCK


class ShardPlan:
    """Column shards: 32-aligned near-equal blocks over `world` ranks
    (parallel.py:162-169).  Row shards for the component step: uniform
    32-aligned chunks (rank g owns rows [g c, min(n, (g+1) c)), c =
    ceil(n / world / 32) * 32), so the row-blocked buffers are simply the
    natural (n, r) layout padded to world * c rows: the reduce-scatter of Y^T
    and the allgather of G need no repacking (the allgather runs in place)."""

    def __init__(self, n, m, world):
        self.n, self.m, self.world = n, m, world
        self.cols = D.block_plan(m, world)
        while len(self.cols) < world:
            self.cols.append((m, m))
        self.row_chunk = max(BLOCK, -(-n // world // BLOCK) * BLOCK) if n else BLOCK
        while self.row_chunk * world < n:
            self.row_chunk += BLOCK
        self.rows = [(min(n, g * self.row_chunk), min(n, (g + 1) * self.row_chunk))
                     for g in range(world)]
        self.padded_rows = self.row_chunk * world

    def col_range(self, rank):
        return self.cols[rank]

    def row_range(self, rank):
        return self.rows[rank]


class PeerExchange:
    """Symmetric device buffers shared by all ranks over NVLink + epoch flags.

    One symmetric allocation (torch symmetric memory; its rendezvous hands out
    every rank's mapping) carved into named regions; `ptrs(name)` lists the
    region's address on every rank.  Flags: world epoch words (one per source
    rank) + an error word, at the end of the allocation."""

    ALIGN = 256

    def __init__(self, regions, device, group=None, timeout_s=60.0):
        import torch.distributed._symmetric_memory as symm

        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world > L.MAX_PEERS:
            raise ValueError(f"peer exchange supports up to {L.MAX_PEERS} ranks")
        gname = (group or dist.group.WORLD).group_name
        self.offsets = {}
        off = 0
        for name, nbytes in list(regions.items()) + [("flags", 8 * (self.world + 1))]:
            self.offsets[name] = (off, int(nbytes))
            off += -(-int(nbytes) // self.ALIGN) * self.ALIGN
        self.buf = symm.empty(max(off, self.ALIGN), dtype=torch.uint8, device=device)
        self.buf.zero_()
        self.handle = symm.rendezvous(self.buf, gname)
        self.bases = [int(p) for p in self.handle.buffer_ptrs]
        if len(self.bases) != self.world:
            raise RuntimeError("symmetric memory rendezvous returned the wrong rank count")
        self.ticket = torch.zeros((1,), dtype=torch.int32, device=device)
        self.flag_ptrs = L.ptr_array(self.ptrs("flags"))
        self.epoch = 0
        self.timeout_s = float(timeout_s)
        torch.cuda.synchronize(device)
        dist.barrier(group)  # every rank's flags are zero before anyone signals

    def ptrs(self, name, byte_offset=0):
        off = self.offsets[name][0] + byte_offset
        return [b + off for b in self.bases]

    def view(self, name, dtype):
        off, nbytes = self.offsets[name]
        return self.buf[off: off + nbytes].view(dtype)

    def put(self, src, name, byte_offset):
        """Copy src (contiguous, 8-byte multiple) to region `name` at
        byte_offset on every rank (no signal)."""
        nbytes = src.numel() * src.element_size()
        L.call("nmfb_peer_put", D.vp(src), nbytes, L.ptr_array(self.ptrs(name, byte_offset)),
               self.world, self.rank, None, None, 0, 0, D.stream_handle())

    def put_barrier(self, src, name, byte_offset):
        """put() + barrier() in one kernel: the copy to every peer, then (after
        all of its CTAs) this rank's epoch flag on every peer; then the wait."""
        self.epoch += 1
        nbytes = src.numel() * src.element_size()
        L.call("nmfb_peer_put", D.vp(src), nbytes, L.ptr_array(self.ptrs(name, byte_offset)),
               self.world, self.rank, self.flag_ptrs, D.vp(self.ticket), self.epoch, 1,
               D.stream_handle())
        L.call("nmfb_peer_wait", self.ptrs("flags")[self.rank], self.world, self.epoch,
               self.timeout_s, D.stream_handle())

    def barrier(self):
        """All writes this rank issued so far (kernels earlier on the stream)
        are visible on every peer, and every peer's on this rank."""
        self.epoch += 1
        L.call("nmfb_peer_put", None, 0, None, self.world, self.rank, self.flag_ptrs,
               D.vp(self.ticket), self.epoch, 1, D.stream_handle())
        L.call("nmfb_peer_wait", self.ptrs("flags")[self.rank], self.world, self.epoch,
               self.timeout_s, D.stream_handle())

    def check(self):
        """Raise if a wait timed out (synchronises)."""
        err = int(self.view("flags", torch.int64)[self.world].item())
        if err:
            raise RuntimeError(f"peer exchange: wait for epoch {err} timed out")


class DistAlternation:
    """One rank's share of the alternation; engine does the local math."""

    def __init__(self, engine, plan: ShardPlan, rank, group=None):
        self.e = engine
        self.plan = plan
        self.rank = rank
        self.group = group
        self.world = plan.world
        # with a process group every collective is issued (also at world 1, so a
        # single-GPU torchrun exercises the NCCL path); without one, world must be 1
        self.comm = dist.is_available() and dist.is_initialized()
        if not self.comm and self.world != 1:
            raise RuntimeError("world > 1 needs an initialised torch.distributed group")

    # -- collectives -------------------------------------------------------
    def _allreduce(self, t):
        if self.comm:
            dist.all_reduce(t, group=self.group)
        return t

    def _reduce_scatter_rows(self, yt_full):
        """Y^T partial -> this rank's rows summed over ranks.  yt_full is either
        the padded (world * chunk, r) buffer (CUDA engine: no repacking) or the
        natural (n, r) array (padded here)."""
        p = self.plan
        chunk = p.row_chunk
        lo, hi = p.row_range(self.rank)
        if not self.comm:
            return yt_full[lo:hi]
        if yt_full.shape[0] != p.padded_rows:
            padded = yt_full.new_zeros((p.padded_rows, yt_full.shape[1]))
            padded[: p.n] = yt_full
            yt_full = padded
        if getattr(self, "_rs_out", None) is None or self._rs_out.dtype != yt_full.dtype:
            self._rs_out = yt_full.new_empty((chunk, yt_full.shape[1]))
        dist.reduce_scatter_tensor(self._rs_out, yt_full, group=self.group)
        return self._rs_out[: hi - lo]

    def _allgather_rows(self, g_pad):
        """In place on the padded (world * chunk, r) G: my block -> everyone."""
        p = self.plan
        if self.comm:
            chunk = p.row_chunk
            mine = g_pad[self.rank * chunk: (self.rank + 1) * chunk]
            dist.all_gather_into_tensor(g_pad, mine, group=self.group)
        return g_pad

    # -- one outer iteration --------------------------------------------------
    def iterate(self, k):
        e, p = self.e, self.plan
        rlo, rhi = p.row_range(self.rank)
        clo, chi = p.col_range(self.rank)
        if getattr(e, "px", None) is not None:
            # peer-memory path: the producers' stores are the exchanges
            e.estep_peer(k, clo)
            e.mstep_peer(k, rlo, rhi)
            e.objective_peer(k, rlo, rhi)
            return
        # Gram of G: partial over my rows, allreduced (first iteration: all rows
        # are already replicated, so every rank's partial covers its own block)
        Qg = self._allreduce(e.gram_rows(rlo, rhi))
        e.set_gram(Qg)
        # coefficient step on my columns; accumulators are partial sums
        Hf_part, yt_part = e.estep(k, clo)
        Hf = self._allreduce(Hf_part)
        yt_rows = self._reduce_scatter_rows(yt_part)
        # component step on my rows, then every rank gets all of G
        e.mstep(k, Hf, yt_rows, rlo, rhi)
        e.set_g(self._allgather_rows(e.g_padded(self.plan)))
        # objective pieces (sum over ranks)
        pieces = self._allreduce(e.objective_pieces(k, yt_rows, rlo, rhi))
        e.store_pieces(k, pieces)


# ---------------------------------------------------------------------------
# CUDA engine: wraps device.Alternation for one rank's column block
# ---------------------------------------------------------------------------
class CudaEngine:
    """Local math of one rank on its GPU (all C-ABI kernels)."""

    def __init__(self, X_block, cfg, G0, FT0_block, max_iters, n_total_cols):
        self.data = D.DeviceData(X_block, cfg.precision)
        self.st = D.Alternation(self.data, cfg, G0, FT0_block, max_iters,
                                precision=cfg.precision, lanes=cfg.lanes, overlap=False)
        self.cfg = cfg
        self.r = cfg.rank
        st = self.st
        dev = self.data.device
        self.Qtmp = torch.zeros((self.r, self.r), dtype=torch.float64, device=dev)
        self.Hf_part = torch.zeros_like(self.Qtmp)
        # dense fast path: split-K partials are summed locally before the
        # reduce-scatter; sparse / fp64: Y^T is already one fp64 buffer
        self.ysplit = self.data.kind == "dense" and st.mode == L.MODE_FAST
        ydt = torch.float32 if self.ysplit else st.ybuf.dtype
        # row-blocked (padded) buffers: G and the Y^T partial live in the
        # (world * chunk, r) layout of the collectives; st.G views the first n rows
        self.g_pad = None
        self.yt_pad = None
        self.yt = torch.zeros((self.data.n, self.r), dtype=ydt, device=dev)
        self.ycode = L.F32 if ydt == torch.float32 else L.F64
        self.n_total_cols = n_total_cols
        self.pieces = torch.zeros((12,), dtype=torch.float64, device=dev)

    def gram_rows(self, lo, hi):
        st = self.st
        if hi > lo:
            L.call("nmfb_gram", st.code, D.vp(st.G[lo:hi]), hi - lo, self.r, self.r,
                   D.vp(self.Qtmp), D.vp(st.gram_ws), D.stream_handle())
        else:
            self.Qtmp.zero_()
        return self.Qtmp

    def set_gram(self, Q):
        self.st.Qg.copy_(Q)
        self.st.qg_valid = True

    def bind_plan(self, plan):
        """Allocate the padded row-blocked buffers of `plan` and move G into one."""
        st, n, r = self.st, self.data.n, self.r
        self.g_pad = torch.zeros((plan.padded_rows, r), dtype=st.G.dtype, device=st.G.device)
        self.g_pad[:n].copy_(st.G)
        st.G = self.g_pad[:n]
        self.yt_pad = torch.zeros((plan.padded_rows, r), dtype=self.yt.dtype,
                                  device=self.yt.device)
        self.yt = self.yt_pad[:n]

    def estep(self, k, col_offset):
        st = self.st
        st.index_base_e = col_offset
        st.estep(k)
        # partial accumulators of my columns: H_f partial, Y^T partial (summed
        # split-K) written straight into the padded collective layout
        self.Hf_part.copy_(st.Hf)
        if self.ysplit:
            L.call("nmfb_sum_parts", D.vp(st.ybuf), st.splits_m, self.data.n * self.r,
                   D.vp(self.yt), D.stream_handle())
        else:
            self.yt.copy_(st.ybuf.view(self.data.n, self.r))
        return self.Hf_part, (self.yt_pad if self.yt_pad is not None else self.yt)

    def mstep(self, k, Hf, yt_rows, lo, hi):
        st = self.st
        st.Hf.copy_(Hf)
        st.rescale(st.Hf, 2.0 * self.cfg.beta2, 1)
        if hi > lo:
            stats = st.stats[k, 1]
            L.call("nmfb_nnls_batch", st.code, st.mode, D.vp(st.Qa[1]), D.vp(st.sa[1]),
                   D.vp(st.act[1]), D.vp(st.active[1]), self.r, self.r, D.vp(st.ra[1]),
                   D.vp(yt_rows), self.ycode, 1, self.r, 0, self.cfg.beta1, D.vp(st.G[lo:hi]),
                   hi - lo, lo, float(self.cfg.epsilon), int(self.cfg.inner_cap), 0.0, None,
                   None, D.vp(stats), st.lanes, D.stream_handle())

    def g_padded(self, plan):
        return self.g_pad

    def set_g(self, G_full):
        pass  # the allgather filled st.G's padded buffer in place

    # -- peer-memory path -------------------------------------------------------
    def enable_peer(self, plan, group=None):
        """Move G and the exchange buffers into symmetric memory (all ranks
        call this together).  Dense fp32 tensor-core path only."""
        st, n, r = self.st, self.data.n, self.r
        if not (self.ysplit and getattr(st, "use_tc", False)):
            raise ValueError("the peer path needs the dense fp32 tensor-core engine")
        world = plan.world
        self.P = st.splits_m  # partial slots per rank (equal column blocks: same on every rank)
        chunk = plan.row_chunk
        regions = {
            "yt": 4 * world * self.P * chunk * r,      # Y^T partial slots, by source rank
            "g": 4 * plan.padded_rows * r,             # replicated G (row-blocked)
            "hf": 8 * world * r * r,                   # F_g F_g^T by source rank
            "pieces": 8 * world * st.max_iters * 12,   # objective pieces [src][k][12]
        }
        px = PeerExchange(regions, self.data.device, group)
        g = px.view("g", torch.float32).view(plan.padded_rows, r)
        g[:n].copy_(st.G)
        st.G = g[:n]
        self.g_pad = g
        self.plan = plan
        self.yt_recv = px.view("yt", torch.float32)
        self.hf_slots = px.view("hf", torch.float64)
        self.piece_slots = px.view("pieces", torch.float64)
        st.yt_out = (L.ptr_array(px.ptrs("yt")), world, chunk, px.rank)
        lo, hi = plan.row_range(px.rank)
        self.g_mirror = L.ptr_array([q for i, q in enumerate(px.ptrs("g", lo * r * 4))
                                     if i != px.rank])
        self.n_mirror = world - 1
        self.iters_done = 0
        torch.cuda.synchronize()
        px.barrier()
        self.px = px

    def estep_peer(self, k, col_offset):
        st, px, r = self.st, self.px, self.r
        st.index_base_e = col_offset
        st.qg_valid = False  # G is replicated exactly: Gram + rescale locally
        st.estep(k)          # the X F^T epilogue stores into the owners' slots
        px.put_barrier(st.Hf, "hf", px.rank * r * r * 8)
        L.call("nmfb_sum_slots_rescale", st.code, D.vp(self.hf_slots), px.world, r * r,
               D.vp(st.Hf), r, 2.0 * self.cfg.beta2, D.vp(st.Qa[1]), D.vp(st.sa[1]),
               D.vp(st.act[1]), D.vp(st.active[1]), D.vp(st.ra[1]), D.stream_handle())

    def mstep_peer(self, k, lo, hi):
        st, px, r = self.st, self.px, self.r
        if hi > lo:
            L.call("nmfb_nnls_batch_peers", st.code, st.mode, D.vp(st.Qa[1]), D.vp(st.sa[1]),
                   D.vp(st.act[1]), D.vp(st.active[1]), r, r, D.vp(st.ra[1]),
                   D.vp(self.yt_recv), L.F32, px.world * self.P, r, self.plan.row_chunk * r,
                   self.cfg.beta1, D.vp(st.G[lo:hi]), hi - lo, lo, float(self.cfg.epsilon),
                   int(self.cfg.inner_cap), 0.0, None, None, D.vp(st.stats[k, 1]), st.lanes,
                   self.g_mirror, self.n_mirror, D.stream_handle())
        px.barrier()  # every rank now holds all of G

    def objective_peer(self, k, lo, hi):
        px = self.px
        p = self.objective_pieces(k, None, lo, hi)
        # slot [src][k]; summed once at finish() (slots are per iteration, so
        # no barrier is needed here)
        px.put(p, "pieces", (px.rank * self.st.max_iters + k) * 12 * 8)
        self.iters_done = max(self.iters_done, k + 1)

    def finish(self):
        """Sum the objective-piece slots of every iteration run so far."""
        px = getattr(self, "px", None)
        if px is None or self.iters_done == 0:
            return
        px.barrier()
        K = self.iters_done
        L.call("nmfb_sum_slots_f64", D.vp(self.piece_slots), px.world, K * 12,
               self.st.max_iters * 12, D.vp(self.st.pieces), D.stream_handle())
        # a timed-out epoch wait left stale slots behind: fail the fit loudly
        px.check()

    def objective_pieces(self, k, yt_rows, lo, hi):
        """Additive per-rank pieces (slot layout of device.Alternation):
        dense residual over my columns; sparse cross <G[R], Y^T[R]> over my
        rows and quad <G^T G, H_f> on rank-0-equivalent terms split by rows;
        penalty sums over my F rows and my G rows."""
        st, cfg, d = self.st, self.cfg, self.data
        p = self.pieces
        p.zero_()
        G = st.G[lo:hi]
        if d.kind == "dense" and getattr(st, "use_i8", False):
            # exact int8 tensor-core residual over my column block (the same
            # kernel as the single-GPU path): 8-bit slices of the full G and of
            # my rows of F^T, X block (n x m_local) row-major
            q = k % 2
            L.call("nmfb_slice_u8", D.vp(st.G), d.n, self.r, self.r, D.vp(st.Gsl[q]),
                   D.stream_handle())
            L.call("nmfb_slice_u8", D.vp(st.FT), d.m, self.r, self.r, D.vp(st.Fsl[q]),
                   D.stream_handle())
            L.call("nmfb_residual_i8", D.vp(d.X), d.n, d.m, D.vp(st.Gsl[q]), D.vp(st.Fsl[q]),
                   self.r, D.vp(p[0:1]), D.vp(st.rq_ws), D.stream_handle())
            if (cfg.beta1 or cfg.beta2) and hi > lo:
                st.dot(G, st.code, None, L.F64, (hi - lo) * self.r, p[1:4])
        elif d.kind == "dense":
            L.call("nmfb_dense_residual", st.code, D.vp(d.XT), d.m, d.n, D.vp(st.G),
                   D.vp(st.FT), self.r, D.vp(p[0:1]), D.vp(st.res_ws), D.stream_handle())
            if (cfg.beta1 or cfg.beta2) and hi > lo:
                st.dot(G, st.code, None, L.F64, (hi - lo) * self.r, p[1:4])
        else:
            if hi > lo:
                st.dot(G, st.code, yt_rows, self.ycode, (hi - lo) * self.r, p[1:4])
                # quad = sum_rows-blocks <G_R^T G_R, H_f>: additive over row blocks
                L.call("nmfb_gram", st.code, D.vp(G), hi - lo, self.r, self.r, D.vp(self.Qtmp),
                       D.vp(st.gram_ws), D.stream_handle())
                st.dot(self.Qtmp, L.F64, st.Hf, L.F64, self.r * self.r, p[7:10])
        if cfg.mu1 or cfg.mu2:
            st.dot(st.FT, st.code, None, L.F64, st.m * self.r, p[4:7])
        return p

    def store_pieces(self, k, pieces):
        self.st.pieces[k].copy_(pieces)


def csc_column_block(X, lo, hi):
    """Columns [lo, hi) of a host CSC matrix (SparseMatrix or the oracle's
    Csc) as a SparseMatrix sharing the index/value arrays."""
    from .matrix import SparseMatrix

    p0, p1 = int(X.indptr[lo]), int(X.indptr[hi])
    return SparseMatrix(X.rows, hi - lo, X.indptr[lo:hi + 1] - p0, X.indices[p0:p1],
                        X.values[p0:p1], validate=False)


class DistFit:
    """bench.py / users: column-sharded fit state on this rank's GPU."""

    def __init__(self, X_block, cfg, init, group=None, m_total=None):
        """X_block: this rank's columns -- dense (n, m_local) or a sparse
        SparseMatrix / ingest.DeviceCsc column block; m_total: the global
        column count (default m_local * world, equal blocks).  The blocks
        must be the ShardPlan's 32-aligned column ranges."""
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        if hasattr(X_block, "shape"):
            n, m_local = X_block.shape
        else:
            n, m_local = X_block.rows, X_block.cols
        m = m_local * world if m_total is None else int(m_total)
        self.plan = ShardPlan(n, m, world)
        clo, chi = self.plan.col_range(rank)
        if chi - clo != m_local:
            raise ValueError("every rank must hold its 32-aligned column block of the shard plan")
        G0, FT0 = init
        self.engine = CudaEngine(X_block, cfg, G0, FT0, cfg.max_outer, m)
        self.peer = False
        if peer_agreed(self.engine, group):
            # every rank is eligible with the same slot layout: the rendezvous
            # below is entered by all ranks or by none; a failure past this
            # point is an error on that rank (no silent per-rank fallback)
            self.engine.enable_peer(self.plan, group)
            self.peer = True
        if not self.peer:
            self.engine.bind_plan(self.plan)
        self.state = _StateView(DistAlternation(self.engine, self.plan, rank, group),
                                self.engine.st)


def peer_agreed(engine, group=None):
    """The peer path is taken only when EVERY rank is eligible and every
    rank derived the same partial-slot count P (the symmetric regions'
    offsets depend on it): an all-gather of (eligible, P) decides it
    collectively, so no rank waits in the symmetric-memory rendezvous while
    another falls back to NCCL."""
    ok = peer_wanted(engine)
    if ok:
        try:  # local prerequisites, checked before the collective decision
            import importlib

            importlib.import_module("torch.distributed._symmetric_memory")
        except Exception:
            ok = False
    P = int(getattr(engine.st, "splits_m", 0)) if ok else 0
    if not (dist.is_initialized() and dist.get_backend(group) == "nccl"):
        return False
    dev = engine.data.device
    mine = torch.tensor([1 if ok else 0, P], dtype=torch.int64, device=dev)
    alls = [torch.empty_like(mine) for _ in range(dist.get_world_size(group))]
    dist.all_gather(alls, mine, group=group)
    got = torch.stack(alls).cpu()
    return bool(got[:, 0].min().item() == 1 and (got[:, 1] == got[0, 1]).all().item())


def peer_wanted(engine):
    """Peer path: dense fp32 tensor-core engine, NCCL group, not disabled."""
    import os

    if os.environ.get("NMFB_DIST_PEER", "1") == "0":
        return False
    if not (dist.is_initialized() and dist.get_backend() == "nccl"):
        return False
    return bool(engine.ysplit and getattr(engine.st, "use_tc", False))


class _StateView:
    """Gives bench.py the same surface as device.Alternation."""

    def __init__(self, da, st):
        self.da = da
        self.st = st
        self.pieces = st.pieces
        self.splits_e = getattr(st, "splits_e", 1)
        self.splits_m = getattr(st, "splits_m", 1)

    def iterate(self, k):
        self.da.iterate(k)

    def join(self):
        fin = getattr(self.da.e, "finish", None)
        if fin is not None:
            fin()
        self.st.join()

    def assemble(self, *a, **kw):
        return self.st.assemble(*a, **kw)
