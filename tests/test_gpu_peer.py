"""Multi-GPU exchange over peer memory (csrc/peer.cu, RowOut in tc_gemm.cu,
the NNLS mirror stores), checked on one GPU.

The rounds' boxes have a single GPU, so the multi-rank ADDRESSING is checked
by simulating the ranks inside one process: every simulated rank's buffers
live on the same device and the producers run one after another (no kernel
waits on another rank's kernel -- the signal of every simulated rank is
issued before any wait).  The layout must be bit-exact: the same kernel and
schedule write the same bits, only to a different place.  The full
torchrun path (symmetric memory rendezvous, epochs, world-1 NCCL group) runs
in a subprocess and must reproduce the single-GPU fit bit for bit."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_1506_08938_b200 import _lib as L
    from paper_1506_08938_b200 import device as D

    return L, D


def _split(L, D, B):
    K, N = B.shape
    dev = D.require_cuda()
    b = torch.from_numpy(np.ascontiguousarray(B, dtype=np.float32)).to(dev)
    hi = torch.empty((N, K), dtype=torch.float32, device=dev)
    lo = torch.empty((N, K), dtype=torch.float32, device=dev)
    L.call("nmfb_split_transpose", D.vp(b), K, N, D.vp(hi), D.vp(lo), D.stream_handle())
    return hi, lo


@pytest.mark.parametrize("M,Kb,N,world", [(1000, 2048, 50, 3), (10000, 4000, 50, 4),
                                           (777, 1024, 64, 2), (1000, 1536, 100, 3),
                                           (4096, 1024, 20, 8)])
def test_tc_gemm_rows_peer_layout_bit_exact(M, Kb, N, world):
    """Each simulated source rank s multiplies its own column block; its
    partial slot p of row i must land at owner o = i // chunk, slot
    s * P + p, row i - o * chunk -- bit-identical to the plain layout."""
    L, D = _lib()
    dev = D.require_cuda()
    rng = np.random.default_rng(M + N + world)
    chunk = -(-M // world // 32) * 32
    while chunk * world < M:
        chunk += 32
    P = L.lib().nmfb_tc_parts(M, Kb, N, 0)
    recv = [torch.full((world * P * chunk * N,), float("nan"), dtype=torch.float32, device=dev)
            for _ in range(world)]
    dst = L.ptr_array([t.data_ptr() for t in recv])
    plain = []
    for s in range(world):
        A = torch.from_numpy(rng.exponential(size=(M, Kb)).astype(np.float32)).to(dev)
        hi, lo = _split(L, D, rng.uniform(size=(Kb, N)))
        C = torch.full((P, M, N), float("nan"), dtype=torch.float32, device=dev)
        L.call("nmfb_tc_gemm", D.vp(A), M, Kb, D.vp(hi), D.vp(lo), N, D.vp(C), 0, 0,
               D.stream_handle())
        L.call("nmfb_tc_gemm_rows", D.vp(A), M, Kb, D.vp(hi), D.vp(lo), N, 0, dst, world, chunk,
               s, D.stream_handle())
        plain.append(C)
    torch.cuda.synchronize()
    for o in range(world):
        rows = min(M, (o + 1) * chunk) - o * chunk
        got = recv[o].view(world * P, chunk, N)
        for s in range(world):
            for p in range(P):
                a = got[s * P + p, :rows]
                b = plain[s][p, o * chunk: o * chunk + rows]
                assert torch.equal(a, b), (o, s, p)
        # rows past M in the last chunk are never written
        if rows < chunk:
            assert torch.isnan(got[:, rows:]).all()


def test_tc_gemm_rows_rejects_bad_layout():
    L, D = _lib()
    dev = D.require_cuda()
    A = torch.zeros((256, 64), dtype=torch.float32, device=dev)
    hi = torch.zeros((16, 64), dtype=torch.float32, device=dev)
    out = torch.zeros((4 * 256 * 16,), dtype=torch.float32, device=dev)
    dst = L.ptr_array([out.data_ptr()] * 2)
    with pytest.raises(ValueError):  # chunk * world < M
        L.call("nmfb_tc_gemm_rows", D.vp(A), 256, 64, D.vp(hi), D.vp(hi), 16, 0, dst, 2, 96, 0,
               D.stream_handle())
    with pytest.raises(ValueError):  # src out of range
        L.call("nmfb_tc_gemm_rows", D.vp(A), 256, 64, D.vp(hi), D.vp(hi), 16, 0, dst, 2, 128, 2,
               D.stream_handle())


@pytest.mark.parametrize("r,count", [(50, 1000), (10, 333), (64, 2048), (100, 500)])
def test_nnls_mirror_rows_equal_solution(r, count):
    """nmfb_nnls_batch_peers: the solution rows (including the x = 0
    short-circuit rows) are also stored in every mirror; the solution equals
    nmfb_nnls_batch's bit for bit."""
    L, D = _lib()
    from gpu_util import rescale

    dev = D.require_cuda()
    rng = np.random.default_rng(r + count)
    Wm = rng.uniform(size=(4 * r, r))
    H = Wm.T @ Wm
    _, _ = rescale(H, 0.0, "fp32")
    b, _ = rescale(H, 0.0, "fp32")
    h = rng.normal(size=(count, r))
    h[::7] = np.abs(h[::7])  # some all-nonnegative rows: x = 0 short-circuit
    hp = torch.from_numpy((1.0 - h).astype(np.float32)).to(dev)  # h = 1 - hp
    warm = torch.from_numpy(rng.uniform(size=(count, r)).astype(np.float32)).to(dev)
    outs = []
    for peers in (False, True):
        x = warm.clone()
        mirrors = [torch.full_like(x, float("nan")) for _ in range(3)] if peers else []
        stats = torch.tensor([0, -1], dtype=torch.int64, device=dev)
        args = [L.F32, L.MODE_FAST, D.vp(b["Qa"]), D.vp(b["sa"]), D.vp(b["act"]),
                D.vp(b["active"]), r, r, D.vp(b["ra"]), D.vp(hp), L.F32, 1, r, 0, 1.0, D.vp(x),
                count, 0, 0.1, 500, 0.0, None, None, D.vp(stats), 0]
        if peers:
            L.call("nmfb_nnls_batch_peers", *args, L.ptr_array([m.data_ptr() for m in mirrors]),
                   len(mirrors), D.stream_handle())
        else:
            L.call("nmfb_nnls_batch", *args, D.stream_handle())
        torch.cuda.synchronize()
        outs.append((x, mirrors, stats.clone()))
    (x0, _, s0), (x1, mir, s1) = outs
    assert torch.equal(x0, x1) and torch.equal(s0, s1)
    for mm in mir:
        assert torch.equal(mm, x1)
    assert (x1[::7] == 0).all()


def test_nnls_mirror_rejected_in_reference_mode():
    L, D = _lib()
    from gpu_util import rescale

    dev = D.require_cuda()
    b, _ = rescale(np.eye(4), 0.0, "fp32")
    x = torch.zeros((32, 4), dtype=torch.float32, device=dev)
    stats = torch.tensor([0, -1], dtype=torch.int64, device=dev)
    with pytest.raises(ValueError):
        L.call("nmfb_nnls_batch_peers", L.F32, L.MODE_REFERENCE, D.vp(b["Qa"]), D.vp(b["sa"]),
               D.vp(b["act"]), D.vp(b["active"]), 4, 4, D.vp(b["ra"]), D.vp(x), L.F32, 0, 4, 0,
               0.0, D.vp(x), 32, 0, 0.1, 10, 0.0, None, None, D.vp(stats), 0,
               L.ptr_array([x.data_ptr()]), 1, D.stream_handle())


@pytest.mark.parametrize("world", [1, 2, 5, 8])
def test_peer_put_signal_wait_simulated_ranks(world):
    """put -> every rank's slot; signal by every simulated rank; then every
    rank's wait returns with no timeout recorded; a wait for a future epoch
    times out (bounded) and records it instead of hanging."""
    L, D = _lib()
    dev = D.require_cuda()
    n = 37 * 2  # doubles per slot
    slots = [torch.full((world * n,), float("nan"), dtype=torch.float64, device=dev)
             for _ in range(world)]
    flags = [torch.zeros((world + 1,), dtype=torch.int64, device=dev) for _ in range(world)]
    tickets = [torch.zeros((1,), dtype=torch.int32, device=dev) for _ in range(world)]
    fptr = L.ptr_array([f.data_ptr() for f in flags])
    srcs = [torch.arange(n, dtype=torch.float64, device=dev) + 1000 * s for s in range(world)]
    for epoch in (1, 2):
        for s in range(world):
            dst = L.ptr_array([t.data_ptr() + s * n * 8 for t in slots])
            L.call("nmfb_peer_put", D.vp(srcs[s]), n * 8, dst, world, s, None, None, 0, 0,
                   D.stream_handle())
            L.call("nmfb_peer_put", None, 0, None, world, s, fptr, D.vp(tickets[s]), epoch, 1,
                   D.stream_handle())
        for s in range(world):
            L.call("nmfb_peer_wait", D.vp(flags[s]), world, epoch, 5.0, D.stream_handle())
        torch.cuda.synchronize()
        for o in range(world):
            assert flags[o][:world].tolist() == [epoch] * world
            assert int(flags[o][world]) == 0
            assert torch.equal(slots[o].view(world, n), torch.stack(srcs))
        assert all(int(t.item()) == 0 for t in tickets)
    # sum of the slots in source order
    out = torch.empty((n,), dtype=torch.float64, device=dev)
    L.call("nmfb_sum_slots_f64", D.vp(slots[0]), world, n, n, D.vp(out), D.stream_handle())
    torch.cuda.synchronize()
    assert torch.equal(out, torch.stack(srcs).sum(0))
    # bounded wait: nobody signals epoch 3
    L.call("nmfb_peer_wait", D.vp(flags[0]), world, 3, 0.05, D.stream_handle())
    torch.cuda.synchronize()
    assert int(flags[0][world]) == 3


def test_peer_put_multi_cta_ticket():
    """A large put spans many CTAs; the flag is stored once, after all."""
    L, D = _lib()
    dev = D.require_cuda()
    n = 1 << 20
    src = torch.arange(n, dtype=torch.float64, device=dev)
    dstt = [torch.zeros((n,), dtype=torch.float64, device=dev) for _ in range(2)]
    flags = [torch.zeros((3,), dtype=torch.int64, device=dev) for _ in range(2)]
    ticket = torch.zeros((1,), dtype=torch.int32, device=dev)
    for epoch in (1, 2, 3):
        L.call("nmfb_peer_put", D.vp(src), n * 8, L.ptr_array([t.data_ptr() for t in dstt]), 2, 1,
               L.ptr_array([f.data_ptr() for f in flags]), D.vp(ticket), epoch, 1,
               D.stream_handle())
        torch.cuda.synchronize()
        assert int(ticket.item()) == 0
        for f in flags:
            assert f.tolist() == [0, epoch, 0]
    for t in dstt:
        assert torch.equal(t, src)


def _torchrun(env_extra, tmp_path, tag):
    out = tmp_path / f"{tag}.json"
    env = dict(os.environ)
    env.update(env_extra)
    env["PYTHONPATH"] = REPO + os.pathsep + env.get("PYTHONPATH", "")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000),
           os.path.join(REPO, "tests", "_dist_fit_check.py"), str(out)]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    return json.loads(out.read_text())


def test_dist_world1_peer_and_nccl_paths_equal_single_gpu(tmp_path):
    """torchrun, one rank: the peer-memory path (symmetric memory, epochs),
    the NCCL path and the single-GPU fit give bit-identical factors and
    objectives."""
    peer = _torchrun({"NMFB_DIST_PEER": "1"}, tmp_path, "peer")
    nccl = _torchrun({"NMFB_DIST_PEER": "0"}, tmp_path, "nccl")
    assert peer["peer"] is True, peer.get("peer_error")
    assert nccl["peer"] is False
    for res in (peer, nccl):
        assert res["G_equal"] and res["FT_equal"], res
        assert res["obj_equal"], res


def test_dist_world1_sparse_block_equals_single_gpu(tmp_path):
    """torchrun, one rank, sparse data through DistFit(m_total=...) with the
    shard plan's CSC column block (bench.py's config 3/5 strong-scaling
    path): bit-identical to the single-GPU fit."""
    res = _torchrun({"NMFB_CHECK_SPARSE": "1", "NMFB_DIST_PEER": "0"}, tmp_path, "sparse")
    assert res["G_equal"] and res["FT_equal"] and res["obj_equal"], res


@pytest.mark.parametrize("comm", ["native", "torch"])
def test_dist_world1_row_sharded_sparse_equals_single_gpu(tmp_path, comm):
    """torchrun, one rank, the ROW-sharded layout for tall sparse data
    (dist_rows.py: Gram / H_f allreduces, reduce-scatter of the partial linear
    terms, allgather of F over NCCL -- through the C-ABI collectives
    nmfb_comm_init / allreduce_r2 / reduce_scatter_panel / allgather_panel, or
    torch.distributed's): bit-identical to the single-GPU fit."""
    res = _torchrun({"NMFB_CHECK_ROWS": "1", "NMFB_COMM": comm}, tmp_path, "rows_" + comm)
    assert res["G_equal"] and res["FT_equal"] and res["obj_equal"], res


def test_comm_c_abi_single_rank():
    """The C-ABI collectives (csrc/comm.cu) on a one-rank NCCL communicator:
    allreduce / reduce-scatter / allgather are the identity (in-place
    allgather included); argument errors are rejected."""
    import ctypes

    import numpy as np
    import torch

    from paper_1506_08938_b200 import _lib as L
    from paper_1506_08938_b200 import device as D

    dev = D.require_cuda()
    assert L.lib().nmfb_comm_available() == 1
    uid = np.zeros(128, dtype=np.uint8)
    L.call("nmfb_comm_unique_id", uid.ctypes.data_as(ctypes.c_void_p))
    comm = ctypes.c_void_p()
    L.call("nmfb_comm_init", uid.ctypes.data_as(ctypes.c_void_p), 0, 1, ctypes.byref(comm))
    try:
        a = torch.arange(40, dtype=torch.float64, device=dev)
        want = a.clone()
        L.call("nmfb_allreduce_r2", comm, D.vp(a), a.numel(), D.stream_handle())
        full = torch.randn(64, 8, device=dev)
        out = torch.empty(64, 8, device=dev)
        L.call("nmfb_reduce_scatter_panel", comm, D.vp(full), D.vp(out), out.numel(), L.F32,
               D.stream_handle())
        g = full.clone()
        L.call("nmfb_allgather_panel", comm, D.vp(g), D.vp(g), g.numel(), L.F32,
               D.stream_handle())
        torch.cuda.synchronize()
        assert torch.equal(a, want) and torch.equal(out, full) and torch.equal(g, full)
        with pytest.raises(ValueError):
            L.call("nmfb_reduce_scatter_panel", comm, D.vp(full), D.vp(out), 8, 7,
                   D.stream_handle())
    finally:
        L.call("nmfb_comm_destroy", comm)
