"""Benchmark of the alternating-NNLS hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 2|3|4|5]

Default workload (BASELINE.json configs[4], "C5", the config its metric is
quoted on "at 1/2/4/8 B200"): sparse text-like NMF, X 1000000 x 200000 CSC at
0.05% density (Zipf rows/columns, tf-idf-scaled Poisson counts, seed 4),
rank 200, fp32 on the GPU.  One step = one outer iteration of nmf.fit (Gram +
rescale, G^T X, NNLS over the 200000 columns, F F^T, X F^T, NNLS over the
1000000 rows, objective by the trace identity), i.e. 1.2 M column/row NNLS
solves.  ``value`` = solves/s over the timed steps with X and the factors
resident in HBM; ``e2e`` = the same metric through the public ``fit()`` call
from the reference's own host input (a float64 SparseMatrix / ndarray):
upload, device CSR build, seeded init, the config's iterations, download of
G, F and the log, all inside the timed region.

--config 3|5 (sparse) at N > 1: strong scaling -- the config's matrix is
split into the shard plan's 32-aligned column blocks (BASELINE: "columns
sharded across 1/2/4/8 GPUs").  --config 2|4 (dense) at N > 1: weak scaling
-- every rank owns a config-shaped column block (G replicated; the r x r Gram
allreduce, the Y^T reduce-scatter and the G allgather as NVLink peer stores
or NCCL; paper_1506_08938_b200/dist.py).

``--impl reference``: the reference's CPU path on this host's cores -- the
oracle port (oracle/, a C + numpy restatement bit-exact to the reference),
multithreaded like the reference's shard workers, on the same config.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

N_ROWS, N_COLS, RANK, SEED = 10000, 20000, 50, 1
WORKLOAD = "C2: dense NMF 10000x20000, rank 50, fp32 (BASELINE.json configs[1])"
WORKLOADS = {
    2: WORKLOAD,
    3: "C3: sparse text-like NMF 100000x50000 CSC 0.1%, rank 100, fp32 (BASELINE.json configs[2])",
    4: "C4: dense L1/L2-regularised NMF 20000x20000, rank 64, mu1=0.1, beta2=0.01, fp32 "
       "(BASELINE.json configs[3])",
    5: "C5: sparse text-like NMF 1000000x200000 CSC 0.05%, rank 200, fp32 (BASELINE.json "
       "configs[4])",
}
# bounded CPU-baseline samples: outer iterations of the oracle port per config
# (~10-25 s of host work on a 16-core box)
CPU_SAMPLE_ITERS = {2: 4, 3: 12, 4: 2, 5: 1}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--config", type=int, default=5, choices=[2, 3, 4, 5],
                   help="BASELINE.json config (default 5 = configs[4], the largest config, "
                        "on which the metric is quoted at 1/2/4/8 GPUs)")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_block(rank, cid=2):
    """This rank's column block: dense configs are weak-scaled (every rank a
    config-shaped block, seeds differ per rank; float64 host, (n, m) Fortran);
    sparse configs are the config's full CSC (N = 1)."""
    from oracle import generators

    c = generators.CONFIGS[cid]
    if c["kind"] == "sparse":
        x, _ = generators.make(cid)
        return x
    n, m = c["shape"]
    seed = SEED if rank == 0 else SEED + 1000 * rank
    return np.asfortranarray(generators.dense_exp(n, m, c["rank"], 0.05, seed))


def config_knobs(cid):
    """NmfConfig keywords of a BASELINE config (rank, seed, penalties)."""
    from oracle import generators

    return dict(generators.CONFIGS[cid]["cfg"])


class Clocks:
    """SM clock + throttle reasons sampled DURING the timed region (the
    recipe's clocks line): NVML polled every ~1 ms from a thread while the
    steps run (nvidia-smi's 100 ms loop would miss a 15 ms region); falls back
    to nvidia-smi if NVML is unavailable."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
               ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4))

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.nvml = None

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.halt = False
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _poll(self):
        nv = self.nvml
        while not self.halt:
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((sm, rs))
            except Exception:
                pass
            time.sleep(0.001)

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.nvml is not None:
            self.halt = True
            self.thread.join(timeout=2)
            sm = [float(r[0]) for r in self.rows]
            reasons = sorted({nm for _, rs in self.rows for nm, bit in self.REASONS if rs & bit})
            return {"sm_mhz": statistics.median(sm) if sm else None,
                    "sm_max_mhz": float(self.max_sm), "reasons": reasons,
                    "samples": len(sm), "source": "nvml"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) > 8:
                for nm, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi"}


def peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6552.6), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def micro_peaks():
    """CUDA-core FMA and L2 read peaks measured on a B200 by tests/micro
    (profiles/r02_micro_peaks.json); spec-derived fallbacks otherwise."""
    path = os.path.join(REPO, "profiles", "r02_micro_peaks.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return (float(d["ffma_tflops"]), float(d["l2_stream_read_gbs"]),
                "measured (tests/micro/fma_peak.cu, l2_bw.cu; profiles/r02_micro_peaks.json)")
    except (OSError, ValueError, KeyError):
        return 148 * 128 * 2 * 1965e6 / 1e12, None, "spec-derived (148 SM x 128 FMA x 2 x 1965 MHz)"


def profile_traffic(cid, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` at
    config `cid` from the committed ncu --set full captures
    (profiles/traffic_r*.json, newest round first: {"C5": {kernel: {...}}}),
    or None."""
    import glob

    for path in sorted(glob.glob(os.path.join(REPO, "profiles", "traffic_r*.json")),
                       reverse=True):
        try:
            with open(path) as f:
                k = json.load(f).get(f"C{cid}", {}).get(kernel)
        except (OSError, ValueError):
            continue
        if k is not None:
            return int(k["dram_bytes_read"]) + int(k["dram_bytes_write"])
    return None


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def st_inner(st, k0, k1):
    """Inner NNLS iterations of steps [k0, k1) from the device stats."""
    stats = getattr(st, "stats", None)
    if stats is None:
        stats = getattr(getattr(st, "st", None), "stats", None)
    if stats is None:
        return 0
    return int(stats[k0:k1, :, 0].sum().item())


def run_ours(args):
    import torch

    from paper_1506_08938_b200 import NmfConfig, _lib
    from paper_1506_08938_b200 import device as D
    from paper_1506_08938_b200.nmf import FitSession, initial_factors_from_mean

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    use_dist = "WORLD_SIZE" in os.environ  # torchrun: NCCL path even at 1 rank
    if use_dist:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cid = args.config
    X = make_block(rank, cid)
    sparse = not isinstance(X, np.ndarray)
    m_total = None
    # sparse configs under torchrun: strong scaling.  Default: the ROW-sharded
    # layout for n > m (dist_rows.py; each rank keeps its 32-aligned row block,
    # panels of r x m move); NMFB_DIST_LAYOUT=cols: the column-sharded DistFit
    rows_layout = sparse and os.environ.get("NMFB_DIST_LAYOUT", "rows") != "cols"
    if sparse:
        from paper_1506_08938_b200 import dist as PDm
        from paper_1506_08938_b200.matrix import SparseMatrix

        n, m_total = X.rows, X.cols
        xmean = float(X.values.sum()) / (n * m_total)
        xsq_total = float(X.values @ X.values)
        full = SparseMatrix(X.rows, X.cols, X.indptr, X.indices, X.values, validate=False)
        if use_dist and not rows_layout:
            lo, hi = PDm.ShardPlan(n, m_total, world).col_range(rank)
            X = PDm.csc_column_block(X, lo, hi)
        else:
            X = full
        m = X.cols
    else:
        n, m = X.shape
        xmean = float(X.mean())
    knobs = config_knobs(cid)
    R = knobs["rank"]
    # iteration slots: warm-up, the timed steps, then the same number of
    # instrumented steps (per-kernel CUDA events) for the kernel shares
    cfg = NmfConfig(max_outer=args.warmup + 2 * args.steps, rel_change_tol=0.0,
                    precision="fp32", **knobs)
    mt = m_total if sparse else m * world
    G0, FT0 = initial_factors_from_mean(n, mt, xmean, cfg)
    if use_dist and rows_layout:
        from paper_1506_08938_b200.dist_rows import RowShardedFit

        sess = RowShardedFit(X, cfg, init=(G0, FT0))
        st = sess.state
        rlo, rhi = sess.plan.row_range(rank)
        clo, chi = sess.plan.col_range(rank)
        n_solve, m_solve = rhi - rlo, chi - clo  # this rank's solves
    elif use_dist:
        from paper_1506_08938_b200 import dist as PD

        clo, chi = PD.ShardPlan(n, mt, world).col_range(rank)
        FT0 = FT0[clo:chi]
        sess = PD.DistFit(X, cfg, init=(G0, FT0), m_total=mt)
        st = sess.state
        n_solve, m_solve = n / world, m
    else:
        sess = FitSession(X, cfg, init=(G0, FT0))
        st = sess.state
        n_solve, m_solve = n, m
    torch.cuda.synchronize()

    def barrier():
        if use_dist:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for k in range(args.warmup):
        st.iterate(k)
    st.join()
    barrier()
    clocks = Clocks(local)
    clocks.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    # timed steps: launch counting, and CUDA events around the roofline
    # kernels' calls only (data products, NNLS) -- their live launch durations
    # (NNLS too on sparse configs, where it is the dominant kernel; on dense
    # ones its ~10 us event pairs would be ~3% of a 0.8 ms step, so its
    # roofline uses the serialised instrumented pass below)
    gemm_names = {"nmfb_tc_gemm", "nmfb_tc_gemm_rows", "nmfb_gemm_tall", "nmfb_csc_linear",
                  "nmfb_csc_linear_blocked", "nmfb_csr_yt_chunked", "nmfb_csr_yt_chunked_blocked"}
    if sparse:
        gemm_names |= {"nmfb_nnls_batch", "nmfb_nnls_batch_peers"}
    with _lib.Recorder(timing=gemm_names) as cnt:
        t0.record()
        for k in range(args.warmup, args.warmup + args.steps):
            st.iterate(k)
        st.join()  # the last objective runs on a side stream
        t1.record()
    barrier()
    clk = clocks.stop()
    ms = t0.elapsed_time(t1)
    # the same number of steps again, SERIALISED (the objective on the main
    # stream, no side-stream overlap) with a CUDA event pair around every
    # C-ABI call: per-kernel durations and shares of the step that add up
    # (these steps are not the timed ones)
    for obj in (st, getattr(st, "st", None)):
        if obj is not None:
            obj.serial = True
    with _lib.Recorder(timing=True) as rec:
        i0 = torch.cuda.Event(enable_timing=True)
        i1 = torch.cuda.Event(enable_timing=True)
        i0.record()
        for k in range(args.warmup + args.steps, args.warmup + 2 * args.steps):
            st.iterate(k)
        st.join()
        i1.record()
    torch.cuda.synchronize()
    for obj in (st, getattr(st, "st", None)):
        if obj is not None:
            obj.serial = False
    ms_instr = i0.elapsed_time(i1)
    if use_dist:
        tt = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = float(tt.item())
    ms_per_step = ms / args.steps
    solves_step = (mt + n)  # per step, all ranks
    value = solves_step * args.steps / (ms / 1e3)
    calls = rec.summary()
    hbm, peak_src = peaks()
    ffma_tf, l2_gbs, micro_src = micro_peaks()
    live = cnt.summary()  # data-product launches inside the timed region
    kernels = {}
    for name, (c, t) in calls.items():
        kernels[name] = {"launches": c, "avg_ms": t / c, "share": round(t / ms_instr, 4)}
    share = {k: round(v[1] / ms_instr, 4) for k, v in calls.items()}
    # inner iterations of the timed steps -> k-bar for the NNLS flop count
    inner = st_inner(st, args.warmup, args.warmup + args.steps)
    kbar = inner / ((m_solve + n_solve) * args.steps) if inner else 1.0
    rooflines = {}
    if not sparse:
        gname = "nmfb_tc_gemm" if "nmfb_tc_gemm" in calls else "nmfb_gemm_tall"
        gemm_calls, gemm_ms = live.get(gname, (0, 0.0))
        if "nmfb_tc_gemm_rows" in live:  # multi-GPU peer path: X F^T stores into the owners
            c2, t2 = live["nmfb_tc_gemm_rows"]
            gemm_calls, gemm_ms = gemm_calls + c2, gemm_ms + t2
        # algorithmic bytes per data-product launch, averaged over the two
        # passes (G^T X: A = X^T, K = n; X F^T: A = X, K = m): X once and the
        # small factor's hi/lo splits (the split-K partial writes are the
        # kernel's own scratch, not algorithmic)
        gemm_bytes = 4.0 * (n * m + 2 * R * (n + m) / 2.0)
        gemm_avg_ms = gemm_ms / max(gemm_calls, 1)
        achieved = gemm_bytes / (gemm_avg_ms / 1e3) / 1e9 if gemm_avg_ms > 0 else 0.0
        rooflines["data_products"] = {
            "kernel": gname + " (G^T X and X F^T passes over X; tcgen05 3xTF32)",
            "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "peak_source": peak_src,
            "algorithmic_bytes_per_launch": gemm_bytes, "avg_launch_ms": gemm_avg_ms,
            "timed": "live CUDA events in the timed steps",
            "traffic": profile_traffic(cid, gname), "share": share.get(gname)}
    else:
        # compulsory bytes of one SpMM pass: values + indices once,
        # the pointer array, both factors read/written once; the factor-row
        # gathers (4 nnz r bytes) are served by L2 -> their roof is the
        # measured L2 read bandwidth
        nnz = X.nnz
        names = ("nmfb_csc_linear", "nmfb_csc_linear_blocked", "nmfb_csr_yt_chunked",
                 "nmfb_csr_yt_chunked_blocked")
        sp_bytes = 8.0 * nnz + 8.0 * (m + 1) + 4.0 * (n + m) * R
        sp_calls = sum(live.get(k, (0, 0.0))[0] for k in names)
        sp_ms = sum(live.get(k, (0, 0.0))[1] for k in names)
        sp_avg = sp_ms / max(sp_calls, 1)
        ach = sp_bytes / (sp_avg / 1e3) / 1e9 if sp_avg > 0 else 0.0
        gbytes = 4.0 * nnz * R
        gach = gbytes / (sp_avg / 1e3) / 1e9 if sp_avg > 0 else 0.0
        rooflines["data_products"] = {
            "kernel": "nmfb_csc_linear[_blocked] + nmfb_csr_yt_chunked (G^T X and X F^T, "
                      "CSC / CSR SpMM with 16-byte factor-row gathers)",
            "bound": "l2" if l2_gbs else "hbm",
            "achieved": gach if l2_gbs else ach, "peak": l2_gbs or hbm, "unit": "GB/s",
            "frac": (gach / l2_gbs) if l2_gbs else ach / hbm,
            "peak_source": micro_src if l2_gbs else peak_src,
            "algorithmic_bytes_per_launch": gbytes, "avg_launch_ms": sp_avg,
            "timed": "live CUDA events in the timed steps",
            "compulsory_bytes_per_launch": sp_bytes, "compulsory_GBps": ach,
            "compulsory_frac_of_hbm": ach / hbm, "hbm_peak": hbm,
            "traffic": profile_traffic(cid, "nmfb_csr_yt_chunked"),
            "share": round(sum(share.get(k, 0.0) for k in names), 4),
            "note": "algorithmic bytes = the factor-row gathers (4 nnz r per pass; every "
                    "nonzero reads its r-row), against the measured L2 read bandwidth"}
    nn_names = ("nmfb_nnls_batch", "nmfb_nnls_batch_peers")
    nn_src = live if sparse else calls
    c = sum(nn_src.get(k, (0, 0.0))[0] for k in nn_names)
    t = sum(nn_src.get(k, (0, 0.0))[1] for k in nn_names)
    if c:
        # 2 r^2 (1 + 2 k) flops per solve (gradient init, Q d per
        # inner iteration, r coordinate-descent column updates per iteration)
        fl = 2.0 * R * R * (1 + 2 * kbar) * (m_solve + n_solve)  # this rank's solves
        nn_ms = t / args.steps  # both NNLS launches of one step
        ach = fl / (nn_ms / 1e3) / 1e12
        # E-only / M-only rates: the step's two NNLS launches in order
        src_rec = cnt if sparse else rec
        seq = [a.elapsed_time(b) for nm, a, b in src_rec.calls if nm in nn_names]
        e_ms = sum(seq[0::2]) / max(len(seq[0::2]), 1)
        m_ms = sum(seq[1::2]) / max(len(seq[1::2]), 1)
        rooflines["nnls"] = {
            "kernel": "nmfb_nnls_batch (E + M solves of one step)", "bound": "fp32",
            "e_step_ms": e_ms, "m_step_ms": m_ms,
            "e_solves_per_s": m_solve / (e_ms / 1e3) if e_ms else None,
            "m_solves_per_s": n_solve / (m_ms / 1e3) if m_ms else None,
            "achieved": ach, "peak": ffma_tf, "unit": "TFLOP/s", "frac": ach / ffma_tf,
            "peak_source": micro_src, "algorithmic_flops_per_step": fl, "k_bar": kbar,
            "ms_per_step": nn_ms, "avg_launch_ms": nn_ms / 2, "share":
                round(sum(share.get(k, 0.0) for k in nn_names), 4),
            "timed": ("live CUDA events in the timed steps" if sparse else
                      "serialised instrumented steps (CUDA events around each call)"),
            "traffic": profile_traffic(cid, "nmfb_nnls_batch"),
            "note": "FMA-counted; the greedy-CD argmax (r compares + a tree per selection) "
                    "and the shuffles are not counted -- issue-slot utilisation is in "
                    "profiles/ (ncu smsp__issue_active)"}
    # Gram products (G^T G over n rows, F F^T over m rows): one read of the
    # factor each, from the serialised instrumented steps
    gr_names = ("nmfb_gram", "nmfb_gram_rescale")
    gc = sum(calls.get(k, (0, 0.0))[0] for k in gr_names)
    gt = sum(calls.get(k, (0, 0.0))[1] for k in gr_names)
    if gc:
        g_bytes = 4.0 * R * (n_solve + m_solve) / 2.0  # per launch, averaged over the two
        g_avg = gt / gc
        g_ach = g_bytes / (g_avg / 1e3) / 1e9
        tc_gram = R % 4 == 0 and 16 <= R <= 224 and os.environ.get("NMFB_GRAM_TC", "1") != "0"
        rooflines["gram"] = {
            "kernel": ("gram_tc_kernel (tcgen05 3xTF32, MN-major operands from one TMA tile) + "
                       "fused reduce/rescale" if tc_gram else
                       "gram_partial_kernel (fp32 slabs folded to fp64) + fused reduce/rescale"),
            "bound": "hbm", "achieved": g_ach, "peak": hbm, "unit": "GB/s", "frac": g_ach / hbm,
            "peak_source": peak_src, "algorithmic_bytes_per_launch": g_bytes,
            "avg_launch_ms": g_avg, "timed": "serialised instrumented steps (CUDA events "
            "around each call, both Gram launches of a step averaged)",
            "traffic": profile_traffic(cid, "nmfb_gram_tc" if tc_gram else "nmfb_gram"),
            "share": round(sum(share.get(k, 0.0) for k in gr_names), 4),
            "note": "tensor pipe 61% active (ncu, profiles/r02_ncu_gram_tc.ncu-rep): bound by "
                    "the ~77 ns issue cost of a tcgen05.mma, 6 per 8 factor rows"
                    if tc_gram else None}
    # the dominant kernel: the largest share of the serialised step
    dom = max(rooflines.items(), key=lambda kv: kv[1].get("share") or 0.0)
    # log sanity: objective decreasing
    pieces = st.pieces[: args.warmup + args.steps].cpu().numpy()
    xsq = xsq_total if sparse else 0.0
    objs = [st.assemble(p, cfg, "sparse" if sparse else "dense", xsq) for p in pieces]
    result = {
        "metric": "column NNLS solves/sec (NMF outer iteration: E+M steps + objective)",
        "value": value,
        "unit": "solves/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "outer_iters_per_sec": 1e3 / ms_per_step,
        "higher_is_better": True,
        "scaling": "strong" if sparse else "weak",
        "vs_baseline": None,
        "dtype": "fp32",
        "data": f"synthetic (seeded generator oracle/generators.py, BASELINE C{cid} shape)",
        "config": config_dict(cid, n, mt),
        "setup": {"m_per_gpu": m, "solves_per_step": solves_step,
                  "step": "one outer iteration of fit(): gram+rescale, G^T X, NNLS(m cols), "
                          "F F^T, X F^T, NNLS(n rows), objective",
                  "l2": ("inputs larger than L2 (X fp32 = %.0f MB per GPU >> 126 MB)"
                         % (n * m * 4 / 1e6)) if not sparse else
                        ("inputs larger than L2 (CSC + CSR of X = %.0f MB, factors %.0f MB)"
                         % (16 * X.nnz / 1e6, 4 * (n + m) * R / 1e6)),
                  "parallelism": (f"dp{world} (row-sharded for n > m: row blocks of X and G "
                                  f"per rank, F replicated; dist_rows.py)" if rows_layout else
                                  f"dp{world} (column-sharded; "
                                  + ("the config's matrix split across ranks)" if sparse
                                     else "a config-shaped block per rank)")),
                  "exchange": ("nvlink peer stores from the producing kernels"
                               if getattr(sess, "peer", False) else
                               ("nccl" if use_dist else "none")),
                  "exchange_bytes_per_rank": (sess.plan.exchange_bytes(R)
                                              if use_dist and rows_layout else None)},
        "roofline": dict(dom[1], name=dom[0]),
        "rooflines": rooflines,
        "step_share": share,
        "kernels": kernels,
        "dominant": dom[0],
        "clocks": clk,
        "gpu_launches": cnt.launches,
        "instrumented_ms_per_step": ms_instr / args.steps,
        "objective_first_last": [objs[0], objs[-1]],
    }
    if rank == 0 and world == 1 and not args.no_e2e:
        result["e2e"] = run_e2e(args, X, cfg)
    if rank == 0 and world == 1 and not args.no_cpu:
        result["cpu_baseline"] = cpu_baseline(X, cid)
    if use_dist:
        torch.distributed.destroy_process_group()
    return result if rank == 0 else None


def config_dict(cid, n, m):
    """The `config` of both arms' lines (identical keys, so the driver can
    pair them)."""
    from oracle import generators

    c = generators.CONFIGS[cid]
    return {"workload": WORKLOADS[cid], "config_id": cid, "n": n, "m": m,
            "rank": c["rank"], "kind": c["kind"]}


def run_e2e(args, X, cfg):
    """Public fit() from the reference's own host input type, as a user of the
    reference calls it: a float64 (n, m) ndarray for dense configs
    (DenseMatrix's array; the host fp32 cast and the pageable upload are
    inside the timed region), the float64 / int64 SparseMatrix CSC for sparse
    ones (upload, index narrowing and the device CSR build inside); seeded
    init, the config's own number of outer iterations (BASELINE.json: C2/C4
    100, C3 50, C5 30), D2H of factors and log.  Dense configs also report the
    pinned fp32 torch-input leg."""
    import torch

    from oracle import generators
    from paper_1506_08938_b200 import NmfConfig, fit
    from paper_1506_08938_b200.matrix import SparseMatrix

    knobs = config_knobs(args.config)
    R = knobs["rank"]
    K = generators.CONFIGS[args.config]["iters"]
    ecfg = NmfConfig(max_outer=K, rel_change_tol=0.0, precision="fp32", **knobs)
    wcfg = NmfConfig(max_outer=2, rel_change_tol=0.0, precision="fp32", **knobs)

    def timed(V):
        # warm-up: one short fit and one with the timed call's own
        # configuration -- the allocator's block cache, the pinned staging and
        # log buffers (sized by max_outer) and the ingest scratch pool only
        # settle during the second call of a process and the first call with
        # this iteration count (~60 ms at C5, ~80 ms at C3 otherwise)
        fit(V, wcfg)
        fit(V, ecfg)
        torch.cuda.synchronize()
        t = time.perf_counter()
        model, log = fit(V, ecfg)
        torch.cuda.synchronize()
        return time.perf_counter() - t, log

    out = {}
    if isinstance(X, SparseMatrix):
        n, m = X.rows, X.cols
        h2d = 8 * (m + 1) + 16 * X.nnz
        dt, log = timed(X)
        call = f"fit(SparseMatrix float64/int64 CSC host arrays, max_outer={K})"
    else:
        n, m = X.shape
        h2d = n * m * X.dtype.itemsize  # the float64 bytes cross the link; cast on device
        dt, log = timed(X)  # the (n, m) float64 array, as DenseMatrix holds it
        call = f"fit(float64 (n,m) ndarray, max_outer={K})"
        XT = torch.from_numpy(np.ascontiguousarray(X.T, dtype=np.float32)).pin_memory()
        dt_p, _ = timed(XT.t())
        out["pinned_fp32_leg"] = {"value": (n + m) * K / dt_p, "unit": "solves/s",
                                  "seconds": dt_p,
                                  "call": f"fit(pinned torch (n,m) fp32 view, max_outer={K})"}
    d2h = (n + m) * R * 8 + K * (12 * 8 + 4 * 8)
    out.update({"value": (n + m) * K / dt, "unit": "solves/s",
                "h2d_bytes_per_step": h2d / K, "d2h_bytes_per_step": d2h / K,
                "steps": K, "seconds": dt, "call": call,
                "final_objective": log.final_objective})
    return out


# ---------------------------------------------------------------------------
# reference arm / cpu baseline: the oracle port on this host's cores
# ---------------------------------------------------------------------------
def cpu_baseline(X, cid):
    """The oracle port (bit-exact restatement of the reference: C kernels +
    numpy/OpenBLAS, one shard worker per host core) on a bounded sample of
    the same workload: CPU_SAMPLE_ITERS[cid] outer iterations of the full
    config matrix from the seeded init."""
    from oracle import nmf_oracle as orc
    from paper_1506_08938_b200.matrix import SparseMatrix

    cores = os.cpu_count() or 1
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(cores))
    sparse = isinstance(X, SparseMatrix)
    if sparse:
        Xo = orc.Csc(X.rows, X.cols, X.indptr, X.indices, X.values)
        n, m = X.rows, X.cols
    else:
        Xo = X
        n, m = X.shape
    iters = CPU_SAMPLE_ITERS[cid]
    knobs = config_knobs(cid)
    cfg = orc.Config(max_outer=iters, rel_change_tol=0.0, workers=cores, **knobs)
    orc.fit(np.ones((64, 64)), orc.Config(rank=4, max_outer=1, seed=0))  # load the C library
    timer = {}
    t = time.perf_counter()
    orc.fit(Xo, cfg, step_timer=timer, chunked_objective=sparse)
    dt = time.perf_counter() - t
    return {"value": (n + m) * iters / dt, "unit": "solves/s", "cores": cores, "kind": "port",
            "sample": f"{iters} outer iteration(s) of the full C{cid} workload ({n}x{m}, "
                      f"r={knobs['rank']}) in float64 by the oracle port (C kernels + "
                      f"numpy/OpenBLAS, {cores} shard threads), objective included",
            "seconds": dt, "em_only_solves_per_s": (n + m) * iters / timer["em_seconds"]}


def run_reference(args):
    """The reference's CPU path (the oracle port: C kernels restating the
    numba shard kernels + numpy/OpenBLAS, as many shard threads as host
    cores) on this arm's config; one step = one outer iteration, the state
    carried between steps.  Sparse configs use the port's threaded C nnz loop
    for the objective's cross term (same formula, matrix.py:240-253) and, at
    config 5 (~22 s per iteration on 16 threads), run at most 2 timed steps
    after no warm-up so the run stays within minutes."""
    world, rank, _ = dist_env()
    if rank != 0:
        return None
    cid = args.config
    X = make_block(0, cid)
    sparse = not isinstance(X, np.ndarray)
    n, m = (X.rows, X.cols) if sparse else X.shape
    from oracle import nmf_oracle as orc

    cores = os.cpu_count() or 1
    knobs = config_knobs(cid)
    steps, warmup = args.steps, args.warmup
    if cid == 5:
        steps, warmup = min(steps, 2), 0
    elif cid in (2, 4):
        steps, warmup = min(steps, 5), min(warmup, 1)
    cfg = orc.Config(max_outer=1, rel_change_tol=0.0, workers=cores, **knobs)
    orc.fit(np.ones((64, 64)), orc.Config(rank=4, max_outer=1, seed=0))  # load the C library
    G, FT = orc.initial_factors(X, cfg)
    times = []
    for k in range(warmup + steps):
        t = time.perf_counter()
        G, FT, _ = orc.fit(X, cfg, init=(G, FT), chunked_objective=sparse)
        times.append(time.perf_counter() - t)
    dt = sum(times[warmup:])
    value = (n + m) * steps / dt
    mt = m * world if not sparse else m
    return {"impl": "reference", "metric": "column NNLS solves/sec (NMF outer iteration: "
            "E+M steps + objective)", "value": value, "unit": "solves/s", "n_gpus": world,
            "steps": steps, "warmup": warmup, "ms_per_step": dt / steps * 1e3,
            "higher_is_better": True, "scaling": "strong" if sparse else "weak",
            "vs_baseline": None, "dtype": "fp64",
            "data": "synthetic (same generator as our arm)",
            "config": config_dict(cid, n, mt),
            "cpu_baseline": {"value": value, "unit": "solves/s", "cores": cores, "kind": "port",
                             "sample": f"{steps} outer iterations of C{cid} (after {warmup} "
                                       f"warm-up), oracle port, {cores} threads"},
            "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    res = run_reference(args) if args.impl == "reference" else run_ours(args)
    if res is not None:
        print(json.dumps(res))


if __name__ == "__main__":
    main()
