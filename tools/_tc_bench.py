"""Micro-benchmark: SIMT gemm_tall vs tcgen05 3xTF32 tc_gemm at C2 pass shapes."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1506_08938_b200 import _lib as L
from paper_1506_08938_b200 import device as D
dev = D.require_cuda()
def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
for (M, K, N) in [(20000, 10000, 50), (10000, 20000, 50), (20000, 20000, 64)]:
    A = torch.rand((M, K), device=dev)
    B = torch.rand((K, N), device=dev)
    Bt = torch.empty((N, K), device=dev); Btl = torch.empty((N, K), device=dev)
    L.call("nmfb_split_transpose", D.vp(B), K, N, D.vp(Bt), D.vp(Btl), D.stream_handle())
    for S in [0, 8]:
        for stages in [2, 4, 6]:
            Ss = L.lib().nmfb_tc_parts(M, K, N, S)
            C = torch.empty((Ss, M, N), device=dev)
            ms = timeit(lambda: L.call("nmfb_tc_gemm", D.vp(A), M, K, D.vp(Bt), D.vp(Btl), N, D.vp(C), S, stages, D.stream_handle()))
            print(f"tc   M={M} K={K} N={N} S={S}/{Ss} stages={stages}: {ms:.3f} ms  {M*K*4/ms/1e6:.0f} GB/s", flush=True)
    Cs = torch.empty((4, M, N), device=dev)
    ms = timeit(lambda: L.call("nmfb_gemm_tall", D.vp(A), 1, M, K, K, D.vp(B), N, N, D.vp(Cs), 4, D.stream_handle()))
    print(f"simt M={M} K={K} N={N} S=4: {ms:.3f} ms  {M*K*4/ms/1e6:.0f} GB/s", flush=True)
    ref = (A.double() @ B.double())
    Ss = L.lib().nmfb_tc_parts(M, K, N, 0)
    C = torch.empty((Ss, M, N), device=dev)
    L.call("nmfb_tc_gemm", D.vp(A), M, K, D.vp(Bt), D.vp(Btl), N, D.vp(C), 0, 0, D.stream_handle())
    torch.cuda.synchronize()
    print("  max rel err tc", float(((C.double().sum(0) - ref).abs() / ref.abs()).max()))
