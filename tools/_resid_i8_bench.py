"""Micro-benchmark: int8 tensor-core residual vs the FFMA residual at C2 shapes."""
import sys, torch
sys.path.insert(0, '.')
from paper_1506_08938_b200 import _lib as L
from paper_1506_08938_b200 import device as D
dev = D.require_cuda()
n, m, r = 10000, 20000, 50
X = torch.rand((n, m), device=dev)
XT = X.t().contiguous()
G = torch.rand((n, r), device=dev); FT = torch.rand((m, r), device=dev)
Gt = G.t().contiguous(); Ft = FT.t().contiguous()
Gsl = torch.zeros((L.lib().nmfb_slice_bytes(n, r),), dtype=torch.uint8, device=dev)
Fsl = torch.zeros((L.lib().nmfb_slice_bytes(m, r),), dtype=torch.uint8, device=dev)
out = torch.zeros(2, dtype=torch.float64, device=dev)
ws = torch.empty((L.lib().nmfb_residual_workspace_bytes(m, n) // 8 + 1,), dtype=torch.float64, device=dev)
ws8 = torch.empty((L.lib().nmfb_residual_i8_workspace_bytes() // 8 + 1,), dtype=torch.float64, device=dev)
def slices():
    L.call("nmfb_slice_u8", D.vp(G), n, r, r, D.vp(Gsl), D.stream_handle())
    L.call("nmfb_slice_u8", D.vp(FT), m, r, r, D.vp(Fsl), D.stream_handle())
def i8():
    L.call("nmfb_residual_i8", D.vp(X), n, m, D.vp(Gsl), D.vp(Fsl), r, D.vp(out[0:1]), D.vp(ws8), D.stream_handle())
def ffma():
    L.call("nmfb_dense_residual_kmajor", D.vp(XT), m, n, D.vp(Gt), D.vp(Ft), r, D.vp(out[1:2]), D.vp(ws), D.stream_handle())
def timeit(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
print(f"slices   {timeit(slices):.4f} ms")
print(f"i8       {timeit(i8):.4f} ms  {n*m*4/timeit(i8)/1e6:.0f} GB/s of X")
print(f"ffma     {timeit(ffma):.4f} ms")
out.zero_(); i8(); ffma(); torch.cuda.synchronize()
print("values", out.tolist(), "rel diff", abs(out[0]-out[1]).item()/out[1].item())
