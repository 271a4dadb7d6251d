"""Micro-benchmark of the fp32 dense residual kernel at C2 shapes."""
import sys, torch
sys.path.insert(0, '.')
from paper_1506_08938_b200 import _lib as L
from paper_1506_08938_b200 import device as D
dev = D.require_cuda()
m, n, r = 20000, 10000, 50
XT = torch.rand((m, n), device=dev)
Gt = torch.rand((r, n), device=dev); Ft = torch.rand((r, m), device=dev)
out = torch.zeros(1, dtype=torch.float64, device=dev)
ws = torch.empty((L.lib().nmfb_residual_workspace_bytes(m, n) // 8 + 1,), dtype=torch.float64, device=dev)
def run():
    L.call("nmfb_dense_residual_kmajor", D.vp(XT), m, n, D.vp(Gt), D.vp(Ft), r, D.vp(out), D.vp(ws), D.stream_handle())
run(); torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): run()
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 10
print(f"residual {ms:.3f} ms  {2*m*n*r/ms/1e9:.1f} TFLOP/s")
