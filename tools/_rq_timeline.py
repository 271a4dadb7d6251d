"""CTA-0 timeline of the int8 residual kernel (NMFB_RQ_DEBUG=64)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1506_08938_b200 import _lib as L
from paper_1506_08938_b200 import device as D
dev = D.require_cuda()
n, m, r = 10000, 20000, 50
X = torch.rand((n, m), device=dev)
G = torch.rand((n, r), device=dev); FT = torch.rand((m, r), device=dev)
Gsl = torch.zeros((L.lib().nmfb_slice_bytes(n, r),), dtype=torch.uint8, device=dev)
Fsl = torch.zeros((L.lib().nmfb_slice_bytes(m, r),), dtype=torch.uint8, device=dev)
L.call("nmfb_slice_u8", D.vp(G), n, r, r, D.vp(Gsl), D.stream_handle())
L.call("nmfb_slice_u8", D.vp(FT), m, r, r, D.vp(Fsl), D.stream_handle())
out = torch.zeros(1, dtype=torch.float64, device=dev)
ws = torch.zeros((L.lib().nmfb_residual_i8_workspace_bytes() // 8 + 1,), dtype=torch.float64, device=dev)
for _ in range(3):
    L.call("nmfb_residual_i8", D.vp(X), n, m, D.vp(Gsl), D.vp(Fsl), r, D.vp(out), D.vp(ws), D.stream_handle())
torch.cuda.synchronize()
t = ws[256:576].cpu().numpy().reshape(5, 64)
t0 = t[0, 0]
names = ["x_issue", "mma_start", "mma_issued", "epi_start", "epi_end"]
for i in range(0, 40):
    print(i, " ".join(f"{names[k]}={t[k, i] - t0:8.0f}" for k in range(5)))
def med(a): return float(np.median(a))
print("tile period (mma_start)", med(np.diff(t[1, 10:60])))
print("mma issue time", med(t[2, 10:60] - t[1, 10:60]))
print("epi duration", med(t[4, 10:60] - t[3, 10:60]))
print("mma_issued -> epi_start", med(t[3, 10:60] - t[2, 10:60]))
print("x issue -> epi_start", med(t[3, 10:60] - t[0, 10:60]))
