"""One tc_gemm launch at a C2 pass shape (for ncu captures)."""
import os, sys, torch
sys.path.insert(0, '.')
from paper_1506_08938_b200 import _lib as L
from paper_1506_08938_b200 import device as D
dev = D.require_cuda()
M, K, N = int(os.environ.get("M", 20000)), int(os.environ.get("K", 10000)), 50
S, stages = int(os.environ.get("S", 0)), int(os.environ.get("STAGES", 4))
A = torch.rand((M, K), device=dev); B = torch.rand((K, N), device=dev)
Bt = torch.empty((N, K), device=dev); Btl = torch.empty((N, K), device=dev)
L.call("nmfb_split_transpose", D.vp(B), K, N, D.vp(Bt), D.vp(Btl), D.stream_handle())
C = torch.empty((L.lib().nmfb_tc_parts(M, K, N, S), M, N), device=dev)
for _ in range(3):
    L.call("nmfb_tc_gemm", D.vp(A), M, K, D.vp(Bt), D.vp(Btl), N, D.vp(C), S, stages, D.stream_handle())
torch.cuda.synchronize()
print("ok")
