"""Dev check: tensor-core Gram (gram_tc.cu) vs the fp64 Gram of the same fp32
values -- max / mean signed relative error and time; run with NMFB_GRAM_TC=0
for the CUDA-core path."""
import os, sys, torch
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
    return a.elapsed_time(b) / reps * 1e3
shapes = [(4096, 32), (20000, 64), (50000, 100), (40000, 128), (65536, 160), (200000, 200), (1000000, 200), (30001, 224), (5000, 16)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in s.split('x')) for s in sys.argv[1:]]
print("NMFB_GRAM_TC =", os.environ.get("NMFB_GRAM_TC", "1"))
for rows, r in shapes:
    torch.manual_seed(rows + r)
    A = torch.rand((rows, r), device=dev) ** 3 * (torch.rand((1, r), device=dev) * 10 + 0.01)
    A[:, r // 2] *= (torch.rand(rows, device=dev) < 0.05)   # a sparse column
    out = torch.zeros((r, r), dtype=torch.float64, device=dev)
    ws = torch.empty((L.lib().nmfb_gram_workspace_bytes(rows, r) // 8 + 1,), dtype=torch.float64, device=dev)
    g = lambda: L.call("nmfb_gram", L.F32, D.vp(A), rows, r, r, D.vp(out), D.vp(ws), D.stream_handle())
    g(); torch.cuda.synchronize()
    A64 = A.double()
    want = A64.T @ A64
    rel = (out - want) / want.abs().clamp_min(1e-300)
    sym = bool((out == out.T).all())
    t = timeit(g)
    print(f"rows={rows} r={r}: max|rel| {rel.abs().max().item():.2e} mean rel {rel.mean().item():+.2e} "
          f"sym {sym}  {t:.1f} us  ({rows*r*4/t/1e3:.0f} GB/s)", flush=True)
