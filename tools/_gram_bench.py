"""Micro-benchmark: nmfb_gram + nmfb_rescale at C2/C3 shapes."""
import sys, torch
sys.path.insert(0, '.')
from paper_1506_08938_b200 import _lib as L
from paper_1506_08938_b200 import device as D
dev = D.require_cuda()
def timeit(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3
for rows, r in [(10000, 50), (20000, 50), (50000, 100), (100000, 100), (20000, 64), (200000, 200)]:
    A = torch.rand((rows, r), device=dev)
    out = torch.zeros((r, r), dtype=torch.float64, device=dev)
    ws = torch.empty((L.lib().nmfb_gram_workspace_bytes(rows, r) // 8 + 1,), dtype=torch.float64, device=dev)
    g = lambda: L.call("nmfb_gram", L.F32, D.vp(A), rows, r, r, D.vp(out), D.vp(ws), D.stream_handle())
    Qa = torch.zeros(r * r, device=dev); sa = torch.zeros(r, device=dev)
    act = torch.zeros(r, dtype=torch.int32, device=dev); active = torch.zeros(r, dtype=torch.uint8, device=dev)
    ra = torch.zeros(1, dtype=torch.int32, device=dev); sc = torch.zeros(r, dtype=torch.float64, device=dev)
    rs = lambda: L.call("nmfb_rescale", L.F32, D.vp(out), r, 0.0, D.vp(Qa), D.vp(sa), D.vp(act), D.vp(active), D.vp(ra), D.vp(sc), D.stream_handle())
    print(f"rows={rows} r={r}: gram {timeit(g):.1f} us  rescale {timeit(rs):.1f} us  ({rows*r*4/timeit(g)/1e3:.0f} GB/s)")
