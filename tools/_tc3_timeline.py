"""CTA-0 per-k-block timeline of tc_gemm3 (NMFB_TC_DEBUG=64)."""
import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1506_08938_b200 import _lib as L
from paper_1506_08938_b200 import device as D
dev = D.require_cuda()
M, K, N = 20000, 10000, 50
A = torch.rand((M, K), device=dev); B = torch.rand((K, N), device=dev)
Bt = torch.empty((N, K), device=dev); Btl = torch.empty((N, K), device=dev)
L.call("nmfb_split_transpose", D.vp(B), K, N, D.vp(Bt), D.vp(Btl), D.stream_handle())
C = torch.empty((L.lib().nmfb_tc_parts(M, K, N, 0), M, N), device=dev)
for _ in range(3):
    L.call("nmfb_tc_gemm", D.vp(A), M, K, D.vp(Bt), D.vp(Btl), N, D.vp(C), 0, 0, D.stream_handle())
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (5 * 256))()
L.lib().nmfb_debug_tc3_timeline(buf)
t = np.array(buf, dtype=np.float64).reshape(5, 256)
t0 = t[0, 0]
names = ["tma_issue", "mma_full", "mma_xlo", "mma_done", "split_start"]
for i in list(range(0, 12)) + list(range(100, 110)):
    print(i, " ".join(f"{names[k]}={t[k, i] - t0:8.0f}" for k in range(5)))
med = lambda a: float(np.median(a))
sl = slice(20, 160)
print("kb period", med(np.diff(t[1, sl])))
print("tma issue -> mma sees full", med(t[1, sl] - t[0, sl]))
print("mma full -> xlo ready", med(t[2, sl] - t[1, sl]))
print("xlo ready -> issued", med(t[3, sl] - t[2, sl]))
print("split start - tma issue", med(t[4, sl] - t[0, sl]))
cb = (ctypes.c_longlong * 320)()
L.lib().nmfb_debug_tc3_cta(cb)
c = np.array(cb, dtype=np.float64).reshape(2, 160)[:, :148]
st, en = c[0] - c[0].min(), c[1] - c[0].min()
print("CTA start spread (ns): min %.0f max %.0f" % (st.min(), st.max()))
print("CTA end (ns): min %.0f median %.0f max %.0f" % (en.min(), np.median(en), en.max()))
order = np.argsort(en)
print("slowest CTAs:", [(int(b), int(en[b])) for b in order[-8:]])
print("fastest CTAs:", [(int(b), int(en[b])) for b in order[:8]])
