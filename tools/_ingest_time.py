"""Timing of the sparse ingest at config 5 (1e8 nonzeros): host numpy CSR
build (the reference's transpose path) vs the device (csrc/ingest.cu)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from oracle import generators
from paper_1506_08938_b200 import SparseMatrix
from paper_1506_08938_b200.ingest import DeviceCsc
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
x, _ = generators.make(cid)
V = SparseMatrix(x.rows, x.cols, x.indptr, x.indices, x.values, validate=False)
torch.cuda.synchronize()
t = time.perf_counter(); V._csr = None; V.csr(); th = time.perf_counter() - t
t = time.perf_counter(); V._validate(); tv = time.perf_counter() - t
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    d = DeviceCsc.from_host(V, dtype=torch.float32); d.csr(); torch.cuda.synchronize()
    td = time.perf_counter() - t
col_of = np.repeat(np.arange(x.cols), np.diff(x.indptr))
i_d = torch.from_numpy(x.indices).cuda(); j_d = torch.from_numpy(col_of).cuda(); v_d = torch.from_numpy(x.values).cuda()
perm = torch.randperm(i_d.numel(), device='cuda')
i_d, j_d, v_d = i_d[perm], j_d[perm], v_d[perm]
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    d2 = DeviceCsc.from_triplets(x.rows, x.cols, i_d, j_d, v_d); torch.cuda.synchronize()
    tt = time.perf_counter() - t
print(f"C{cid} nnz {V.nnz}: host csr() {th:.2f} s, host _validate {tv:.2f} s; device upload+narrow+validate+csr {td*1e3:.1f} ms; device from_triplets (shuffled, device-resident) {tt*1e3:.1f} ms")
