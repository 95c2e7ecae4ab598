"""K-split INT pair kernel timeline (SERQ_DIAG_TS build) at C1: per cluster (items 0..31 = upper K
halves / publishers, 32..63 = lower halves / finishers) the MMA start / end and epilogue phases, ns."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2603_08185_b200 import build, _lib
diag = os.path.join(os.path.dirname(build.OUT), "libserq_b200_diag.so")
subprocess.run([build.nvcc()] + build.NVCC_FLAGS + ["-DSERQ_DIAG_TS", "-o", diag, build.SRC], check=True)
lib = _lib.load(diag); _lib._lib = lib
from paper_2603_08185_b200 import benchmarks as B, device as D
M = 512
R = int(os.environ.get("R", "64"))
lin = B.device_int_linear(4096, 4096, R, "dense" if R else "none")
x = B.outlier_x(M, 4096); act = lin.quantize(x, 4, True); y = torch.empty((M, 4096), dtype=torch.bfloat16, device="cuda")
ts = torch.zeros(6000, dtype=torch.int64, device="cuda")
for _ in range(3): lin.gemm(act, y)
torch.cuda.synchronize()
print(D.last_kernel())
lib.serq_set_debug_timestamps(ts.data_ptr()); lin.gemm(act, y); torch.cuda.synchronize(); lib.serq_set_debug_timestamps(None)
t = ts.cpu().numpy()
tl = t[512:512 + 74 * 64].reshape(74, 8, 8)
base = tl[:, 0, 0][tl[:, 0, 0] > 0].min()
print("cluster: mma_start, mma_end | epi_wait_start, tmem_full, epi_end  (ns from first MMA start)")
for c in list(range(0, 64, 4)):
    r = tl[c, 0]
    print(c, (r[[0, 2]] - base).tolist(), "|", (r[3:6] - base).tolist(), "| x", (r[6:8] - base).tolist())
st = t[:256].reshape(32, 8)
c0 = st[0, 5]
print("CTA0 per step (cycles): issued, next-full", [(int(st[g, 5] - c0), int(st[g, 6] - c0)) for g in range(16)])
