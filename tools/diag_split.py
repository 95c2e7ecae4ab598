import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_08185_b200 import build, _lib
diag = os.path.join(os.path.dirname(build.OUT), "libserq_b200_diag.so")
subprocess.run([build.nvcc()] + build.NVCC_FLAGS + ["-DSERQ_DIAG_TS", "-o", diag, build.SRC], check=True)
lib = _lib.load(diag); _lib._lib = lib
from paper_2603_08185_b200 import benchmarks as B
lin = B.device_mx_linear(4096, 4096, 64)
x = B.outlier_x(4096, 4096); act = lin.quantize(x); y = torch.empty((4096, 4096), dtype=torch.bfloat16, device="cuda")
ts = torch.zeros(512, dtype=torch.int64, device="cuda")
for _ in range(3): lin.gemm(act, y)
torch.cuda.synchronize()
lib.serq_set_debug_timestamps(ts.data_ptr()); lin.gemm(act, y); torch.cuda.synchronize(); lib.serq_set_debug_timestamps(None)
t = ts.cpu().numpy()
t0 = t[510]
print("kernel span (MMA warp CTA0):", (t[511] - t[510]) / 1e3, "us")
e = t[256:496].reshape(40, 6)
for row in e:
    if row[0] == 0: continue
    r = (row[:5] - t0) / 1e3
    print(f"half={row[5]:2d} wait_start={r[0]:7.2f} full={r[1]:7.2f} partial_done={r[2]:7.2f} atomic={r[3]:7.2f} end={r[4]:7.2f}")
