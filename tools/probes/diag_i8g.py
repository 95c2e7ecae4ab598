"""Per-unit epilogue timeline of the grouped INT kernel (SERQ_DIAG_TS build), CTA 0 warp 4."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2603_08185_b200 import build, _lib
diag = os.path.join(os.path.dirname(build.OUT), "libserq_b200_diag.so")
subprocess.run([build.nvcc()] + build.NVCC_FLAGS + ["-DSERQ_DIAG_TS", "-o", diag, build.SRC], check=True)
lib = _lib.load(diag); _lib._lib = lib
from paper_2603_08185_b200 import benchmarks as B
g = int(os.environ.get("G", "128"))
lin = B.device_int_linear(4096, 11008, 128, "int", group=g)
x = B.outlier_x(2048, 4096)
act = lin.quantize(x, 8, False)
y = torch.empty((2048, 11008), dtype=torch.bfloat16, device="cuda")
ts = torch.zeros(64 * 8, dtype=torch.int64, device="cuda")
for _ in range(3):
    lin.gemm(act, y)
torch.cuda.synchronize()
lib.serq_set_debug_timestamps(ts.data_ptr())
lin.gemm(act, y)
torch.cuda.synchronize()
lib.serq_set_debug_timestamps(None)
t = ts.cpu().numpy().reshape(64, 8).astype(np.float64)
base = t[0, 0]
print("unit: wait_start acc_full first_ld chunks_done barrier_done (cycles from unit 0 start)")
for u in range(40):
    print(u, " ".join(f"{(v - base):8.0f}" for v in t[u, :5]))
