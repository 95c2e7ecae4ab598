"""C-ABI host pipeline spans (SERQ_DIAG build, SERQ_E2E_TRACE): C2 (M = K = N = 4096) through
serq_forward_mx_host with pinned buffers; SERQ_E2E_ROWS sets the chunk rows."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2603_08185_b200 import build, _lib
diag = os.path.join(os.path.dirname(build.OUT), "libserq_b200_diag.so")
subprocess.run([build.nvcc()] + build.NVCC_FLAGS + ["-DSERQ_DIAG", "-o", diag, build.SRC], check=True)
lib = _lib.load(diag); _lib._lib = lib
from paper_2603_08185_b200 import benchmarks as B
lin = B.device_mx_linear(4096, 4096, 64)
x = B.outlier_x(4096, 4096)
xh = x.cpu().pin_memory()
yh = torch.empty((4096, 4096), dtype=torch.bfloat16).pin_memory()
for _ in range(3):
    lin.forward_host(xh, yh)
os.environ["SERQ_E2E_TRACE"] = "1"
lin.forward_host(xh, yh)
torch.cuda.synchronize()
