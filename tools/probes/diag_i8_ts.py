import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2603_08185_b200 import build, _lib
diag = os.path.join(os.path.dirname(build.OUT), "libserq_b200_diag.so")
subprocess.run([build.nvcc()] + build.NVCC_FLAGS + ["-DSERQ_DIAG_TS", "-o", diag, build.SRC], check=True)
lib = _lib.load(diag); _lib._lib = lib
from paper_2603_08185_b200 import benchmarks as B
lin = B.device_int_linear(4096, 11008, 128, "int")
x = B.outlier_x(2048, 4096); act = lin.quantize(x, 8, False); y = torch.empty((2048, 11008), dtype=torch.bfloat16, device="cuda")
ts = torch.zeros(512, dtype=torch.int64, device="cuda")
for _ in range(2): lin.gemm(act, y)
torch.cuda.synchronize()
lib.serq_set_debug_timestamps(ts.data_ptr()); lin.gemm(act, y); torch.cuda.synchronize(); lib.serq_set_debug_timestamps(None)
t = ts.cpu().numpy()[:256].reshape(32, 8)
base = t[0, 0]
print("step: tr_start bpk_landed unpacked fullA arrived | mma_before_wait mma_after_wait")
for g in range(0, 20):
    r = t[g] - base
    print(g, r[:5].tolist(), "|", r[5:7].tolist())
