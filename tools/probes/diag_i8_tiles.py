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
ts = torch.zeros(6000, dtype=torch.int64, device="cuda")
fl = B.Flusher()
for _ in range(2): lin.gemm(act, y)
fl(); torch.cuda.synchronize()
lib.serq_set_debug_timestamps(ts.data_ptr()); lin.gemm(act, y); torch.cuda.synchronize(); lib.serq_set_debug_timestamps(None)
t = ts.cpu().numpy()[512:512 + 74 * 64].reshape(74, 8, 8)
base = t[:, 0, 0][t[:, 0, 0] > 0].min()
print("cluster tile: mma_start mma_go mma_end | epi_wait epi_go epi_end   (ns rel. to first start)")
for c in (0, 1, 37, 73):
    for i in range(5):
        r = t[c, i]
        if r[0] == 0: continue
        print(c, i, (r[:3] - base).tolist(), "|", (r[3:6] - base).tolist())
ends = t[:, :, 5]
print("kernel span ns:", ends.max() - base)
e = ts.cpu().numpy()[5300:5300 + 64].reshape(8, 8)[:, [0, 4, 5, 1, 2, 3]]
print("tile1 epilogue chunks (ns from chunk0 start): start ldwait0 ldwait1 math_done staged_free stored")
for c in range(8):
    print(c, (e[c] - e[0, 0]).tolist())
