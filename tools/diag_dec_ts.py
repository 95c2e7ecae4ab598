import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_08185_b200 import build, _lib
diag = os.path.join(os.path.dirname(build.OUT), "libserq_b200_diag.so")
subprocess.run([build.nvcc()] + build.NVCC_FLAGS + ["-DSERQ_DIAG_TS", "-o", diag, build.SRC], check=True)
lib = _lib.load(diag); _lib._lib = lib
from paper_2603_08185_b200 import benchmarks as B
for K in (256, 4096):
    lin = B.device_mx_linear(K, 11008, 64 if K > 256 else 0)
    x = B.outlier_x(16, K); act = lin.quantize(x); y = torch.empty((16, 11008), dtype=torch.bfloat16, device="cuda")
    ts = torch.zeros(2048, dtype=torch.int64, device="cuda")
    for _ in range(3): lin.gemm(act, y)
    torch.cuda.synchronize()
    lib.serq_set_debug_timestamps(ts.data_ptr())
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); lin.gemm(act, y); e.record(); e.synchronize()
    lib.serq_set_debug_timestamps(None)
    t = ts.cpu().numpy().reshape(-1, 2); t = t[t[:, 0] > 0]
    ent, ex = t[:, 0] - t[:, 0].min(), t[:, 1] - t[:, 0].min()
    print(f"K={K}: ctas={len(t)} event={s.elapsed_time(e)*1e3:.1f}us  entry spread={ent.max()/1e3:.2f}us  "
          f"first exit={ex.min()/1e3:.2f}us  last exit={ex.max()/1e3:.2f}us  median CTA life={(np.median(ex-ent))/1e3:.2f}us")
