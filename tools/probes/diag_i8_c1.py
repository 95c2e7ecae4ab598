"""C1 (M=512, K=N=4096, A4 sym, dense R r=64): INT pair kernel timeline with the SERQ_DIAG_TS build --
per-K-step MMA-warp clocks of CTA 0 (issue done / next stage full) and per-cluster tile times."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2603_08185_b200 import build, _lib
diag = os.path.join(os.path.dirname(build.OUT), "libserq_b200_diag.so")
subprocess.run([build.nvcc()] + build.NVCC_FLAGS + ["-DSERQ_DIAG_TS", "-o", diag, build.SRC], check=True)
lib = _lib.load(diag); _lib._lib = lib
from paper_2603_08185_b200 import benchmarks as B
M = int(os.environ.get("M", "512"))
lin = B.device_int_linear(4096, 4096, 64, "dense")
x = B.outlier_x(M, 4096); act = lin.quantize(x, 4, True); y = torch.empty((M, 4096), dtype=torch.bfloat16, device="cuda")
ts = torch.zeros(6000, dtype=torch.int64, device="cuda")
fl = B.Flusher()
for _ in range(2): lin.gemm(act, y)
for mode in ("cold", "warm"):
    if mode == "cold": fl()
    else: lin.gemm(act, y)
    torch.cuda.synchronize()
    ts.zero_()
    lib.serq_set_debug_timestamps(ts.data_ptr()); lin.gemm(act, y); torch.cuda.synchronize(); lib.serq_set_debug_timestamps(None)
    t = ts.cpu().numpy()
    st = t[:256].reshape(32, 8)
    c0 = st[0, 5]
    print(mode, "CTA0 per step (cycles from step-0 issue): issued, next-full")
    print([(int(st[g, 5] - c0), int(st[g, 6] - c0)) for g in range(32)])
    tl = t[512:512 + 74 * 64].reshape(74, 8, 8)
    base = tl[:, 0, 0][tl[:, 0, 0] > 0].min()
    print(mode, "cluster: mma_start mma_end | epi (ns rel. to first mma start)")
    for c in (0, 1, 31, 63):
        r = tl[c, 0]
        print(c, (r[[0, 2]] - base).tolist(), "|", (r[3:6] - base).tolist())
    print(mode, "span ns", int(tl[:, :, 5].max() - base))
e = ts.cpu().numpy()[5300:5300 + 64].reshape(8, 8)[:, [0, 4, 5, 1, 2, 3]]
print("epilogue chunks of cluster 0 (ns from chunk0 start): start ldwait0 ldwait1 math_done staged_free stored")
for c in range(4):
    print(c, (e[c] - e[0, 0]).tolist())
