"""Timeline of a CUDA-graph chain of decode linears (quantize + cluster decode kernel per
layer; SERQ_DIAG_TS build): per layer, min/median/max over CTAs of the kernel's stamps."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2603_08185_b200 import build, _lib
diag = os.path.join(os.path.dirname(build.OUT), "libserq_b200_diag.so")
subprocess.run([build.nvcc()] + build.NVCC_FLAGS + ["-DSERQ_DIAG_TS", "-o", diag, build.SRC], check=True)
lib = _lib.load(diag); _lib._lib = lib
from paper_2603_08185_b200 import benchmarks as B
L = 8
names = ["entry", "after pdl_wait", "first stage", "last MMA issued", "acc done", "epi done", "exit"]
for K, N in ((4096, 11008), (11008, 4096)):
    lins = [B.device_mx_linear(K, N, 64, seed=1 + i) for i in range(L)]
    M = int(os.environ.get("M", "1"))
    x = B.outlier_x(M, K)
    acts = [l.quantize(x) for l in lins]
    ys = [torch.empty((M, N), dtype=torch.bfloat16, device="cuda") for _ in lins]
    ts = torch.zeros((L, 1024 * 8 + 384), dtype=torch.int64, device="cuda")
    fused = bool(os.environ.get("FUSED"))
    lib.serq_set_debug_flags(0 if fused else (1 << 23))
    def chain():
        for i in range(L):
            lib.serq_set_debug_timestamps(ts[i].data_ptr())
            if fused:
                lins[i].forward(x, acts[i], ys[i])
            else:
                lins[i].quantize(x, acts[i])
                lins[i].gemm(acts[i], ys[i])
        lib.serq_set_debug_timestamps(None)
    g = B.graph_of(chain)
    for _ in range(3):
        ts.zero_(); torch.cuda.synchronize(); g.replay(); torch.cuda.synchronize()
    tt = ts.cpu().numpy()
    t = tt[:, :8192].reshape(L, 1024, 8).astype(np.float64)
    ok = t[:, :, 0] > 0
    t0 = t[0][ok[0]][:, 0].min()
    print(f"fused={fused} K={K} N={N} M={M}: ctas/layer={ok[0].sum()} (us from layer 0's first entry)")
    for i in range(L):
        v = (t[i][ok[i]] - t0) / 1e3
        print(f"  layer {i}: " + "  ".join(f"{n}={np.median(v[:, c]):.2f}[{v[:, c].max():.2f}]" for c, n in enumerate(names)))
    st = tt[1, 8192:].reshape(6, 64).astype(np.float64)
    base = st[2, 0]
    kinds = ["w issued", "x issued", "mma start", "cv xfull", "cv empty", "cv arrived"]
    print("  layer 1 CTA 0 per-step SM-clock (kcycles from first MMA):")
    for c, n in enumerate(kinds):
        v = st[c]; v = v[v > 0]
        print(f"    {n:10s} " + " ".join(f"{(a - base) / 1e3:6.2f}" for a in v[:24]))
    del lins
