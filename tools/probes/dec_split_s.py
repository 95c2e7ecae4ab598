"""Decode: CTAs per 128-row tile (S) for the fused q/k/v (3 x 4096) and gate/up (2 x 11008) handles and
single layers at M = 1 (SERQ_DIAG build: SERQ_DEC_S overrides the default S)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2603_08185_b200 import build, _lib
diag = os.path.join(os.path.dirname(build.OUT), "libserq_b200_diag.so")
subprocess.run([build.nvcc()] + build.NVCC_FLAGS + ["-DSERQ_DIAG", "-o", diag, build.SRC], check=True)
lib = _lib.load(diag); _lib._lib = lib
from paper_2603_08185_b200 import benchmarks as B, device as D
rng = np.random.default_rng(5)
K, r, L = 4096, 64, 8
for name, ns in (("qkv", (4096, 4096, 4096)), ("gate_up", (11008, 11008)), ("o_proj", (4096,)), ("up", (11008,))):
    fused = [D.FusedMxLinear([B.device_mx_parts(K, n, r, seed=100 * i + j, salient_idx=np.sort(rng.permutation(K)[:r]))
                              for j, n in enumerate(ns)]) if len(ns) > 1 else
             D.MxLinear(*B.device_mx_parts(K, ns[0], r, seed=100 * i)) for i in range(L)]
    x = B.outlier_x(1, K)
    N = sum(ns)
    ys = [torch.empty((1, N), dtype=torch.bfloat16, device="cuda") for _ in range(L)]
    res = {}
    for S in ("", "1", "2", "3"):
        if S:
            os.environ["SERQ_DEC_S"] = S
        else:
            os.environ.pop("SERQ_DEC_S", None)
        if len(ns) > 1:
            acts = [f.fused._activation(1, x.device) for f in fused]
            fn = lambda i: fused[i % L].fused.forward(x, acts[i % L], ys[i % L])
        else:
            acts = [f._activation(1, x.device) for f in fused]
            fn = lambda i: fused[i % L].forward(x, acts[i % L], ys[i % L])
        res[S or "default"] = round(B.time_steps(fn, 16) * 1e3, 2)
    print(name, res)
