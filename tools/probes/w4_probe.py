"""Packed-INT4 (W4) INT linear at C3 with loader diagnostics (SERQ_DIAG build): flags 0,
1<<10 (no weight loads), 1<<11 (no operand stores), both; and the int8 feed for reference."""
import json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08185_b200 import build, _lib
diag = os.path.join(os.path.dirname(build.OUT), "libserq_b200_diag.so")
subprocess.run([build.nvcc()] + build.NVCC_FLAGS + ["-DSERQ_DIAG", "-o", diag, build.SRC], check=True)
lib = _lib.load(diag)
_lib._lib = lib
import torch
from paper_2603_08185_b200 import benchmarks as B, device as D
import numpy as np

K, N, M, r = 4096, 11008, 2048, 128
g = torch.Generator(device="cuda").manual_seed(1)
w = torch.randn((K, N), generator=g, device="cuda", dtype=torch.float64) * 0.02
s = w.abs().amax(dim=0) / 7.0
codes = torch.clamp(torch.round(w / s), -7, 7).to(torch.int32)
resid = w[:r] - codes[:r].double() * s
sr = resid.abs().amax(dim=0) / 7.0
rc = torch.clamp(torch.round(resid / sr), -7, 7).to(torch.int32)
lins = {f: D.IntLinear(codes, s, 4, r_codes=rc, r_scales=sr, salient_idx=np.arange(r), weight_format=f) for f in ("int8", "int4")}
xs = [B.outlier_x(M, K, seed=i) for i in range(4)]
acts = [lins["int8"].quantize(x, 8, False) for x in xs]
y = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
for fmt, flags in [("int8", 0), ("int4", 0), ("int4", 1 << 10), ("int4", 1 << 11), ("int4", 3 << 10)]:
    lib.serq_set_debug_flags(flags)
    t = B.time_steps(lambda i: lins[fmt].gemm(acts[i % 4], y), 16)
    print(json.dumps({"fmt": fmt, "flags": flags, "linear_us": round(t * 1e3, 2)}), flush=True)
lib.serq_set_debug_flags(0)
