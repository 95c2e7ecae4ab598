"""MX linear with a gathered salient set at 4096^3 (pair3 gather variant, ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2603_08185_b200 import benchmarks as B
idx = np.sort(np.random.default_rng(0).permutation(4096)[:64])
lin = B.device_mx_linear(4096, 4096, 64, salient_idx=idx)
x = B.outlier_x(4096, 4096)
act = lin.quantize(x)
y = torch.empty((4096, 4096), dtype=torch.bfloat16, device="cuda")
for _ in range(4):
    lin.gemm(act, y)
torch.cuda.synchronize()
print("ok")
