"""Run the C3 INT linear (W4A8 asym, M=2048, K=4096, N=11008, r=128 int R) a few times (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2603_08185_b200 import benchmarks as B
g = int(os.environ.get("GROUP", "0")) or None  # GROUP=128: group-wise weights
lin = B.device_int_linear(4096, 11008, 128, "int", group=g)
x = B.outlier_x(2048, 4096, frac=0.005, mag=100.0)
act = lin.quantize(x, 8, False)
y = torch.empty((2048, 11008), dtype=torch.bfloat16, device="cuda")
for _ in range(5):
    lin.gemm(lin.quantize(x, 8, False), y)
torch.cuda.synchronize()
print("ok")
