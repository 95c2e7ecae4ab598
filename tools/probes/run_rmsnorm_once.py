"""Run the fused RMSNorm -> MX quantizer at 4096 x 4096 a few times (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2603_08185_b200 import benchmarks as B, device as D
x = B.outlier_x(4096, 4096)
g = torch.rand(4096, device="cuda", dtype=torch.float64) + 0.5
a = D.rmsnorm_quantize_mx(x, g)
for _ in range(4):
    D.rmsnorm_quantize_mx(x, g, 1e-6, a)
torch.cuda.synchronize()
print("ok")
