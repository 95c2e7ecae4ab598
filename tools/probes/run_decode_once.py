import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2603_08185_b200 import benchmarks as B
lin = B.device_mx_linear(4096, 11008, 64)
M = int(os.environ.get("M", "16"))
x = B.outlier_x(M, 4096)
act = lin.quantize(x)
y = torch.empty((M, 11008), dtype=torch.bfloat16, device="cuda")
for _ in range(5):
    if os.environ.get("FORWARD"):  # serq_forward_mx: fused quantizer for M <= 4
        lin.forward(x, act, y)
    else:
        lin.gemm(act, y)
torch.cuda.synchronize()
print("ok")
