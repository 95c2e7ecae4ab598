import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_08185_b200 import benchmarks as B
lin = B.device_mx_linear(4096, 11008, 64)
x = B.outlier_x(16, 4096)
act = lin.quantize(x)
y = torch.empty((16, 11008), dtype=torch.bfloat16, device="cuda")
for _ in range(5):
    lin.gemm(act, y)
torch.cuda.synchronize()
print("ok")
