"""C1 INT linear (M=512, K=N=4096, sym A4, bf16 L r=64) a few times (ncu target: 128-column tiles)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2603_08185_b200 import benchmarks as B
lin = B.device_int_linear(4096, 4096, 64, "dense")
x = B.outlier_x(512, 4096)
act = lin.quantize(x, 4, True)
y = torch.empty((512, 4096), dtype=torch.bfloat16, device="cuda")
for _ in range(4):
    lin.gemm(act, y)
torch.cuda.synchronize()
print("ok")
