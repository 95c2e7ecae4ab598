"""INT per-token quantizer once (ncu target): C3 activations 2048 x 4096, asym A8."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2603_08185_b200 import benchmarks as B, device as D
x = B.outlier_x(2048, 4096, frac=0.005, mag=100.0)
for _ in range(4):
    D.quantize_int(x, 8, False)
torch.cuda.synchronize()
print("ok")
