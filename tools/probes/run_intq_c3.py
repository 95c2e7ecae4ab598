"""One-shot K1-INT launches at C3's shape (2048 x 4096 bf16, A8 asymmetric) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_08185_b200 import benchmarks as B, device as D  # noqa: E402

xs = [B.outlier_x(2048, 4096, seed=i) for i in range(4)]
for i in range(8):
    D.quantize_int(xs[i % 4], 8, False)
torch.cuda.synchronize()
print("ok")
