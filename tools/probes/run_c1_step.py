"""C1 steps (INT4 symmetric per-token activations, dense bf16 L, M=512, K=N=4096) through the
single-call entry, for an ncu launch list: which kernels a step runs and how long each takes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_08185_b200 import benchmarks as B  # noqa: E402

lin = B.device_int_linear(4096, 4096, 64, "dense")
xs = [B.outlier_x(512, 4096, seed=i) for i in range(4)]
y = torch.empty((512, 4096), dtype=torch.bfloat16, device="cuda")
for i in range(8):
    lin.forward(xs[i % 4], 4, True, None, y)
torch.cuda.synchronize()
print("ok")
