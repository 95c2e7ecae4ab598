"""One-shot INT decode launches (Llama-2-7B up_proj, int R r = 128, M = 1) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_08185_b200 import benchmarks as B  # noqa: E402

lin = B.device_int_linear(4096, 11008, 128, "int")
x = B.outlier_x(1, 4096)
act = lin.quantize(x, 8, False)
y = torch.empty((1, 11008), dtype=torch.bfloat16, device="cuda")
for _ in range(4):
    lin.gemm(act, y)
torch.cuda.synchronize()
print("ok")
