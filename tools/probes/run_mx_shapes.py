"""One-shot MX linear launches for ncu: argv[1] = "c2" (pair3, 4096^3, r=64) or "c5qkv"
(the CTA-pair kernel for r != 64 at C5's qkv shape: M=8192, K=8192, N=10240, r=128)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_08185_b200 import benchmarks as B  # noqa: E402

M, K, N, r = {"c2": (4096, 4096, 4096, 64), "c5qkv": (8192, 8192, 10240, 128)}[sys.argv[1]]
lin = B.device_mx_linear(K, N, r)
x = B.outlier_x(M, K)
act = lin.quantize(x)
y = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
for _ in range(4):
    lin.gemm(act, y)
torch.cuda.synchronize()
print("ok")
