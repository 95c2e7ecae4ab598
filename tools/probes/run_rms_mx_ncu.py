"""One-shot RMSNorm -> MX producer launches at 4096 x 4096 bf16 for ncu (rmsnorm_mx_encode_kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_08185_b200 import benchmarks as B, device as D  # noqa: E402

xs = [B.outlier_x(4096, 4096, seed=i) for i in range(4)]
g = torch.rand(4096, device="cuda", dtype=torch.float64) + 0.5
acts = [D.quantize_mx(x) for x in xs]
for i in range(6):
    D.rmsnorm_quantize_mx(xs[i % 4], g, 1e-6, acts[i % 4])
torch.cuda.synchronize()
print("ok")
