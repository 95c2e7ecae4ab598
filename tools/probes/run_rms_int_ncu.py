"""One-shot RMSNorm -> INT producer launches at C3's shape (2048 x 4096 bf16, A8 asymmetric) for ncu:
argv[1] = "fast" (the f32-bounded kernel) or "f64" (the all-f64 kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_08185_b200 import benchmarks as B, device as D  # noqa: E402

xs = [B.outlier_x(2048, 4096, seed=i) for i in range(4)]
g = torch.rand(4096, device="cuda", dtype=torch.float64) + 0.5
for i in range(6):
    D.rmsnorm_quantize_int(xs[i % 4], g, 1e-6, 8, False, exact_f64=sys.argv[1] == "f64")
torch.cuda.synchronize()
print("ok")
