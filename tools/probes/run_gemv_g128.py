"""One-shot group-wise (g = 128) INT decode gemv launches for ncu: Llama-2-7B down_proj
(11008 -> 4096, integer R r = 128), M = argv[1] (default 1), 8 distinct weight sets."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_08185_b200 import benchmarks as B  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1
lins = [B.device_int_linear(11008, 4096, 128, "int", seed=1 + i, group=128) for i in range(8)]
x = B.outlier_x(M, 11008)
act = lins[0].quantize(x, 8, False)
y = torch.empty((M, 4096), dtype=torch.bfloat16, device="cuda")
for i in range(16):
    lins[i % 8].gemm(act, y)
torch.cuda.synchronize()
print("ok")
