"""One-shot INT decode gemv launches for ncu: argv[1] = "int8" | "int4", argv[2] = M; Llama-2-7B
up_proj (4096 -> 11008, integer R r = 128), 8 distinct weight sets."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_08185_b200 import benchmarks as B  # noqa: E402

wf, M = sys.argv[1], int(sys.argv[2])
K, N = int(os.environ.get("K", 4096)), int(os.environ.get("N", 11008))
lins = [B.device_int_linear(K, N, 128, "int", seed=1 + i, weight_format=wf) for i in range(8)]
x = B.outlier_x(M, K)
act = lins[0].quantize(x, 8, False)
y = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
for i in range(16):
    lins[i % 8].gemm(act, y)
torch.cuda.synchronize()
print("ok")
