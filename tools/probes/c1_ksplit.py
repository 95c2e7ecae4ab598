"""C1 linear timing with and without the K-split workspace (cold weights, 8 sets)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_08185_b200 import _lib, benchmarks as B, device as D  # noqa: E402

M, K, N, r = 512, 4096, 4096, 64
lins = [B.device_int_linear(K, N, r, "dense", seed=1 + i) for i in range(8)]
xs = [B.outlier_x(M, K, seed=i) for i in range(8)]
acts = [lins[0].quantize(x, 4, True) for x in xs]
ys = [torch.empty((M, N), dtype=torch.bfloat16, device="cuda") for _ in xs]
out = {}
out["ksplit_linear_us"] = B.time_steps(lambda i: lins[i % 8].gemm(acts[i % 8], ys[i % 8]), 16) * 1e3
out["ksplit_kernel"] = D.last_kernel()
out["ksplit_step_us"] = B.time_steps(lambda i: lins[i % 8].forward(xs[i % 8], 4, True, acts[i % 8], ys[i % 8]), 16) * 1e3
for lin in lins:
    _lib.call("serq_linear_set_workspace", lin._h.ptr, None, 0)
out["narrow_linear_us"] = B.time_steps(lambda i: lins[i % 8].gemm(acts[i % 8], ys[i % 8]), 16) * 1e3
print(json.dumps(out))
