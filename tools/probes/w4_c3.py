"""C3 linear with INT4-packed weights (weight_format="int4") vs int8 weights (8 weight sets, cold)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_08185_b200 import benchmarks as B, device as D  # noqa: E402

M, K, N, r = 2048, 4096, 11008, 128
out = {}
for fmt in ("int8", "int4"):
    lins = []
    for i in range(8):
        g = torch.Generator(device="cuda").manual_seed(1 + i)
        codes = torch.randint(-7, 8, (K, N), generator=g, device="cuda", dtype=torch.int32)
        s = torch.rand(N, generator=g, device="cuda", dtype=torch.float64) * 0.01 + 0.01
        rc = torch.randint(-7, 8, (r, N), generator=g, device="cuda", dtype=torch.int32)
        lins.append(D.IntLinear(codes, s, 4, r_codes=rc, r_scales=s, salient_idx=np.arange(r), weight_format=fmt))
    xs = [B.outlier_x(M, K, seed=i) for i in range(8)]
    acts = [lins[0].quantize(x, 8, False) for x in xs]
    ys = [torch.empty((M, N), dtype=torch.bfloat16, device="cuda") for _ in xs]
    out[fmt + "_linear_us"] = B.time_steps(lambda i: lins[i % 8].gemm(acts[i % 8], ys[i % 8]), 16) * 1e3
    out[fmt + "_kernel"] = D.last_kernel()
print(json.dumps(out))
