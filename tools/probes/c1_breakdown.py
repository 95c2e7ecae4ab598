"""C1 (M=512, K=N=4096, A4 sym, dense R r=64) step breakdown: quantizer alone, linear alone, two calls,
the single call, in CUDA graphs over 8 weight / activation sets (cold weights every step)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_08185_b200 import benchmarks as B, device as D  # noqa: E402

M, K, N, r = 512, 4096, 4096, 64
lins = [B.device_int_linear(K, N, r, "dense", seed=1 + i) for i in range(8)]
xs = [B.outlier_x(M, K, seed=i) for i in range(8)]
acts = [lins[0].quantize(x, 4, True) for x in xs]
ys = [torch.empty((M, N), dtype=torch.bfloat16, device="cuda") for _ in xs]
out = {
    "quant_only_us": B.time_steps(lambda i: D.quantize_int(xs[i % 8], 4, True, None, r, 1), 16) * 1e3,
    "linear_only_us": B.time_steps(lambda i: lins[i % 8].gemm(acts[i % 8], ys[i % 8]), 16) * 1e3,
    "two_call_us": B.time_steps(lambda i: lins[i % 8].gemm(lins[i % 8].quantize(xs[i % 8], 4, True), ys[i % 8]),
                                16) * 1e3,
    "single_call_us": B.time_steps(lambda i: lins[i % 8].forward(xs[i % 8], 4, True, acts[i % 8], ys[i % 8]),
                                   16) * 1e3,
}
print(json.dumps(out))
