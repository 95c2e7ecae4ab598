"""F8 probe: step time of the MX linear at C2's shape with the permuted (contiguous)
salient layout vs an arbitrary salient index set (gather fallback: the quantizer
also encodes x[:, idx], the CTA-pair kernel reads it as a side operand)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2603_08185_b200 import benchmarks as B

M = K = N = 4096
r = 64
out = {}
for name, idx in (("contiguous", None), ("gather", np.sort(np.random.default_rng(0).permutation(K)[:r]))):
    lins = [B.device_mx_linear(K, N, r, seed=1 + i, salient_idx=idx) for i in range(4)]
    xs = [B.outlier_x(M, K, seed=i) for i in range(8)]
    acts = [lins[0].quantize(x) for x in xs]
    ys = [torch.empty((M, N), dtype=torch.bfloat16, device="cuda") for _ in xs]
    t = B.time_steps(lambda i: lins[i % 4].forward(xs[i % 8], acts[i % 8], ys[i % 8]), 16)
    tq = B.time_steps(lambda i: lins[i % 4].quantize(xs[i % 8], acts[i % 8]), 16)
    tl = B.time_steps(lambda i: lins[i % 4].gemm(acts[i % 8], ys[i % 8]), 16)
    out[name] = {"step_us": round(t * 1e3, 2), "quant_us": round(tq * 1e3, 2), "linear_us": round(tl * 1e3, 2),
                 "step_tflops": round(2.0 * M * N * (K + r) / (t * 1e-3) / 1e12, 1)}
print(json.dumps(out))
