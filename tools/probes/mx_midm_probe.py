"""MX linear at 16 < M <= 256 (between the decode kernel and the CTA-pair kernel's home ground):
per-layer time in an 8-layer graph of distinct weights, and which kernel runs."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
from paper_2603_08185_b200 import benchmarks as B, device as D  # noqa: E402

L = 8
for K, N, r in ((4096, 11008, 64), (11008, 4096, 64), (4096, 4096, 64)):
    lins = [B.device_mx_linear(K, N, r, seed=1 + i) for i in range(L)]
    for M in [int(v) for v in os.environ.get("MS", "17,32,64,128,129,256").split(",")]:
        x = B.outlier_x(M, K)
        acts = [lin.quantize(x) for lin in lins]
        ys = [torch.empty((M, N), dtype=torch.bfloat16, device="cuda") for _ in lins]
        t = B.time_steps(lambda i: lins[i % L].gemm(acts[i % L], ys[i % L]), 2 * L) * 1e3
        print(json.dumps({"K": K, "N": N, "M": M, "linear_us": round(t, 2), "kernel": D.last_kernel()}), flush=True)
    del lins
    torch.cuda.empty_cache()
