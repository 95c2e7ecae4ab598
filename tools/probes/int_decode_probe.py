"""INT linear at decode sizes (M = 1 / 4 / 16): which kernel runs and how long it takes (8 layers of
distinct weights per graph, so weights stream from HBM every step)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_08185_b200 import benchmarks as B, device as D  # noqa: E402

WF = os.environ.get("WF", "int8,int4").split(",")
for (K, N, r, mode), wf in [(c, f) for c in [(4096, 11008, 128, "int"), (11008, 4096, 128, "int"),
                                             (4096, 4096, 64, "dense")] for f in WF]:
    lins = [B.device_int_linear(K, N, r, mode, seed=1 + i, weight_format=wf) for i in range(8)]
    wb = lins[0].weight_bytes()[0]
    for M in [int(v) for v in os.environ.get("MS", "1,4,16").split(",")]:
        xs = [B.outlier_x(M, K, seed=i) for i in range(8)]
        acts = [lins[0].quantize(x, 8, False) for x in xs]
        ys = [torch.empty((M, N), dtype=torch.bfloat16, device="cuda") for _ in xs]
        t = B.time_steps(lambda i: lins[i % 8].gemm(acts[i % 8], ys[i % 8]), 16) * 1e3
        kern = D.last_kernel()
        print(json.dumps({"K": K, "N": N, "r": r, "mode": mode, "weights": wf, "M": M, "linear_us": t,
                          "kernel": kern, "hbm_tbps": (wb + N * r) / (t * 1e-6) / 1e12}))
