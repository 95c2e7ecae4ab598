"""Decode (M = 1 / 4 / 16) per-layer time and HBM fraction for fused-width layers: what a
q/k/v (4096 -> 12288) or gate/up (4096 -> 22016) launch would stream vs the single layers."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2603_08185_b200 import benchmarks as B

hbm = 6550.1
for K, N in ((4096, 11008), (4096, 22016), (4096, 12288), (11008, 4096)):
    layers = 8
    lins = [B.device_mx_linear(K, N, 64, seed=1 + i) for i in range(layers)]
    for M in (1, 16):
        x = B.outlier_x(M, K)
        acts = [lin.quantize(x) for lin in lins]
        ys = [torch.empty((M, N), dtype=torch.bfloat16, device="cuda") for _ in lins]

        def lin_all():
            for lin, a, y in zip(lins, acts, ys):
                lin.gemm(a, y)

        t = B.time_in_graph(lin_all, None, n=10) / layers
        byts = N * K / 2 + N * K / 32 + N * 64 / 2 + N * 64 / 32 + M * K / 2 + M * K / 32 + 2 * M * N
        print(json.dumps({"K": K, "N": N, "M": M, "linear_us": round(t * 1e3, 2),
                          "hbm_frac": round(byts / (t * 1e-3) / 1e9 / hbm, 3)}), flush=True)
    del lins
    torch.cuda.empty_cache()
