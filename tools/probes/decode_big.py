"""Decode linear streaming ceiling: one big layer (N large) vs Llama shapes, 4 layers per graph."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2603_08185_b200 import benchmarks as B, _lib
for flags in (0, 1 << 19):
    _lib.call("serq_set_debug_flags", flags)
    for K, N in ((4096, 11008), (4096, 65536), (8192, 57344)):
        lins = [B.device_mx_linear(K, N, 64, seed=1 + i) for i in range(4)]
        x = B.outlier_x(1, K)
        acts = [l.quantize(x) for l in lins]
        ys = [torch.empty((1, N), dtype=torch.bfloat16, device="cuda") for _ in lins]
        def run():
            for l, a, y in zip(lins, acts, ys):
                l.gemm(a, y)
        t = B.time_graph(B.graph_of(run), None, n=10) / 4 * 1e-3
        byts = N * K / 2 + N * K / 32
        print(json.dumps({"flags": flags, "K": K, "N": N, "us": round(t * 1e6, 2), "gbs": round(byts / t / 1e9)}), flush=True)
        del lins
        torch.cuda.empty_cache()
_lib.call("serq_set_debug_flags", 0)
