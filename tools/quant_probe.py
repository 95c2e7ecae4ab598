"""Quantizer probe: MX encode of bf16 X [M, K] (graph replay, L2 flushed) for
the streaming kernel (flags 0) and the 2-D grid kernel (flags 1<<20)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_08185_b200 import _lib, benchmarks as B, device as D

flush = B.Flusher()
for (M, K) in [(4096, 4096), (2048, 4096), (8192, 8192), (8192, 28672), (16, 4096), (4096, 11008)]:
    x = B.outlier_x(M, K)
    act = D.quantize_mx(x)
    out = {"M": M, "K": K}
    for f in (0, 1 << 20):
        _lib.load().serq_set_debug_flags(f)
        g = B.graph_of(lambda: D.quantize_mx(x, None, act))
        t = B.time_graph(g, flush) * 1e-3
        byts = 2 * M * K + M * K / 2 + M * K / 32
        out[f"f{f}_us"] = round(t * 1e6, 2)
        out[f"f{f}_gbs"] = round(byts / t / 1e9, 1)
    _lib.load().serq_set_debug_flags(0)
    print(json.dumps(out), flush=True)
