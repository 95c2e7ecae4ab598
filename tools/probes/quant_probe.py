"""Quantizer probe: MX encode of bf16 X [M, K], 16 launches back to back over 8
activation sets (cold operands), for the debug-flag variants of the 2-D grid kernel (flags 1<<20)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2603_08185_b200 import _lib, benchmarks as B, device as D

flush = B.Flusher()
for (M, K) in [(4096, 4096), (2048, 4096), (8192, 8192), (8192, 28672), (16, 4096), (4096, 11008)]:
    nx = max(2, min(8, int(512e6 // (2 * M * K))))
    xs = [B.outlier_x(M, K, seed=i) for i in range(nx)]
    acts = [D.quantize_mx(x) for x in xs]
    out = {"M": M, "K": K}
    for f in (0, 1 << 22, 1 << 30):
        _lib.load().serq_set_debug_flags(f)
        t = B.time_steps(lambda i: D.quantize_mx(xs[i % nx], None, acts[i % nx]), 16) * 1e-3
        byts = 2 * M * K + M * K / 2 + M * K / 32
        out[f"f{f}_us"] = round(t * 1e6, 2)
        out[f"f{f}_gbs"] = round(byts / t / 1e9, 1)
    _lib.load().serq_set_debug_flags(0)
    print(json.dumps(out), flush=True)
