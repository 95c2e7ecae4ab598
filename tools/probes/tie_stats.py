"""How often the INT quantizer's fp32 fast path defers to the f64 path (near-.5 ties), on the
probe's activations; float32 arithmetic as in int_quant_bf16_kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2603_08185_b200 import benchmarks as B
for (M, K, bits, sym) in [(512, 4096, 4, True), (2048, 4096, 8, False)]:
    x = B.outlier_x(M, K, seed=0).float().cpu().numpy().astype(np.float32)
    xd = x.astype(np.float64)
    if sym:
        s = np.abs(xd).max(1, keepdims=True) / ((1 << (bits - 1)) - 1)
    else:
        s = (xd.max(1, keepdims=True) - xd.min(1, keepdims=True)) / ((1 << bits) - 1)
    inv32 = (1.0 / s).astype(np.float32)
    q = (x * inv32).astype(np.float32)
    M_ = np.float32(12582912.0)
    n = ((q + M_) - M_).astype(np.float32)
    d = (q - n).astype(np.float32)
    margin = (np.abs(q) * np.float32(2.0 ** -21) + np.float32(2.0 ** -40)).astype(np.float32)
    bad = ~((np.abs(q) < 2 ** 21) & (np.abs(np.abs(d) - np.float32(0.5)) > margin))
    # kernel layout: thread t of a row owns 8-element groups t, t + 64, ...
    per_thread = bad.reshape(M, -1, 64, 8).any(axis=(1, 3))
    print(M, K, bits, sym, "elements", bad.mean(), "threads", per_thread.mean(), "rows", bad.any(1).mean())
