"""INT per-token quantizer probe (C1: 512 x 4096 sym A4, C3: 2048 x 4096 asym A8, C5-like 8192 x 8192)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08185_b200 import _lib, benchmarks as B, device as D

for f in (0, 1 << 21):
  _lib.load().serq_set_debug_flags(f)
  for (M, K, bits, sym) in [(512, 4096, 4, True), (2048, 4096, 8, False), (8192, 8192, 8, False), (4096, 4096, 4, False)]:
    xs = [B.outlier_x(M, K, seed=i) for i in range(8)]
    t = B.time_steps(lambda i: D.quantize_int(xs[i % 8], bits, sym), 16) * 1e-3
    byts = 2 * M * K + M * K + 16 * M
    print(json.dumps({"flags": f, "M": M, "K": K, "bits": bits, "sym": sym, "us": round(t * 1e6, 2),
                      "gbs": round(byts / t / 1e9)}), flush=True)
