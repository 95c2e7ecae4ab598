"""K1-INT cold timing (16 activation sets, steps back to back in one graph) with a given library
build (argv[1]) -- used to pick the per-SM row-loop CTA count (-DSERQ_INTQ_CTAS_PER_SM)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08185_b200 import _lib
if len(sys.argv) > 1:
    _lib._lib = _lib.load(os.path.abspath(sys.argv[1]))
from paper_2603_08185_b200 import benchmarks as B, device as D

tag = sys.argv[1] if len(sys.argv) > 1 else "default"
for M, K, bits, sym in [(2048, 4096, 8, False), (512, 4096, 4, True), (8192, 8192, 8, False)]:
    xs = [B.outlier_x(M, K, seed=i) for i in range(16)]
    t = B.time_steps(lambda i: D.quantize_int(xs[i % 16], bits, sym), 32)
    ib = 2 * M * K + M * K + 16 * M
    print(json.dumps({"lib": tag, "M": M, "K": K, "us": round(t * 1e3, 2), "tbs": round(ib / t / 1e9, 2)}), flush=True)
