"""K1-INT timing at C3 (2048 x 4096, A8 asym) and C1 (512 x 4096, A4 sym), 8 activation sets."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08185_b200 import benchmarks as B, device as D  # noqa: E402

out = {}
for name, M, bits, sym in (("c3", 2048, 8, False), ("c1", 512, 4, True)):
    xs = [B.outlier_x(M, 4096, seed=i) for i in range(8)]
    out[name + "_us"] = B.time_steps(lambda i: D.quantize_int(xs[i % 8], bits, sym), 16) * 1e3
print(json.dumps(out))
