"""C3 with group-wise weights (g = 128 / 256) through the i8g pair kernel, for A/B runs of library
variants (SERQ_B200_LIB)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08185_b200 import benchmarks as B  # noqa: E402

fl = B.Flusher()
out = {}
for g in (128, 256):
    pt = B.int_linear_point(2048, 4096, 11008, 128, "int", 8, False, fl, group=g)
    out[f"g{g}_linear_us"] = round(pt["linear_us"], 2)
print(os.environ.get("SERQ_B200_LIB", "new"), json.dumps(out))
