"""C3 with group-wise weights (g = 128): linear / step timing (benchmarks.int_linear_point)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08185_b200 import benchmarks as B  # noqa: E402

out = B.int_linear_point(2048, 4096, 11008, 128, "int", 8, False, None, group=128)
out.pop("e2e", None)
print(json.dumps(out))
