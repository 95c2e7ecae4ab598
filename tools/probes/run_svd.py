"""SVD-baseline step timing at C3's shape (benchmarks.svd_baseline_point): fused vs cuBLAS two-GEMM."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08185_b200 import benchmarks as B  # noqa: E402

print(json.dumps(B.svd_baseline_point(2048, 4096, 11008, 128)))
