"""RMSNorm -> MX producer timing (benchmarks.rmsnorm_quant_point) at 4096^2 and 2048 x 8192."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08185_b200 import benchmarks as B  # noqa: E402

for M, K in [(4096, 4096), (2048, 8192), (512, 4096)]:
    print(json.dumps(B.rmsnorm_quant_point(M, K, 6550.0)))
