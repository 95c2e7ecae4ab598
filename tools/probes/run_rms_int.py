"""RMSNorm -> INT producer timing (benchmarks.rmsnorm_int_quant_point) at C3's and C1's shapes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08185_b200 import benchmarks as B  # noqa: E402

for M, K, bits, sym in [(2048, 4096, 8, False), (512, 4096, 4, True), (4096, 4096, 8, False)]:
    print(json.dumps(B.rmsnorm_int_quant_point(M, K, bits, sym, 6550.0)))
