"""benchmarks.decode_fused_points alone."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08185_b200 import benchmarks as B
for p in B.decode_fused_points(6550.1):
    print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in p.items()}), flush=True)
