import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08185_b200 import benchmarks as B
pts = B.decode_points(6534.8)
for p in pts:
    print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in p.items()}))
