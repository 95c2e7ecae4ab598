"""benchmarks.int_decode_points on its own."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08185_b200 import benchmarks as B
for p in B.int_decode_points(6550.1):
    print(json.dumps(p))
