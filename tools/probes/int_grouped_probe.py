"""Grouped (g=128) vs per-output-channel INT SERQ linear at the C3 shape
(M=2048, K=4096, N=11008, W4A8 asym, integer R r=128)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08185_b200 import benchmarks as B

for group in (None, 128, 256):
    r = B.int_linear_point(2048, 4096, 11008, 128, "int", 8, False, group=group)
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
r = B.int_linear_point(512, 4096, 4096, 64, "dense", 4, True, group=128)
print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
