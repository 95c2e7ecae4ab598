"""benchmarks.llama7b_block_point (fused linears) at M = 1 / 16 / 2048."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08185_b200 import benchmarks as B
for M in (1, 16, 2048):
    print(json.dumps(B.llama7b_block_point(M, fused=True)))
