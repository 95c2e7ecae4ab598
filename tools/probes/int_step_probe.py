"""C1 / C3 INT steps (quantize + linear) and linear alone, bench methodology."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08185_b200 import benchmarks as B
for args, kw in (((512, 4096, 4096, 64, "dense", 4, True), {}), ((2048, 4096, 11008, 128, "int", 8, False), {}),
                 ((2048, 4096, 11008, 128, "int", 8, False), {"group": 128})):
    r = B.int_linear_point(*args, **kw)
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
