import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08185_b200 import benchmarks as B, _lib
for f in (0, 1 << 30):
    _lib.call("serq_set_debug_flags", f)
    for M, K in ((4096, 4096), (2048, 8192)):
        r = B.rmsnorm_quant_point(M, K, 6550.1)
        r["flags"] = f
        print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
_lib.call("serq_set_debug_flags", 0)
