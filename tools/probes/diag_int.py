import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08185_b200 import benchmarks as B, _lib
fl = B.Flusher()
flags = [int(f) for f in sys.argv[1:]] or [0]
for f in flags:
    _lib.load().serq_set_debug_flags(f)
    for args in [(512, 4096, 4096, 64, "dense", 4, True), (2048, 4096, 11008, 128, "int", 8, False)]:
        p = B.int_linear_point(*args, fl)
        print(f, json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in p.items()}))
_lib.load().serq_set_debug_flags(0)
