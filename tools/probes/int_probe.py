"""INT linear probe (C1, C3): direct int8 weight feed (flags 0) vs packed INT4 widened in
shared memory (flags 1<<28), steady state over cold operand sets."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08185_b200 import _lib, benchmarks as B

for f in [int(v) for v in os.environ.get("FLAGS", "0,268435456").split(",")]:
    _lib.load().serq_set_debug_flags(f)
    c1 = B.int_linear_point(512, 4096, 4096, 64, "dense", 4, True)
    c3 = B.int_linear_point(2048, 4096, 11008, 128, "int", 8, False)
    print(json.dumps({"flags": f, "c1_linear_us": round(c1["linear_us"], 2), "c1_tops": round(c1["linear_tops"]),
                      "c3_linear_us": round(c3["linear_us"], 2), "c3_tops": round(c3["linear_tops"]),
                      "c3_step_us": round(c3["step_us"], 2)}), flush=True)
_lib.load().serq_set_debug_flags(0)
