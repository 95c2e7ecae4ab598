"""INT CTA-pair linear (C1, C3) timing with a given library build (argv[1]): used to
compare epilogue-warp counts (-DSERQ_I8_EPI=1/2/4).  Same measurement as the bench's
other_configs (steps back to back in one CUDA graph over > L2 operand sets)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08185_b200 import _lib
if len(sys.argv) > 1:
    _lib._lib = _lib.load(os.path.abspath(sys.argv[1]))
from paper_2603_08185_b200 import benchmarks as B

tag = sys.argv[1] if len(sys.argv) > 1 else "default"
for name, args in [("c1", (512, 4096, 4096, 64, "dense", 4, True)), ("c3", (2048, 4096, 11008, 128, "int", 8, False))]:
    pt = B.int_linear_point(*args)
    print(json.dumps({"lib": tag, "cfg": name, "step_us": round(pt["step_us"], 2), "linear_us": round(pt["linear_us"], 2),
                      "linear_tops": round(pt["linear_tops"], 1)}), flush=True)
