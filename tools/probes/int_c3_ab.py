"""C3 / C1 INT linear timing (benchmarks.int_linear_point) for A/B runs of library variants
(SERQ_B200_LIB)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08185_b200 import benchmarks as B  # noqa: E402

fl = B.Flusher()
c3 = B.int_linear_point(2048, 4096, 11008, 128, "int", 8, False, fl)
c1 = B.int_linear_point(512, 4096, 4096, 64, "dense", 4, True, fl)
print(os.environ.get("SERQ_B200_LIB", "new"), json.dumps({"c3_linear_us": c3["linear_us"], "c3_step_us": c3["step_us"],
                                                           "c1_linear_us": c1["linear_us"]}))
