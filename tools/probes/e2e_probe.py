"""e2e probe: serq_forward_mx_host wall / CPU time vs chunk rows (SERQ_E2E_ROWS)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2603_08185_b200 import benchmarks as B

M = K = N = 4096
lin = B.device_mx_linear(K, N, 64)
x = B.outlier_x(M, K)
xh = x.cpu().pin_memory()
yh = torch.empty((M, N), dtype=torch.bfloat16).pin_memory()
plans = os.environ.get("PLANS")
for rows in ([p for p in plans.split(";")] if plans else [int(v) for v in os.environ.get("ROWS_LIST", "0,512,1024,2048").split(",")]):
    if isinstance(rows, str):
        os.environ["SERQ_E2E_PLAN"] = rows
    elif rows:
        os.environ["SERQ_E2E_ROWS"] = str(rows)
    else:
        os.environ.pop("SERQ_E2E_ROWS", None)  # default plan
    for _ in range(2):
        lin.forward_host(xh, yh)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        lin.forward_host(xh, yh)
        ts.append(time.perf_counter() - t0)
    print(json.dumps({"rows": rows, "ms": sorted(ts)[2] * 1e3}), flush=True)
