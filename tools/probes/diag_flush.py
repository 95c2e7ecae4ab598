import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2603_08185_b200 import benchmarks as B
lin = B.device_mx_linear(4096, 11008, 64)
x = B.outlier_x(16, 4096)
act = lin.quantize(x)
y = torch.empty((16, 11008), dtype=torch.bfloat16, device="cuda")
g = B.graph_of(lambda: lin.gemm(act, y))
fa = torch.empty(64 << 20, device="cuda"); fb = torch.ones(64 << 20, device="cuda"); fc = torch.ones(64 << 20, device="cuda")
def wflush(): fa.zero_(); fb.sum()
def rflush(): fb.sum(); fc.sum()
def wflush_idle(): fa.zero_(); fb.sum(); torch.cuda.synchronize(); torch.cuda._sleep(2000000)
res = {}
for name, fl in [("write+read", wflush), ("read-only", rflush), ("write+read+sleep", wflush_idle), ("none", None)]:
    res[name] = round(B.time_graph(g, fl, n=30) * 1e3, 3)
# many back-to-back launches (weights L2 resident): per-launch time
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(50): g.replay()
e.record(); e.synchronize()
res["b2b_per_launch"] = round(s.elapsed_time(e) / 50 * 1e3, 3)
# tiny K: fixed overhead
lin2 = B.device_mx_linear(256, 11008, 0)
x2 = B.outlier_x(16, 256); a2 = lin2.quantize(x2); y2 = torch.empty((16, 11008), dtype=torch.bfloat16, device="cuda")
g2 = B.graph_of(lambda: lin2.gemm(a2, y2))
res["K256_none"] = round(B.time_graph(g2, None, n=30) * 1e3, 3)
print(json.dumps(res))
