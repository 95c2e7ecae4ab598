"""Does device compute slow pinned H2D / D2H?  32 MB copies alone vs while the C2 linear runs in a
loop on another stream."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2603_08185_b200 import benchmarks as B

n = 32 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
lin = B.device_mx_linear(4096, 4096, 64)
x = B.outlier_x(4096, 4096)
act = lin.quantize(x)
y = torch.empty((4096, 4096), dtype=torch.bfloat16, device="cuda")
s_cp, s_k = torch.cuda.Stream(), torch.cuda.Stream()


def h2d_ms():
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s_cp):
        a.record()
        d_in.copy_(h_in, non_blocking=True)
        b.record()
    b.synchronize()
    return a.elapsed_time(b)


out = {"alone": min(h2d_ms() for _ in range(5))}
with torch.cuda.stream(s_k):
    for _ in range(60):
        lin.gemm(act, y)
out["with_linear_loop"] = h2d_ms()
torch.cuda.synchronize()
with torch.cuda.stream(s_k):
    for _ in range(200):
        lin.quantize(x, act)
out["with_quantizer_loop"] = h2d_ms()
torch.cuda.synchronize()
print(json.dumps({k: round(v, 3) for k, v in out.items()}))
