"""Step probe at C2: fused serq_forward_mx (flags) vs quantize-then-linear."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_08185_b200 import _lib, benchmarks as B

flush = B.Flusher()
M = K = N = 4096
lin = B.device_mx_linear(K, N, 64)
x = B.outlier_x(M, K)
act = lin.quantize(x)
y = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
out = {}
for f in [0, 1 << 21, 131072]:
    _lib.load().serq_set_debug_flags(f)
    g = B.graph_of(lambda: lin.forward(x, act, y))
    out[f"fused_f{f}_us"] = round(B.time_graph(g, flush, n=30) * 1e3, 2)
_lib.load().serq_set_debug_flags(0)
g = B.graph_of(lambda: (lin.quantize(x, act), lin.gemm(act, y)))
out["two_launch_us"] = round(B.time_graph(g, flush, n=30) * 1e3, 2)
g = B.graph_of(lambda: lin.gemm(act, y))
out["gemm_us"] = round(B.time_graph(g, flush, n=30) * 1e3, 2)
g = B.graph_of(lambda: lin.quantize(x, act))
out["quant_us"] = round(B.time_graph(g, flush, n=30) * 1e3, 2)
g = B.graph_of(lambda: None)
print(json.dumps(out))
