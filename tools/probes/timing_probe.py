"""Timing-floor probe: in-graph event timing of an empty region, one tiny
kernel, and 1 / 2 / 4 back-to-back MX quantizer launches at 4096^2."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2603_08185_b200 import benchmarks as B, device as D

flush = B.Flusher()
xs = B.outlier_x(16, 4096)
a_s = D.quantize_mx(xs)
x = B.outlier_x(4096, 4096)
acts = [D.quantize_mx(x) for _ in range(4)]
z = torch.zeros(1, device="cuda")
out = {
    "empty_us": B.time_in_graph(lambda: None, flush) * 1e3,
    "tiny_torch_kernel_us": B.time_in_graph(lambda: z.add_(1), flush) * 1e3,
    "quant16_us": B.time_in_graph(lambda: D.quantize_mx(xs, None, a_s), flush) * 1e3,
}
for n in (1, 2, 4):
    out[f"quant4096_x{n}_us"] = B.time_in_graph(lambda: [D.quantize_mx(x, None, acts[i]) for i in range(n)], flush) * 1e3
out["quant4096_x1_noflush_us"] = B.time_in_graph(lambda: D.quantize_mx(x, None, acts[0]), None) * 1e3
print(json.dumps({k: round(v, 2) for k, v in out.items()}))
