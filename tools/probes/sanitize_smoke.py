"""Small calls of the new kernels for compute-sanitizer (memcheck / racecheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2603_08185_b200 import device as D, benchmarks as B
from oracle import serq_oracle as O
for M, K in ((3, 1024), (130, 4096), (257, 8192)):
    x = B.outlier_x(M, K, seed=M)
    D.quantize_mx(x)
    for bits, sym in ((8, False), (4, True)):
        D.quantize_int(x, bits, sym)
w = np.random.default_rng(1).standard_normal((1024, 264)) * 0.02
main, comp = O.build_grouped_int(w, np.arange(128), 128, 4, "col")
lin = D.IntLinear(main.codes, main.scales, 4, group_size=128, r_dense=O.dequantize(comp.r_q),
                  salient_idx=np.arange(128), r_split=True)
x = B.outlier_x(70, 1024)
lin.gemm(lin.quantize(x, 8, False))
lin2 = B.device_mx_linear(1024, 384, 64)
for M in (1, 5, 8):
    xx = B.outlier_x(M, 1024)
    lin2.forward(xx, lin2.quantize(xx))
torch.cuda.synchronize()
print("ok")
# round 2 paths: packed-INT4 loaders, the INT single-call / host entries, K-sharded ranges,
# decode with r = 128 / 32 (zero-padded R), the pipelined TP backend (one rank)
w = np.random.default_rng(2).standard_normal((512, 264)) * 0.02
main, comp = O.build_per_channel_int(w, np.arange(64), 4, r_mode="int")
for fmt in ("int8", "int4"):
    lin3 = D.IntLinear(main.codes, main.scales, 4, r_codes=comp.r_q.codes, r_scales=comp.r_q.scales,
                       salient_idx=np.arange(64), weight_format=fmt)
    x = B.outlier_x(300, 512)
    lin3.forward(x, 8, False)
    xh = x.cpu().pin_memory()
    yh = torch.empty((300, 264), dtype=torch.bfloat16).pin_memory()
    lin3.forward_host(xh, yh, 8, False)
rng = D.int_token_ranges(x[:, :256].contiguous())
D.quantize_int_with_range(x[:, :256].contiguous(), rng, 8, False)
for r in (128, 32):
    lin4 = B.device_mx_linear(1024, 296, r)
    for M in (1, 16):
        xx = B.outlier_x(M, 1024)
        lin4.forward(xx, lin4.quantize(xx))
        lin4.gemm(lin4.quantize(xx))
torch.cuda.synchronize()
print("ok2")
