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
