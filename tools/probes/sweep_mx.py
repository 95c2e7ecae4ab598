"""Shape sweep: our fused MX SERQ linear (gemm only, L2 flushed, CUDA graph)
vs cuBLASLt NVFP4 (torch._scaled_mm, same MMA rate, no R term) -- diagnostic."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

from paper_2603_08185_b200 import _lib
from paper_2603_08185_b200 import benchmarks as B

flush = B.Flusher()
flags = [int(f) for f in os.environ.get("FLAGS", "0").split(",")]
shapes = [tuple(int(v) for v in s.split("x")) for s in os.environ.get(
    "SHAPES", "4096x4096x4096,8192x8192x8192,8192x4096x4096,4096x8192x4096,4096x4096x8192,2048x4096x11008").split(",")]
for (M, K, N) in shapes:
    r = int(os.environ.get("R", "64"))
    lin = B.device_mx_linear(K, N, r)
    x = B.outlier_x(M, K)
    act = lin.quantize(x)
    y = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    out = {"M": M, "K": K, "N": N, "r": r}
    for f in flags:
        _lib.load().serq_set_debug_flags(f)
        g = B.graph_of(lambda: lin.gemm(act, y))
        t = B.time_graph(g, flush) * 1e-3
        out[f"ours_f{f}_us"] = round(t * 1e6, 2)
        out[f"ours_f{f}_tflops"] = round(2.0 * M * N * (K + r) / t / 1e12, 1)
    _lib.load().serq_set_debug_flags(0)
    a = torch.randint(0, 256, (M, K // 2), dtype=torch.uint8, device="cuda").view(torch.float4_e2m1fn_x2)
    b = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device="cuda").view(torch.float4_e2m1fn_x2)
    sa = torch.full((M * K // 16,), 56, dtype=torch.uint8, device="cuda").view(torch.float8_e4m3fn)
    sb = torch.full((N * K // 16,), 56, dtype=torch.uint8, device="cuda").view(torch.float8_e4m3fn)
    g = B.graph_of(lambda: torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16))
    t = B.time_graph(g, flush) * 1e-3
    out["cublaslt_nvfp4_us"] = round(t * 1e6, 2)
    out["cublaslt_nvfp4_tflops"] = round(2.0 * M * N * K / t / 1e12, 1)
    print(json.dumps(out), flush=True)
    del lin
