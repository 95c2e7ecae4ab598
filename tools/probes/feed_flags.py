"""K2 (pair3) feed-rate experiments with diagnostic flags (SERQ_DIAG builds only):
1024 = no MMAs (feed alone); 1<<25 = A and B as flat 256-B-row boxes (contiguous copies,
garbage data -- timing only); 1<<19 = no narrow last round."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2603_08185_b200 import _lib, benchmarks as B

lib = _lib.load()
FL = [int(f) for f in os.environ.get("FLAGS", "0,1024,524288,34078720,34079744").split(",")]
for M, K, N in [(4096, 4096, 4096), (8192, 8192, 8192)]:
    lins = [B.device_mx_linear(K, N, 64, seed=1 + i) for i in range(4)]
    xs = [B.outlier_x(M, K, seed=i) for i in range(4)]
    acts = [lins[0].quantize(x) for x in xs]
    y = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    for flags in FL:
        lib.serq_set_debug_flags(flags)
        t = B.time_steps(lambda i: lins[i % 4].gemm(acts[i % 4], y), 16)
        print(f"{M}x{K}x{N} flags={flags:9d}: {t*1e3:8.2f} us/launch  {2*M*N*(K+64)/t/1e9:8.1f} TFLOP/s-equiv", flush=True)
    lib.serq_set_debug_flags(0)
    del lins, xs, acts
    torch.cuda.empty_cache()
