"""Pair3 narrow last-round tiles (256 x 128) vs the full-tile schedule (debug flag 1<<19): bit-equal outputs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

from paper_2603_08185_b200 import _lib
from paper_2603_08185_b200 import benchmarks as B

shapes = [tuple(int(v) for v in s.split("x")) for s in os.environ.get("SHAPES", "2600x512x4096,4096x4096x4096").split(",")]
for (M, K, N) in shapes:
    lin = B.device_mx_linear(K, N, 64)
    x = B.outlier_x(M, K)
    act = lin.quantize(x)
    ys = []
    for f in [1 << 19] + [int(v) for v in os.environ.get("FL", "0").split(",")]:
        _lib.load().serq_set_debug_flags(f)
        y = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda")
        lin.gemm(act, y)
        torch.cuda.synchronize()
        ys.append(y)
        print(M, K, N, "flag", f, "ok", flush=True)
    _lib.load().serq_set_debug_flags(0)
    for y in ys[1:]:
        print(M, K, N, "equal", torch.equal(ys[0], y), "nan", int(torch.isnan(y.float()).sum()),
              "cols-equal", [bool(torch.equal(ys[0][:, c:c + 128], y[:, c:c + 128])) for c in range(0, N, 128)][:4], flush=True)
