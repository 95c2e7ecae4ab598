"""Where the MX SVD-baseline step (device.SvdMxLinear) spends its time at C2 (4096^3, r = 64):
each piece timed alone in a graph, 8 weight / activation sets."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_08185_b200 import _lib, benchmarks as B, device as D  # noqa: E402

M = K = N = 4096
r = 64
rng = np.random.default_rng(6)
l1 = rng.standard_normal((K, r)) * 0.01
l2 = rng.standard_normal((r, N)) * 0.01
svds = []
for i in range(8):
    codes, exps, *_ = B.device_mx_parts(K, N, 0, seed=1 + i)
    svds.append(D.SvdMxLinear(codes, exps, l1, l2))
xs = [B.outlier_x(M, K, seed=i) for i in range(8)]
acts = [svds[0].lin.quantize(x) for x in xs]
xh = [D.mx_decode_bf16(a) for a in acts]
us = [x @ svds[0].l1 for x in xh]
cs = [torch.mm(u, svds[0].l2, out_dtype=torch.float32) for u in us]
ys = [torch.empty((M, N), dtype=torch.bfloat16, device="cuda") for _ in xs]
out = {}
out["quantize"] = B.time_steps(lambda i: svds[i % 8].lin.quantize(xs[i % 8], acts[i % 8]), 16)
out["decode"] = B.time_steps(lambda i: D.mx_decode_bf16(acts[i % 8]), 16)
out["u_gemm"] = B.time_steps(lambda i: xh[i % 8] @ svds[0].l1, 16)
out["c_gemm_f32out"] = B.time_steps(lambda i: torch.mm(us[i % 8], svds[0].l2, out_dtype=torch.float32), 16)
out["linear_addend"] = B.time_steps(lambda i: _lib.call(
    "serq_linear_mx_addend", svds[i % 8].lin._h.ptr, acts[i % 8].codes.data_ptr(), acts[i % 8].sf.data_ptr(), M,
    cs[i % 8].data_ptr(), ys[i % 8].data_ptr(), N, D._stream()), 16)
out["linear_plain"] = B.time_steps(lambda i: svds[i % 8].lin.gemm(acts[i % 8], ys[i % 8]), 16)
out["whole"] = B.time_steps(lambda i: svds[i % 8].forward(xs[i % 8], ys[i % 8]), 16)
print(json.dumps({k: round(v * 1e3, 2) for k, v in out.items()}))
