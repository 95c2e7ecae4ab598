"""K1-MX / K1-INT timing, cold (16 activation sets > L2) vs warm (one set), 4096 x 4096 and
C3's 2048 x 4096: bytes moved per launch / time against the measured HBM copy rate."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2603_08185_b200 import benchmarks as B, device as D

for M, K in [(4096, 4096), (8192, 8192), (2048, 4096)]:
    xs = [B.outlier_x(M, K, seed=i) for i in range(16)]
    acts = [D.quantize_mx(x) for x in xs]
    byts = 2 * M * K + M * K // 2 + M * K // 32
    cold = B.time_steps(lambda i: D.quantize_mx(xs[i % 16], None, acts[i % 16]), 32)
    warm = B.time_steps(lambda i: D.quantize_mx(xs[0], None, acts[0]), 32)
    ib = 2 * M * K + M * K + 16 * M
    icold = B.time_steps(lambda i: D.quantize_int(xs[i % 16], 8, False), 32)
    print(json.dumps({"M": M, "K": K, "mx_cold_us": round(cold * 1e3, 2), "mx_cold_tbs": round(byts / cold / 1e9, 2),
                      "mx_warm_us": round(warm * 1e3, 2), "int8_cold_us": round(icold * 1e3, 2),
                      "int8_cold_tbs": round(ib / icold / 1e9, 2)}), flush=True)
    del xs, acts
    torch.cuda.empty_cache()
