"""K1-INT (A8 asym) cold timing at C3 / C1 / 4096^2 / 8192^2 -- run once per library variant
(SERQ_B200_LIB) to compare rows-per-CTA settings."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
from paper_2603_08185_b200 import benchmarks as B, device as D  # noqa: E402

out = {}
for M, K, bits, sym in [(2048, 4096, 8, False), (512, 4096, 4, True), (4096, 4096, 8, False), (8192, 8192, 8, False)]:
    xs = [B.outlier_x(M, K, seed=i) for i in range(16)]
    out[f"{M}x{K}"] = round(B.time_steps(lambda i: D.quantize_int(xs[i % 16], bits, sym), 32) * 1e3, 2)
    del xs
    torch.cuda.empty_cache()
print(os.environ.get("SERQ_B200_LIB", "default"), json.dumps(out))
