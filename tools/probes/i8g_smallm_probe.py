"""Group-wise INT weights (g = 128) at decode / small M: per-layer time in an 8-layer graph and the
kernel that runs (Llama-2-7B up_proj / down_proj, integer R r = 128)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
from paper_2603_08185_b200 import benchmarks as B, device as D  # noqa: E402

L = 8
for K, N in ((4096, 11008), (11008, 4096)):
    if K % 128:
        continue
    lins = [B.device_int_linear(K, N, 128, "int", seed=1 + i, group=128) for i in range(L)]
    for M in [int(v) for v in os.environ.get("MS", "1,16,64").split(",")]:
        xs = [B.outlier_x(M, K, seed=i) for i in range(L)]
        acts = [lins[0].quantize(x, 8, False) for x in xs]
        ys = [torch.empty((M, N), dtype=torch.bfloat16, device="cuda") for _ in xs]
        t = B.time_steps(lambda i: lins[i % L].gemm(acts[i % L], ys[i % L]), 2 * L) * 1e3
        print(json.dumps({"K": K, "N": N, "M": M, "linear_us": round(t, 2), "kernel": D.last_kernel(),
                          "tbps": round((K * N + 128 * N + 4 * N * K / 128) / (t * 1e-6) / 1e12, 2)}), flush=True)
    del lins
    torch.cuda.empty_cache()
