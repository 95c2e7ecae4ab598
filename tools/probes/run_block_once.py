"""One Llama-2-7B-shaped device block forward at M tokens (ncu launch-list target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2603_08185_b200 import benchmarks as B
from paper_2603_08185_b200.block import DeviceBlock
M = int(os.environ.get("M", "1"))
H, F, r = 4096, 11008, 64
rng = np.random.default_rng(9)
def lin(k, n, gather, s):
    idx = np.sort(rng.permutation(k)[:r]) if gather else None
    return B.device_mx_linear(k, n, r, seed=s, salient_idx=idx)
lins = {"q_proj": lin(H, H, True, 1), "k_proj": lin(H, H, True, 2), "v_proj": lin(H, H, True, 3),
        "o_proj": lin(H, H, False, 4), "up_proj": lin(H, F, True, 5), "gate_proj": lin(H, F, True, 6),
        "down_proj": lin(F, H, False, 7)}
blk = DeviceBlock(lins, {"ln1": np.ones(H), "ln2": np.ones(H)}, 128)
x = B.outlier_x(M, H).float()
for _ in range(3):
    blk(x)
torch.cuda.synchronize()
print("ok")
