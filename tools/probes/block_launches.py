"""Kernel launch list of one fused-linear Llama-2-7B block forward at M tokens (as in the bench's
c4_block_fused point, fast attention) -- for ncu --metrics gpu__time_duration.sum."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2603_08185_b200 import benchmarks as B, device as D
from paper_2603_08185_b200.block import DeviceBlock
M = int(os.environ.get("M", "1"))
H, F, r, hd = 4096, 11008, 64, 128
rng = np.random.default_rng(9)
def parts(k, n, gather, s):
    idx = np.sort(rng.permutation(k)[:r]) if gather else None
    return B.device_mx_parts(k, n, r, seed=s, salient_idx=idx)
pq, pk, pv, pu, pg = parts(H, H, True, 1), parts(H, H, True, 2), parts(H, H, True, 3), parts(H, F, True, 5), parts(H, F, True, 6)
lins = {"qkv_proj": D.FusedMxLinear([pq, pk, pv]), "up_gate_proj": D.FusedMxLinear([pu, pg]),
        "o_proj": D.MxLinear(*parts(H, H, False, 4)), "down_proj": D.MxLinear(*parts(F, H, False, 7))}
blk = DeviceBlock(lins, {"ln1": np.ones(H), "ln2": np.ones(H)}, hd, fast_attention=True)
x = B.outlier_x(M, H).float()
for _ in range(2):
    blk(x)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()  # ncu --profile-from-start off: one forward only
blk(x)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
