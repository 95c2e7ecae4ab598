import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
from oracle import serq_oracle as O
from paper_2603_08185_b200 import bundle as BD
from paper_2603_08185_b200.block import DeviceBlock, rmsnorm
import test_bundle as TB
g = np.load("/root/repo/tests/golden/golden.npz")
bdir = "/root/repo/tests/golden/block_mx"
lins, gains = TB._oracle_block_linears(bdir)
b = BD.load_bundle_device(bdir)
x = g["block_x"]
h1 = O.rmsnorm(x, gains["ln1"])
h1d = rmsnorm(torch.from_numpy(x).cuda().float(), torch.from_numpy(gains["ln1"]).cuda().float())
print("h1 rel", np.abs(h1d.double().cpu().numpy() - h1).max() / np.abs(h1).max())
for name in ("q_proj", "k_proj", "v_proj"):
    yo = O.forward_mx(h1, *lins[name])
    yd = b.linears[name].linear(torch.from_numpy(h1).cuda().float()).double().cpu().numpy()
    print(name, O.parity_errors(yd, yo))
    # with bf16 input
    yd2 = b.linears[name].linear(torch.from_numpy(h1).cuda().bfloat16()).double().cpu().numpy()
    print(name, "bf16-in", O.parity_errors(yd2, O.forward_mx(O.bf16_round(h1), *lins[name])))
from paper_2603_08185_b200.block import attention_mix
hd = int(g["block_head_dim"])
def lo(name, xin): return O.forward_mx(xin, *lins[name])
def ld(name, xin): return b.linears[name].linear(torch.from_numpy(np.ascontiguousarray(xin)).cuda().float()).double().cpu().numpy()
q, k, v = lo("q_proj", h1), lo("k_proj", h1), lo("v_proj", h1)
ao = O.attention_mix(q, k, v, hd)
ad = attention_mix(torch.from_numpy(q).cuda().float(), torch.from_numpy(k).cuda().float(), torch.from_numpy(v).cuda().float(), hd).double().cpu().numpy()
print("attn rel", np.abs(ad - ao).max() / np.abs(ao).max())
res1 = x + lo("o_proj", ao)
print("o_proj", O.parity_errors(ld("o_proj", ao), lo("o_proj", ao)))
h2 = O.rmsnorm(res1, gains["ln2"])
for n in ("up_proj", "gate_proj"):
    print(n, O.parity_errors(ld(n, h2), lo(n, h2)))
mid = O.silu(lo("gate_proj", h2)) * lo("up_proj", h2)
print("down", O.parity_errors(ld("down_proj", mid), lo("down_proj", mid)))
blk = DeviceBlock.from_bundle(b, hd)
y = blk(torch.from_numpy(x).cuda().float()).double().cpu().numpy()
yo = O.forward_block_mx(x, lins, gains, hd)
print("block", np.abs(y - yo).max() / np.abs(yo).max(), np.abs(y - yo).mean() / np.abs(yo).mean())
print("golden vs oracle", np.abs(g["block_y_quant"] - yo).max())
