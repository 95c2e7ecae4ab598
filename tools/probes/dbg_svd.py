import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
from oracle import serq_oracle as O
from paper_2603_08185_b200 import device as D, _lib
g = np.load("tests/golden/golden.npz")
lin = D.SvdMxLinear(g["fmx_main_codes"], g["fmx_main_exps"], g["fmxsvd_l1"], g["fmxsvd_l2"])
x = torch.from_numpy(g["fmx_x"]).cuda().to(torch.bfloat16)
y = lin(x).double().cpu().numpy()
act = lin.lin.quantize(x)
y0 = lin.lin.gemm(act).double().cpu().numpy()
main_t = O.MxT(g["fmx_main_codes"], g["fmx_main_exps"], 32, g["fmx_main_codes"].shape)
ymain = O.forward_mx(g["fmx_x"], main_t, None)
yref = g["fmxsvd_y"]
print("main parity", O.parity_errors(y0, ymain))
print("y vs main only", np.abs(y - y0).max(), "corr size", np.abs(yref - ymain).max(), np.abs(ymain).max())
xhat = D.mx_decode_bf16(act).double().cpu().numpy()
print("xhat exact", np.array_equal(xhat, O.mx_decode(O.mx_encode(g["fmx_x"], 32))))
c = (xhat @ g["fmxsvd_l1"]) @ g["fmxsvd_l2"]
print("corr vs ref", np.abs(c - (yref - ymain)).max())
print("y - y0 vs c", np.abs((y - y0) - c).max())
print(D.last_kernel())
