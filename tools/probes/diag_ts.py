import os, sys, json, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2603_08185_b200 import build, _lib
# diagnostic build with timestamps compiled in, loaded from a separate path
diag = os.path.join(os.path.dirname(build.OUT), "libserq_b200_diag.so")
subprocess.run([build.nvcc()] + build.NVCC_FLAGS + ["-DSERQ_DIAG_TS", "-o", diag, build.SRC], check=True)
lib = _lib.load(diag)
_lib._lib = lib
from paper_2603_08185_b200 import device as D, api, workload as WL
M = K = N = 4096; R = 64
wl = WL.make_linear(K, N, M, R)
main_t, comp = api.build_serq_rtn_mx(wl.w, np.arange(R))
lin = D.MxLinear(main_t.element_codes, main_t.block_scale_exponents, comp.r_q.element_codes, comp.r_q.block_scale_exponents, np.arange(R))
x = torch.from_numpy(wl.x).to("cuda", torch.bfloat16)
act = lin.quantize(x); y = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
ts = torch.zeros(512, dtype=torch.int64, device="cuda")
np.set_printoptions(linewidth=200)
for flags in [int(f) for f in os.environ.get("FLAGS", "0,15").split(",")]:
    lib.serq_set_debug_flags(flags)
    lib.serq_set_debug_timestamps(None)
    for _ in range(5): lin.gemm(act, y)
    lib.serq_set_debug_timestamps(ts.data_ptr())
    lin.gemm(act, y); torch.cuda.synchronize()
    lib.serq_set_debug_timestamps(None)
    full = ts.cpu().numpy()
    cyc, ns = full[509] - full[508], full[511] - full[510]
    print(f"flags={flags}: MMA warp of CTA 0: {cyc} cycles in {ns} ns -> {cyc / ns:.3f} GHz")
    t = full[:400].reshape(100, 4)
    d = np.diff(t, axis=1)
    print("unit: [issue part1, wait next, last mma+commit], gap to next unit")
    for u in range(0, 20):
        print(u, d[u].tolist(), int(t[u + 1, 0] - t[u, 3]))
