"""Per-CTA timeline of the CTA-pair MX linear at 4096^3 (SERQ_DIAG_TS build),
whole tiles only (flags 0) vs the split last wave (flags 8192): per work item,
when its accumulator was complete and when its epilogue ended (us from the
first CTA entry), and the kernel's first entry / last exit."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2603_08185_b200 import build, _lib
diag = os.path.join(os.path.dirname(build.OUT), "libserq_b200_diag.so")
subprocess.run([build.nvcc()] + build.NVCC_FLAGS + ["-DSERQ_DIAG_TS", "-o", diag, build.SRC], check=True)
lib = _lib.load(diag); _lib._lib = lib
from paper_2603_08185_b200 import benchmarks as B
lin = B.device_mx_linear(4096, 4096, 64)
x = B.outlier_x(4096, 4096); act = lin.quantize(x); y = torch.empty((4096, 4096), dtype=torch.bfloat16, device="cuda")
for flags in [int(f) for f in os.environ.get('FLAGS', '0,8192').split(',')]:
    lib.serq_set_debug_flags(flags)
    ts = torch.zeros(8192, dtype=torch.int64, device="cuda")
    for _ in range(3): lin.gemm(act, y)
    torch.cuda.synchronize()
    lib.serq_set_debug_timestamps(ts.data_ptr()); lin.gemm(act, y); torch.cuda.synchronize()
    lib.serq_set_debug_timestamps(None)
    t = ts.cpu().numpy().astype(np.float64)
    ent = t[1024 + 148 * 24::2][:148]; ex = t[1024 + 148 * 24 + 1::2][:148]
    t0 = ent[ent > 0].min()
    print(f"flags={flags}: entry spread {(ent.max()-t0)/1e3:.2f} us, exit first/median/last "
          f"{(ex.min()-t0)/1e3:.2f}/{(np.median(ex)-t0)/1e3:.2f}/{(ex.max()-t0)/1e3:.2f} us")
    items = t[1024:1024 + 148 * 24].reshape(148, 6, 4)
    for i in range(6):
        v = items[:, i, :]
        ok = v[:, 1] > 0
        if not ok.any(): continue
        full = (v[ok, 1] - t0) / 1e3; end = (v[ok, 2] - t0) / 1e3; half = v[ok, 3]
        print(f"  item {i}: ctas={ok.sum():3d} halves={int((half >= 0).sum()):3d} acc done min/med/max "
              f"{full.min():6.2f}/{np.median(full):6.2f}/{full.max():6.2f}  epi end {end.min():6.2f}/{np.median(end):6.2f}/{end.max():6.2f}")
    sk = t[1024 + 148 * 24 + 296:1024 + 148 * 24 + 296 + 148 * 8].reshape(148, 8)[:, :6]
    ok = sk[:, 0] > 0
    if ok.any():
        names = ["publish issued", "publish landed", "flag raised", "partner flag seen", "partner partial in", "done"]
        for k, nm in enumerate(names):
            col = (sk[ok, k] - t0) / 1e3
            print(f"    split {nm:18s} min/med/max {col.min():6.2f}/{np.median(col):6.2f}/{col.max():6.2f}")
lib.serq_set_debug_flags(0)
