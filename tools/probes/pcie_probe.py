"""PCIe probe: pinned H2D alone, D2H alone, and both at once on two streams."""
import json
import torch

n = 32 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=10):
    import time
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d(); d2h()


out = {"bytes": n}
for name, fn in [("h2d", h2d), ("d2h", d2h), ("both", both)]:
    dt = t(fn)
    out[name + "_ms"] = dt * 1e3
    out[name + "_gbs"] = (2 * n if name == "both" else n) / dt / 1e9
print(json.dumps(out))
