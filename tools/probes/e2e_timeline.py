"""Timeline of the chunked host pipeline (same plan as serq_forward_mx_host), rebuilt with
timing events on three streams: per chunk H2D / compute / D2H spans in us."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2603_08185_b200 import benchmarks as B

M = K = N = 4096
lin = B.device_mx_linear(K, N, 64)
x = B.outlier_x(M, K)
xh = x.cpu().pin_memory()
yh = torch.empty((M, N), dtype=torch.bfloat16).pin_memory()
xd = torch.empty((M, K), dtype=torch.bfloat16, device="cuda")
yd = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
plan = [int(v) for v in os.environ.get("PLAN", "256,512,1024,1024,512,512,256").split(",")]
s_in, s_c, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
acts = []
r0 = 0
for mc in plan:
    acts.append(lin.quantize(xd[r0:r0 + mc]))
    r0 += mc


def run(record):
    ev = {k: [] for k in ("h0", "h1", "c0", "c1", "o0", "o1")}
    E = lambda: torch.cuda.Event(enable_timing=True)
    start = E()
    start.record(torch.cuda.current_stream())
    s_in.wait_stream(torch.cuda.current_stream())
    r0 = 0
    for mc in plan:
        a, b = E(), E()
        a.record(s_in)
        xd[r0:r0 + mc].copy_(xh[r0:r0 + mc], non_blocking=True) if False else None
        with torch.cuda.stream(s_in):
            xd[r0:r0 + mc].copy_(xh[r0:r0 + mc], non_blocking=True)
        b.record(s_in)
        ev["h0"].append(a); ev["h1"].append(b)
        r0 += mc
    r0 = 0
    for c, mc in enumerate(plan):
        s_c.wait_event(ev["h1"][c])
        a, b = E(), E()
        a.record(s_c)
        with torch.cuda.stream(s_c):
            lin.forward(xd[r0:r0 + mc], acts[c], yd[r0:r0 + mc])
        b.record(s_c)
        ev["c0"].append(a); ev["c1"].append(b)
        s_out.wait_event(b)
        a2, b2 = E(), E()
        a2.record(s_out)
        with torch.cuda.stream(s_out):
            yh[r0:r0 + mc].copy_(yd[r0:r0 + mc], non_blocking=True)
        b2.record(s_out)
        ev["o0"].append(a2); ev["o1"].append(b2)
        r0 += mc
    torch.cuda.synchronize()
    if record:
        for c in range(len(plan)):
            print(json.dumps({"chunk": c, "rows": plan[c],
                              **{k: round(start.elapsed_time(ev[k][c]) * 1e3, 1) for k in ev}}), flush=True)
        print("total_us", round(start.elapsed_time(ev["o1"][-1]) * 1e3, 1))


for i in range(3):
    run(i == 2)
