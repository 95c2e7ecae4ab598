"""Chunked pinned H2D (the host pipeline's plan) alone, and with the D2H chunks interleaved on a
second stream (each D2H after its H2D), timed with events: is the chunking itself slow?"""
import json
import torch

plan = [256, 512, 1024, 1024, 512, 512, 256]
row = 4096 * 2
n = sum(plan) * row
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_x = torch.empty(n, dtype=torch.uint8, device="cuda")
d_y = torch.empty(n, dtype=torch.uint8, device="cuda")
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
E = lambda: torch.cuda.Event(enable_timing=True)


def run(with_d2h):
    t0 = E()
    t0.record()
    s_in.wait_stream(torch.cuda.current_stream())
    s_out.wait_stream(torch.cuda.current_stream())
    ends_in, ends_out = [], []
    off = 0
    for mc in plan:
        b = mc * row
        with torch.cuda.stream(s_in):
            d_x[off:off + b].copy_(h_in[off:off + b], non_blocking=True)
            e = E()
            e.record()
            ends_in.append(e)
        if with_d2h:
            with torch.cuda.stream(s_out):
                s_out.wait_event(e)
                h_out[off:off + b].copy_(d_y[off:off + b], non_blocking=True)
                e2 = E()
                e2.record()
                ends_out.append(e2)
        off += b
    torch.cuda.synchronize()
    return [round(t0.elapsed_time(e) * 1e3, 1) for e in ends_in], [round(t0.elapsed_time(e) * 1e3, 1) for e in ends_out]


for w in (False, True, False, True):
    print(json.dumps(run(w)))

# two streams per direction (chunks alternate)
s_in2, s_out2 = torch.cuda.Stream(), torch.cuda.Stream()


def run2():
    t0 = E()
    t0.record()
    for s in (s_in, s_in2, s_out, s_out2):
        s.wait_stream(torch.cuda.current_stream())
    ends_in, ends_out = [], []
    off = 0
    for i, mc in enumerate(plan):
        b = mc * row
        si, so = (s_in, s_out) if i % 2 == 0 else (s_in2, s_out2)
        with torch.cuda.stream(si):
            d_x[off:off + b].copy_(h_in[off:off + b], non_blocking=True)
            e = E()
            e.record()
            ends_in.append(e)
        with torch.cuda.stream(so):
            so.wait_event(e)
            h_out[off:off + b].copy_(d_y[off:off + b], non_blocking=True)
            e2 = E()
            e2.record()
            ends_out.append(e2)
        off += b
    torch.cuda.synchronize()
    return [round(t0.elapsed_time(e) * 1e3, 1) for e in ends_in], [round(t0.elapsed_time(e) * 1e3, 1) for e in ends_out]


for _ in range(2):
    print("2x2", json.dumps(run2()))
plan = [128] * 32
for w in (True, True):
    print("128-row chunks", json.dumps(run(w))[-60:])
