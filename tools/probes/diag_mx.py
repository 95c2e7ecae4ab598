"""Roofline diagnostics for the MX linear (not a bench line): times the linear
with operand loads / output stores disabled to separate the MMA ceiling from
the feed, and the quantizer with and without an L2 flush."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2603_08185_b200 import device as D, _lib, api, workload as WL

M = int(os.environ.get("M", 4096)); K = int(os.environ.get("K", 4096)); N = int(os.environ.get("N", 4096)); R = 64
wl = WL.make_linear(K, N, M, R)
main_t, comp = api.build_serq_rtn_mx(wl.w, np.arange(R))
lin = D.MxLinear(main_t.element_codes, main_t.block_scale_exponents, comp.r_q.element_codes, comp.r_q.block_scale_exponents, np.arange(R))
x = torch.from_numpy(wl.x).to("cuda", torch.bfloat16)
act = lin.quantize(x); y = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
fa = torch.empty(64 << 20, device="cuda"); fb = torch.ones(64 << 20, device="cuda")
def flush():
    fa.zero_(); fb.sum()
def timeit(fn, n=20, fl=True):
    ts = []
    for i in range(n + 3):
        if fl: flush()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); fn(); e.record(); e.synchronize()
        if i >= 3: ts.append(s.elapsed_time(e))
    return statistics.median(ts) * 1e3
fl = 2.0 * M * N * (K + R)
out = {}
for flags in [int(f) for f in os.environ.get('FLAGS', '0,1,2,3').split(',')]:
    _lib.load().serq_set_debug_flags(flags)
    gg = torch.cuda.CUDAGraph()
    with torch.cuda.stream(torch.cuda.Stream()):
        lin.gemm(act, y); torch.cuda.synchronize()
        with torch.cuda.graph(gg):
            lin.gemm(act, y)
    t = timeit(lambda: gg.replay())
    out[f"linear_dbg{flags}_us"] = t; out[f"linear_dbg{flags}_tflops"] = fl / t / 1e6
qb = M * K * 2 + M * K // 2 + M * K // 32
for qf in (0,):
    _lib.load().serq_set_debug_flags(qf)
    for f in (True, False):
        t = timeit(lambda: lin.quantize(x, act), fl=f)
        out[f"quant{qf}_flush{int(f)}_us"] = t; out[f"quant{qf}_flush{int(f)}_GBs"] = qb / t / 1e3
_lib.load().serq_set_debug_flags(0)
print(json.dumps(out, indent=1))

# host-overhead check: back-to-back launches and CUDA-graph replay
def timed_loop(fn, n=20):
    torch.cuda.synchronize(); flush(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(n): fn()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / n * 1e3
res = {}
res["gemm_b2b_us"] = timed_loop(lambda: lin.gemm(act, y))
res["quant_b2b_us"] = timed_loop(lambda: lin.quantize(x, act))
g = torch.cuda.CUDAGraph()
s_ = torch.cuda.Stream()
with torch.cuda.stream(s_):
    lin.gemm(act, y); torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s_):
        lin.gemm(act, y)
res["gemm_graph_us"] = timed_loop(lambda: g.replay())
g2 = torch.cuda.CUDAGraph()
with torch.cuda.stream(s_):
    with torch.cuda.graph(g2, stream=s_):
        lin.quantize(x, act)
res["quant_graph_us"] = timed_loop(lambda: g2.replay())
res["gemm_graph_tflops"] = fl / res["gemm_graph_us"] / 1e6
res["quant_graph_GBs"] = qb / res["quant_graph_us"] / 1e3
# flushed + graph
def tf(gr):
    ts = []
    for i in range(23):
        flush()
        a_, b_ = torch.cuda.Event(True), torch.cuda.Event(True)
        a_.record(); gr.replay(); b_.record(); b_.synchronize()
        if i >= 3: ts.append(a_.elapsed_time(b_))
    return statistics.median(ts) * 1e3
res["gemm_graph_flushed_us"] = tf(g); res["quant_graph_flushed_us"] = tf(g2)
print(json.dumps(res, indent=1))
# HBM calibration: same harness, plain torch kernels over X (32 MiB bf16)
y2 = torch.empty_like(x)
cal = {}
cal["torch_copy_64MB_us"] = timeit(lambda: y2.copy_(x))
cal["torch_sum_32MB_us"] = timeit(lambda: x.sum(dtype=torch.float32))
xb = torch.empty(256 << 20, dtype=torch.uint8, device="cuda"); yb = torch.empty_like(xb)
cal["torch_copy_512MB_us"] = timeit(lambda: yb.copy_(xb), n=5)
cal["copy_64MB_GBs"] = 64 * 2**20 / cal["torch_copy_64MB_us"] / 1e3
cal["sum_32MB_GBs"] = 32 * 2**20 / cal["torch_sum_32MB_us"] / 1e3
cal["copy_512MB_GBs"] = 512 * 2**20 / cal["torch_copy_512MB_us"] / 1e3
print(json.dumps(cal, indent=1))
