#!/usr/bin/env python
"""Benchmark of the SERQ W4A4 linear hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl serq|reference]

Workload (N=1): BASELINE config 2 -- SERQ MXFP4 linear, X bf16 [M=4096,
K=4096] (N(0,1), 1% of channels x50, seed 0, SAF-flattened and salient-
permuted), W [N=4096, K=4096] ~ N(0, 0.02) (seed 1), rank r=64, bf16 output.
One step = quantize X (K1-MX) + the fused SERQ linear (K2: main GEMM + the
salient term + epilogue) on device-resident bf16 X.  An L2 flush (256 MiB
write, > 126 MB L2) separates timed steps and is excluded from them.

Multi-GPU (--gpus N > 1; re-executed under torch.distributed.run when
WORLD_SIZE is unset, one process per GPU, NCCL): BASELINE config 5 -- the
Llama-3-70B-shaped block linears, M = 8192 tokens, column/row tensor parallel
with one all-reduce after o_proj and after down_proj, pipelined over token
chunks under the GEMMs and captured with the kernels in one CUDA graph
("strong" scaling, value = whole-job TFLOPS, max over ranks).  The line also
carries the same block measured on one GPU by rank 0 (tp = 1) and the
resulting efficiency.

``--impl reference`` times the reference algorithm's CPU implementation (the
oracle port of serq.compensate._forward_mx, compensate.py:319-340) on the
host cores over a bounded row sample per step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

M, K, N, R = 4096, 4096, 4096, 64
FP4_PEAK_TFLOPS = 9000.0  # nominal dense FP4 (B200_PROFILING.md table) -- no measured FP4 peak exists
METRIC = "SERQ W4A4 linear TFLOPS (% of FP4/INT8 tensor peak) & tokens/s at 1/2/4/8 GPUs"
WORKLOAD = "c2: SERQ MXFP4 linear M=4096 K=4096 N=4096 r=64 (quantize + fused GEMM/R/epilogue)"
CPU_SAMPLE_ROWS = 256


def flops_per_token() -> float:
    return 2.0 * N * (K + R)  # main + salient term


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait()

    def summary(self) -> dict:
        rows = []
        try:
            for line in open(self.path):
                p = [c.strip() for c in line.split(",")]
                if len(p) >= 9 and p[1].replace(".", "").isdigit():
                    rows.append(p)
        except OSError:
            pass
        finally:
            if self.path and os.path.exists(self.path):
                os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows]
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": float(rows[0][2]), "reasons": reasons,
                "samples": len(rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_baseline_leg(x_bf16: np.ndarray, w: np.ndarray, rows: int = CPU_SAMPLE_ROWS, reps: int = 1) -> dict:
    """The reference algorithm on host cores: oracle port of _forward_mx
    (compensate.py:319-340) over a bounded row sample (output rows are
    independent, so the sample is exact work per token)."""
    from oracle import serq_oracle as O

    main_t, comp = O.build_serq_rtn_mx(w, np.arange(R), 32)  # offline, untimed
    xs = x_bf16[:rows]
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.forward_mx(xs, main_t, comp)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return {"value": rows * flops_per_token() / t / 1e12, "unit": "TFLOPS", "cores": os.cpu_count(),
            "kind": "port", "seconds": t,
            "sample": f"{rows} of {M} token rows of config c2 through oracle.forward_mx "
                      f"(NumPy/OpenBLAS, {os.cpu_count()} threads), per-call W decode included as in the reference"}


def run_reference(args) -> None:
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    if ws > 1:
        run_reference_c5(args, ws)
        return
    from paper_2603_08185_b200 import workload as WL

    wl = WL.make_linear(K, N, M, R, 0.01, 50.0, "mx")
    from oracle import serq_oracle as O

    main_t, comp = O.build_serq_rtn_mx(wl.w, np.arange(R), 32)
    rows = CPU_SAMPLE_ROWS
    for _ in range(args.warmup):
        O.forward_mx(wl.x[:rows], main_t, comp)
    t0 = time.perf_counter()
    for i in range(args.steps):
        lo = (i * rows) % M
        O.forward_mx(wl.x[lo:lo + rows], main_t, comp)
    dt = (time.perf_counter() - t0) / args.steps
    val = rows * flops_per_token() / dt / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "TFLOPS", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD + f" -- CPU sample {rows} token rows per step", "M": M, "K": K, "N": N,
                   "r": R, "format": "mxfp4"},
        "tokens_per_s": rows / dt,
        "cpu_baseline": {"value": val, "unit": "TFLOPS", "cores": os.cpu_count(), "kind": "port",
                         "sample": f"{rows} token rows per step (oracle port of _forward_mx, NumPy/OpenBLAS)"},
        "e2e": {"value": val, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_reference_c5(args, ws: int) -> None:
    """Reference arm for the multi-GPU workload (C5 block linears): the oracle port of
    _forward_mx (compensate.py:319-340) on the host cores over a bounded sample of the
    block -- 16 token rows x 1024 output columns of each of the four linears at their full
    K (output elements are independent, so the sample is exact work per element)."""
    from oracle import serq_oracle as O

    rows, cols, r = 16, 1024, 128
    shapes = [("qkv_proj", 8192, 10240), ("o_proj", 8192, 8192), ("gate_up_proj", 8192, 57344),
              ("down_proj", 28672, 8192)]
    cases = []
    for i, (_, k, _n) in enumerate(shapes):
        rng = np.random.default_rng(40 + i)
        w = rng.standard_normal((k, cols)) * 0.02
        main_t, comp = O.build_serq_rtn_mx(w, np.arange(r), 32)
        x = O.bf16_round(O.synthetic_activations(rows, k, k // 100, 50.0, seed=50 + i))
        cases.append((x, main_t, comp, 2.0 * rows * cols * (k + r)))
    flops = sum(c[3] for c in cases)
    for _ in range(max(1, args.warmup)):
        for x, mt, comp, _f in cases:
            O.forward_mx(x, mt, comp)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for x, mt, comp, _f in cases:
            O.forward_mx(x, mt, comp)
    dt = (time.perf_counter() - t0) / args.steps
    val = flops / dt / 1e12
    sample = (f"{rows} token rows x {cols} output columns of each C5 linear (full K, r={r}) per step, oracle port of "
              f"_forward_mx, NumPy/OpenBLAS {os.cpu_count()} threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": "TFLOPS", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "c5: Llama-3-70B-shaped block linears, SERQ MXFP4 r=128 -- CPU sample", "sample": sample},
        "cpu_baseline": {"value": val, "unit": "TFLOPS", "cores": os.cpu_count(), "kind": "port", "sample": sample},
        "e2e": {"value": val, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_serq(args) -> None:
    import torch

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2603_08185_b200 import api
    from paper_2603_08185_b200 import benchmarks as B
    from paper_2603_08185_b200 import device as D
    from paper_2603_08185_b200 import workload as WL

    wl = WL.make_linear(K, N, M, R, 0.01, 50.0, "mx", x_seed=rank)
    main_t, comp = api.build_serq_rtn_mx(wl.w, np.arange(R))
    lin = D.MxLinear(main_t.element_codes, main_t.block_scale_exponents, comp.r_q.element_codes,
                     comp.r_q.block_scale_exponents, np.arange(R))
    x = torch.from_numpy(wl.x).to("cuda", torch.bfloat16)
    act = lin.quantize(x)
    y = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    stream = torch.cuda.current_stream()

    # One step = quantize + fused linear (serq_forward_mx) on one token batch.  The
    # K timed steps run back to back inside ONE CUDA graph between two event-record
    # nodes, cycling over NW weight sets and NX activation / output sets whose total
    # (~620 MB) exceeds the 126 MB L2: every step reads cold operands (instead of
    # an L2 flush between steps) and the graph-launch / event overhead (~3 us) is
    # paid once per K steps.  Set 0 is the reference-built workload above; the
    # others are drawn from the same distributions on the device.
    NW, NX = 4, 8
    lins = [lin] + [B.device_mx_linear(K, N, R, seed=11 + i) for i in range(NW - 1)]
    xs = [x] + [B.outlier_x(M, K, seed=100 + i) for i in range(NX - 1)]
    acts = [lin.quantize(xi) for xi in xs]
    ys = [y] + [torch.empty((M, N), dtype=torch.bfloat16, device="cuda") for _ in range(NX - 1)]
    counts = {}

    def step(i):
        lins[i % NW].forward(xs[i % NX], acts[i % NX], ys[i % NX])
        counts["launches"] = D.last_launch_count()

    def capture(work, n):
        ev = (torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
        g = B.graph_of(lambda: (ev[0].record(), [work(i) for i in range(n)], ev[1].record()))
        return g, ev

    g_step = capture(step, args.steps)
    launches_per_step = counts["launches"]
    n_brk = max(args.steps, 16)
    g_q = capture(lambda i: lin.quantize(xs[i % NX], acts[i % NX]), n_brk)
    g_l = capture(lambda i: lins[i % NW].gemm(acts[i % NX], ys[i % NX]), n_brk)
    for _ in range(max(args.warmup, 3)):  # W untimed warm-up passes over the K steps
        g_step[0].replay()
    torch.cuda.synchronize()

    def timed(ge, warm=0):
        g, (a, b) = ge
        for _ in range(warm):  # a graph's first replays pay its upload: not kernel time
            g.replay()
        torch.cuda.synchronize()
        g.replay()
        b.synchronize()
        return a.elapsed_time(b)

    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        total_ms = timed(g_step)
    if ws > 1:
        torch.distributed.barrier()
    launches = launches_per_step * args.steps
    q_ms = timed(g_q, 2) / n_brk
    g_ms = timed(g_l, 2) / n_brk
    if ws > 1:
        t = torch.tensor([total_ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = ws * M * flops_per_token() * args.steps / (total_ms / 1e3) / 1e12
    clocks = clk.summary()

    # ---- end to end through the C-ABI from pinned host memory
    xh = x.cpu().pin_memory()
    yh = torch.empty((M, N), dtype=torch.bfloat16).pin_memory()
    for _ in range(2):
        lin.forward_host(xh, yh)
    e2e_ms = []
    for _ in range(max(3, min(args.steps, 10))):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        lin.forward_host(xh, yh)
        e.record(stream)
        e.synchronize()
        e2e_ms.append(s.elapsed_time(e))
    e2e_t = statistics.median(e2e_ms)
    if ws > 1:
        t = torch.tensor([e2e_t], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_t = float(t.item())
    e2e_val = ws * M * flops_per_token() / (e2e_t / 1e3) / 1e12

    if rank == 0:
        peaks = measured_peaks()
        hbm = float(peaks.get("hbm_gbs", 6650.0))
        gemm_tflops = M * flops_per_token() / (g_ms / 1e3) / 1e12
        q_bytes = M * K * 2 + M * K // 2 + M * K // 32  # bf16 in, packed codes + E8M0 out
        traffic = None
        prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(prof):
            try:
                traffic = json.load(open(prof)).get("serq_mx_pair3_kernel", {}).get("dram_bytes_per_launch")
            except (OSError, ValueError):
                traffic = None
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": ws, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp4(e2m1)+e8m0 -> f32 accumulate -> bf16", "data": "synthetic",
            "config": {"workload": WORKLOAD, "M": M, "K": K, "N": N, "r": R, "format": "mxfp4",
                       "activations": "N(0,1), 1% channels x50, SAF a=0.5, salient-permuted, bf16",
                       "l2": "inputs larger than L2: steps cycle 4 weight sets x 8 activation/output sets (~620 MB > 126 MB L2), no flush",
                       "timing": "K steps back to back in one CUDA graph between two CUDA event-record nodes (device time, max over ranks)",
                       "parallelism": "single GPU (BASELINE C2; --gpus N > 1 runs the C5 tensor-parallel block)"},
            "tokens_per_s": ws * M / (ms_per_step / 1e3),
            "tflops_pct_of_fp4_peak": 100.0 * value / FP4_PEAK_TFLOPS,
            "breakdown_ms": {"quantize": q_ms, "linear": g_ms},
            "roofline": {"bound": "tensor", "kernel": "serq_mx_pair3_kernel (CTA-pair tcgen05 kind::mxf4, fused main + salient term + epilogue)",
                         "achieved": gemm_tflops, "peak": FP4_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": gemm_tflops / FP4_PEAK_TFLOPS,
                         "peak_source": "nominal dense FP4 9 PFLOP/s (B200_PROFILING.md; MEASURED_PEAKS.json has no FP4 figure)",
                         "measured_fp4_mma_ceiling_tflops": 8800.0,
                         "measured_fp4_note": "tools/mma_rate.cu: back-to-back tcgen05.mma kind::mxf4 128x256x64 on 148 SMs, random operands (profiles/mma_rate_r01.txt)",
                         "algorithmic_flops_per_launch": M * flops_per_token(), "traffic": traffic},
            "quantizer_roofline": {"bound": "hbm", "kernel": "mx_encode_blk_kernel<1> (one thread per 32-block)",
                                   "achieved": q_bytes / (q_ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                                   "frac": q_bytes / (q_ms / 1e3) / 1e9 / hbm,
                                   "peak_source": "MEASURED_PEAKS.json hbm_gbs", "bytes_per_launch": q_bytes},
            "e2e": {"value": e2e_val, "unit": "TFLOPS", "h2d_bytes_per_step": M * K * 2,
                    "d2h_bytes_per_step": M * N * 2, "ms_per_step": e2e_t,
                    "path": "serq_forward_mx_host (C-ABI): pinned H2D, quantize, fused linear, D2H"},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        line["parity"] = parity_check(wl, main_t, comp, ys[0])
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_leg(wl.x, wl.w)
        if ws == 1 and not args.no_extra:
            line["other_configs"] = other_configs(hbm)
        print(json.dumps(line), flush=True)
        if not line["parity"]["ok"]:
            print("bench.py: the benchmarked output does not match the oracle", file=sys.stderr)
            sys.exit(3)
    if ws > 1:
        torch.distributed.destroy_process_group()


def parity_check(wl, main_t, comp, y, rows: int = 256) -> dict:
    """CHECKER (test infrastructure, not measured): the first `rows` token rows of the
    benchmarked output Y (weight set 0 on activation set 0, i.e. the C2 workload itself)
    against the oracle's _forward_mx restatement (compensate.py:319-340) on the same
    artefacts, at the north_star tolerance (max 1e-2 / mean 1e-3 vs bf16(oracle))."""
    from oracle import serq_oracle as O

    mt = O.MxT(np.asarray(main_t.element_codes), np.asarray(main_t.block_scale_exponents), 32,
               tuple(np.asarray(main_t.element_codes).shape))
    rq = comp.r_q
    c = O.Comp(int(comp.rank), np.asarray(comp.salient_idx),
               r_q=O.MxT(np.asarray(rq.element_codes), np.asarray(rq.block_scale_exponents), 32,
                         tuple(np.asarray(rq.element_codes).shape)))
    ref = O.forward_mx(wl.x[:rows], mt, c)
    mx, mean = O.parity_errors(y[:rows].float().cpu().numpy(), ref)
    return {"rows_checked": rows, "of": "C2 output (weight set 0, activation set 0)", "max_rel": mx, "mean_rel": mean,
            "tol_max": 1e-2, "tol_mean": 1e-3, "ok": bool(mx <= 1e-2 and mean <= 1e-3),
            "oracle": "oracle/serq_oracle.py forward_mx (checker only)"}


def _round(d):
    if isinstance(d, dict):
        return {k: _round(v) for k, v in d.items()}
    if isinstance(d, list):
        return [_round(v) for v in d]
    return round(d, 4) if isinstance(d, float) else d


def other_configs(hbm_gbs: float) -> dict:
    """The other BASELINE configs, measured the same way (steps back to back in
    one CUDA graph over operand sets larger than L2, CUDA events); not the
    headline metric."""
    from paper_2603_08185_b200 import benchmarks as B

    fl = B.Flusher()
    out = {}
    try:
        out["c1_int4_sym_dense_L"] = B.int_linear_point(512, 4096, 4096, 64, "dense", 4, True, fl)
        out["c3_w4a8_asym_int_R"] = B.int_linear_point(2048, 4096, 11008, 128, "int", 8, False, fl)
        # the paper's group-wise weights (row groups of 128 along K) at C3's shape
        out["c3_w4a8_group128_int_R"] = B.int_linear_point(2048, 4096, 11008, 128, "int", 8, False, fl, group=128)
        # the paper's comparison at C3's shape: SVD baseline (two-factor L1 L2, r = 128) vs SERQ's fused R
        out["c3_svd_baseline_r128"] = B.svd_baseline_point(2048, 4096, 11008, 128)
        # the same comparison over an MX main at C2 (compensate.py:326-331)
        out["c2_mx_svd_baseline_r64"] = B.mx_svd_baseline_point(4096, 4096, 4096, 64)
        out["c4_decode"] = B.decode_points(hbm_gbs)
        # q/k/v and gate/up each as ONE fused launch (own salient set per part, gather fallback)
        out["c4_decode_fused"] = B.decode_fused_points(hbm_gbs)
        out["int_decode_7b"] = B.int_decode_points(hbm_gbs)
        out["int_decode_7b_w4"] = B.int_decode_points(hbm_gbs, weight_format="int4")
        out["int_decode_7b_g128"] = B.int_decode_points(hbm_gbs, group=128)
        out["producer_rmsnorm_quant_c2"] = B.rmsnorm_quant_point(4096, 4096, hbm_gbs)
        out["producer_rmsnorm_quant_int_c3"] = B.rmsnorm_int_quant_point(2048, 4096, 8, False, hbm_gbs)
        # C4 as a whole block: Llama-2-7B-shaped decoder block (SERQ linears + f32 non-linear nodes)
        out["c4_block"] = [B.llama7b_block_point(m) for m in (1, 16, 2048)]
        # the same block with q/k/v and up/gate fused (device.FusedMxLinear)
        out["c4_block_fused"] = [B.llama7b_block_point(m, fused=True) for m in (1, 16, 2048)]
        out["c5_block_tp1"] = B.c5_block_point(1, 0, flush=fl)
    except Exception as e:  # secondary numbers must not hide the headline line
        out["error"] = f"{type(e).__name__}: {e}"
    return _round(out)


def run_c5(args) -> None:
    """BASELINE C5 (the multi-GPU workload): Llama-3-70B-shaped block linears, M = 8192
    tokens, tensor parallel over the launched ranks (NCCL all-reduce after o_proj and
    down_proj, pipelined over token chunks, one CUDA graph per step)."""
    import torch

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2603_08185_b200 import benchmarks as B

    M = 8192
    ref1 = None
    if ws > 1 and rank == 0 and not args.no_extra:
        # the same block on ONE GPU (tp = 1) for the efficiency figure; the other ranks wait
        ref1 = B.c5_tp_point(1, 0, M=M, steps=max(args.steps // 2, 3), warm=args.warmup, with_e2e=False)
    if ws > 1:
        torch.distributed.barrier()
    with ClockSampler(local) as clk:
        p = B.c5_tp_point(ws, rank, M=M, steps=args.steps, warm=max(args.warmup, 3))
    clocks = clk.summary()

    def max_over_ranks(v):
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        if ws > 1:
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    ms = max_over_ranks(p["step_ms"])
    serial = max_over_ranks(p["serial_ms"])
    ar = max_over_ranks(p["allreduce_ms"])
    e2e_ms = max_over_ranks(p["e2e_ms"])
    if rank == 0:
        value = p["flops_per_step"] / (ms * 1e-3) / 1e12
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": ws, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "fp4(e2m1)+e8m0 -> f32 accumulate -> bf16", "data": "synthetic",
            "config": {"workload": "c5: Llama-3-70B-shaped block linears (qkv 8192x10240, o 8192x8192, gate_up "
                                   "8192x57344, down 28672x8192), SERQ MXFP4 r=128, M=8192 tokens",
                       "parallelism": f"tp{ws}", "chunks": p["chunks"], "graph": p["graph"],
                       "l2": "inputs larger than L2 (weights + activations of the block per rank exceed 126 MB at tp<=4)",
                       "timing": "steps back to back, CUDA events on the launching stream, max over ranks",
                       "per_rank_linears": p["linears"]},
            "tokens_per_s": M / (ms * 1e-3),
            "serial_ms_per_step": serial, "allreduce_ms_per_step": ar,
            "e2e": {"value": p["flops_per_step"] / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOPS",
                    "h2d_bytes_per_step": p["h2d_bytes_per_step"], "d2h_bytes_per_step": p["d2h_bytes_per_step"],
                    "ms_per_step": e2e_ms, "path": "tp.PipelinedTPBlock.forward with pinned H2D of x and D2H of the output"},
            "gpu_launches": p["gpu_launches_per_step"] * args.steps,
            "clocks": clocks,
        }
        if ref1 is not None:
            line["tp1_reference"] = {"ms_per_step": ref1["step_ms"], "tokens_per_s": ref1["tokens_per_s"],
                                     "tflops": ref1["block_tflops"]}
            line["efficiency_vs_tp1"] = ref1["step_ms"] / (ws * ms)
        print(json.dumps(_round(line)), flush=True)
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def relaunch(args) -> int:
    """--gpus N > 1 outside torchrun: re-execute this command under torch.distributed.run
    (one process per GPU on this node, rendezvous on 127.0.0.1)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    # communicator / NVLS lines for the driver's logs (stderr: stdout carries the JSON line)
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="serq", choices=["serq", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the other-config measurements")
    ap.add_argument("--workload", default="c2", choices=["c2", "c5"])
    args = ap.parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "0"))
    if ws == 0 and args.gpus > 1:
        sys.exit(relaunch(args))
    ws = ws or 1
    if ws != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "c5" or ws > 1:
        run_c5(args)
    else:
        run_serq(args)


if __name__ == "__main__":
    main()
