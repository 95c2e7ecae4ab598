"""Secondary measurements reported beside the headline bench line (BASELINE
configs other than C2): decode (C4), integer linears (C1, C3) and the
Llama-70B-shaped block linears (C5, tp=1 on one GPU).

Every measurement replays a CUDA graph of the hot path (quantize + fused
linear) with the L2 flushed before each replay, timed with CUDA events on the
launching stream.  Weights are synthetic N(0, 0.02) encoded on the device;
activations follow the reference's outlier recipe (tensorio.py:157-168).
"""

from __future__ import annotations

import statistics

import numpy as np
import torch

from . import device as D


class Flusher:
    def __init__(self):
        self.a = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
        self.b = torch.ones(64 << 20, dtype=torch.float32, device="cuda")

    def __call__(self):
        self.a.zero_()
        self.b.sum()


def graph_of(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.synchronize()
    return g


def time_in_graph(fn, flush: Flusher | None = None, n=20, warm=3) -> float:
    """Median device time (ms) of fn() measured by CUDA event-record nodes INSIDE
    one captured graph [flush, event, fn, event]: excludes the graph launch
    latency (~6 us for a one-kernel graph on this box) and the L2 flush."""
    a = torch.cuda.Event(enable_timing=True, external=True)
    b = torch.cuda.Event(enable_timing=True, external=True)

    def body():
        if flush is not None:
            flush()
        a.record()
        fn()
        b.record()

    g = graph_of(body)
    ts = []
    for i in range(n + warm):
        g.replay()
        torch.cuda.synchronize()
        if i >= warm:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def time_steps(step, n_steps: int, warm: int = 2) -> float:
    """Device time per step (ms): ONE captured graph [event, step(0), ...,
    step(n_steps - 1), event], replayed once after `warm` untimed replays.  The
    caller's step(i) cycles over input / weight sets whose total size exceeds
    the 126 MB L2, so every step reads cold operands (the alternative to an L2
    flush between steps); the two event nodes add ~3 us once per graph, not per
    step (a one-kernel graph timed alone reads ~6 us above the kernel)."""
    a = torch.cuda.Event(enable_timing=True, external=True)
    b = torch.cuda.Event(enable_timing=True, external=True)

    def body():
        a.record()
        for i in range(n_steps):
            step(i)
        b.record()

    g = graph_of(body)
    for _ in range(warm):
        g.replay()
    torch.cuda.synchronize()
    g.replay()
    b.synchronize()
    return a.elapsed_time(b) / n_steps


def time_graph(g, flush: Flusher | None, n=20, warm=3):
    ts = []
    for i in range(n + warm):
        if flush is not None:
            flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        if i >= warm:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def device_mx_linear(K: int, N: int, r: int, seed: int = 1, salient_idx=None):
    """Synthetic SERQ MX linear built on the device: W ~ N(0, 0.02) [K, N],
    main_t = mx_encode(W^T), R = exact residual of the first r rows (the
    salient rows after the offline permutation), encoded [N, r].  With
    ``salient_idx`` (length r) R covers those rows instead (gather fallback)."""
    return D.MxLinear(*device_mx_parts(K, N, r, seed, salient_idx))


def device_mx_parts(K: int, N: int, r: int, seed: int = 1, salient_idx=None):
    """The artefacts of device_mx_linear: (codes [N, K], exps, r_codes [N, r], r_exps, salient_idx)."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    wt = torch.randn((N, K), generator=g, device="cuda", dtype=torch.float32) * 0.02
    act = D.quantize_mx(wt)
    codes, exps = D.unpack_mx(act.codes, act.sf, N, K)
    if r:
        mags = torch.tensor([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0], device="cuda")
        cols = torch.arange(r, device="cuda") if salient_idx is None else torch.as_tensor(
            np.asarray(salient_idx), device="cuda", dtype=torch.long)
        c = codes[:, cols].long()
        dec = torch.where((c & 8) != 0, -1.0, 1.0) * mags[c & 7]
        dec = dec * torch.exp2(exps[:, cols // 32].float())
        resid = (wt[:, cols] - dec).contiguous()
        ra = D.quantize_mx(resid)
        rc, re_ = D.unpack_mx(ra.codes, ra.sf, N, r)
    else:
        rc = re_ = None
    del wt
    return codes, exps, rc, re_, (np.arange(r) if salient_idx is None else np.asarray(salient_idx)) if r else None


def outlier_x(M: int, K: int, seed: int = 0, frac=0.01, mag=50.0) -> torch.Tensor:
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn((M, K), generator=g, device="cuda")
    n = max(1, int(round(frac * K)))
    cols = torch.randperm(K, generator=g, device="cuda")[:n]
    x[:, cols] *= mag
    return x.to(torch.bfloat16)


def mx_linear_point(lin, M: int, flush: Flusher) -> dict:
    x = outlier_x(M, lin.K)
    act = lin.quantize(x)
    y = torch.empty((M, lin.N), dtype=torch.bfloat16, device="cuda")
    t_step = time_in_graph(lambda: lin.forward(x, act, y), flush)
    t_lin = time_in_graph(lambda: lin.gemm(act, y), flush)
    K, N, r = lin.K, lin.N, lin.r
    flops = 2.0 * M * N * (K + r)
    w_bytes = N * K / 2 + N * K / 32 + N * r / 2 + N * r / 32
    io_bytes = M * K / 2 + M * K / 32 + 2 * M * N
    return {"M": M, "K": K, "N": N, "r": r, "step_us": t_step * 1e3, "linear_us": t_lin * 1e3,
            "linear_tflops": flops / (t_lin * 1e-3) / 1e12, "step_tflops": flops / (t_step * 1e-3) / 1e12,
            "linear_hbm_gbs": (w_bytes + io_bytes) / (t_lin * 1e-3) / 1e9, "tokens_per_s": M / (t_step * 1e-3)}


def decode_points(hbm_peak_gbs: float, layers: int = 16) -> list:
    """BASELINE C4 decode: Llama-2-7B up_proj (4096 x 11008) and down_proj
    (11008 x 4096), M in {1, 4, 16}, r = 64.  Steady state: ONE graph runs the
    step (serq_forward_mx: quantize + linear) over ``layers`` distinct weight sets whose total
    size (~390 MB) exceeds the 126 MB L2, so every layer streams its weights
    from HBM; per-step time = graph time / layers."""
    out = []
    for K, N in ((4096, 11008), (11008, 4096)):
        lins = [device_mx_linear(K, N, 64, seed=1 + i) for i in range(layers)]
        for M in (1, 4, 16):
            x = outlier_x(M, K)
            acts = [lin.quantize(x) for lin in lins]
            ys = [torch.empty((M, N), dtype=torch.bfloat16, device="cuda") for _ in lins]

            def run_all():
                # the public call (serq_forward_mx): quantizer fused into the decode kernel for M <= 4
                for lin, a, y in zip(lins, acts, ys):
                    lin.forward(x, a, y)

            def lin_all():
                for lin, a, y in zip(lins, acts, ys):
                    lin.gemm(a, y)

            t_step = time_in_graph(run_all, None, n=10) / layers
            t_lin = time_in_graph(lin_all, None, n=10) / layers
            r = 64
            flops = 2.0 * M * N * (K + r)
            w_bytes = N * K / 2 + N * K / 32 + N * r / 2 + N * r / 32
            io_bytes = M * K / 2 + M * K / 32 + 2 * M * N
            out.append({"M": M, "K": K, "N": N, "r": r, "layers_in_graph": layers, "step_us": t_step * 1e3,
                        "linear_us": t_lin * 1e3, "linear_hbm_gbs": (w_bytes + io_bytes) / (t_lin * 1e-3) / 1e9,
                        "linear_hbm_frac": (w_bytes + io_bytes) / (t_lin * 1e-3) / 1e9 / hbm_peak_gbs,
                        "step_tflops": flops / (t_step * 1e-3) / 1e12, "tokens_per_s": M / (t_step * 1e-3)})
        del lins
        torch.cuda.empty_cache()
    return out


def int_decode_points(hbm_peak_gbs: float, layers: int = 8, weight_format: str = "int8",
                      group: int | None = None) -> list:
    """INT decode (serq_i8_gemv_kernel): Llama-2-7B up_proj / down_proj with int8 or packed INT4
    (``weight_format``) weights -- per output channel, or in row groups of ``group`` (int8) -- and
    an integer R (r = 128), A8 asymmetric tokens, M = 1 / 4 / 16; ``layers`` distinct weight sets
    per graph (> L2).  Bytes = resident weights + R + scales / colsums + activations + outputs."""
    out = []
    for K, N in ((4096, 11008), (11008, 4096)):
        lins = [device_int_linear(K, N, 128, "int", seed=1 + i, weight_format=weight_format, group=group)
                for i in range(layers)]
        wbytes = lins[0].weight_bytes()[0] + (4 * N * (K // group) if group else 0)  # + fp32 group scales
        for M in (1, 4, 16):
            xs = [outlier_x(M, K, seed=i) for i in range(layers)]
            acts = [lins[0].quantize(x, 8, False) for x in xs]
            ys = [torch.empty((M, N), dtype=torch.bfloat16, device="cuda") for _ in xs]
            t_lin = time_steps(lambda i: lins[i % layers].gemm(acts[i % layers], ys[i % layers]), 2 * layers)
            t_step = time_steps(lambda i: lins[i % layers].forward(xs[i % layers], 8, False, acts[i % layers],
                                                                  ys[i % layers]), 2 * layers)
            byts = wbytes + 128 * N + 16 * N + M * K + 8 * M + 2 * M * N
            out.append({"M": M, "K": K, "N": N, "r": 128, "weights": weight_format, "group": group or K,
                        "kernel": D.last_kernel(),
                        "step_us": t_step * 1e3, "linear_us": t_lin * 1e3,
                        "linear_hbm_gbs": byts / (t_lin * 1e-3) / 1e9,
                        "linear_hbm_frac": byts / (t_lin * 1e-3) / 1e9 / hbm_peak_gbs})
    return out


def decode_fused_points(hbm_peak_gbs: float, layers: int = 8) -> list:
    """Decode through FUSED linears (device.FusedMxLinear): Llama-2-7B gate/up (2 x 11008) and
    q/k/v (3 x 4096) as one handle each, every part with its own salient set (the gather
    fallback these layers take in the reference's block), against the same parts as
    separate linears.  ``layers`` distinct weight sets chained in one graph (> L2); per-layer
    time = graph time / layers; bytes = every part's weights + R + activations + outputs."""
    out = []
    rng = np.random.default_rng(5)
    r, K = 64, 4096
    for name, ns in (("gate_up_proj", (11008, 11008)), ("qkv_proj", (4096, 4096, 4096))):
        fused, sep = [], []
        for i in range(layers):
            parts = [device_mx_parts(K, n, r, seed=100 * i + j, salient_idx=np.sort(rng.permutation(K)[:r]))
                     for j, n in enumerate(ns)]
            fused.append(D.FusedMxLinear(parts))
            sep.append([D.MxLinear(*p) for p in parts])
        N = sum(ns)
        for M in (1, 4, 16):
            x = outlier_x(M, K)
            ys = [torch.empty((M, N), dtype=torch.bfloat16, device="cuda") for _ in range(layers)]
            acts = [f.fused._activation(M, x.device) for f in fused]
            acts_s = [[lin._activation(M, x.device) for lin in ls] for ls in sep]

            def run_fused():
                for f, a, y in zip(fused, acts, ys):
                    f.fused.forward(x, a, y)

            def run_sep():
                for ls, aa, y in zip(sep, acts_s, ys):
                    for j, (lin, a) in enumerate(zip(ls, aa)):
                        lin.forward(x, a, y[:, sum(ns[:j]):sum(ns[:j + 1])])

            t_f = time_in_graph(run_fused, None, n=10) / layers
            t_s = time_in_graph(run_sep, None, n=10) / layers
            byts = N * K / 2 + N * K / 32 + N * r / 2 + N * r / 32 + M * K / 2 + M * K / 32 + 2 * M * N
            out.append({"linear": name, "parts": list(ns), "M": M, "K": K, "r": r, "layers_in_graph": layers,
                        "fused_step_us": t_f * 1e3, "separate_step_us": t_s * 1e3,
                        "fused_hbm_gbs": byts / (t_f * 1e-3) / 1e9,
                        "fused_hbm_frac": byts / (t_f * 1e-3) / 1e9 / hbm_peak_gbs,
                        "tokens_per_s": M / (t_f * 1e-3)})
        del fused, sep
        torch.cuda.empty_cache()
    return out


def device_int_linear(K: int, N: int, r: int, r_mode: str, seed: int = 1, group: int | None = None,
                      weight_format: str = "int8"):
    """Synthetic SERQ INT4 linear (SURVEY F4 composition): W ~ N(0, 0.02) [K, N];
    main = symmetric INT4 with one scale per output column (``group`` None) or
    per (row group of ``group`` input rows, column); R = residual
    of the first r rows, dense bf16 (``r_mode='dense'``) or INT4 with one scale
    per output column (``'int'``)."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    w = torch.randn((K, N), generator=g, device="cuda", dtype=torch.float64) * 0.02
    gs = K if group is None else group
    wg = w.view(K // gs, gs, N)
    s = wg.abs().amax(dim=1) / 7.0  # [G, N]
    s = torch.where(s == 0, torch.ones_like(s), s)
    codes = torch.clamp(torch.round(wg / s[:, None, :]), -7, 7).to(torch.int32).view(K, N)
    kw = {}
    if r:
        resid = w[:r] - (codes.view(K // gs, gs, N).double() * s[:, None, :]).view(K, N)[:r]
        if r_mode == "dense":
            kw = dict(r_dense=resid.to(torch.bfloat16).double(), salient_idx=np.arange(r))
        else:
            sr = resid.abs().amax(dim=0) / 7.0
            sr = torch.where(sr == 0, torch.ones_like(sr), sr)
            kw = dict(r_codes=torch.clamp(torch.round(resid / sr), -7, 7).to(torch.int32), r_scales=sr,
                      salient_idx=np.arange(r))
    return D.IntLinear(codes, s if group is not None else s.reshape(-1), 4, group_size=gs,
                       weight_format=weight_format, **kw)


def int_linear_point(M, K, N, r, r_mode, bits, symmetric, flush: Flusher | None = None, n_steps: int = 16,
                     group: int | None = None) -> dict:
    """Steady state over n_steps steps cycling 8 weight sets x 8 activation sets
    (> L2 at these shapes: cold operands every step, no flush)."""
    lins = [device_int_linear(K, N, r, r_mode, seed=1 + i, group=group) for i in range(8)]
    xs = [outlier_x(M, K, seed=i) for i in range(8)]
    acts = [lins[0].quantize(x, bits, symmetric) for x in xs]
    ys = [torch.empty((M, N), dtype=torch.bfloat16, device="cuda") for _ in xs]

    def step(i):
        lins[i % 8].gemm(lins[i % 8].quantize(xs[i % 8], bits, symmetric), ys[i % 8])

    def lin_only(i):
        lins[i % 8].gemm(acts[i % 8], ys[i % 8])

    def fwd(i):  # the public single call (serq_forward_int): quantizer + PDL-chained linear
        lins[i % 8].forward(xs[i % 8], bits, symmetric, acts[i % 8], ys[i % 8])

    t_step = time_steps(step, n_steps)
    t_fwd = time_steps(fwd, n_steps)
    t_lin = time_steps(lin_only, n_steps)
    flops = 2.0 * M * N * (K + r)
    out = {"M": M, "K": K, "N": N, "r": r, "r_mode": r_mode, "act_bits": bits, "act_symmetric": symmetric,
           "weight_group": group or K, "step_us": t_fwd * 1e3, "two_call_step_us": t_step * 1e3,
           "linear_us": t_lin * 1e3, "linear_tops": flops / (t_lin * 1e-3) / 1e12,
           "step_tops": flops / (t_fwd * 1e-3) / 1e12, "tokens_per_s": M / (t_fwd * 1e-3)}
    # end to end through the C-ABI from pinned host memory (serq_forward_int_host)
    xh = xs[0].cpu().pin_memory()
    yh = torch.empty((M, N), dtype=torch.bfloat16).pin_memory()
    for _ in range(2):
        lins[0].forward_host(xh, yh, bits, symmetric)
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        lins[0].forward_host(xh, yh, bits, symmetric)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    e2e = statistics.median(ts)
    out["e2e"] = {"us": e2e * 1e3, "tops": flops / (e2e * 1e-3) / 1e12, "h2d_bytes": M * K * 2, "d2h_bytes": M * N * 2,
                  "path": "serq_forward_int_host (C-ABI): pinned H2D, quantize, fused linear, D2H"}
    return out


def svd_baseline_point(M, K, N, r, bits=8, n_steps: int = 16) -> dict:
    """The paper's L2QER-style comparison (SVD baseline, compensate.py:209-224,
    304-310) at an INT shape, two ways: (a) device.SvdIntLinear -- the quantizer's
    exact bf16 (codes - zp), one bf16 GEMM U = (codes - zp) L1, and U L2 as the fused
    INT kernel's dense side term (our kernel); (b) the correction as two fp32 cuBLAS
    GEMMs added in the INT kernel's epilogue from an [M, N] fp32 buffer.  Factors are
    random with the right shapes (only the cost is measured here; parity is a test)."""
    rng = np.random.default_rng(5)
    mains = []
    for i in range(8):
        w = np.random.default_rng(1 + i).integers(-7, 8, (K, N))
        mains.append((w, np.random.default_rng(2 + i).uniform(0.01, 0.02, N)))
    l1 = rng.standard_normal((K, r)) * 0.01
    l2 = rng.standard_normal((r, N)) * 0.01
    svds = [D.SvdIntLinear(w, s, 4, l1, l2) for w, s in mains]
    xs = [outlier_x(M, K, seed=i, frac=0.005, mag=100.0) for i in range(8)]
    ys = [torch.empty((M, N), dtype=torch.bfloat16, device="cuda") for _ in xs]
    t_fused = time_steps(lambda i: svds[i % 8].forward(xs[i % 8], bits, False, ys[i % 8]), n_steps)
    lins = [device_int_linear(K, N, 0, "dense", seed=1 + i) for i in range(8)]
    l1t = torch.from_numpy(l1).to("cuda", torch.float32)
    l2t = torch.from_numpy(l2).to("cuda", torch.float32)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False

    def two_gemm(i):
        lin = lins[i % 8]
        act = lin.quantize(xs[i % 8], bits, False)
        corr = (D.IntLinear.dequantize(act) @ l1t) @ l2t
        lin.gemm(act, ys[i % 8], addend=corr)

    try:
        t_lib = time_steps(two_gemm, n_steps)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return {"M": M, "K": K, "N": N, "r": r, "act_bits": bits, "step_us": t_fused * 1e3, "aux_matmuls": 2,
            "tokens_per_s": M / (t_fused * 1e-3), "cublas_two_gemm_addend_step_us": t_lib * 1e3}

def mx_svd_baseline_point(M, K, N, r, n_steps: int = 16) -> dict:
    """The SVD baseline over an MX main (compensate.py:326-331, device.SvdMxLinear: K1-MX,
    exact bf16 mx_decode, two cuBLAS GEMMs for the correction, the MX kernel with the fp32
    addend) against SERQ's MX linear with its fused salient term (device.MxLinear.forward) at
    the same shape and rank; 8 weight / activation sets (cold).  Factors are random with the
    right shapes (cost only; parity is a test)."""
    rng = np.random.default_rng(6)
    l1 = rng.standard_normal((K, r)) * 0.01
    l2 = rng.standard_normal((r, N)) * 0.01
    svds, serq = [], []
    for i in range(8):
        codes, exps, rc, re_, idx = device_mx_parts(K, N, r, seed=1 + i)
        svds.append(D.SvdMxLinear(codes, exps, l1, l2))
        serq.append(D.MxLinear(codes, exps, rc, re_, idx))
    xs = [outlier_x(M, K, seed=i) for i in range(8)]
    ys = [torch.empty((M, N), dtype=torch.bfloat16, device="cuda") for _ in xs]
    t_svd = time_steps(lambda i: svds[i % 8].forward(xs[i % 8], ys[i % 8]), n_steps)
    t_serq = time_steps(lambda i: serq[i % 8].forward(xs[i % 8], None, ys[i % 8]), n_steps)
    return {"M": M, "K": K, "N": N, "r": r, "svd_step_us": t_svd * 1e3, "serq_step_us": t_serq * 1e3,
            "svd_aux_matmuls": 2, "serq_aux_matmuls": 1}


def rmsnorm_quant_point(M: int, K: int, hbm_peak_gbs: float, n_steps: int = 16) -> dict:
    """Producer fusion: rmsnorm(x, gain) -> MX codes in one
    kernel vs the plain MX quantizer on an already-normalised bf16 X, same shape,
    8 activation sets (cold).  Bytes per launch: 2MK in, MK/2 + MK/32 out."""
    xs = [outlier_x(M, K, seed=i) for i in range(8)]
    gain = (torch.rand(K, device="cuda", dtype=torch.float64) + 0.5)
    acts = [D.quantize_mx(x) for x in xs]
    t_f = time_steps(lambda i: D.rmsnorm_quantize_mx(xs[i % 8], gain, 1e-6, acts[i % 8]), n_steps)
    t_q = time_steps(lambda i: D.quantize_mx(xs[i % 8], None, acts[i % 8]), n_steps)
    # the unfused alternative: torch RMSNorm to a bf16 tensor, then the quantizer (its codes are
    # not the reference's: the normalised row is rounded to bf16 before encoding)
    g16 = gain.to(torch.bfloat16)
    hs = [torch.empty_like(x) for x in xs]

    def unfused(i):
        hs[i % 8].copy_(torch.nn.functional.rms_norm(xs[i % 8], (K,), g16, 1e-6))
        D.quantize_mx(hs[i % 8], None, acts[i % 8])

    t_u = time_steps(unfused, n_steps)
    byts = 2 * M * K + M * K / 2 + M * K / 32
    return {"M": M, "K": K, "rmsnorm_quant_us": t_f * 1e3, "quant_only_us": t_q * 1e3,
            "unfused_torch_rmsnorm_then_quant_us": t_u * 1e3,
            "rmsnorm_quant_hbm_frac": byts / (t_f * 1e-3) / 1e9 / hbm_peak_gbs,
            "unfused_extra_bytes": 4 * M * K}


def rmsnorm_int_quant_point(M: int, K: int, bits: int, symmetric: bool, hbm_peak_gbs: float,
                            n_steps: int = 16) -> dict:
    """Producer fusion for the integer formats: rmsnorm(x, gain) -> per-token INT codes with the
    reference's f64 scales (serq_rmsnorm_quant_int) vs the plain K1-INT quantizer on the same
    shape, and vs torch RMSNorm to bf16 + K1-INT (whose scales are not the reference's).  Bytes
    per launch: 2MK in, MK codes + 12M (f64 + f32 scales) [+ 4M zero points] out."""
    xs = [outlier_x(M, K, seed=i) for i in range(8)]
    gain = (torch.rand(K, device="cuda", dtype=torch.float64) + 0.5)
    t_f = time_steps(lambda i: D.rmsnorm_quantize_int(xs[i % 8], gain, 1e-6, bits, symmetric), n_steps)
    t_q = time_steps(lambda i: D.quantize_int(xs[i % 8], bits, symmetric), n_steps)
    g16 = gain.to(torch.bfloat16)
    hs = [torch.empty_like(x) for x in xs]

    def unfused(i):
        hs[i % 8].copy_(torch.nn.functional.rms_norm(xs[i % 8], (K,), g16, 1e-6))
        D.quantize_int(hs[i % 8], bits, symmetric)

    t_u = time_steps(unfused, n_steps)
    byts = 2 * M * K + M * K + 12 * M + (0 if symmetric else 4 * M)
    return {"M": M, "K": K, "bits": bits, "symmetric": symmetric, "rmsnorm_quant_us": t_f * 1e3,
            "quant_only_us": t_q * 1e3, "unfused_torch_rmsnorm_then_quant_us": t_u * 1e3,
            "rmsnorm_quant_hbm_frac": byts / (t_f * 1e-3) / 1e9 / hbm_peak_gbs}


def llama7b_block_point(M: int, n_blocks: int = 4, r: int = 64, fused: bool = False) -> dict:
    """Whole Llama-2-7B-shaped decoder block on the device (block.DeviceBlock: SERQ MXFP4
    linears + f32 RMSNorm / attention / SiLU), ``n_blocks`` distinct blocks chained in ONE
    CUDA graph (~400 MB of weights > L2, so every block streams its weights).  q/k/v and
    gate/up use the gather fallback (their inputs come from the residual
    stream), o/down the permuted layout; the (non-SERQ) token-batch attention runs as bf16
    flash attention.  Tokens/s = M / per-block time."""
    from .block import DeviceBlock

    H, F, hd = 4096, 11008, 128
    rng = np.random.default_rng(9)
    blocks = []
    for b in range(n_blocks):
        def parts(k, n, gather, s):
            idx = np.sort(rng.permutation(k)[:r]) if gather else None
            return device_mx_parts(k, n, r, seed=100 * b + s, salient_idx=idx)
        pq, pk, pv = parts(H, H, True, 1), parts(H, H, True, 2), parts(H, H, True, 3)
        pu, pg = parts(H, F, True, 5), parts(H, F, True, 6)
        lins = {"o_proj": D.MxLinear(*parts(H, H, False, 4)), "down_proj": D.MxLinear(*parts(F, H, False, 7))}
        if fused:  # q/k/v and up/gate as one launch each (own salient set per part)
            lins["qkv_proj"] = D.FusedMxLinear([pq, pk, pv])
            lins["up_gate_proj"] = D.FusedMxLinear([pu, pg])
        else:
            lins.update({"q_proj": D.MxLinear(*pq), "k_proj": D.MxLinear(*pk), "v_proj": D.MxLinear(*pv),
                         "up_proj": D.MxLinear(*pu), "gate_proj": D.MxLinear(*pg)})
        gains = {"ln1": np.abs(rng.standard_normal(H)) + 0.5, "ln2": np.abs(rng.standard_normal(H)) + 0.5}
        blocks.append(DeviceBlock(lins, gains, hd, fast_attention=True))
    x = outlier_x(M, H).float()

    def step():
        h = x
        for blk in blocks:
            h = blk(h)
        return h

    t = time_in_graph(step, None, n=10) / n_blocks
    flops = 2.0 * M * (4 * H * (H + r) + 2 * H * (F + r) + F * (H + r))
    return {"M": M, "hidden": H, "ffn": F, "r": r, "fused_qkv_up_gate": fused, "blocks_in_graph": n_blocks,
            "block_us": t * 1e3,
            "tokens_per_s": M / (t * 1e-3), "linear_tflops_equiv": flops / (t * 1e-3) / 1e12}


def c5_block_point(world: int = 1, rank: int = 0, M: int = 8192, r: int = 128, group=None, steps: int = 5,
                   flush: Flusher | None = None) -> dict:
    """BASELINE C5: Llama-3-70B-shaped decoder-block linears (hidden 8192,
    FFN 28672, GQA kv 1024), SERQ W4A4 MXFP4, M tokens, tensor parallel over
    ``world`` ranks with one all-reduce after o_proj and after down_proj
    (tp.TPBlockLinears).  q/k/v and gate/up are fused (one salient plan each);
    row-parallel layers hold salient_per_rank(r) channels per rank.  The
    attention output and SiLU(gate)*up feeding o/down are synthetic tensors of
    the right shape (non-linear ops are out of scope for this path)."""
    from . import tp

    specs = tp.block_specs(8192, 28672, 1024)
    lins, feeds, acts = {}, {}, {}
    for spec in specs:
        if spec.kind == "column":
            n0, n1 = tp.column_shard(spec.n, world, rank)
            lins[spec.name] = device_mx_linear(spec.k, n1 - n0, r, seed=hash(spec.name) % 1000)
        else:
            k0, k1 = tp.row_shard(spec.k, world, rank)
            lins[spec.name] = device_mx_linear(k1 - k0, spec.n, tp.salient_per_rank(r, world),
                                               seed=hash(spec.name) % 1000)
            feeds[spec.name] = outlier_x(M, k1 - k0, seed=7)
    x = outlier_x(M, 8192, seed=3)
    outs = {s.name: torch.empty((M, lins[s.name].N), dtype=torch.bfloat16, device="cuda") for s in specs}

    def run_linear(name):
        def f(xin):
            lin = lins[name]
            a = acts.get(name)
            acts[name] = lin.quantize(xin, a)
            return lin.gemm(acts[name], outs[name])
        return f

    drv = tp.TPBlockLinears(specs, {s.name: run_linear(s.name) for s in specs}, world, rank, group)

    def step():
        drv.forward(x, feeds)

    step()
    torch.cuda.synchronize()
    use_graph = world == 1  # NCCL collectives are kept outside graphs here
    g = graph_of(step) if use_graph else None
    ts = []
    for i in range(steps + 2):
        if flush is not None:
            flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay() if use_graph else step()
        b.record()
        b.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    t = statistics.median(ts)
    flops = 0.0
    for s in specs:
        lin = lins[s.name]
        flops += 2.0 * M * lin.N * (lin.K + lin.r)
    return {"M": M, "tp": world, "r": r, "block_ms": t, "tokens_per_s": M / (t * 1e-3),
            "rank_tflops": flops / (t * 1e-3) / 1e12, "graph": use_graph,
            "linears": {s.name: [lins[s.name].K, lins[s.name].N, lins[s.name].r] for s in specs}}


def c5_tp_point(world: int = 1, rank: int = 0, M: int = 8192, r: int = 128, group=None, steps: int = 10,
                chunks: int = 4, warm: int = 3, with_e2e: bool = True) -> dict:
    """BASELINE C5 tensor parallel: this rank's shard of the Llama-3-70B-shaped block linears
    (qkv / gate_up column-parallel, o / down row-parallel with salient_per_rank(r) channels
    per rank), token-chunk pipelined all-reduces (tp.PipelinedTPBlock on tp.DeviceBackend),
    the whole step -- quantizers, fused GEMMs, NCCL all-reduces -- in ONE CUDA graph.

    Times (device, CUDA events, the caller takes the max over ranks):
      step_ms        one block step, ``steps`` graph replays back to back
      serial_ms      the same with one chunk (no communication / compute overlap)
      allreduce_ms   the two all-reduces of [M, hidden] bf16 alone
      e2e_ms         pinned H2D of x + the step + D2H of the block output (public API)"""
    import torch.distributed as dist

    from . import tp

    specs = tp.block_specs(8192, 28672, 1024)
    lins, feeds = {}, {}
    for spec in specs:
        if spec.kind == "column":
            n0, n1 = tp.column_shard(spec.n, world, rank)
            lins[spec.name] = device_mx_linear(spec.k, n1 - n0, r, seed=101 + len(lins))
        else:
            k0, k1 = tp.row_shard(spec.k, world, rank)
            lins[spec.name] = device_mx_linear(k1 - k0, spec.n, tp.salient_per_rank(r, world), seed=101 + len(lins))
            feeds[spec.name] = outlier_x(M, k1 - k0, seed=7 + len(feeds))
    x = outlier_x(M, 8192, seed=3)

    def timed_graph(fn, n):
        fn()
        torch.cuda.synchronize()
        graph = True
        try:
            g = graph_of(fn)
        except Exception:  # a collective that cannot be captured: eager replay
            g, graph = None, False
        run = g.replay if g is not None else fn
        for _ in range(warm):
            run()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier(group=group)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            run()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / n, graph

    coll = world > 1  # a tp = 1 reference inside a multi-rank job must not issue collectives
    be = tp.DeviceBackend(lins, group, collectives=coll)
    blk = tp.PipelinedTPBlock(specs, be, chunks=chunks)
    step_ms, graph = timed_graph(lambda: blk.forward(x, feeds), steps)
    launches = be.launches_per_forward
    be1 = tp.DeviceBackend(lins, group, collectives=coll)
    blk1 = tp.PipelinedTPBlock(specs, be1, chunks=1)
    serial_ms, _ = timed_graph(lambda: blk1.forward(x, feeds), max(3, steps // 2))
    outs = blk.forward(x, feeds)
    ar_ms = 0.0
    if coll:
        ar_ms, _ = timed_graph(lambda: (tp.allreduce_sum_(outs["o_proj"], group),
                                        tp.allreduce_sum_(outs["down_proj"], group)), max(3, steps // 2))
    flops = sum(2.0 * M * s.n * (s.k + r) for s in specs)  # the full block (padding of per-rank salient sets not counted)
    out = {"M": M, "tp": world, "r": r, "chunks": len(tp.chunk_bounds(M, chunks)), "graph": graph,
           "step_ms": step_ms, "serial_ms": serial_ms, "allreduce_ms": ar_ms, "block_tflops": flops / (step_ms * 1e-3) / 1e12,
           "tokens_per_s": M / (step_ms * 1e-3), "flops_per_step": flops, "gpu_launches_per_step": launches,
           "linears": {s.name: [lins[s.name].K, lins[s.name].N, lins[s.name].r] for s in specs}}
    if with_e2e:
        xh = x.cpu().pin_memory()
        yh = torch.empty((M, lins["down_proj"].N), dtype=torch.bfloat16).pin_memory()
        xd = torch.empty_like(x)

        def e2e():
            xd.copy_(xh, non_blocking=True)
            o = blk.forward(xd, feeds)
            yh.copy_(o["down_proj"], non_blocking=True)

        ts = []
        for i in range(warm + max(3, steps // 2)):
            if world > 1:
                dist.barrier(group=group)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            e2e()
            b.record()
            b.synchronize()
            if i >= warm:
                ts.append(a.elapsed_time(b))
        out["e2e_ms"] = statistics.median(ts)
        out["h2d_bytes_per_step"] = xh.numel() * 2
        out["d2h_bytes_per_step"] = yh.numel() * 2
    del lins, feeds
    torch.cuda.empty_cache()
    return out
