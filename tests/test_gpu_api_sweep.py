"""GPU sweep over the public entry points with seeded random shapes: the single C-ABI calls
(quantizer + linear), the end-to-end host paths, fused linears, the RMSNorm producers and the
quantizers on f32 / f64 input -- each against the oracle (codes / scales / accumulators exact,
Y at the north_star tolerance)."""

import numpy as np
import pytest

from oracle import serq_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_MAX, TOL_MEAN = 1e-2, 1e-3
MS = [1, 3, 8, 16, 17, 64, 128, 129, 256, 300, 1100]


@pytest.fixture(scope="module")
def D():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_08185_b200 import device

    return device


def _x(M, K, seed):
    return O.bf16_round(O.synthetic_activations(M, K, max(1, K // 100), 50.0, seed))


def _cuda(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


def _cases(seed, n):
    rng = np.random.default_rng(seed)
    return [(int(rng.choice(MS)), int(rng.choice([512, 1024, 2048])), int(rng.choice([256, 640, 1024])),
             bool(rng.random() < 0.5)) for _ in range(n)]


@pytest.mark.parametrize("M,K,N,gather", _cases(31, 16))
def test_mx_single_call_and_host(D, M, K, N, gather):
    rng = np.random.default_rng(M + K + N)
    r = 64
    x = _x(M, K, seed=M)
    w = rng.standard_normal((K, N)) * 0.02
    idx = np.sort(rng.choice(K, r, replace=False)) if gather else np.arange(r)
    main_t, comp = O.build_serq_rtn_mx(w, idx, 32)
    lin = D.MxLinear(main_t.element_codes, main_t.block_scale_exponents, comp.r_q.element_codes,
                     comp.r_q.block_scale_exponents, idx)
    ref = O.forward_mx(x, main_t, comp)
    y = lin.forward(_cuda(x, torch.bfloat16)).float().cpu().numpy()
    mx, mean = O.parity_errors(y, ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (D.last_kernel(), mx, mean)
    xh = torch.from_numpy(x).to(torch.bfloat16).pin_memory()
    yh = torch.empty((M, N), dtype=torch.bfloat16).pin_memory()
    lin.forward_host(xh, yh)
    assert np.array_equal(yh.float().numpy(), y)  # the host path runs the same kernels per chunk


@pytest.mark.parametrize("M,K,N,gather", _cases(32, 16))
def test_int_single_call_and_host(D, M, K, N, gather):
    rng = np.random.default_rng(M * 3 + K + N)
    r = 64
    x = _x(M, K, seed=M + 1)
    w = rng.standard_normal((K, N)) * 0.02
    idx = np.sort(rng.choice(K, r, replace=False)) if gather else np.arange(r)
    main, comp = O.build_per_channel_int(w, idx, r_mode="int")
    lin = D.IntLinear(main.codes, main.scales, 4, r_codes=comp.r_q.codes, r_scales=comp.r_q.scales, salient_idx=idx)
    y_ref, _ = O.forward_int(x, main, comp, O.IntCfg(8, False, "per-row"))
    y = lin.forward(_cuda(x, torch.bfloat16), 8, False).float().cpu().numpy()
    mx, mean = O.parity_errors(y, y_ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (D.last_kernel(), mx, mean)
    xh = torch.from_numpy(x).to(torch.bfloat16).pin_memory()
    yh = torch.empty((M, N), dtype=torch.bfloat16).pin_memory()
    lin.forward_host(xh, yh, 8, False)
    mx, mean = O.parity_errors(yh.float().numpy(), y_ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN, ("host", mx, mean)


@pytest.mark.parametrize("M", [1, 4, 16, 40, 300])
def test_fused_mx_linear_random_parts(D, M):
    # 2-3 parts, each with its own random salient set (the gather fallback), vs each part's oracle
    rng = np.random.default_rng(M)
    K, r = 1024, 64
    ns = [int(v) for v in rng.choice([128, 256, 384], size=int(rng.integers(2, 4)))]
    x = _x(M, K, seed=M + 7)
    parts, refs = [], []
    for j, n in enumerate(ns):
        w = rng.standard_normal((K, n)) * 0.02
        idx = np.sort(rng.choice(K, r, replace=False))
        main_t, comp = O.build_serq_rtn_mx(w, idx, 32)
        parts.append((main_t.element_codes, main_t.block_scale_exponents, comp.r_q.element_codes,
                      comp.r_q.block_scale_exponents, idx))
        refs.append(O.forward_mx(x, main_t, comp))
    fused = D.FusedMxLinear(parts)
    y = fused.forward(_cuda(x, torch.bfloat16)).float().cpu().numpy()
    mx, mean = O.parity_errors(y, np.concatenate(refs, axis=1))
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (D.last_kernel(), mx, mean)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("M,K", [(1, 512), (33, 1024), (300, 2048)])
def test_quantizers_on_f32_f64_input(D, dtype, M, K):
    rng = np.random.default_rng(M + K)
    x = _x(M, K, seed=K) + rng.standard_normal((M, K)) * 1e-3
    if dtype == "f32":
        x = x.astype(np.float32).astype(np.float64)
    tdt = torch.float32 if dtype == "f32" else torch.float64
    act = D.quantize_mx(_cuda(x, tdt))
    c, e = D.unpack_mx(act.codes, act.sf, M, K)
    ref = O.mx_encode(x, 32)
    assert np.array_equal(e.cpu().numpy(), ref.block_scale_exponents)
    assert np.array_equal(c.cpu().numpy(), ref.element_codes)
    for bits, sym in ((8, False), (4, True)):
        a = D.quantize_int(_cuda(x, tdt), bits, sym)
        cfg = O.IntCfg(bits, sym, "per-row")
        q = O.quantize_symmetric(x, cfg) if sym else O.quantize_asymmetric(x, cfg)
        codes = a.codes.cpu().numpy()
        codes = codes.astype(np.int32) if sym else codes.view(np.uint8).astype(np.int32)
        assert np.array_equal(a.scale64.cpu().numpy(), q.scales[:, 0])
        assert np.array_equal(codes, q.codes)


def test_threads_and_streams_share_a_layer(D):
    # SPEC: pure functions, results independent of the thread count -- four host threads drive
    # one MX and one INT layer on their own streams; every result equals the sequential one
    import threading

    K, N, r = 1024, 512, 64
    rng = np.random.default_rng(77)
    w = rng.standard_normal((K, N)) * 0.02
    main_t, comp = O.build_serq_rtn_mx(w, np.arange(r), 32)
    mxl = D.MxLinear(main_t.element_codes, main_t.block_scale_exponents, comp.r_q.element_codes,
                     comp.r_q.block_scale_exponents, np.arange(r))
    main, icomp = O.build_per_channel_int(w, np.arange(r), r_mode="int")
    il = D.IntLinear(main.codes, main.scales, 4, r_codes=icomp.r_q.codes, r_scales=icomp.r_q.scales,
                     salient_idx=np.arange(r))
    xs = [_cuda(_x(m, K, seed=m), torch.bfloat16) for m in (1, 16, 200, 513)]
    seq = [(mxl.forward(x).clone(), il.forward(x, 8, False).clone()) for x in xs]
    torch.cuda.synchronize()
    out = [None] * len(xs)

    def work(i):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(5):
                out[i] = (mxl.forward(xs[i]), il.forward(xs[i], 8, False))
        s.synchronize()

    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(xs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    torch.cuda.synchronize()
    for (a, b), (c, d) in zip(out, seq):
        assert torch.equal(a, c) and torch.equal(b, d)
