"""GPU shape sweep: seeded random (M, K, N, r, mode) across every dispatch regime -- decode
(M <= 16), the small-M kernels, the CTA-pair kernels with ragged M / N tiles -- for the MX and
INT linears, against the oracle: INT accumulators bit-exact, Y at the north_star tolerance.
Guards the dispatch boundaries (M = 16 / 17, 128 / 129, 255 / 256) and ragged tiles."""

import numpy as np
import pytest

from oracle import serq_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_MAX, TOL_MEAN = 1e-2, 1e-3
MS = [1, 5, 16, 17, 100, 128, 129, 255, 256, 300, 513]


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


def _mx_cases(n=64):
    rng = np.random.default_rng(2026)
    return [(int(rng.choice(MS)), int(rng.choice([256, 512, 1024, 1536])), int(rng.choice([128, 384, 520, 1000])),
             int(rng.choice([0, 32, 64, 96, 128])), bool(rng.random() < 0.4)) for _ in range(n)]


def _int_cases(n=64):
    rng = np.random.default_rng(2027)
    return [(int(rng.choice(MS)), int(rng.choice([256, 512, 1024, 1536])), int(rng.choice([136, 256, 520, 1000])),
             str(rng.choice(["int", "dense", "none"])), int(rng.choice([16, 64, 128])), bool(rng.random() < 0.3),
             bool(rng.random() < 0.5)) for _ in range(n)]


@pytest.mark.parametrize("M,K,N,r,gather", _mx_cases())
def test_mx_shape_sweep(D, M, K, N, r, gather):
    rng = np.random.default_rng(M * 7 + K + N + r)
    x = _x(M, K, seed=M + N)
    w = rng.standard_normal((K, N)) * 0.02
    idx = np.sort(rng.choice(K, r, replace=False)) if (gather and r) else np.arange(r)
    main_t, comp = O.build_serq_rtn_mx(w, idx, 32)
    lin = D.MxLinear(main_t.element_codes, main_t.block_scale_exponents,
                     comp.r_q.element_codes if r else None, comp.r_q.block_scale_exponents if r else None,
                     idx if r else None)
    y = lin(_cuda(x, torch.bfloat16)).float().cpu().numpy()
    ref = O.forward_mx(x, main_t, comp if r else None)
    mx, mean = O.parity_errors(y, ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (D.last_kernel(), mx, mean)


@pytest.mark.parametrize("M,K,N,r_mode,r,gather,sym", _int_cases())
def test_int_shape_sweep(D, M, K, N, r_mode, r, gather, sym):
    rng = np.random.default_rng(M * 5 + K + N + r)
    x = _x(M, K, seed=M + K)
    w = rng.standard_normal((K, N)) * 0.02
    bits = 4 if sym else 8
    if r_mode == "none":
        main = O.quantize_symmetric(w, O.IntCfg(4, True, K, "row"))
        comp, kw, idx = None, {}, None
    else:
        idx = np.sort(rng.choice(K, r, replace=False)) if gather else np.arange(r)
        main, comp = O.build_per_channel_int(w, idx, r_mode=r_mode)
        kw = dict(r_dense=comp.r_dense) if r_mode == "dense" else dict(r_codes=comp.r_q.codes, r_scales=comp.r_q.scales)
        kw["salient_idx"] = idx
    lin = D.IntLinear(main.codes, main.scales, 4, **kw)
    act = lin.quantize(_cuda(x, torch.bfloat16), bits, sym)
    acc = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    accr = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    y = lin.gemm(act, acc_dump=acc, accr_dump=accr).float().cpu().numpy()
    kern = D.last_kernel()
    cfg = O.IntCfg(bits, sym, "per-row")
    y_ref, xq = O.forward_int(x, main, comp, cfg, symmetric_act=sym)
    _, parts = O.int_gemm(xq, main, return_partials=True)
    assert np.array_equal(acc.cpu().numpy().astype(np.int64), parts[0][1]), kern
    if r_mode == "int":
        _, rp = O.int_gemm(O.gather_columns(xq, idx), comp.r_q, return_partials=True)
        assert np.array_equal(accr.cpu().numpy().astype(np.int64), rp[0][1]), kern
    mx, mean = O.parity_errors(y, y_ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (kern, mx, mean)


def _grouped_cases(n=16):
    rng = np.random.default_rng(2028)
    return [(int(rng.choice(MS)), int(rng.choice([512, 1024, 1536])), int(rng.choice([136, 256, 520])),
             int(rng.choice([128, 256])), str(rng.choice(["int", "dense", "none"])), bool(rng.random() < 0.5))
            for _ in range(n)]


@pytest.mark.parametrize("M,K,N,g,r_mode,single_call", _grouped_cases())
def test_int_grouped_shape_sweep(D, M, K, N, g, r_mode, single_call):
    # group-wise weight scales (gptq.py:98-146): one promoted partial per group; Y vs the oracle,
    # through gemm() or the single C-ABI call (quantizer + linear)
    if K % g:
        pytest.skip("group does not divide K")
    rng = np.random.default_rng(M + K + N + g)
    x = _x(M, K, seed=M * 3 + g)
    w = rng.standard_normal((K, N)) * 0.02
    main = O.quantize_symmetric(w, O.IntCfg(4, True, g, "row"))
    r = 64
    comp, kw = None, {}
    if r_mode != "none":
        resid = w[:r] - O.dequantize(main)[:r]
        if r_mode == "dense":
            comp = O.Comp(r, salient_idx=np.arange(r), r_dense=O.bf16_round(resid))
            kw = dict(r_dense=comp.r_dense, salient_idx=np.arange(r))
        else:
            rq = O.quantize_symmetric(resid, O.IntCfg(4, True, r, "row"))
            comp = O.Comp(r, salient_idx=np.arange(r), r_q=rq)
            kw = dict(r_codes=rq.codes, r_scales=rq.scales, salient_idx=np.arange(r))
    lin = D.IntLinear(main.codes, main.scales.reshape(K // g, N), 4, group_size=g, **kw)
    xt = _cuda(x, torch.bfloat16)
    if single_call:
        y = lin.forward(xt, 8, False).float().cpu().numpy()
    else:
        y = lin.gemm(lin.quantize(xt, 8, False)).float().cpu().numpy()
    y_ref, _ = O.forward_int(x, main, comp, O.IntCfg(8, False, "per-row"))
    mx, mean = O.parity_errors(y, y_ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (D.last_kernel(), mx, mean)


def _odd_k_cases(n=24):
    # K not a multiple of the 128-byte / 256-element steps (partial last K-step, padded SF chunks)
    rng = np.random.default_rng(2029)
    return [(int(rng.choice(MS)), int(rng.choice([96, 544, 2080])), int(rng.choice([16, 272, 1040])),
             int(rng.choice([128, 520]))) for _ in range(n)]


@pytest.mark.parametrize("M,Kmx,Kint,N", _odd_k_cases())
def test_odd_k_sweep(D, M, Kmx, Kint, N):
    rng = np.random.default_rng(M + Kmx + Kint + N)
    # MX (K % 32 == 0): r = 32 salient columns
    x = _x(M, Kmx, seed=M + 11)
    w = rng.standard_normal((Kmx, N)) * 0.02
    main_t, comp = O.build_serq_rtn_mx(w, np.arange(32), 32)
    lin = D.MxLinear(main_t.element_codes, main_t.block_scale_exponents, comp.r_q.element_codes,
                     comp.r_q.block_scale_exponents, np.arange(32))
    y = lin(_cuda(x, torch.bfloat16)).float().cpu().numpy()
    mx, mean = O.parity_errors(y, O.forward_mx(x, main_t, comp))
    assert mx <= TOL_MAX and mean <= TOL_MEAN, ("mx", D.last_kernel(), mx, mean)
    # INT (K % 16 == 0): integer R at r = 16
    x = _x(M, Kint, seed=M + 12)
    w = rng.standard_normal((Kint, N)) * 0.02
    main, comp = O.build_per_channel_int(w, np.arange(16), r_mode="int")
    lin = D.IntLinear(main.codes, main.scales, 4, r_codes=comp.r_q.codes, r_scales=comp.r_q.scales,
                      salient_idx=np.arange(16))
    act = lin.quantize(_cuda(x, torch.bfloat16), 8, False)
    acc = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    y = lin.gemm(act, acc_dump=acc).float().cpu().numpy()
    y_ref, xq = O.forward_int(x, main, comp, O.IntCfg(8, False, "per-row"))
    _, parts = O.int_gemm(xq, main, return_partials=True)
    assert np.array_equal(acc.cpu().numpy().astype(np.int64), parts[0][1]), ("int", D.last_kernel())
    mx, mean = O.parity_errors(y, y_ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN, ("int", D.last_kernel(), mx, mean)
