"""GPU parity: the sm_100a kernels (through the C-ABI) vs the oracle.

Integer outputs (codes, scales, zero points, E8M0 exponents, integer
accumulators) must be bit-exact.  bf16 outputs are compared with
bf16_rne(Y_oracle) at tolerance max 1e-2 / mean 1e-3
(BASELINE.json north_star), written here as TOL_MAX / TOL_MEAN.
"""

import numpy as np
import pytest

from oracle import serq_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_MAX, TOL_MEAN = 1e-2, 1e-3


@pytest.fixture(scope="module")
def D():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_08185_b200 import device

    return device


def _bf16_outlier_x(M, K, seed=0, n_out=None, mag=50.0):
    n_out = max(1, K // 100) if n_out is None else n_out
    return O.bf16_round(O.synthetic_activations(M, K, n_out, mag, seed))


def _cuda(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


def _check_mx_encode(D, x, dtype):
    M, K = x.shape
    act = D.quantize_mx(_cuda(x, dtype))
    c, e = D.unpack_mx(act.codes, act.sf, M, K)
    ref = O.mx_encode(x, 32)
    assert np.array_equal(e.cpu().numpy(), ref.block_scale_exponents)
    assert np.array_equal(c.cpu().numpy(), ref.element_codes)


# ---------------------------------------------------------------- K1-MX


@pytest.mark.parametrize("dtype", ["bf16", "f32", "f64"])
def test_mx_encode_bitexact_outliers(D, dtype):
    x = _bf16_outlier_x(300, 1024, seed=1)
    if dtype == "f64":
        x = x + np.random.default_rng(2).standard_normal(x.shape) * 1e-9  # not bf16-representable
    tdt = {"bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64}[dtype]
    _check_mx_encode(D, x, tdt)


def test_mx_encode_golden(D, golden):
    for i in range(int(golden["mx_count"])):
        x = golden[f"mx_x_{i}"]
        act = D.quantize_mx(_cuda(x, torch.float64))
        c, e = D.unpack_mx(act.codes, act.sf, *x.shape)
        assert np.array_equal(c.cpu().numpy(), golden[f"mx_codes_{i}"]), i
        assert np.array_equal(e.cpu().numpy(), golden[f"mx_exps_{i}"]), i


def test_mx_encode_every_bf16_value(D):
    # all 65536 bf16 bit patterns (minus NaN/Inf), shuffled into 32-blocks
    bits = np.arange(65536, dtype=np.uint32)
    vals = (bits << 16).view(np.float32).astype(np.float64)
    vals = vals[np.isfinite(vals)]
    rng = np.random.default_rng(3)
    for perm in range(3):
        v = vals[rng.permutation(vals.size)] if perm else vals.copy()
        v = v[: (v.size // 256) * 256].reshape(-1, 256)
        _check_mx_encode(D, v, torch.bfloat16)


def test_mx_encode_acceptance_grid(D):
    # acceptance criterion 04 grid (test_acceptance.py:158-179) in blocks with max 6 -> e = 0
    grid = np.linspace(-8.0, 8.0, 100_001)[:99_968].reshape(-1, 32).copy()
    grid[:, 0] = 6.0  # pin the block exponent to 0 so codes are the plain E2M1 rounding
    _check_mx_encode(D, grid, torch.float64)
    _check_mx_encode(D, grid.astype(np.float32).astype(np.float64), torch.float32)


# ---------------------------------------------------------------- K1-INT


@pytest.mark.parametrize("M,K", [(1, 11008), (3, 16384), (200, 9216)])
def test_int_quant_long_rows_bitexact(D, M, K):
    # rows above 8192 elements (down_proj's 11008): the 256-thread kernel with 8 chunks per thread
    x = _bf16_outlier_x(M, K, seed=K)
    for bits, sym in ((8, False), (4, True)):
        act = D.quantize_int(_cuda(x, torch.bfloat16), bits, sym)
        cfg = O.IntCfg(bits, sym, "per-row")
        ref = O.quantize_symmetric(x, cfg) if sym else O.quantize_asymmetric(x, cfg)
        codes = act.codes.cpu().numpy()
        codes = codes.astype(np.int32) if sym else codes.view(np.uint8).astype(np.int32)
        assert np.array_equal(act.scale64.cpu().numpy(), ref.scales[:, 0])
        assert np.array_equal(codes, ref.codes)


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("symmetric", [True, False])
@pytest.mark.parametrize("dtype", ["bf16", "f64"])
def test_int_quant_bitexact(D, bits, symmetric, dtype):
    x = _bf16_outlier_x(257, 1024, seed=bits)
    if dtype == "f64":
        x = x * 1.000000123
    xt = _cuda(x, torch.bfloat16 if dtype == "bf16" else torch.float64)
    act = D.quantize_int(xt, bits, symmetric)
    cfg = O.IntCfg(bits, symmetric, "per-row")
    ref = O.quantize_symmetric(x, cfg) if symmetric else O.quantize_asymmetric(x, cfg)
    codes = act.codes.cpu().numpy()
    codes = codes.astype(np.int32) if symmetric else codes.view(np.uint8).astype(np.int32)
    assert np.array_equal(act.scale64.cpu().numpy(), ref.scales[:, 0])
    if not symmetric:
        assert np.array_equal(act.zp.cpu().numpy(), ref.zero_points[:, 0])
    assert np.array_equal(codes, ref.codes)


@pytest.mark.parametrize("K", [1024, 4096, 8192, 11008, 16384])
def test_int_quant_exact_ties(D, K):
    # rows built so that x / s lands EXACTLY on k + 1/2 for many elements (s a power of two),
    # plus values a few ulps off the ties: the fast path must hand every one of them to the
    # exact path and reproduce rint's half-to-even (quantcore.py:116, 131-132)
    rng = np.random.default_rng(K)
    M = 96
    x = np.zeros((M, K))
    for m in range(M):
        e = -int(rng.integers(2, 9))
        if m % 2 == 0:  # asymmetric A8: lo = 0, hi = 255 * 2^e -> s = 2^e
            ties = (rng.integers(0, 127, K) + 0.5) * 2.0**e
            x[m] = ties
            x[m, 0], x[m, 1] = 0.0, 255 * 2.0**e
        else:  # symmetric A4: amax = 7 * 2^e -> s = 2^e
            ties = (rng.integers(-6, 6, K) + 0.5) * 2.0**e
            x[m] = ties
            x[m, 0] = 7 * 2.0**e
        near = rng.random(K) < 0.1  # neighbours of the ties (next bf16 up / down)
        x[m, near] = np.nextafter(x[m, near].astype(np.float32), np.float32(np.inf)).astype(np.float64)
    x = O.bf16_round(x)
    xt = _cuda(x, torch.bfloat16)
    for sym, bits, rows in ((False, 8, slice(0, None, 2)), (True, 4, slice(1, None, 2))):
        xr = np.ascontiguousarray(x[rows])
        act = D.quantize_int(_cuda(xr, torch.bfloat16), bits, sym)
        cfg = O.IntCfg(bits, sym, "per-row")
        ref = O.quantize_symmetric(xr, cfg) if sym else O.quantize_asymmetric(xr, cfg)
        codes = act.codes.cpu().numpy()
        codes = codes.astype(np.int32) if sym else codes.view(np.uint8).astype(np.int32)
        assert np.array_equal(act.scale64.cpu().numpy(), ref.scales[:, 0])
        assert np.array_equal(codes, ref.codes), int((codes != ref.codes).sum())
    del xt


def test_int_quant_golden(D, golden):
    for i in range(int(golden["q_count"])):
        x = golden[f"q_x_{i}"]
        if x.shape[1] % 16:
            continue
        for bits in (2, 4, 8):
            s = D.quantize_int(_cuda(x, torch.float64), bits, True)
            a = D.quantize_int(_cuda(x, torch.float64), bits, False)
            assert np.array_equal(s.codes.cpu().numpy().astype(np.int32), golden[f"q_sym{bits}_codes_{i}"])
            assert np.array_equal(s.scale64.cpu().numpy(), golden[f"q_sym{bits}_scales_{i}"][:, 0])
            assert np.array_equal(a.codes.cpu().numpy().view(np.uint8).astype(np.int32),
                                  golden[f"q_asym{bits}_codes_{i}"])
            assert np.array_equal(a.zp.cpu().numpy(), golden[f"q_asym{bits}_zps_{i}"][:, 0])


# ---------------------------------------------------------------- K2 MX linear


def _mx_case(M, K, N, r, seed=0):
    x = _bf16_outlier_x(M, K, seed=seed)
    w = np.random.default_rng(seed + 1).standard_normal((K, N)) * 0.02
    w[:r] *= 8  # salient rows carry more error
    main_t, comp = O.build_serq_rtn_mx(w, np.arange(r), 32)
    return x, main_t, comp


@pytest.mark.parametrize("M,K,N,r", [(256, 1024, 512, 64), (100, 512, 384, 32), (128, 256, 256, 0),
                                     (384, 2048, 768, 128), (17, 4096, 256, 256)])
def test_mx_linear_parity(D, M, K, N, r):
    x, main_t, comp = _mx_case(M, K, N, r, seed=M)
    lin = D.MxLinear(main_t.element_codes, main_t.block_scale_exponents,
                     comp.r_q.element_codes if r else None, comp.r_q.block_scale_exponents if r else None,
                     np.arange(r) if r else None)
    y = lin(_cuda(x, torch.bfloat16)).float().cpu().numpy()
    mx, mean = O.parity_errors(y, O.forward_mx(x, main_t, comp))
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


def test_mx_linear_golden_and_gather(D, golden):
    x = golden["fmx_x"]
    lin = D.MxLinear(golden["fmx_main_codes"], golden["fmx_main_exps"], golden["fmx_r_codes"],
                     golden["fmx_r_exps"], golden["fmx_idx"])
    y = lin(_cuda(x, torch.bfloat16)).float().cpu().numpy()
    mx, mean = O.parity_errors(y, golden["fmx_y"])
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)
    lin_g = D.MxLinear(golden["fmx_main_codes"], golden["fmx_main_exps"], golden["fmx_r_codes"],
                       golden["fmx_r_exps"], golden["fmx_gidx"])
    assert not lin_g.contiguous
    y = lin_g(_cuda(x, torch.bfloat16)).float().cpu().numpy()
    mx, mean = O.parity_errors(y, golden["fmx_y_gather"])
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


# ---------------------------------------------------------------- K3 INT linear


@pytest.mark.parametrize("bits,symmetric,r_mode", [(4, True, "dense"), (8, False, "int"), (4, False, "int"),
                                                   (8, False, "dense"), (4, True, "none")])
def test_int_linear_parity(D, bits, symmetric, r_mode):
    M, K, N, r = 200, 1024, 512, 64
    x = _bf16_outlier_x(M, K, seed=bits + 10)
    w = np.random.default_rng(5).standard_normal((K, N)) * 0.02
    main, comp = O.build_per_channel_int(w, np.arange(r), r_mode="dense" if r_mode == "none" else r_mode)
    if r_mode == "none":
        comp = None
    kw = {}
    if r_mode == "dense":
        kw = dict(r_dense=comp.r_dense, salient_idx=np.arange(r))
    elif r_mode == "int":
        kw = dict(r_codes=comp.r_q.codes, r_scales=comp.r_q.scales, salient_idx=np.arange(r))
    lin = D.IntLinear(main.codes, main.scales, 4, **kw)
    xt = _cuda(x, torch.bfloat16)
    act = lin.quantize(xt, bits, symmetric)
    acc = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    accr = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    y = lin.gemm(act, acc_dump=acc, accr_dump=accr).float().cpu().numpy()
    cfg = O.IntCfg(bits, symmetric, "per-row")
    y_ref, xq = O.forward_int(x, main, comp, cfg, symmetric_act=symmetric)
    _, parts = O.int_gemm(xq, main, return_partials=True)
    assert np.array_equal(acc.cpu().numpy().astype(np.int64), parts[0][1])
    if r_mode == "int":
        _, rp = O.int_gemm(O.gather_columns(xq, np.arange(r)), comp.r_q, return_partials=True)
        assert np.array_equal(accr.cpu().numpy().astype(np.int64), rp[0][1])
    mx, mean = O.parity_errors(y, y_ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


@pytest.mark.parametrize("M,K,N,r", [(300, 1024, 512, 128), (1024, 2048, 1536, 96), (260, 512, 264, 72)])
def test_int_linear_dense_r_above_64_pair_kernel(D, M, K, N, r):
    # dense R with r > 64 on the CTA-pair kernel: ceil(r / 64) side tiles staged with spread
    # K-steps into one TMEM accumulator; partial last side tile (72, 96), many tiles per pair
    x = _bf16_outlier_x(M, K, seed=r)
    w = np.random.default_rng(r).standard_normal((K, N)) * 0.02
    main, comp = O.build_per_channel_int(w, np.arange(r), r_mode="dense")
    lin = D.IntLinear(main.codes, main.scales, 4, r_dense=comp.r_dense, salient_idx=np.arange(r))
    act = lin.quantize(_cuda(x, torch.bfloat16), 8, False)
    acc = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    y = lin.gemm(act, acc_dump=acc).float().cpu().numpy()
    assert D.last_kernel().startswith("serq_i8_pair_kernel"), D.last_kernel()
    y_ref, xq = O.forward_int(x, main, comp, O.IntCfg(8, False, "per-row"))
    _, parts = O.int_gemm(xq, main, return_partials=True)
    assert np.array_equal(acc.cpu().numpy().astype(np.int64), parts[0][1])
    mx, mean = O.parity_errors(y, y_ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


@pytest.mark.parametrize("M", [1, 3, 8, 16])
@pytest.mark.parametrize("r_mode,contiguous,bits,sym", [("int", True, 8, False), ("int", False, 8, False),
                                                       ("dense", True, 4, True), ("none", True, 8, False)])
def test_int_decode_gemv_parity(D, M, r_mode, contiguous, bits, sym):
    # M <= 16: the CUDA-core weight-stream kernel (dp4a, exact s32) -- accumulators bit-exact
    K, N, r = 1536, 1000, 64
    rng = np.random.default_rng(M + K)
    x = _bf16_outlier_x(M, K, seed=M)
    w = rng.standard_normal((K, N)) * 0.02
    idx = np.arange(r) if contiguous else np.sort(rng.choice(K, r, replace=False))
    if r_mode == "none":
        main = O.quantize_symmetric(w, O.IntCfg(4, True, K, "row"))
        comp, kw = None, {}
    else:
        main, comp = O.build_per_channel_int(w, idx, r_mode=r_mode)
        kw = (dict(r_dense=comp.r_dense) if r_mode == "dense" else dict(r_codes=comp.r_q.codes, r_scales=comp.r_q.scales))
        kw["salient_idx"] = idx
    lin = D.IntLinear(main.codes, main.scales, 4, **kw)
    act = lin.quantize(_cuda(x, torch.bfloat16), bits, sym)
    acc = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    accr = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    y = lin.gemm(act, acc_dump=acc, accr_dump=accr).float().cpu().numpy()
    assert D.last_kernel() == "serq_i8_gemv_kernel"
    cfg = O.IntCfg(bits, sym, "per-row")
    y_ref, xq = O.forward_int(x, main, comp, cfg, symmetric_act=sym)
    _, parts = O.int_gemm(xq, main, return_partials=True)
    assert np.array_equal(acc.cpu().numpy().astype(np.int64), parts[0][1])
    if r_mode == "int":
        _, rp = O.int_gemm(O.gather_columns(xq, idx), comp.r_q, return_partials=True)
        assert np.array_equal(accr.cpu().numpy().astype(np.int64), rp[0][1])
    mx, mean = O.parity_errors(y, y_ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)
    # the single call (quantizer + gemv) gives the same Y
    y1 = lin.forward(_cuda(x, torch.bfloat16), bits, sym).float().cpu().numpy()
    assert np.array_equal(y1, y)


@pytest.mark.parametrize("M", [1, 5, 16, 24])  # 24: two 16-token groups (few tiles: the gemv up to 32)
@pytest.mark.parametrize("K,N", [(1536, 1000), (1552, 264), (11008, 520)])
@pytest.mark.parametrize("r_mode,bits,sym", [("int", 8, False), ("dense", 4, True), ("none", 8, True)])
def test_int_decode_gemv_w4_parity(D, M, K, N, r_mode, bits, sym):
    # packed INT4 weights (0.5 B / weight) at decode sizes: the gemv widens the CTA-pair kernel's
    # tiled nibbles in registers; ragged K (1552 = 12 * 128 + 16) reads the zero-padded tail
    r = 64
    rng = np.random.default_rng(M + K + N)
    x = _bf16_outlier_x(M, K, seed=M + 1)
    w = rng.standard_normal((K, N)) * 0.02
    idx = np.arange(r)
    if r_mode == "none":
        main = O.quantize_symmetric(w, O.IntCfg(4, True, K, "row"))
        comp, kw = None, {}
    else:
        main, comp = O.build_per_channel_int(w, idx, r_mode=r_mode)
        kw = (dict(r_dense=comp.r_dense) if r_mode == "dense" else dict(r_codes=comp.r_q.codes, r_scales=comp.r_q.scales))
        kw["salient_idx"] = idx
    lin = D.IntLinear(main.codes, main.scales, 4, weight_format="int4", **kw)
    nbytes, packed = lin.weight_bytes()
    assert packed and nbytes == -(-N // 128) * -(-K // 128) * 128 * 64
    act = lin.quantize(_cuda(x, torch.bfloat16), bits, sym)
    acc = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    accr = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    y = lin.gemm(act, acc_dump=acc, accr_dump=accr).float().cpu().numpy()
    assert D.last_kernel() == "serq_i8_gemv_kernel"
    cfg = O.IntCfg(bits, sym, "per-row")
    y_ref, xq = O.forward_int(x, main, comp, cfg, symmetric_act=sym)
    _, parts = O.int_gemm(xq, main, return_partials=True)
    assert np.array_equal(acc.cpu().numpy().astype(np.int64), parts[0][1])
    if r_mode == "int":
        _, rp = O.int_gemm(O.gather_columns(xq, idx), comp.r_q, return_partials=True)
        assert np.array_equal(accr.cpu().numpy().astype(np.int64), rp[0][1])
    mx, mean = O.parity_errors(y, y_ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)
    # same Y as the int8-resident copy of the same weights
    lin8 = D.IntLinear(main.codes, main.scales, 4, **kw)
    assert np.array_equal(lin8.gemm(act).float().cpu().numpy(), y)


@pytest.mark.parametrize("M,K,N,r", [(5, 512, 264, 48), (300, 1024, 520, 128), (2048, 4096, 1024, 64)])
def test_mx_svd_baseline_matches_oracle(D, M, K, N, r):
    # SVD baseline over an MX main (compensate.py:326-331): x_hat = mx_decode(x_mx) exact in bf16,
    # (x_hat L1) L2 as the MX kernel's fp32 addend; Y vs the oracle at the north_star tolerance
    rng = np.random.default_rng(M + N)
    x = _bf16_outlier_x(M, K, seed=M)
    w = rng.standard_normal((K, N)) * 0.02
    main_t = O.mx_encode(w.T, 32)
    u, sv, vt = np.linalg.svd(w - O.mx_decode(main_t).T, full_matrices=False)
    l1, l2 = u[:, :r] * np.sqrt(sv[:r]), np.sqrt(sv[:r])[:, None] * vt[:r]
    lin = D.SvdMxLinear(main_t.element_codes, main_t.block_scale_exponents, l1, l2)
    xt = _cuda(x, torch.bfloat16)
    # the decoded activation is exactly the oracle's mx_decode(mx_encode(x))
    xhat = D.mx_decode_bf16(lin.lin.quantize(xt)).double().cpu().numpy()
    assert np.array_equal(xhat, O.mx_decode(O.mx_encode(x, 32)))
    y = lin(xt).float().cpu().numpy()
    y_ref = O.forward_mx(x, main_t, O.Comp(r, l1=l1, l2=l2))
    mx, mean = O.parity_errors(y, y_ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


def test_mx_decode_bf16_many_rows_and_extremes(D):
    # serq_mx_decode_bf16 past the 65535-row grid limit (grid-stride rows) and at the exponent
    # extremes (subnormal-range blocks take the ldexpf path): exact vs the oracle's mx_decode
    rng = np.random.default_rng(17)
    x = rng.standard_normal((70000, 64)).astype(np.float32)
    x[:8] *= np.float32(2.0 ** -120)  # blocks whose smallest values are bf16 subnormals
    x[8:16] *= np.float32(2.0 ** 100)
    xt = torch.from_numpy(x).cuda()
    act = D.quantize_mx(xt)
    got = D.mx_decode_bf16(act).double().cpu().numpy()
    ref = O.mx_decode(O.mx_encode(x.astype(np.float64), 32))
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("M,K,N,r", [(3, 512, 264, 32), (300, 1024, 520, 64), (1024, 2048, 1024, 128)])
def test_mx_dense_r_matches_oracle(D, M, K, N, r):
    # MX main + unquantized R at an arbitrary salient set (compensate.py:335-339)
    rng = np.random.default_rng(M + r)
    x = _bf16_outlier_x(M, K, seed=M + 2)
    w = rng.standard_normal((K, N)) * 0.02
    main_t = O.mx_encode(w.T, 32)
    idx = np.sort(rng.choice(K, r, replace=False))
    r_dense = (w - O.mx_decode(main_t).T)[idx]
    lin = D.MxDenseRLinear(main_t.element_codes, main_t.block_scale_exponents, r_dense, idx)
    y = lin(_cuda(x, torch.bfloat16)).float().cpu().numpy()
    y_ref = O.forward_mx(x, main_t, O.Comp(r, idx, r_dense=r_dense))
    mx, mean = O.parity_errors(y, y_ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


@pytest.mark.parametrize("M,K,N,r", [(300, 1024, 512, 128), (2048, 4096, 1024, 128), (40, 512, 256, 8)])
def test_svd_baseline_fused_matches_oracle(D, M, K, N, r):
    # SVD baseline (compensate.py:304-310): U = (codes - zp) L1 by one bf16 GEMM, U L2 as the
    # fused kernel's dense side term; vs the oracle's f64 (x_hat L1) L2 at the north_star tolerance
    rng = np.random.default_rng(M + r)
    x = _bf16_outlier_x(M, K, seed=7)
    w = rng.standard_normal((K, N)) * 0.02
    main = O.quantize_symmetric(w, O.IntCfg(4, True, K, "row"))
    err = w - O.dequantize(main)
    u, sv, vt = np.linalg.svd(err, full_matrices=False)
    l1, l2 = u[:, :r] * sv[:r], vt[:r]
    lin = D.SvdIntLinear(main.codes, main.scales, 4, l1, l2)
    y = lin.forward(_cuda(x, torch.bfloat16), 8, False).float().cpu().numpy()
    y_ref, _ = O.forward_int(x, main, O.Comp(r, l1=l1, l2=l2), O.IntCfg(8, False, "per-row"))
    mx, mean = O.parity_errors(y, y_ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


@pytest.mark.parametrize("M,N,r_mode", [(300, 520, "int"), (257, 1000, "dense"), (129, 136, "int")])
def test_int_linear_ragged_narrow_tiles(D, M, N, r_mode):
    # few tiles -> the 128-column CTA-pair tiles; ragged M and N (partial last tiles)
    K, r = 1024, 64
    x = _bf16_outlier_x(M, K, seed=M + N)
    w = np.random.default_rng(N).standard_normal((K, N)) * 0.02
    main, comp = O.build_per_channel_int(w, np.arange(r), r_mode=r_mode)
    kw = dict(r_dense=comp.r_dense) if r_mode == "dense" else dict(r_codes=comp.r_q.codes, r_scales=comp.r_q.scales)
    lin = D.IntLinear(main.codes, main.scales, 4, salient_idx=np.arange(r), **kw)
    act = lin.quantize(_cuda(x, torch.bfloat16), 8, False)
    acc = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    y = lin.gemm(act, acc_dump=acc).float().cpu().numpy()
    y_ref, xq = O.forward_int(x, main, comp, O.IntCfg(8, False, "per-row"))
    _, parts = O.int_gemm(xq, main, return_partials=True)
    assert np.array_equal(acc.cpu().numpy().astype(np.int64), parts[0][1])
    mx, mean = O.parity_errors(y, y_ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


def test_int_linear_golden(D, golden):
    x, w = golden["fint_x"], golden["fint_w"]
    main, comp = O.build_per_channel_int(w, np.arange(32), r_mode="int")
    lin = D.IntLinear(main.codes, main.scales, 4, r_codes=comp.r_q.codes, r_scales=comp.r_q.scales,
                      salient_idx=np.arange(32))
    for bits in (4, 8):
        act = lin.quantize(_cuda(x, torch.bfloat16), bits, False)
        acc = torch.zeros((x.shape[0], w.shape[1]), dtype=torch.int32, device="cuda")
        accr = torch.zeros_like(acc)
        y = lin.gemm(act, acc_dump=acc, accr_dump=accr).float().cpu().numpy()
        assert np.array_equal(acc.cpu().numpy(), golden[f"fint_acc_a{bits}"])
        assert np.array_equal(accr.cpu().numpy(), golden[f"fint_accr_a{bits}"])
        mx, mean = O.parity_errors(y, golden[f"fint_y_a{bits}"])
        assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


def test_int_linear_gather_int_r(D):
    M, K, N, r = 64, 512, 256, 32
    x = _bf16_outlier_x(M, K, seed=21)
    w = np.random.default_rng(22).standard_normal((K, N)) * 0.02
    idx = np.random.default_rng(23).permutation(K)[:r]
    main, comp = O.build_per_channel_int(w, idx, r_mode="int")
    lin = D.IntLinear(main.codes, main.scales, 4, r_codes=comp.r_q.codes, r_scales=comp.r_q.scales, salient_idx=idx)
    assert not lin.contiguous
    act = lin.quantize(_cuda(x, torch.bfloat16), 8, False)
    y = lin.gemm(act).float().cpu().numpy()
    y_ref, _ = O.forward_int(x, main, comp, O.IntCfg(8, False, "per-row"))
    mx, mean = O.parity_errors(y, y_ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


# ---------------------------------------------------------------- K3 with group-wise weight scales


@pytest.mark.parametrize("M,K,N,g,r,bits,symmetric,r_mode", [
    (300, 1024, 512, 128, 64, 8, False, "int"),
    (200, 2048, 768, 128, 128, 4, False, "int"),
    (100, 1024, 1000, 256, 64, 8, False, "dense"),
    (512, 1024, 512, 128, 64, 4, True, "col"),
    (70, 512, 264, 128, 0, 8, False, "none"),
    (600, 3072, 512, 1024, 32, 8, False, "int"),
    (256, 2048, 512, 128, 128, 8, False, "col"),    # the paper's g = r = 128 with default_r_config R
    (130, 1024, 776, 256, 96, 4, False, "dense"),
    (300, 1024, 512, 128, 128, 8, False, "split"),  # dequantize(col-grouped R) as bf16 hi + lo
    (64, 2048, 256, 2048, 64, 8, False, "split"),   # one group spanning K: the split R on a per-channel main
    # decode sizes (M <= 16): the group-wise gemv (whole groups per warp, fp32 promotion)
    (1, 1024, 520, 128, 128, 8, False, "int"),
    (5, 2048, 264, 256, 64, 4, True, "dense"),
    (16, 1024, 512, 128, 128, 8, False, "split"),
    (3, 4096, 1000, 128, 64, 8, False, "none"),
    # 16 < M <= 64: the same gemv over 16-token groups (grid rows)
    (24, 1024, 520, 128, 128, 8, False, "int"),
    (32, 2048, 264, 256, 64, 4, True, "dense"),
    (64, 2048, 264, 256, 64, 4, True, "dense"),  # past the token-grouped gemv: the i8g pair kernel
])
def test_int_grouped_linear_parity(D, M, K, N, g, r, bits, symmetric, r_mode):
    # int_gemm_reference row-grouped branch: one exact integer partial per group
    # (acc_dump [G, M, N]), promoted with the group's scales in fp32
    x = _bf16_outlier_x(M, K, seed=M + g)
    w = np.random.default_rng(K + g).standard_normal((K, N)) * 0.02
    main, comp = O.build_grouped_int(w, np.arange(r), g, 4, {"none": "int", "split": "col"}.get(r_mode, r_mode))
    if r_mode == "none":
        comp = None
    kw = {}
    if r_mode == "dense":
        kw = dict(r_dense=comp.r_dense, salient_idx=np.arange(r))
    elif r_mode == "col":
        kw = dict(r_dense=O.dequantize(comp.r_q), salient_idx=np.arange(r))
    elif r_mode == "split":
        kw = dict(r_dense=O.dequantize(comp.r_q), salient_idx=np.arange(r), r_split=True)
    elif r_mode == "int":
        kw = dict(r_codes=comp.r_q.codes, r_scales=comp.r_q.scales, salient_idx=np.arange(r))
    lin = D.IntLinear(main.codes, main.scales, 4, group_size=g, **kw)
    act = lin.quantize(_cuda(x, torch.bfloat16), bits, symmetric)
    G = K // g
    acc = torch.zeros((G, M, N), dtype=torch.int32, device="cuda")
    accr = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    for _ in range(2):
        y = lin.gemm(act, acc_dump=acc, accr_dump=accr).float().cpu().numpy()
        cfg = O.IntCfg(bits, symmetric, "per-row")
        y_ref, xq = O.forward_int(x, main, comp, cfg, symmetric_act=symmetric)
        _, parts = O.int_gemm(xq, main, return_partials=True)
        assert len(parts) == G
        for gi in range(G):
            assert np.array_equal(acc[gi].cpu().numpy().astype(np.int64), parts[gi][1]), gi
        if r_mode == "int":
            _, rp = O.int_gemm(O.gather_columns(xq, np.arange(r)), comp.r_q, return_partials=True)
            assert np.array_equal(accr.cpu().numpy().astype(np.int64), rp[0][1])
        mx, mean = O.parity_errors(y, y_ref)
        assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)
    assert D.last_kernel() == ("serq_i8_gemv_kernel" if M <= 32 else "serq_i8g_pair_kernel")


def test_int_grouped_rejects_unsupported_groups(D):
    from paper_2603_08185_b200.errors import ValidationError

    K, N = 512, 256
    w = np.random.default_rng(3).standard_normal((K, N)) * 0.02
    for g in (64, 32):
        main = O.quantize_symmetric(w, O.IntCfg(4, True, g, "row"))
        with pytest.raises(ValidationError):
            D.IntLinear(main.codes, main.scales, 4, group_size=g)


# ---------------------------------------------------------------- decode (M <= 16): swap-AB split-K kernel


@pytest.mark.parametrize("M,K,N,r", [(1, 2048, 1536, 64), (4, 4096, 1024, 64), (16, 2048, 1000, 64),
                                     (3, 1024, 512, 0), (16, 11008 // 32 * 32, 768, 64),
                                     # stream-K partitions: whole tiles per CTA (K=256), tiles split over
                                     # several CTAs (few tiles, long K), ragged N, 86 tiles on 148 SMs
                                     (7, 256, 11008, 0), (2, 512, 20000, 64), (16, 11008, 256, 64),
                                     (5, 8192, 200, 32), (1, 4096, 11008, 64), (16, 11008, 4096, 64),
                                     (1, 32768, 128, 64),  # one tile over many CTAs (slot cap 32)
                                     # R zero-padded to 64 / 128 columns (two K = 64 salient MMAs)
                                     (1, 4096, 1024, 128), (16, 2048, 768, 96), (4, 8192, 512, 128),
                                     (8, 4096, 296, 128), (3, 1024, 384, 32)])
def test_mx_decode_parity(D, M, K, N, r):
    x, main_t, comp = _mx_case(M, K, N, r, seed=K + M)
    lin = D.MxLinear(main_t.element_codes, main_t.block_scale_exponents,
                     comp.r_q.element_codes if r else None, comp.r_q.block_scale_exponents if r else None,
                     np.arange(r) if r else None)
    xt = _cuda(x, torch.bfloat16)
    ref = O.forward_mx(x, main_t, comp)
    # the split-K partials meet through the narrow DSMEM buffer or, when they do not fit it
    # (e.g. M = 16 with many CTAs per tile), through the drained pipeline stages
    for _ in range(2):
        # serq_forward_mx: for M <= 8 the quantizer runs inside the decode kernel; Y and
        # the activation codes it reports
        act = D.MxActivation(torch.empty(D.mx_sizes(M, K)[0], dtype=torch.uint8, device="cuda"),
                             torch.empty(D.mx_sizes(M, K)[1], dtype=torch.uint8, device="cuda"), M, K)
        y = lin.forward(xt, act).float().cpu().numpy()
        assert D.last_kernel().startswith("serq_mx_decode_cl_kernel")
        # two-kernel path (quantizer, then the linear on codes)
        y2 = lin.gemm(lin.quantize(xt)).float().cpu().numpy()
        mx, mean = O.parity_errors(y, ref)
        assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)
        c, e = D.unpack_mx(act.codes, act.sf, M, K)
        enc = O.mx_encode(x, 32)
        assert np.array_equal(c.cpu().numpy(), enc.element_codes)
        assert np.array_equal(e.cpu().numpy(), enc.block_scale_exponents)
        assert np.array_equal(y2, y)


@pytest.mark.parametrize("M,K,N,gather", [(2560, 1024, 2048, False), (2600, 512, 4096, False),
                                          (4096, 1024, 4096, False), (2600, 512, 4096, True)])
def test_mx_linear_narrow_last_round(D, M, K, N, gather):
    # the leftover tiles of the last partial round run as 256 x 128 tiles (two per tile);
    # gather: an arbitrary salient set (the salient MMA's A operand from the quantizer's slice)
    r = 64
    idx = np.sort(np.random.default_rng(7).choice(K, r, replace=False)) if gather else np.arange(r)
    x = _bf16_outlier_x(M, K, seed=M + N)
    w = np.random.default_rng(M + N + 1).standard_normal((K, N)) * 0.02
    main_t, comp = O.build_serq_rtn_mx(w, idx, 32)
    lin = D.MxLinear(main_t.element_codes, main_t.block_scale_exponents, comp.r_q.element_codes,
                     comp.r_q.block_scale_exponents, idx)
    xt = _cuda(x, torch.bfloat16)
    y = lin(xt).float().cpu().numpy()
    assert D.last_kernel() == ("serq_mx_pair3_kernel<gather>" if gather else "serq_mx_pair3_kernel")
    assert np.array_equal(lin(xt).float().cpu().numpy(), y)  # deterministic
    rows = np.r_[0:64, M - 300:M]  # oracle on the first rows and on the last (narrow-tile) rows
    ref = O.forward_mx(x[rows], main_t, comp)
    mx, mean = O.parity_errors(y[rows], ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


@pytest.mark.parametrize("M", [1000, 300, 4096])
def test_mx_forward_host_chunked(D, M):
    # serq_forward_mx_host pipelines H2D / quantize+linear / D2H over 256-row
    # chunks: rows land in the same tiles' K order as the device path, so the
    # output equals the device path exactly when every chunk runs the pair kernel
    K, N, r = 1024, 512, 64
    x, main_t, comp = _mx_case(M, K, N, r, seed=M + 5)
    lin = D.MxLinear(main_t.element_codes, main_t.block_scale_exponents, comp.r_q.element_codes,
                     comp.r_q.block_scale_exponents, np.arange(r))
    xh = torch.from_numpy(x).to(torch.bfloat16).pin_memory()
    yh = torch.empty((M, N), dtype=torch.bfloat16).pin_memory()
    lin.forward_host(xh, yh)
    y = yh.float().numpy()
    mx, mean = O.parity_errors(y, O.forward_mx(x, main_t, comp))
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)
    if M % 256 == 0 or M % 256 > 128:
        yd = lin(xh.to("cuda")).cpu()
        assert torch.equal(yd, yh)


@pytest.mark.parametrize("M", [1000, 2600])
def test_mx_forward_host_chunked_gather(D, M):
    # the host pipeline on a non-contiguous salient set: the salient slice is
    # re-encoded per chunk and every chunk reaches the gather variant of the linear
    K, N, r = 1024, 512, 64
    x = _bf16_outlier_x(M, K, seed=M + 9)
    w = np.random.default_rng(M).standard_normal((K, N)) * 0.02
    idx = np.random.default_rng(M + 1).permutation(K)[:r]
    main_t, comp = O.build_serq_rtn_mx(w, idx, 32)
    lin = D.MxLinear(main_t.element_codes, main_t.block_scale_exponents, comp.r_q.element_codes,
                     comp.r_q.block_scale_exponents, idx)
    assert not lin.contiguous
    xh = torch.from_numpy(x).to(torch.bfloat16).pin_memory()
    yh = torch.empty((M, N), dtype=torch.bfloat16).pin_memory()
    lin.forward_host(xh, yh)
    mx, mean = O.parity_errors(yh.float().numpy(), O.forward_mx(x, main_t, comp))
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


@pytest.mark.parametrize("M,K,N", [(4096, 1024, 1024), (1000, 2048, 768), (2600, 512, 4096)])
def test_mx_forward_fused_equals_two_launches(D, M, K, N):
    # serq_forward_mx (one C-ABI call, PDL between the two kernels) must equal
    # quantize-then-linear exactly, on every call
    r = 64
    x, main_t, comp = _mx_case(M, K, N, r, seed=M + 7)
    lin = D.MxLinear(main_t.element_codes, main_t.block_scale_exponents, comp.r_q.element_codes,
                     comp.r_q.block_scale_exponents, np.arange(r))
    xt = _cuda(x, torch.bfloat16)
    y2 = lin.gemm(lin.quantize(xt))
    for _ in range(3):
        y1 = lin.forward(xt)
        assert torch.equal(y1, y2)
    mx, mean = O.parity_errors(y2.float().cpu().numpy(), O.forward_mx(x, main_t, comp))
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


def _near_midpoint(y, bs=32, rel=1e-12):
    """Elements whose scaled magnitude lies within `rel` of an E2M1 rounding
    midpoint, or whose block amax is within `rel` of a power of two: the only
    places a last-ulp difference in the f64 normalisation can change a code."""
    M, K = y.shape
    blk = np.abs(y).reshape(M, K // bs, bs)
    amax = blk.max(axis=2, keepdims=True)
    with np.errstate(divide="ignore"):
        lg = np.log2(np.where(amax > 0, amax, 1.0))
    e_edge = np.abs(lg - np.round(lg)) < rel * 4
    e = np.where(amax > 0, np.floor(lg) - 2, 0)
    s = blk / np.exp2(e)
    mids = np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0])
    near = (np.abs(s[..., None] - mids) <= rel * np.maximum(s[..., None], 1e-300)).any(axis=-1)
    return (near | e_edge).reshape(M, K)


@pytest.mark.parametrize("dtype,M,K", [("bf16", 300, 4096), ("f32", 64, 1024), ("bf16", 5, 8192)])
def test_rmsnorm_quant_mx_matches_reference_order(D, dtype, M, K):
    rng = np.random.default_rng(M + K)
    x = O.bf16_round(_bf16_outlier_x(M, K, seed=K) * 3.0)
    if dtype == "f32":
        x = x + rng.standard_normal(x.shape) * 1e-3
        x = x.astype(np.float32).astype(np.float64)
    gain = (np.abs(rng.standard_normal(K)) + 0.5) / np.exp2(rng.uniform(-2, 2, K))  # ln weight / SAF scales
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    act = D.rmsnorm_quantize_mx(_cuda(x, tdt), torch.from_numpy(gain).to("cuda"), 1e-6)
    c, e = D.unpack_mx(act.codes, act.sf, M, K)
    yref = O.rmsnorm(x, gain, 1e-6)
    ref = O.mx_encode(yref, 32)
    eb = np.repeat(e.cpu().numpy() != ref.block_scale_exponents, 32, axis=1)
    diff = (c.cpu().numpy() != ref.element_codes) | eb
    allowed = _near_midpoint(yref)
    assert not (diff & ~allowed).any(), int((diff & ~allowed).sum())


def test_rmsnorm_fused_linear_parity(D):
    M, K, N, r = 512, 2048, 768, 64
    x, main_t, comp = _mx_case(M, K, N, r, seed=31)
    gain = np.abs(np.random.default_rng(32).standard_normal(K)) + 0.5
    lin = D.MxLinear(main_t.element_codes, main_t.block_scale_exponents, comp.r_q.element_codes,
                     comp.r_q.block_scale_exponents, np.arange(r))
    y = lin.forward_rmsnorm(_cuda(x, torch.bfloat16), torch.from_numpy(gain).to("cuda")).float().cpu().numpy()
    mx, mean = O.parity_errors(y, O.forward_mx(O.rmsnorm(x, gain), main_t, comp))
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


@pytest.mark.parametrize("M,K,r", [(300, 4096, 64), (17, 1024, 128), (130, 8192, 32)])
def test_rmsnorm_quant_mx_gather(D, M, K, r):
    # the gather fallback inside the producer fusion: rmsnorm(x)[:, idx] encoded by the same kernel
    # (compensate.py:335 re-encodes the salient columns of the normalised row)
    rng = np.random.default_rng(M + r)
    x = O.bf16_round(_bf16_outlier_x(M, K, seed=r) * 2.0)
    gain = np.abs(rng.standard_normal(K)) + 0.5
    idx = rng.permutation(K)[:r]
    act = D.rmsnorm_quantize_mx(_cuda(x, torch.bfloat16), torch.from_numpy(gain).to("cuda"), 1e-6,
                                gather_idx=torch.from_numpy(idx.astype(np.int32)).to("cuda"), r=r)
    yref = O.rmsnorm(x, gain, 1e-6)
    for codes, sf, cols, ref_y in ((act.codes, act.sf, K, yref), (act.xs_codes, act.xs_sf, r, yref[:, idx])):
        c, e = D.unpack_mx(codes, sf, M, cols)
        ref = O.mx_encode(np.ascontiguousarray(ref_y), 32)
        eb = np.repeat(e.cpu().numpy() != ref.block_scale_exponents, 32, axis=1)
        diff = (c.cpu().numpy() != ref.element_codes) | eb
        assert not (diff & ~_near_midpoint(np.ascontiguousarray(ref_y))).any()


def test_rmsnorm_fused_linear_gather_parity(D):
    M, K, N, r = 400, 2048, 512, 64
    x = O.bf16_round(_bf16_outlier_x(M, K, seed=51))
    w = np.random.default_rng(52).standard_normal((K, N)) * 0.02
    idx = np.random.default_rng(53).permutation(K)[:r]
    main_t, comp = O.build_serq_rtn_mx(w, idx, 32)
    gain = np.abs(np.random.default_rng(54).standard_normal(K)) + 0.5
    lin = D.MxLinear(main_t.element_codes, main_t.block_scale_exponents, comp.r_q.element_codes,
                     comp.r_q.block_scale_exponents, idx)
    assert not lin.contiguous
    y = lin.forward_rmsnorm(_cuda(x, torch.bfloat16), torch.from_numpy(gain).to("cuda")).float().cpu().numpy()
    mx, mean = O.parity_errors(y, O.forward_mx(O.rmsnorm(x, gain), main_t, comp))
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


def test_rmsnorm_quant_mx_exact_fallback_blocks(D):
    # rows built so many blocks sit exactly on E2M1 decision points / power-of-two maxima after
    # normalisation: the kernel must send them through its exact f64 path
    K = 256
    base = np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0, 6.0] * (K // 8))
    x = np.stack([base * 2.0 ** k for k in range(-3, 5)])
    x = O.bf16_round(x)
    gain = np.ones(K)
    act = D.rmsnorm_quantize_mx(_cuda(x, torch.bfloat16), torch.from_numpy(gain).to("cuda"), 0.0)
    c, e = D.unpack_mx(act.codes, act.sf, *x.shape)
    ref = O.mx_encode(O.rmsnorm(x, gain, 0.0), 32)
    assert np.array_equal(e.cpu().numpy(), ref.block_scale_exponents)
    assert np.array_equal(c.cpu().numpy(), ref.element_codes)


# ---------------------------------------------------------------- RMSNorm -> INT producer


def _check_rms_int(D, x, tdt, gain, eps, bits, symmetric, exact_f64=False):
    act = D.rmsnorm_quantize_int(_cuda(x, tdt), torch.from_numpy(gain).to("cuda"), eps, bits, symmetric,
                                 exact_f64=exact_f64)
    cfg = O.IntCfg(bits, symmetric, "per-row")
    y = O.rmsnorm(x, gain, eps)
    ref = O.quantize_symmetric(y, cfg) if symmetric else O.quantize_asymmetric(y, cfg)
    codes = act.codes.cpu().numpy()
    codes = codes.astype(np.int32) if symmetric else codes.view(np.uint8).astype(np.int32)
    assert np.array_equal(act.scale64.cpu().numpy(), ref.scales[:, 0])
    if not symmetric:
        assert np.array_equal(act.zp.cpu().numpy(), ref.zero_points[:, 0])
    assert np.array_equal(codes, ref.codes), int((codes != ref.codes).sum())


# K % 8 != 0 (100, 4100) runs the all-f64 kernel, the rest the f32-bounded fast kernel
@pytest.mark.parametrize("dtype,K", [("bf16", 100), ("bf16", 1000), ("bf16", 1024), ("f32", 2560), ("bf16", 3008),
                                     ("bf16", 4096), ("f32", 4100), ("bf16", 6144), ("f32", 8192), ("bf16", 8192)])
@pytest.mark.parametrize("bits,symmetric", [(8, False), (4, True), (4, False)])
def test_rmsnorm_quant_int_bitexact(D, dtype, K, bits, symmetric):
    # codes, f64 scales and zero points of quantize_*(rmsnorm(x, gain)) bit for bit: the kernel
    # replays NumPy's pairwise row sum, so even the f64 rms equals the reference's
    M = 67
    rng = np.random.default_rng(K + bits)
    x = O.bf16_round(_bf16_outlier_x(M, K, seed=K) * 3.0)
    if dtype == "f32":
        x = (x + rng.standard_normal(x.shape) * 1e-3).astype(np.float32).astype(np.float64)
    gain = (np.abs(rng.standard_normal(K)) + 0.5) / np.exp2(rng.uniform(-2, 2, K))
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    _check_rms_int(D, x, tdt, gain, 1e-6, bits, symmetric)
    if K in (1024, 3008):
        _check_rms_int(D, x, tdt, gain, 1e-6, bits, symmetric, exact_f64=True)


@pytest.mark.parametrize("symmetric", [True, False])
@pytest.mark.parametrize("K", [1024, 4096])
def test_rmsnorm_quant_int_fast_kernel_ties_and_slow_rows(D, symmetric, K):
    # rows built to stress the fast kernel's bounds: (a) exact .5 ties of y / s (|x| = 2 with
    # eps = 0: rms = 2, y = +-1, s = 2/255 -> y / s = +-127.5), (b) values so small that the f32
    # pass would go denormal (whole row in f64), (c) huge values, (d) an f32-denormal gain entry
    # and zero rows (eps > 0)
    rng = np.random.default_rng(5)
    x = O.bf16_round(rng.standard_normal((5, K)))
    x[0] = np.where(rng.random(K) < 0.5, -2.0, 2.0)
    x[1] = O.bf16_round(rng.standard_normal(K) * 1e-33)
    x[2] = O.bf16_round(rng.standard_normal(K) * 1e30)
    x[3, ::3] = 0.0
    gain = np.ones(K)
    _check_rms_int(D, x, torch.bfloat16, gain, 0.0, 8, symmetric)
    x2 = x.copy()
    x2[4] = 0.0
    gain2 = np.abs(rng.standard_normal(K)) + 0.5
    gain2[7] = 1e-40
    gain2[9] = 0.0
    _check_rms_int(D, x2, torch.bfloat16, gain2, 1e-6, 8, symmetric)


@pytest.mark.parametrize("dtype,K", [("bf16", 4096), ("f32", 2048)])
def test_rmsnorm_quant_int_fast_matches_f64_kernel(D, dtype, K):
    # the two kernels agree on a larger sample (the fast one's exactness argument, checked)
    M = 1024
    x = _bf16_outlier_x(M, K, seed=21) * 1.7
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    xt = _cuda(x, tdt)
    g = torch.from_numpy(np.random.default_rng(2).uniform(0.3, 3.0, K)).to("cuda")
    for bits, sym in ((8, False), (4, True), (2, False)):
        a = D.rmsnorm_quantize_int(xt, g, 1e-6, bits, sym)
        b = D.rmsnorm_quantize_int(xt, g, 1e-6, bits, sym, exact_f64=True)
        assert torch.equal(a.codes, b.codes) and torch.equal(a.scale64, b.scale64)
        if not sym:
            assert torch.equal(a.zp, b.zp)


@pytest.mark.parametrize("r_mode,contiguous", [("int", True), ("dense", True), ("int", False)])
def test_rmsnorm_fused_int_linear_matches_two_step(D, r_mode, contiguous):
    # linear(rmsnorm(x)) with the norm fused into K1-INT == the linear on the reference's rmsnorm
    # output quantized by the plain K1-INT (same codes -> identical bf16 Y), incl. the xs slices
    M, K, N, r = 300, 2048, 512, 64
    rng = np.random.default_rng(3)
    x = O.bf16_round(_bf16_outlier_x(M, K, seed=9) * 2.0)
    gain = np.abs(rng.standard_normal(K)) + 0.5
    w = rng.standard_normal((K, N)) * 0.02
    idx = np.arange(r) if contiguous else np.sort(rng.choice(K, r, replace=False))
    main, comp = O.build_per_channel_int(w, idx, r_mode=r_mode)
    kw = dict(r_dense=comp.r_dense) if r_mode == "dense" else dict(r_codes=comp.r_q.codes, r_scales=comp.r_q.scales)
    lin = D.IntLinear(main.codes, main.scales, 4, salient_idx=idx, **kw)
    y1 = lin.forward_rmsnorm(_cuda(x, torch.bfloat16), torch.from_numpy(gain).to("cuda"), 1e-6, 8, False)
    y2 = lin.gemm(lin.quantize(_cuda(O.rmsnorm(x, gain, 1e-6), torch.float64), 8, False))
    assert torch.equal(y1, y2)


def test_rmsnorm_quant_int_constant_and_zero_rows(D):
    # all-zero rows (rms = sqrt(eps), scale 0 -> 1) and constant rows (hi == lo)
    K = 1024
    x = np.zeros((4, K))
    x[1] = 3.0
    x[2, ::2] = -1.5
    x[3] = _bf16_outlier_x(1, K, seed=4)[0]
    gain = np.ones(K)
    for sym in (True, False):
        act = D.rmsnorm_quantize_int(_cuda(x, torch.bfloat16), torch.from_numpy(gain).to("cuda"), 1e-6, 8, sym)
        cfg = O.IntCfg(8, sym, "per-row")
        y = O.rmsnorm(x, gain, 1e-6)
        ref = O.quantize_symmetric(y, cfg) if sym else O.quantize_asymmetric(y, cfg)
        codes = act.codes.cpu().numpy()
        codes = codes.astype(np.int32) if sym else codes.view(np.uint8).astype(np.int32)
        assert np.array_equal(act.scale64.cpu().numpy(), ref.scales[:, 0])
        assert np.array_equal(codes, ref.codes)


@pytest.mark.parametrize("world", [2, 4])
def test_tp_shards_on_device_match_single_device(D, world):
    # SURVEY 8(e) with the real kernels: the per-rank shards of a column-parallel and a
    # row-parallel MX linear, run one after another on this GPU, reproduce the unsharded
    # layer -- column shards concatenate bit-exactly, row shards sum (the all-reduce, in
    # bf16 as NCCL would) to the single-device oracle within tolerance
    from paper_2603_08185_b200 import tp

    rng = np.random.default_rng(40 + world)
    M, K, N, r_rank = 300, 1024, 512, 32
    w = rng.standard_normal((K, N)) * 0.02
    x = O.bf16_round(O.synthetic_activations(M, K, 8, 50.0, 41))
    xt = _cuda(x, torch.bfloat16)
    # column parallel: shard N, X replicated
    main_t, comp = O.build_serq_rtn_mx(w, np.arange(64), 32)
    full = D.MxLinear(main_t.element_codes, main_t.block_scale_exponents, comp.r_q.element_codes,
                      comp.r_q.block_scale_exponents, np.arange(64))(xt)
    parts = []
    for rank in range(world):
        n0, n1 = tp.column_shard(N, world, rank)
        c, e, rc, re_ = tp.shard_columns_mx(main_t.element_codes, main_t.block_scale_exponents,
                                            comp.r_q.element_codes, comp.r_q.block_scale_exponents, n0, n1)
        parts.append(D.MxLinear(c, e, rc, re_, np.arange(64))(xt))
    assert torch.equal(torch.cat(parts, dim=1), full)
    # row parallel: each rank's K-slice leads with its own salient channels; one all-reduce
    perm, _ = tp.row_parallel_salient_layout(np.abs(w).max(axis=1), world, r_rank)
    wp, xp = w[perm], x[:, perm]
    acc = None
    for rank in range(world):
        k0, k1 = tp.row_shard(K, world, rank)
        mt, cp = O.build_serq_rtn_mx(wp[k0:k1], np.arange(r_rank), 32)
        lin = D.MxLinear(mt.element_codes, mt.block_scale_exponents, cp.r_q.element_codes,
                         cp.r_q.block_scale_exponents, np.arange(r_rank))
        y = lin(_cuda(np.ascontiguousarray(xp[:, k0:k1]), torch.bfloat16)).float()
        acc = y if acc is None else acc + y  # the all-reduce, accumulated in fp32
    union = np.concatenate([tp.row_shard(K, world, rk)[0] + np.arange(r_rank) for rk in range(world)])
    mg, cg = O.build_serq_rtn_mx(wp, union, 32)
    mx, mean = O.parity_errors(acc.bfloat16().float().cpu().numpy(), O.forward_mx(xp, mg, cg))
    # each rank's partial is rounded to bf16 before the reduction (world extra roundings of
    # magnitude ~|Y| / sqrt(world)): the mean tolerance scales with the number of partials
    assert mx <= TOL_MAX and mean <= TOL_MEAN * world, (mx, mean)


@pytest.mark.parametrize("M,K,N", [(1, 1024, 768), (5, 4096, 1024), (16, 2048, 11008 // 128 * 128)])
def test_mx_decode_gather_parity(D, M, K, N):
    # decode (M <= 16) with an arbitrary salient set (SURVEY F8's common case): the salient
    # term's B operand is the quantizer's x[:, idx] slice loaded next to R
    r = 64
    rng = np.random.default_rng(M + K)
    x = _bf16_outlier_x(M, K, seed=M + 3)
    w = rng.standard_normal((K, N)) * 0.02
    idx = np.sort(rng.permutation(K)[:r])
    w[idx] *= 8
    main_t, comp = O.build_serq_rtn_mx(w, idx, 32)
    lin = D.MxLinear(main_t.element_codes, main_t.block_scale_exponents, comp.r_q.element_codes,
                     comp.r_q.block_scale_exponents, idx)
    assert not lin.contiguous
    for _ in range(2):
        y = lin(_cuda(x, torch.bfloat16)).float().cpu().numpy()
        mx, mean = O.parity_errors(y, O.forward_mx(x, main_t, comp))
        assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


# ---------------------------------------------------------------- INT single-call and host entry points


@pytest.mark.parametrize("M,K,N,r,r_mode,bits,sym,gather,group", [
    (2048, 4096, 1024, 128, "int", 8, False, False, None),   # C3-like, per-channel, integer R
    (512, 1024, 768, 64, "dense", 4, True, False, None),     # C1-like, symmetric A4, bf16 L
    (300, 1024, 512, 32, "int", 8, False, True, None),       # non-contiguous salient set, integer R
    (1000, 1024, 512, 64, "int", 8, False, False, 128),      # group-wise weights
    (5, 512, 256, 32, "dense", 8, False, True, None),        # small M (1-CTA kernel), gathered dense R
])
def test_int_forward_single_call_and_host(D, M, K, N, r, r_mode, bits, sym, gather, group):
    # serq_forward_int (quantize + linear in one call) == quantize then gemm, bit for bit;
    # serq_forward_int_host (pinned host in / out, chunked) == the device forward
    x = _bf16_outlier_x(M, K, seed=M + K)
    w = np.random.default_rng(N).standard_normal((K, N)) * 0.02
    idx = np.sort(np.random.default_rng(K).choice(K, r, replace=False)) if gather else np.arange(r)
    if group:
        main, comp = O.build_grouped_int(w, idx, group, 4, r_mode=r_mode)
    else:
        main, comp = O.build_per_channel_int(w, idx, 4, r_mode=r_mode)
    kw = dict(r_dense=comp.r_dense) if r_mode == "dense" else dict(r_codes=comp.r_q.codes, r_scales=comp.r_q.scales)
    lin = D.IntLinear(main.codes, main.scales, 4, salient_idx=idx, group_size=group, **kw)
    xt = _cuda(x, torch.bfloat16)
    y1 = lin.forward(xt, bits, sym)
    assert D.last_launch_count() == 2
    y2 = lin.gemm(lin.quantize(xt, bits, sym))
    assert torch.equal(y1, y2)
    xh = xt.cpu().pin_memory()
    yh = torch.empty((M, N), dtype=torch.bfloat16).pin_memory()
    lin.forward_host(xh, yh, bits, sym)
    assert torch.equal(yh, y1.cpu())
    cfg = O.IntCfg(bits, sym, "per-row")
    y_ref, _ = O.forward_int(x, main, comp, cfg, symmetric_act=sym)
    mx, mean = O.parity_errors(y1.float().cpu().numpy(), y_ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


@pytest.mark.parametrize("bits,sym,world", [(8, False, 2), (4, True, 4), (8, False, 8)])
def test_int_k_sharded_quantizer_and_accumulators(D, bits, sym, world):
    # row-parallel INT layer, ranks emulated on one GPU: per-slice ranges, the MIN / MAX
    # reduction (what tp.int_token_range_allreduce does over NCCL), per-slice quantization on
    # the global range -> the unsharded codes / scales / zero points, and per-slice integer
    # accumulators that sum EXACTLY to the single-device ones (int_gemm_reference, mxfmt.py:177-195)
    M, K, N = 300, 4096, 512
    x = _bf16_outlier_x(M, K, seed=world + bits)
    w = np.random.default_rng(world).standard_normal((K, N)) * 0.02
    main = O.quantize_symmetric(w, O.IntCfg(4, True, K, "row"))
    xt = _cuda(x, torch.bfloat16)
    full = D.quantize_int(xt, bits, sym)
    ks = K // world
    rngs = [D.int_token_ranges(xt[:, i * ks:(i + 1) * ks].contiguous()) for i in range(world)]
    g = torch.stack(rngs)
    glob = torch.stack([g[:, 0].amin(0), g[:, 1].amax(0)]).contiguous()
    acc_sum = torch.zeros((M, N), dtype=torch.int64, device="cuda")
    for i in range(world):
        xs_i = xt[:, i * ks:(i + 1) * ks].contiguous()
        a = D.quantize_int_with_range(xs_i, glob, bits, sym)
        assert torch.equal(a.codes, full.codes[:, i * ks:(i + 1) * ks])
        assert torch.equal(a.scale64, full.scale64)
        if not sym:
            assert torch.equal(a.zp, full.zp)
        lin = D.IntLinear(main.codes[i * ks:(i + 1) * ks], main.scales, 4)
        acc = torch.zeros((M, N), dtype=torch.int32, device="cuda")
        lin.gemm(a, acc_dump=acc)
        acc_sum += acc.long()
    cfg = O.IntCfg(bits, sym, "per-row")
    xq = O.quantize_symmetric(x, cfg) if sym else O.quantize_asymmetric(x, cfg)
    _, parts = O.int_gemm(xq, main, return_partials=True)
    assert np.array_equal(acc_sum.cpu().numpy(), parts[0][1])


@pytest.mark.parametrize("M,N,w_bits,r_mode,fmt", [(600, 1024, 8, "int", "int8"),   # 8-bit weights, int8 feed
                                                   (64, 520, 4, "int", "int4"),    # W4 handle at small M
                                                   (1000, 4104, 4, "dense", "int4"),  # W4, ragged N, multi-tile
                                                   (1000, 4104, 4, "dense", "int8")])
def test_int_weight_storage_paths(D, M, N, w_bits, r_mode, fmt):
    # W4 (packed INT4 widened in the SM) and int8 weight feeds of the CTA-pair kernel: exact
    # accumulators against the oracle and the resident weight bytes
    K, r = 2048, 64
    x = _bf16_outlier_x(M, K, seed=M + w_bits)
    w = np.random.default_rng(N + w_bits).standard_normal((K, N)) * 0.02
    main = O.quantize_symmetric(w, O.IntCfg(w_bits, True, K, "row"))
    resid = w[:r] - O.dequantize(main)[:r]
    if r_mode == "dense":
        comp = O.Comp(r, np.arange(r), r_dense=O.bf16_round(resid))
        kw = dict(r_dense=comp.r_dense)
    else:
        comp = O.Comp(r, np.arange(r), r_q=O.quantize_symmetric(resid, O.IntCfg(4, True, r, "row")))
        kw = dict(r_codes=comp.r_q.codes, r_scales=comp.r_q.scales)
    lin = D.IntLinear(main.codes, main.scales, w_bits, salient_idx=np.arange(r), weight_format=fmt, **kw)
    nbytes, packed = lin.weight_bytes()
    if fmt == "int4":
        assert packed and nbytes == -(-N // 128) * 128 * K // 2
    else:
        assert not packed and nbytes == N * K
    act = lin.quantize(_cuda(x, torch.bfloat16), 8, False)
    acc = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    y = lin.gemm(act, acc_dump=acc).float().cpu().numpy()
    if M > 128 or fmt == "int4":
        assert D.last_kernel().startswith("serq_i8_pair_kernel") and D.last_kernel().endswith(",w4>") == (fmt == "int4")
    xq = O.quantize_asymmetric(x, O.IntCfg(8, False, "per-row"))
    _, parts = O.int_gemm(xq, main, return_partials=True)
    assert np.array_equal(acc.cpu().numpy().astype(np.int64), parts[0][1])
    y_ref, _ = O.forward_int(x, main, comp, O.IntCfg(8, False, "per-row"))
    mx, mean = O.parity_errors(y, y_ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


# ---------------------------------------------------------------- fused linears (q/k/v, gate/up)


@pytest.mark.parametrize("M", [1, 5, 16, 64, 300])
@pytest.mark.parametrize("r", [64, 128])
def test_fused_linears_per_part_salient_sets(D, M, r):
    # two (or three) linears reading the same activation, each with its own salient set, packed as
    # ONE handle: one quantizer launch, one kernel (decode / CTA pair) or per-part views -- every
    # part equals the oracle forward of that linear alone (compensate.py:319-340)
    K = 1024
    ns = [512, 768] if r == 64 else [256, 512, 384]
    rng = np.random.default_rng(M + r)
    x = _bf16_outlier_x(M, K, seed=M + 7)
    parts, refs = [], []
    for j, n in enumerate(ns):
        w = rng.standard_normal((K, n)) * 0.02
        idx = np.sort(rng.choice(K, r, replace=False))
        w[idx] *= 8
        main_t, comp = O.build_serq_rtn_mx(w, idx, 32)
        parts.append((main_t.element_codes, main_t.block_scale_exponents, comp.r_q.element_codes,
                      comp.r_q.block_scale_exponents, idx))
        refs.append(O.forward_mx(x, main_t, comp))
    fl = D.FusedMxLinear(parts, prefill_one_kernel=True)
    y = fl(_cuda(x, torch.bfloat16))
    assert D.last_launch_count() >= 1
    if M <= 16 and r == 64:
        assert D.last_kernel().startswith("serq_mx_decode_cl_kernel")
    elif M > 128 and r == 64:
        assert D.last_kernel() == "serq_mx_pair3_kernel<gather>"
    for j, yj in enumerate(fl.split(y)):
        mx, mean = O.parity_errors(yj.float().cpu().numpy(), refs[j])
        assert mx <= TOL_MAX and mean <= TOL_MEAN, (j, mx, mean)


@pytest.mark.parametrize("M", [1, 8, 300])
def test_device_block_fused_linears_match_separate(D, M):
    # the block with q/k/v and up/gate as FusedMxLinear (one quantizer + one kernel each) against
    # the same block with seven separate linears: same artefacts, same math (tolerance: the fused
    # decode kernel splits K differently)
    from paper_2603_08185_b200 import benchmarks as B
    from paper_2603_08185_b200.block import DeviceBlock

    H, F, r = 512, 1024, 64
    rng = np.random.default_rng(M)

    def parts(k, n, s):
        return B.device_mx_parts(k, n, r, seed=s, salient_idx=np.sort(rng.permutation(k)[:r]))

    pq, pk, pv, pu, pg = parts(H, H, 1), parts(H, H, 2), parts(H, H, 3), parts(H, F, 5), parts(H, F, 6)
    po, pd = B.device_mx_parts(H, H, r, seed=4), B.device_mx_parts(F, H, r, seed=7)
    gains = {"ln1": np.abs(rng.standard_normal(H)) + 0.5, "ln2": np.abs(rng.standard_normal(H)) + 0.5}
    sep = DeviceBlock({"q_proj": D.MxLinear(*pq), "k_proj": D.MxLinear(*pk), "v_proj": D.MxLinear(*pv),
                       "o_proj": D.MxLinear(*po), "up_proj": D.MxLinear(*pu), "gate_proj": D.MxLinear(*pg),
                       "down_proj": D.MxLinear(*pd)}, gains, 128)
    fus = DeviceBlock({"qkv_proj": D.FusedMxLinear([pq, pk, pv]), "up_gate_proj": D.FusedMxLinear([pu, pg]),
                       "o_proj": D.MxLinear(*po), "down_proj": D.MxLinear(*pd)}, gains, 128)
    # no outlier channels here: with them the attention logits reach the hundreds and one bf16 ulp
    # of q or k (the fused decode kernel splits K differently) moves the softmax weights visibly --
    # the linears themselves are checked against the oracle in test_fused_linears_per_part_salient_sets
    # Both blocks are valid implementations; their linears differ only in the fp32 summation order
    # of split-K partials, so a bf16 output flips by one ulp now and then (mean ~1.5e-3 of |Y| after
    # five linears): the block-vs-block bound is 1e-2 max / 4e-3 mean.
    x = B.outlier_x(M, H, mag=1.0).float()
    a, b = sep(x).cpu().numpy(), fus(x).cpu().numpy()
    mx, mean = O.parity_errors(b, a)
    assert mx <= TOL_MAX and mean <= 4e-3, (mx, mean)


@pytest.mark.parametrize("M", [1, 5, 16])
def test_block_glue_kernels_match_torch_ops(D, M):
    # the decode-size glue (csrc/serq_block.cuh) against the PyTorch ops it replaces, f32
    from paper_2603_08185_b200 import _lib
    from paper_2603_08185_b200.block import attention_mix, rmsnorm

    H, F, hd = 1024, 2048, 128
    g = torch.Generator(device="cuda").manual_seed(M)
    x = torch.randn((M, H), device="cuda", generator=g) * 3
    o = (torch.randn((M, H), device="cuda", generator=g)).to(torch.bfloat16)
    gain = torch.rand(H, device="cuda", generator=g) + 0.5
    res, h = torch.empty_like(x), torch.empty_like(x)
    _lib.call("serq_block_add_rmsnorm", x.data_ptr(), o.data_ptr(), H, M, H, gain.data_ptr(), 1e-6, res.data_ptr(),
              h.data_ptr(), 0)
    torch.cuda.synchronize()
    r_ref = x + o
    assert torch.equal(res, r_ref)
    torch.testing.assert_close(h, rmsnorm(r_ref, gain, 1e-6), rtol=2e-6, atol=1e-6)
    qkv = (torch.randn((M, 3 * H), device="cuda", generator=g) * 2).to(torch.bfloat16)
    q, k, v = qkv[:, :H], qkv[:, H:2 * H], qkv[:, 2 * H:]
    att = torch.empty((M, H), device="cuda")
    _lib.call("serq_block_attention", q.data_ptr(), q.stride(0), k.data_ptr(), k.stride(0), v.data_ptr(), v.stride(0),
              M, H // hd, hd, 1.0 / hd ** 0.5, att.data_ptr(), H, 0)
    torch.cuda.synchronize()
    torch.testing.assert_close(att, attention_mix(q.contiguous(), k.contiguous(), v.contiguous(), hd), rtol=1e-4,
                               atol=1e-5)
    gate = torch.randn((M, 2 * F), device="cuda", generator=g).to(torch.bfloat16)
    up, gt = gate[:, :F], gate[:, F:]
    mid = torch.empty((M, F), device="cuda")
    _lib.call("serq_block_silu_mul", gt.data_ptr(), gt.stride(0), up.data_ptr(), up.stride(0), M, F, mid.data_ptr(), 0)
    torch.cuda.synchronize()
    torch.testing.assert_close(mid, torch.nn.functional.silu(gt.float()) * up, rtol=2e-6, atol=1e-6)


@pytest.mark.parametrize("M", [1, 3, 16])
@pytest.mark.parametrize("H", [4096, 6144, 8192, 1002])
def test_block_add_rmsnorm_shapes(D, M, H):
    # register-resident residual add + RMSNorm (one or two float4 chunks per thread) and the
    # looped fallback (H = 1002: rows not 16-B aligned), with and without the bf16 addend / res
    from paper_2603_08185_b200 import _lib
    from paper_2603_08185_b200.block import rmsnorm

    g = torch.Generator(device="cuda").manual_seed(M + H)
    x = torch.randn((M, H), device="cuda", generator=g) * 3
    o = (torch.randn((M, H), device="cuda", generator=g)).to(torch.bfloat16)
    gain = torch.rand(H, device="cuda", generator=g) + 0.5
    for with_o in (True, False):
        res, h = torch.empty_like(x), torch.empty_like(x)
        _lib.call("serq_block_add_rmsnorm", x.data_ptr(), o.data_ptr() if with_o else None, H, M, H, gain.data_ptr(),
                  1e-6, res.data_ptr(), h.data_ptr(), 0)
        torch.cuda.synchronize()
        r_ref = x + o if with_o else x
        assert torch.equal(res, r_ref)
        torch.testing.assert_close(h, rmsnorm(r_ref, gain, 1e-6), rtol=2e-6, atol=1e-6)
    # the residual add alone (h NULL): the block's output
    out = torch.empty_like(x)
    _lib.call("serq_block_add_rmsnorm", x.data_ptr(), o.data_ptr(), H, M, H, None, 1e-6, out.data_ptr(), None, 0)
    torch.cuda.synchronize()
    assert torch.equal(out, x + o)


@pytest.mark.parametrize("M", [1, 4, 16])
def test_device_block_glue_path_matches_torch_path(D, M):
    # the whole block at decode size: glue kernels vs the PyTorch glue, same SERQ linears
    from paper_2603_08185_b200 import benchmarks as B
    from paper_2603_08185_b200.block import DeviceBlock

    H, F, r = 512, 1024, 64
    rng = np.random.default_rng(M + 100)

    def parts(k, n, s):
        return B.device_mx_parts(k, n, r, seed=s, salient_idx=np.sort(rng.permutation(k)[:r]))

    lins = {"qkv_proj": D.FusedMxLinear([parts(H, H, 1), parts(H, H, 2), parts(H, H, 3)]),
            "up_gate_proj": D.FusedMxLinear([parts(H, F, 5), parts(H, F, 6)]),
            "o_proj": D.MxLinear(*B.device_mx_parts(H, H, r, seed=4)),
            "down_proj": D.MxLinear(*B.device_mx_parts(F, H, r, seed=7))}
    gains = {"ln1": np.abs(rng.standard_normal(H)) + 0.5, "ln2": np.abs(rng.standard_normal(H)) + 0.5}
    glue = DeviceBlock(lins, gains, 128)
    ref = DeviceBlock(lins, gains, 128, glue_kernels=False)
    x = B.outlier_x(M, H, mag=1.0).float()
    a, b = glue(x).cpu().numpy(), ref(x).cpu().numpy()
    # the two f32 RMSNorms sum in different orders; a last-ulp difference of an activation moves
    # an MX code at an E2M1 decision point now and then and one bf16 output ulp propagates through
    # five linears (as between the fused and separate blocks above): 1e-2 max / 4e-3 mean
    mx, mean = O.parity_errors(a, b)
    assert mx <= TOL_MAX and mean <= 4e-3, (mx, mean)
