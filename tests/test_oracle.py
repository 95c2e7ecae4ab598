"""Pin the CPU oracle (oracle/serq_oracle.py) before trusting it.

Two anchors: (1) golden vectors produced by running the reference package
itself (tests/golden/make_golden.py), and (2) restatements of the
reference's own known-answer tests for this path (test_quantcore.py,
test_mxfmt.py, test_compensate.py, test_acceptance.py criteria 03/04).
"""

import numpy as np
import pytest

from oracle import serq_oracle as O


# --------------------------------------------------------------- golden vectors


def test_quantizers_match_reference_golden(golden):
    for i in range(int(golden["q_count"])):
        x = golden[f"q_x_{i}"]
        for bits in (2, 4, 8):
            s = O.quantize_symmetric(x, O.IntCfg(bits, True, "per-row"))
            a = O.quantize_asymmetric(x, O.IntCfg(bits, False, "per-row"))
            assert np.array_equal(s.codes, golden[f"q_sym{bits}_codes_{i}"]), (i, bits)
            assert np.array_equal(s.scales, golden[f"q_sym{bits}_scales_{i}"])
            assert np.array_equal(a.codes, golden[f"q_asym{bits}_codes_{i}"]), (i, bits)
            assert np.array_equal(a.scales, golden[f"q_asym{bits}_scales_{i}"])
            assert np.array_equal(a.zero_points, golden[f"q_asym{bits}_zps_{i}"])


def test_e2m1_grid_matches_reference_golden(golden):
    c, v = O.e2m1_nearest(golden["e2m1_grid"])
    assert np.array_equal(c, golden["e2m1_codes"])
    assert np.array_equal(v, golden["e2m1_vals"])


def test_mx_encode_matches_reference_golden(golden):
    for i in range(int(golden["mx_count"])):
        t = O.mx_encode(golden[f"mx_x_{i}"], 32)
        assert np.array_equal(t.element_codes, golden[f"mx_codes_{i}"]), i
        assert np.array_equal(t.block_scale_exponents, golden[f"mx_exps_{i}"]), i


def test_mx_file_bytes_match_reference_golden(golden):
    t = O.mx_encode(golden["mxfile_src"], 32)
    assert np.frombuffer(O.pack_mx_file_bytes(t), np.uint8).tolist() == golden["mxfile_bytes"].tolist()


def test_int_gemm_matches_reference_golden(golden):
    for i in range(6):
        k, gs, bits = golden[f"ig_meta_{i}"].tolist()
        xq = O.quantize_asymmetric(golden[f"ig_x_{i}"], O.IntCfg(bits, False, "per-row"))
        wq = O.quantize_symmetric(golden[f"ig_w_{i}"], O.IntCfg(4, True, gs, "row"))
        out, parts = O.int_gemm(xq, wq, return_partials=True)
        assert np.array_equal(np.stack([p[1] for p in parts]), golden[f"ig_parts_{i}"])
        assert np.array_equal(out, golden[f"ig_out_{i}"])
    xq = O.quantize_symmetric(golden["igpc_x"], O.IntCfg(4, True, "per-row"))
    wq = O.quantize_symmetric(golden["igpc_w"], O.IntCfg(4, True, 128, "row"))
    assert np.array_equal(wq.codes, golden["igpc_wcodes"])
    out, parts = O.int_gemm(xq, wq, return_partials=True)
    assert np.array_equal(parts[0][1], golden["igpc_acc"])
    assert np.array_equal(out, golden["igpc_out"])


def test_mx_gemm_matches_reference_golden(golden):
    x = O.MxT(golden["mg_xc"], golden["mg_xe"], 32, golden["mg_xc"].shape)
    w = O.MxT(golden["mg_wc"], golden["mg_we"], 32, golden["mg_wc"].shape)
    assert np.array_equal(O.mx_gemm(x, w), golden["mg_out"])


def test_mx_forward_matches_reference_golden(golden):
    main_t, comp = O.build_serq_rtn_mx(golden["fmx_w"], golden["fmx_idx"], 32)
    assert np.array_equal(main_t.element_codes, golden["fmx_main_codes"])
    assert np.array_equal(main_t.block_scale_exponents, golden["fmx_main_exps"])
    assert np.array_equal(comp.r_q.element_codes, golden["fmx_r_codes"])
    assert np.array_equal(comp.r_q.block_scale_exponents, golden["fmx_r_exps"])
    y = O.forward_mx(golden["fmx_x"], main_t, comp)
    assert np.array_equal(y, golden["fmx_y"])
    comp_g = O.Comp(64, golden["fmx_gidx"], r_q=comp.r_q)
    assert np.array_equal(O.forward_mx(golden["fmx_x"], main_t, comp_g), golden["fmx_y_gather"])


def test_mx_dense_r_forward_matches_reference_golden(golden):
    # MX main with an unquantized R (compensate.py:338-339): mx_decode(mx_encode(x[:, idx])) @ r_dense
    main_t, _ = O.build_serq_rtn_mx(golden["fmx_w"], golden["fmx_idx"], 32)
    comp = O.Comp(64, golden["fmx_idx"], r_dense=golden["fmx_r_dense"])
    assert np.array_equal(O.forward_mx(golden["fmx_x"], main_t, comp), golden["fmx_y_dense"])


def test_mx_svd_baseline_forward_matches_reference_golden(golden):
    # SVD baseline over an MX main (compensate.py:326-331): y + (mx_decode(x_mx) L1) L2
    main_t, _ = O.build_serq_rtn_mx(golden["fmx_w"], golden["fmx_idx"], 32)
    comp = O.Comp(48, l1=golden["fmxsvd_l1"], l2=golden["fmxsvd_l2"])
    assert np.array_equal(O.forward_mx(golden["fmx_x"], main_t, comp), golden["fmxsvd_y"])
    assert int(golden["fmxsvd_aux"]) == 2


def test_int_forward_matches_reference_golden(golden):
    xi, wi = golden["fint_x"], golden["fint_w"]
    main, comp = O.build_per_channel_int(wi, np.arange(32), r_mode="int")
    for bits in (4, 8):
        y, xq = O.forward_int(xi, main, comp, O.IntCfg(bits, False, "per-row"))
        assert np.array_equal(y, golden[f"fint_y_a{bits}"])
        _, mp = O.int_gemm(xq, main, return_partials=True)
        assert np.array_equal(mp[0][1], golden[f"fint_acc_a{bits}"])
    main_d, comp_d = O.build_per_channel_int(wi, np.arange(32), r_mode="dense")
    y, _ = O.forward_int(xi, main_d, comp_d, O.IntCfg(8, False, "per-row"))
    np.testing.assert_array_equal(y, golden["fint_y_dense_a8"])


def test_grouped_int_builder_and_forward_match_reference_golden(golden):
    # build_serq_rtn with row groups of 128 and the GPTQ-swapped forward
    xg, wg = golden["fgrp_x"], golden["fgrp_w"]
    k, n = wg.shape
    for tag in ("col", "int"):
        main, comp = O.build_grouped_int(wg, np.arange(128), 128, 4, tag)
        assert np.array_equal(main.codes, golden[f"fgrp_{tag}_codes"])
        assert np.array_equal(main.scales, golden[f"fgrp_{tag}_scales"])
        assert np.array_equal(comp.r_q.codes, golden[f"fgrp_{tag}_r_codes"])
        assert np.array_equal(comp.r_q.scales, golden[f"fgrp_{tag}_r_scales"])
        y, xq = O.forward_int(xg, main, comp, O.IntCfg(8, False, "per-row"))
        np.testing.assert_allclose(y, golden[f"fgrp_{tag}_y_a8"], rtol=1e-12, atol=1e-12)
        _, parts = O.int_gemm(xq, main, return_partials=True)
        assert np.array_equal(np.stack([a for _, a in parts]), golden[f"fgrp_{tag}_acc_a8"])
    main = O.IntQ(golden["fgptq_codes"], golden["fgptq_scales"], None, O.IntCfg(4, True, 128, "row"), (k, n))
    rq = O.IntQ(golden["fgptq_r_codes"], golden["fgptq_r_scales"], None, O.default_r_config(n, 4, 128), (128, n))
    comp = O.Comp(128, np.arange(128), r_q=rq)
    for bits in (4, 8):
        y, _ = O.forward_int(xg, main, comp, O.IntCfg(bits, False, "per-row"))
        np.testing.assert_allclose(y, golden[f"fgptq_y_a{bits}"], rtol=1e-12, atol=1e-12)


def test_svd_baseline_forward_matches_reference_golden(golden):
    # build_svd_baseline main is per-output-channel INT4 (compensate.py:209-224); the
    # forward adds (dequantize(xq) @ L1) @ L2 (compensate.py:304-310), two aux products
    xi = golden["fint_x"]
    k, n = golden["fsvd_codes"].shape
    main = O.IntQ(golden["fsvd_codes"], golden["fsvd_scales"], None, O.IntCfg(4, True, k, "row"), (k, n))
    comp = O.Comp(8, l1=golden["fsvd_l1"], l2=golden["fsvd_l2"])
    y, _ = O.forward_int(xi, main, comp, O.IntCfg(8, False, "per-row"))
    np.testing.assert_array_equal(y, golden["fsvd_y_a8"])
    assert int(golden["fsvd_aux"]) == 2


# ------------------------------------------- the reference's known-answer tests


def test_symmetric_hand_cases():
    # test_quantcore.py:21-32
    q = O.quantize_symmetric(np.array([[7.0, -7.0, 3.5]]), O.IntCfg(4))
    assert q.scales[0, 0] == 1.0 and q.codes.tolist() == [[7, -7, 4]]
    q = O.quantize_symmetric(np.zeros((1, 4)), O.IntCfg(4))
    assert q.scales[0, 0] == 1.0 and not q.codes.any()


def test_asymmetric_hand_cases():
    # test_quantcore.py:51-65
    q = O.quantize_asymmetric(np.array([[0.0, 15.0]]), O.IntCfg(4, False))
    assert q.scales[0, 0] == 1.0 and q.zero_points[0, 0] == 0 and q.codes.tolist() == [[0, 15]]
    q = O.quantize_asymmetric(np.full((1, 5), -3.0), O.IntCfg(4, False))
    assert np.array_equal(O.dequantize(q), np.full((1, 5), -3.0))


def _nearest_exhaustive(v):
    """test_mxfmt.py:26-41 restated: all 16 codes, ties -> even mantissa -> +0."""
    best = None
    for code in range(16):
        mag = O.E2M1_MAG[code & 7]
        val = -mag if code & 8 else mag
        key = (abs(v - val), code & 1, code)
        if best is None or key < best[0]:
            best = (key, code, val)
    code, val = best[1], best[2]
    return (0 if val == 0.0 else code), val


def test_e2m1_exhaustive_grid():
    # test_mxfmt.py:72-78 (20,001 points) + tie table :57-64
    grid = np.linspace(-8, 8, 20001)
    c, v = O.e2m1_nearest(grid)
    for g_, cc, vv in zip(grid, c, v):
        oc, ov = _nearest_exhaustive(float(g_))
        assert (cc, vv) == (oc, ov), g_
    for v_, e in [(0.25, 0.0), (0.75, 1.0), (1.25, 1.0), (1.75, 2.0), (2.5, 2.0), (3.5, 4.0), (5.0, 4.0)]:
        assert O.e2m1_nearest(v_)[1] == e and O.e2m1_nearest(-v_)[1] == -e


def test_mx_nibble_layout():
    # test_mxfmt.py:266-280
    x = np.zeros((1, 32))
    x[0, 0], x[0, 1] = 1.0, -1.0
    t = O.mx_encode(x, 32)
    assert t.block_scale_exponents[0, 0] == -2
    raw = O.pack_mx_file_bytes(t)
    assert raw[28] == 125 and raw[29] & 0xF == 6 and raw[29] >> 4 == 14


def test_int_partials_bigint():
    # test_acceptance.py:124-155 (criterion 03) with the oracle, 20 seeds
    for seed in range(20):
        rng = np.random.default_rng(seed)
        k = int(rng.choice([64, 128, 256]))
        gs = int(rng.choice([g for g in (16, 32, 64) if k % g == 0]))
        x = rng.standard_normal((4, k)) * 3
        w = rng.standard_normal((k, 12))
        xq = O.quantize_asymmetric(x, O.IntCfg(int(rng.choice([4, 8])), False))
        wq = O.quantize_symmetric(w, O.IntCfg(4, True, gs, "row"))
        xc = xq.codes.astype(object) - np.repeat(xq.zero_points.astype(object), k, axis=1)
        _, parts = O.int_gemm(xq, wq, return_partials=True)
        for (a, b), acc in parts:
            assert np.array_equal(xc[:, a:b] @ wq.codes.astype(object)[a:b, :], acc.astype(object))


def test_bf16_round_matches_torch():
    torch = pytest.importorskip("torch")
    x = np.random.default_rng(0).standard_normal(100000) * np.exp(np.random.default_rng(1).uniform(-20, 20, 100000))
    # torch rounds f32 -> bf16; feed f32-exact values so both are a single rounding
    x32 = x.astype(np.float32).astype(np.float64)
    t = torch.from_numpy(x32.astype(np.float32)).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(O.bf16_round(x32), t)


def test_rmsnorm_matches_reference_golden(golden):
    # saliency.py:194-196, the producer of q/k/v and gate/up inputs (fused into the quantizer on the GPU)
    y = O.rmsnorm(golden["rms_x"], golden["rms_gain"])
    assert np.array_equal(y, golden["rms_y"])
    assert np.array_equal(O.mx_encode(y, 32).element_codes, golden["rms_codes"])
