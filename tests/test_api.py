"""The reference-facing mirror (paper_2603_08185_b200.api): same names,
dataclasses, argument meaning and error behaviour as serq.compensate /
serq.quantcore / serq.mxfmt for the hot path."""

import types

import numpy as np
import pytest

from oracle import serq_oracle as O
from paper_2603_08185_b200 import api
from paper_2603_08185_b200.errors import ValidationError

torch = pytest.importorskip("torch")

TOL_MAX, TOL_MEAN = 1e-2, 1e-3


# ---------------------------------------------------------------- CPU: preconditions fail loudly, before the GPU


def test_validation_error_is_value_error():
    assert issubclass(ValidationError, ValueError)


def test_config_validation_mirrors_reference():
    # quantcore.py:35-43
    with pytest.raises(ValidationError):
        api.IntQuantConfig(bits=9)
    with pytest.raises(ValidationError):
        api.IntQuantConfig(axis="diag")
    with pytest.raises(ValidationError):
        api.IntQuantConfig(group_size=0)
    assert api.per_token_config(8) == api.IntQuantConfig(8, False, "per-row")


def test_forward_requires_asymmetric_act_cfg():
    # compensate.py:298-299
    main = api.QuantizedTensor(np.zeros((8, 4), np.int32), np.ones((1, 4)), None,
                               api.IntQuantConfig(4, True, 8, "row"), (8, 4))
    with pytest.raises(ValidationError, match="asymmetric"):
        api.forward_reconstructed(np.ones((2, 8)), main, None, api.IntQuantConfig(4, True))
    with pytest.raises(ValidationError, match="main rows"):
        api.forward_reconstructed(np.ones((2, 7)), main, None, api.per_token_config(8))


def test_layouts_integer_cores_cannot_evaluate_are_rejected():
    # per-row (per input channel) main scales vary along K
    main = api.QuantizedTensor(np.zeros((8, 4), np.int32), np.ones((8, 1)), None,
                               api.IntQuantConfig(4, True, "per-row"), (8, 4))
    with pytest.raises(ValidationError, match="GPU-native"):
        api.SerqLinear(main, None, api.per_token_config(8))
    # row groups that are not a multiple of 128 (or above 1024) are rejected too
    main_g = api.QuantizedTensor(np.zeros((256, 8), np.int32), np.ones((4, 8)), None,
                                 api.IntQuantConfig(4, True, 64, "row"), (256, 8))
    with pytest.raises(ValidationError, match="GPU-native"):
        api.SerqLinear(main_g, None, api.per_token_config(8))
    with pytest.raises(ValidationError):
        api.forward_reconstructed(np.ones((2, 8)), main, None, api.per_token_config(8))


def test_svd_compensator_validation():
    with pytest.raises(ValidationError, match="two factors"):
        api.Compensator(api.SVD_BASELINE, 2, l1=np.ones((8, 2)))
    with pytest.raises(ValidationError, match="residual"):
        api.Compensator(api.SVD_BASELINE, 2, l1=np.ones((8, 2)), l2=np.ones((2, 4)), r_dense=np.ones((2, 4)))
    comp = api.Compensator(api.SVD_BASELINE, 2, l1=np.ones((8, 2)), l2=np.ones((2, 4)))
    main = api.MxBlockTensor(np.zeros((4, 32), np.uint8), np.zeros((4, 1), np.int32), 32, (4, 32))
    with pytest.raises(ValidationError, match="SVD"):
        api.SerqLinear(main, comp)


def test_nonfinite_input_rejected():
    main = api.MxBlockTensor(np.zeros((4, 32), np.uint8), np.zeros((4, 1), np.int32), 32, (4, 32))
    with pytest.raises(ValidationError, match="non-finite"):
        api.forward_reconstructed(np.full((2, 32), np.nan), main, None, None)


def test_single_matrix_compensator_invariant():
    with pytest.raises(ValidationError, match="exactly one R"):
        api.Compensator(api.RTN_RESIDUAL, 4, np.arange(4))


# ---------------------------------------------------------------- GPU: drop-in parity


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    api.clear_cache()
    return True


def _mx_artifacts(golden, idx_key="fmx_idx"):
    main = api.MxBlockTensor(golden["fmx_main_codes"], golden["fmx_main_exps"], 32, golden["fmx_main_codes"].shape)
    rq = api.MxBlockTensor(golden["fmx_r_codes"], golden["fmx_r_exps"], 32, golden["fmx_r_codes"].shape)
    comp = api.Compensator(api.RTN_RESIDUAL, 64, np.asarray(golden[idx_key]), r_q=rq)
    return main, comp


@pytest.mark.gpu
def test_forward_reconstructed_mx_golden(gpu, golden):
    main, comp = _mx_artifacts(golden)
    probe = api.OpProbe()
    y = api.forward_reconstructed(golden["fmx_x"], main, comp, None, probe)
    assert probe.aux_matmuls == 1  # one auxiliary product (compensate.py:336-337)
    mx, mean = O.parity_errors(y, golden["fmx_y"])
    assert y.dtype == np.float64 and mx <= TOL_MAX and mean <= TOL_MEAN
    # gather fallback
    main_g, comp_g = _mx_artifacts(golden, "fmx_gidx")
    y = api.forward_reconstructed(golden["fmx_x"], main_g, comp_g, None)
    mx, mean = O.parity_errors(y, golden["fmx_y_gather"])
    assert mx <= TOL_MAX and mean <= TOL_MEAN


@pytest.mark.gpu
def test_forward_reconstructed_mx_dense_r_golden(gpu, golden):
    # MX main + unquantized R ("test mode", compensate.py:338-339), reference-built golden
    main = api.MxBlockTensor(golden["fmx_main_codes"], golden["fmx_main_exps"], 32, golden["fmx_main_codes"].shape)
    comp = api.Compensator(api.RTN_RESIDUAL, 64, np.asarray(golden["fmx_idx"]), r_dense=golden["fmx_r_dense"])
    probe = api.OpProbe()
    y = api.forward_reconstructed(golden["fmx_x"], main, comp, None, probe)
    assert probe.aux_matmuls == 1
    mx, mean = O.parity_errors(y, golden["fmx_y_dense"])
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


@pytest.mark.gpu
def test_forward_reconstructed_mx_svd_baseline_golden(gpu, golden):
    # SVD baseline over an MX main (compensate.py:326-331), reference-built golden: two aux
    # products and no probe note (unlike the integer branch)
    main = api.MxBlockTensor(golden["fmx_main_codes"], golden["fmx_main_exps"], 32, golden["fmx_main_codes"].shape)
    comp = api.Compensator(api.SVD_BASELINE, 48, l1=golden["fmxsvd_l1"], l2=golden["fmxsvd_l2"])
    probe = api.OpProbe()
    y = api.forward_reconstructed(golden["fmx_x"], main, comp, None, probe)
    assert probe.aux_matmuls == int(golden["fmxsvd_aux"]) == 2 and probe.notes == []
    mx, mean = O.parity_errors(y, golden["fmxsvd_y"])
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


@pytest.mark.gpu
def test_forward_reconstructed_int_golden(gpu, golden):
    x, w = golden["fint_x"], golden["fint_w"]
    main, comp = api.build_per_channel_int(w, np.arange(32), r_mode="int")
    for bits in (4, 8):
        y = api.forward_reconstructed(x, main, comp, api.per_token_config(bits))
        mx, mean = O.parity_errors(y, golden[f"fint_y_a{bits}"])
        assert mx <= TOL_MAX and mean <= TOL_MEAN, (bits, mx, mean)
    main_d, comp_d = api.build_per_channel_int(w, np.arange(32), r_mode="dense")
    y = api.forward_reconstructed(x, main_d, comp_d, api.per_token_config(8))
    mx, mean = O.parity_errors(y, golden["fint_y_dense_a8"])
    assert mx <= TOL_MAX and mean <= TOL_MEAN


@pytest.mark.gpu
def test_gpu_quantizers_and_builders_match_oracle(gpu, golden):
    x = golden["q_x_13"]
    for bits in (2, 4, 8):
        s = api.quantize_symmetric(x, api.IntQuantConfig(bits, True, "per-row"))
        a = api.quantize_asymmetric(x, api.per_token_config(bits))
        assert np.array_equal(s.codes, golden[f"q_sym{bits}_codes_13"])
        assert np.array_equal(a.codes, golden[f"q_asym{bits}_codes_13"])
        assert np.array_equal(a.zero_points, golden[f"q_asym{bits}_zps_13"])
    # per-output-channel weights: group_size == rows, axis 'row' (one scale per column)
    wq = api.quantize_symmetric(golden["igpc_w"], api.IntQuantConfig(4, True, 128, "row"))
    assert np.array_equal(wq.codes, golden["igpc_wcodes"]) and np.array_equal(wq.scales, golden["igpc_wscales"])
    # mx_encode (f64 exact) and the MX builder
    for i in range(int(golden["mx_count"])):
        t = api.mx_encode(golden[f"mx_x_{i}"], 32)
        assert np.array_equal(t.element_codes, golden[f"mx_codes_{i}"])
        assert np.array_equal(t.block_scale_exponents, golden[f"mx_exps_{i}"])
    main_t, comp = api.build_serq_rtn_mx(golden["fmx_w"], golden["fmx_idx"])
    assert np.array_equal(main_t.element_codes, golden["fmx_main_codes"])
    assert np.array_equal(comp.r_q.element_codes, golden["fmx_r_codes"])
    assert np.array_equal(comp.r_q.block_scale_exponents, golden["fmx_r_exps"])


@pytest.mark.gpu
def test_passthrough_mode(gpu):
    # quantization-disabled mode (compensate.py:288-293)
    rng = np.random.default_rng(0)
    x, w = rng.standard_normal((5, 16)), rng.standard_normal((16, 8))
    np.testing.assert_allclose(api.forward_reconstructed(x, w, None, None), x @ w, rtol=1e-12)


@pytest.mark.gpu
def test_serq_linear_module_and_linear_fn(gpu, golden):
    main, comp = _mx_artifacts(golden)
    lin = api.SerqLinear(main, comp)
    xt = torch.from_numpy(golden["fmx_x"]).to("cuda", torch.bfloat16)
    y = lin(xt)
    assert y.dtype == torch.bfloat16 and y.shape == (golden["fmx_x"].shape[0], main.shape[0])
    mx, mean = O.parity_errors(y.float().cpu().numpy(), golden["fmx_y"])
    assert mx <= TOL_MAX and mean <= TOL_MEAN
    # graph_forward(linear_fn=...) hook with a bundle-shaped object
    bundle = types.SimpleNamespace(linears={"down_proj": types.SimpleNamespace(main=main, comp=comp, act_cfg=None)})
    fn = api.make_linear_fn(bundle)
    mx, mean = O.parity_errors(fn("down_proj", golden["fmx_x"]), golden["fmx_y"])
    assert mx <= TOL_MAX and mean <= TOL_MEAN


@pytest.mark.gpu
def test_symmetric_activation_composition_c1_style(gpu):
    # BASELINE C1 composition: symmetric per-token INT4 activations, bf16 L
    rng = np.random.default_rng(7)
    x = O.bf16_round(O.synthetic_activations(96, 512, 5, 50.0, 7))
    w = rng.standard_normal((512, 256)) * 0.02
    main, comp = api.build_per_channel_int(w, np.arange(64), r_mode="dense")
    y = api.forward_symmetric_act(x, main, comp, api.IntQuantConfig(4, True, "per-row"))
    main_o, comp_o = O.build_per_channel_int(w, np.arange(64), r_mode="dense")
    y_ref, _ = O.forward_int(x, main_o, comp_o, O.IntCfg(4, True, "per-row"), symmetric_act=True)
    mx, mean = O.parity_errors(y, y_ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN


@pytest.mark.gpu
def test_forward_reconstructed_svd_baseline_golden(gpu, golden):
    # build_svd_baseline artefacts (reference-built golden): INT main through the fused kernel,
    # (x_hat @ L1) @ L2 as two fp32 GEMMs added in the epilogue; two aux products (compensate.py:307-309)
    x = golden["fint_x"]
    k, n = golden["fsvd_codes"].shape
    main = api.QuantizedTensor(golden["fsvd_codes"], golden["fsvd_scales"], None,
                               api.IntQuantConfig(4, True, k, "row"), (k, n))
    comp = api.Compensator(api.SVD_BASELINE, 8, l1=golden["fsvd_l1"], l2=golden["fsvd_l2"])
    probe = api.OpProbe()
    y = api.forward_reconstructed(x, main, comp, api.per_token_config(8), probe)
    assert probe.aux_matmuls == int(golden["fsvd_aux"]) == 2
    mx, mean = O.parity_errors(y, golden["fsvd_y_a8"])
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)
    # the large-M CTA-pair kernel takes the same addend
    xb = np.tile(x, (40, 1))[:300]
    yb = api.forward_reconstructed(xb, main, comp, api.per_token_config(8))
    ref, _ = O.forward_int(xb, O.IntQ(main.codes, main.scales, None, O.IntCfg(4, True, k, "row"), (k, n)),
                           O.Comp(8, l1=comp.l1, l2=comp.l2), O.IntCfg(8, False, "per-row"))
    mx, mean = O.parity_errors(yb, ref)
    assert mx <= TOL_MAX and mean <= TOL_MEAN, (mx, mean)


@pytest.mark.gpu
def test_thread_count_invariance(gpu, golden):
    # the reference's harness runs forwards from a thread pool and requires results independent of the
    # thread count (test_harness.py:133-140): the device path is stream-ordered and keeps no per-call
    # state in the shared artefact handle
    from concurrent.futures import ThreadPoolExecutor

    main, comp = _mx_artifacts(golden, "fmx_idx")
    xs = [golden["fmx_x"] * s for s in (1.0, 0.5, 2.0, -1.0, 0.25, 4.0)]
    single = [api.forward_reconstructed(x, main, comp, None) for x in xs]
    with ThreadPoolExecutor(4) as ex:
        multi = list(ex.map(lambda x: api.forward_reconstructed(x, main, comp, None), xs))
    for a, b in zip(single, multi):
        assert np.array_equal(a, b)


@pytest.mark.gpu
def test_serq_beats_rtn_and_rank_monotone(gpu):
    # test_toymodel.py:76-99 at the linear level on the device: the salient compensation lowers the error
    # against the unquantized product, and more salient rows lower it further
    rng = np.random.default_rng(5)
    K, N, M = 512, 256, 64
    x = O.bf16_round(O.synthetic_activations(M, K, 8, 30.0, 6))
    w = rng.standard_normal((K, N)) * 0.02
    w[:64] *= 6.0  # the permuted salient rows (largest quantization error)
    exact = x @ w
    errs = []
    for r in (0, 32, 64):
        main_t, comp = api.build_serq_rtn_mx(w, np.arange(r))
        y = api.forward_reconstructed(x, main_t, comp if r else None, None)
        errs.append(np.linalg.norm(y - exact) / np.linalg.norm(exact))
    assert errs[0] > errs[1] > errs[2], errs


@pytest.mark.gpu
def test_forward_reconstructed_grouped_and_gptq_golden(gpu, golden):
    # group-wise INT weights through the drop-in: RTN with row groups of 128 (default_r_config
    # R and integer R) and the GPTQ-swapped artefacts, all built by the reference
    xg, wg = golden["fgrp_x"], golden["fgrp_w"]
    k, n = wg.shape
    r = 128
    plan = type("Plan", (), {"scores": np.arange(k, 0, -1.0), "rank": r, "salient_idx": np.arange(r)})()
    for tag, rcfg in (("col", api.IntQuantConfig(4, True, 96, "col")), ("int", api.IntQuantConfig(4, True, r, "row"))):
        main, comp = api.build_serq_rtn(wg, plan, api.IntQuantConfig(4, True, 128, "row"), rcfg)
        # the device quantizers reproduce the reference artefacts bit for bit
        assert np.array_equal(main.codes, golden[f"fgrp_{tag}_codes"])
        assert np.array_equal(main.scales, golden[f"fgrp_{tag}_scales"])
        assert np.array_equal(comp.r_q.codes, golden[f"fgrp_{tag}_r_codes"])
        assert np.array_equal(comp.r_q.scales, golden[f"fgrp_{tag}_r_scales"])
        probe = api.OpProbe()
        y = api.forward_reconstructed(xg, main, comp, api.per_token_config(8), probe)
        assert probe.aux_matmuls == int(golden[f"fgrp_{tag}_aux"])
        mx, mean = O.parity_errors(y, golden[f"fgrp_{tag}_y_a8"])
        assert mx <= TOL_MAX and mean <= TOL_MEAN, (tag, mx, mean)
    main = api.QuantizedTensor(golden["fgptq_codes"], golden["fgptq_scales"], None,
                               api.IntQuantConfig(4, True, 128, "row"), (k, n))
    rq = api.QuantizedTensor(golden["fgptq_r_codes"], golden["fgptq_r_scales"], None,
                             api.IntQuantConfig(4, True, 96, "col"), (r, n))
    comp = api.Compensator(api.GPTQ_SWAPPED, r, np.arange(r), r_q=rq)
    for bits in (4, 8):
        y = api.forward_reconstructed(xg, main, comp, api.per_token_config(bits))
        mx, mean = O.parity_errors(y, golden[f"fgptq_y_a{bits}"])
        assert mx <= TOL_MAX and mean <= TOL_MEAN, (bits, mx, mean)


@pytest.mark.gpu
def test_layer_forward_golden(gpu, golden):
    # pipeline.quantize_layer artefacts built by the reference (SAF smoothing, a salient plan that
    # is not the permuted front: the gather fallback) through the layer_forward drop-in
    from types import SimpleNamespace

    x = golden["flayer_x"]
    k = x.shape[1]
    for fmt in ("mxfp4", "int"):
        t = f"flayer_{fmt}"
        idx = golden[f"{t}_idx"]
        r = idx.size
        if fmt == "mxfp4":
            n = golden[f"{t}_codes"].shape[0]
            main = api.MxBlockTensor(golden[f"{t}_codes"], golden[f"{t}_exps"], 32, (n, k))
            rq = api.MxBlockTensor(golden[f"{t}_r_codes"], golden[f"{t}_r_exps"], 32, (n, r))
            act_cfg = None
        else:
            n = golden[f"{t}_codes"].shape[1]
            main = api.QuantizedTensor(golden[f"{t}_codes"], golden[f"{t}_scales"], None,
                                       api.IntQuantConfig(4, True, 128, "row"), (k, n))
            rq = api.QuantizedTensor(golden[f"{t}_r_codes"], golden[f"{t}_r_scales"], None,
                                     api.IntQuantConfig(4, True, n, "col"), (r, n))
            act_cfg = api.per_token_config(8)
        art = SimpleNamespace(main=main, comp=api.Compensator(api.RTN_RESIDUAL, r, idx, r_q=rq), act_cfg=act_cfg,
                              smoothing=SimpleNamespace(s=golden[f"{t}_s"]))
        y = api.layer_forward(art, x)
        mx, mean = O.parity_errors(y, golden[f"{t}_y"])
        assert mx <= TOL_MAX and mean <= TOL_MEAN, (fmt, mx, mean)


def test_predict_validation_mirrors_estimator():
    # estimators.py:86-97: not fitted / wrong feature count raise before any device work
    from types import SimpleNamespace

    with pytest.raises(ValidationError, match="not fitted"):
        api.predict(SimpleNamespace(), np.ones((2, 8)))
    est = SimpleNamespace(artifacts_=None, n_features_in_=8)
    with pytest.raises(ValidationError, match="features"):
        api.predict(est, np.ones((2, 7)))


def test_empty_input_rejected_like_reference():
    # _validation.as_matrix (reference): "x must be non-empty" before any device work
    main = api.MxBlockTensor(np.zeros((32, 64), np.uint8), np.zeros((32, 2), np.int32), 32, (32, 64))
    with pytest.raises(ValidationError, match="non-empty"):
        api.forward_reconstructed(np.zeros((0, 64)), main, None, None)
