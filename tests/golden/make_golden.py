"""Generate golden vectors from the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the reference read-only, evaluates the hot-path functions on
seeded inputs and writes ``tests/golden/golden.npz``.  The reference does
not exist on the GPU box, so these committed fixtures are how the oracle
(``oracle/serq_oracle.py``) is pinned there and here.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from serq.compensate import (  # noqa: E402
    Compensator,
    OpProbe,
    build_serq_gptq_swapped,
    build_serq_rtn,
    default_r_config,
    build_svd_baseline,
    build_serq_rtn_mx,
    forward_reconstructed,
)
from serq.mxfmt import (  # noqa: E402
    e2m1_nearest,
    mx_decode,
    int_gemm_reference,
    mx_encode,
    mx_gemm_reference,
    save_mx,
)
from serq.quantcore import (  # noqa: E402
    IntQuantConfig,
    dequantize,
    gather_columns,
    per_token_config,
    quantize_asymmetric,
    quantize_symmetric,
)
from serq.saliency import build_plan, score_rows  # noqa: E402
from serq.pipeline import layer_forward, quantize_layer  # noqa: E402
from serq.gptq import GptqConfig, HessianState, accumulate_hessian  # noqa: E402
from serq.tensorio import SyntheticSpec, gen_synthetic_activations  # noqa: E402
from serq.flatten import compute_smoothing_scales  # noqa: E402
from serq.tensorio import collect_calib_stats  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def bf16(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def main():
    g = {}
    # -- quantizers: hand cases and random rows across bit widths ------------
    rng = np.random.default_rng(100)
    qx = [np.array([[7.0, -7.0, 3.5]]), np.zeros((1, 4)), np.array([[0.0, 15.0]]),
          np.full((1, 5), 3.0), np.full((1, 5), -3.0)]
    for i in range(8):
        qx.append(rng.standard_normal((6, 64)) * 10.0 ** float(rng.integers(-3, 4)))
    # bf16-valued outlier rows like the benchmark activations
    spec = SyntheticSpec(rows=64, cols=256, n_outlier_channels=3, outlier_magnitude=50, seed=7)
    qx.append(bf16(gen_synthetic_activations(spec)))
    for i, x in enumerate(qx):
        g[f"q_x_{i}"] = x
        for bits in (2, 4, 8):
            s = quantize_symmetric(x, IntQuantConfig(bits, True, "per-row"))
            a = quantize_asymmetric(x, per_token_config(bits))
            g[f"q_sym{bits}_codes_{i}"] = s.codes
            g[f"q_sym{bits}_scales_{i}"] = s.scales
            g[f"q_asym{bits}_codes_{i}"] = a.codes
            g[f"q_asym{bits}_scales_{i}"] = a.scales
            g[f"q_asym{bits}_zps_{i}"] = a.zero_points
    g["q_count"] = np.array(len(qx))

    # -- E2M1 grid (acceptance 04 grid) --------------------------------------
    grid = np.linspace(-8.0, 8.0, 100_001)
    c, v = e2m1_nearest(grid)
    g["e2m1_grid"] = grid
    g["e2m1_codes"] = c
    g["e2m1_vals"] = v

    # -- MX encode: random, zero blocks, tiny/huge magnitudes -----------------
    mx_inputs = [rng.standard_normal((8, 128)) * 5, np.zeros((2, 64)),
                 rng.standard_normal((4, 96)) * 1e-30, rng.standard_normal((4, 64)) * 1e30,
                 bf16(gen_synthetic_activations(spec))]
    tiny = np.zeros((1, 64))
    tiny[0, :32] = np.ldexp(1.0, -140) * np.arange(1, 33)  # block amax < 2^-126
    mx_inputs.append(tiny)
    for i, x in enumerate(mx_inputs):
        t = mx_encode(x, 32)
        g[f"mx_x_{i}"] = x
        g[f"mx_codes_{i}"] = t.element_codes
        g[f"mx_exps_{i}"] = t.block_scale_exponents
    g["mx_count"] = np.array(len(mx_inputs))

    # on-disk MX bytes (mxfmt.py:228-251)
    import tempfile

    t = mx_encode(mx_inputs[0][:4, :64], 32)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "t.mx")
        save_mx(p, t)
        g["mxfile_bytes"] = np.frombuffer(open(p, "rb").read(), dtype=np.uint8)
    g["mxfile_src"] = mx_inputs[0][:4, :64]

    # -- int GEMM partials (criterion-03 style) --------------------------------
    for i in range(6):
        r2 = np.random.default_rng(200 + i)
        k = int(r2.choice([64, 128, 256]))
        gs = int(r2.choice([16, 32, 64]))
        x = r2.standard_normal((5, k)) * 3
        w = r2.standard_normal((k, 24))
        bits = int(r2.choice([4, 8]))
        xq = quantize_asymmetric(x, per_token_config(bits))
        wq = quantize_symmetric(w, IntQuantConfig(4, True, gs, "row"))
        out, parts = int_gemm_reference(xq, wq, return_partials=True)
        g[f"ig_x_{i}"] = x
        g[f"ig_w_{i}"] = w
        g[f"ig_meta_{i}"] = np.array([k, gs, bits])
        g[f"ig_out_{i}"] = out
        g[f"ig_parts_{i}"] = np.stack([p[1] for p in parts])
    # per-output-channel weights (group_size=K): one integer group
    x = rng.standard_normal((7, 128))
    w = rng.standard_normal((128, 40)) * 0.02
    xq = quantize_symmetric(x, IntQuantConfig(4, True, "per-row"))
    wq = quantize_symmetric(w, IntQuantConfig(4, True, 128, "row"))
    out, parts = int_gemm_reference(xq, wq, return_partials=True)
    g["igpc_x"], g["igpc_w"], g["igpc_out"], g["igpc_acc"] = x, w, out, parts[0][1]
    g["igpc_wcodes"], g["igpc_wscales"] = wq.codes, wq.scales

    # -- MX GEMM ---------------------------------------------------------------
    xa = mx_encode(rng.standard_normal((6, 128)) * 4, 32)
    wa = mx_encode(rng.standard_normal((9, 128)), 32)
    g["mg_xc"], g["mg_xe"] = xa.element_codes, xa.block_scale_exponents
    g["mg_wc"], g["mg_we"] = wa.element_codes, wa.block_scale_exponents
    g["mg_out"] = mx_gemm_reference(xa, wa)

    # -- full decomposed forward, MX (reference builder + forward) -------------
    spec2 = SyntheticSpec(rows=128 + 64, cols=512, n_outlier_channels=5, outlier_magnitude=50, seed=0)
    pool = gen_synthetic_activations(spec2)
    calib, x = pool[:128], pool[128:]
    w = np.random.default_rng(1).standard_normal((512, 384)) * 0.02
    s = compute_smoothing_scales(collect_calib_stats(calib), w, 0.5).s
    wt, xt = s[:, None] * w, x / s
    plan = build_plan(score_rows(wt), 64)
    wp, xp = wt[plan.permutation], bf16(xt[:, plan.permutation])
    plan_p = build_plan(score_rows(wp), 64)
    main_t, comp = build_serq_rtn_mx(wp, plan_p, 32)
    g["fmx_x"], g["fmx_w"] = xp, wp
    g["fmx_idx"] = plan_p.salient_idx
    g["fmx_main_codes"], g["fmx_main_exps"] = main_t.element_codes, main_t.block_scale_exponents
    g["fmx_r_codes"], g["fmx_r_exps"] = comp.r_q.element_codes, comp.r_q.block_scale_exponents
    g["fmx_y"] = forward_reconstructed(xp, main_t, comp, None)
    # gather fallback: same artefacts, arbitrary salient index set
    idx = np.random.default_rng(3).permutation(512)[:64]
    comp_g = Compensator("rtn_residual", 64, idx, r_q=comp.r_q)
    g["fmx_gidx"] = idx
    g["fmx_y_gather"] = forward_reconstructed(xp, main_t, comp_g, None)
    # MX main with a dense (unquantized, "test mode") R: y + mx_decode(mx_encode(x[:, idx])) @ r_dense
    # (compensate.py:338-339)
    err = wp - mx_decode(main_t).T
    comp_dr = Compensator("rtn_residual", 64, plan_p.salient_idx.copy(), r_dense=err[plan_p.salient_idx])
    g["fmx_y_dense"] = forward_reconstructed(xp, main_t, comp_dr, None)
    g["fmx_r_dense"] = comp_dr.r_dense
    # SVD baseline over an MX main (compensate.py:326-331): (mx_decode(x_mx) L1) L2, two aux products
    u, sv, vt = np.linalg.svd(err, full_matrices=False)
    root = np.sqrt(sv[:48])
    comp_svd = Compensator("svd_baseline", 48, l1=u[:, :48] * root[None, :], l2=root[:, None] * vt[:48])
    probe = OpProbe()
    g["fmxsvd_y"] = forward_reconstructed(xp, main_t, comp_svd, None, probe)
    g["fmxsvd_aux"] = np.array(probe.aux_matmuls)
    g["fmxsvd_l1"], g["fmxsvd_l2"] = comp_svd.l1, comp_svd.l2

    # -- full decomposed forward, INT (asym A8, per-output-channel W, int R) ---
    k, n, r = 256, 96, 32
    xi = bf16(np.random.default_rng(11).standard_normal((9, k)) * 2)
    wi = np.random.default_rng(12).standard_normal((k, n)) * 0.02
    main = quantize_symmetric(wi, IntQuantConfig(4, True, k, "row"))
    resid = wi[:r] - dequantize(main)[:r]
    rq = quantize_symmetric(resid, IntQuantConfig(4, True, r, "row"))
    comp_i = Compensator("rtn_residual", r, np.arange(r), r_q=rq)
    for bits in (4, 8):
        yv = forward_reconstructed(xi, main, comp_i, per_token_config(bits))
        xq = quantize_asymmetric(xi, per_token_config(bits))
        _, mp = int_gemm_reference(xq, main, return_partials=True)
        _, rp = int_gemm_reference(gather_columns(xq, np.arange(r)), rq, return_partials=True)
        g[f"fint_y_a{bits}"] = yv
        g[f"fint_acc_a{bits}"] = mp[0][1]
        g[f"fint_accr_a{bits}"] = rp[0][1]
    g["fint_x"], g["fint_w"] = xi, wi
    # dense-R variant (r_dense, "L in bf16")
    comp_d = Compensator("rtn_residual", r, np.arange(r), r_dense=bf16(resid))
    g["fint_y_dense_a8"] = forward_reconstructed(xi, main, comp_d, per_token_config(8))
    # the per-row default builder path (float branch) for the drop-in rejection test
    plan_i = build_plan(score_rows(wi), r)
    m2, c2 = build_serq_rtn(wi, plan_i, IntQuantConfig(4, True, 16, "row"),
                            IntQuantConfig(4, True, r, "row"))
    g["fint_g16_y"] = forward_reconstructed(xi, m2, c2, per_token_config(8))
    g["fint_g16_idx"] = plan_i.salient_idx

    # -- SVD baseline (two-factor L1 L2 over the full quantization error, compensate.py:209-224, 304-310)
    main_s, comp_s = build_svd_baseline(wi, IntQuantConfig(4, True, k, "row"), 8)
    probe = OpProbe()
    g["fsvd_y_a8"] = forward_reconstructed(xi, main_s, comp_s, per_token_config(8), probe)
    g["fsvd_aux"] = np.array(probe.aux_matmuls)
    g["fsvd_l1"], g["fsvd_l2"] = comp_s.l1, comp_s.l2
    g["fsvd_codes"], g["fsvd_scales"] = main_s.codes, main_s.scales

    # -- group-wise INT weights (the paper's g = r = 128): reference builders
    #    build_serq_rtn with row groups of 128 and build_serq_gptq_swapped (GPTQ group 128), R from
    #    default_r_config (column groups: the float branch) or row groups of r (integer)
    kg, ng, rg = 256, 96, 128
    xg = bf16(np.random.default_rng(31).standard_normal((9, kg)) * 2)
    wg = np.random.default_rng(32).standard_normal((kg, ng)) * 0.02
    plan_g = build_plan(np.arange(kg, 0, -1.0), rg)  # salient rows = arange(r) (permuted layout)
    wcfg_g = IntQuantConfig(4, True, 128, "row")
    for tag, rcfg in (("col", default_r_config(ng, 4, 128)), ("int", IntQuantConfig(4, True, rg, "row"))):
        mg, cg = build_serq_rtn(wg, plan_g, wcfg_g, rcfg)
        g[f"fgrp_{tag}_codes"], g[f"fgrp_{tag}_scales"] = mg.codes, mg.scales
        g[f"fgrp_{tag}_r_codes"], g[f"fgrp_{tag}_r_scales"] = cg.r_q.codes, cg.r_q.scales
        probe = OpProbe()
        g[f"fgrp_{tag}_y_a8"] = forward_reconstructed(xg, mg, cg, per_token_config(8), probe)
        g[f"fgrp_{tag}_aux"] = np.array(probe.aux_matmuls)
        _, parts = int_gemm_reference(quantize_asymmetric(xg, per_token_config(8)), mg, return_partials=True)
        g[f"fgrp_{tag}_acc_a8"] = np.stack([acc for _, acc in parts])
    calib_g = np.random.default_rng(33).standard_normal((64, kg))
    hess = accumulate_hessian(HessianState.zeros(kg), calib_g)
    mq, cq = build_serq_gptq_swapped(wg, plan_g, GptqConfig(4, 128), default_r_config(ng, 4, 128), hess)
    g["fgptq_codes"], g["fgptq_scales"] = mq.codes, mq.scales
    g["fgptq_r_codes"], g["fgptq_r_scales"] = cq.r_q.codes, cq.r_q.scales
    for bits in (4, 8):
        g[f"fgptq_y_a{bits}"] = forward_reconstructed(xg, mq, cq, per_token_config(bits))
    g["fgrp_x"], g["fgrp_w"] = xg, wg

    # -- pipeline.quantize_layer / layer_forward (SAF smoothing + salient plan built by the
    #    reference; the layer's salient set is NOT the permuted front: the gather fallback)
    calib_l = gen_synthetic_activations(SyntheticSpec(rows=64 + 12, cols=256, n_outlier_channels=3,
                                                      outlier_magnitude=50.0, seed=5))
    w_l = np.random.default_rng(6).standard_normal((256, 128)) * 0.02
    x_l = bf16(calib_l[64:])
    for fmt, rank in (("mxfp4", 64), ("int", 128)):
        art = quantize_layer(w_l, calib_l[:64], rank=rank, fmt=fmt, weight_group=128 if fmt == "int" else "per-row")
        tag = f"flayer_{fmt}"
        g[f"{tag}_s"] = art.smoothing.s
        g[f"{tag}_idx"] = art.comp.salient_idx
        if fmt == "mxfp4":
            g[f"{tag}_codes"], g[f"{tag}_exps"] = art.main.element_codes, art.main.block_scale_exponents
            g[f"{tag}_r_codes"], g[f"{tag}_r_exps"] = art.comp.r_q.element_codes, art.comp.r_q.block_scale_exponents
        else:
            g[f"{tag}_codes"], g[f"{tag}_scales"] = art.main.codes, art.main.scales
            g[f"{tag}_r_codes"], g[f"{tag}_r_scales"] = art.comp.r_q.codes, art.comp.r_q.scales
        g[f"{tag}_y"] = layer_forward(art, x_l)
    g["flayer_x"] = x_l

    # -- a small bundle written by the reference's own save_bundle (bundleio.py:73-126), for the
    #    device bundle loader: MX main + MX R, INT main + INT R, INT main + SVD factors
    from serq.bundleio import save_bundle
    from serq.toymodel import LinearBundle, QuantizedBlockBundle

    bdir = os.path.join(os.path.dirname(OUT), "bundle")
    wb = np.random.default_rng(21).standard_normal((256, 128)) * 0.02
    mx_main, mx_comp = build_serq_rtn_mx(wb, build_plan(score_rows(wb), 32), 32)
    int_main = quantize_symmetric(wb, IntQuantConfig(4, True, 256, "row"))
    rb = wb[:32] - dequantize(int_main)[:32]
    int_comp = Compensator("rtn_residual", 32, np.arange(32), r_q=quantize_symmetric(rb, IntQuantConfig(4, True, 32, "row")))
    svd_main, svd_comp = build_svd_baseline(wb, IntQuantConfig(4, True, 256, "row"), 4)
    linears = {"up_proj": LinearBundle(mx_main, mx_comp, None),
               "down_proj": LinearBundle(int_main, int_comp, per_token_config(8)),
               "o_proj": LinearBundle(svd_main, svd_comp, per_token_config(8))}
    gains = {"ln1": np.abs(np.random.default_rng(22).standard_normal(256)) + 0.5}
    save_bundle(bdir, QuantizedBlockBundle(linears=linears, nl_weights=gains, plans={}, rank=32, fmt="mixed"))
    xb = bf16(np.random.default_rng(23).standard_normal((40, 256)))
    g["bundle_x"] = xb
    for name, lb in linears.items():
        g[f"bundle_y_{name}"] = forward_reconstructed(xb, lb.main, lb.comp, lb.act_cfg)
    g["bundle_up_codes"], g["bundle_up_exps"] = mx_main.element_codes, mx_main.block_scale_exponents
    g["bundle_up_rcodes"], g["bundle_up_rexps"] = mx_comp.r_q.element_codes, mx_comp.r_q.block_scale_exponents

    # -- producer RMSNorm (saliency.py:194-196) feeding the fused quantizer
    from serq.saliency import rmsnorm

    xr = bf16(np.random.default_rng(31).standard_normal((16, 512)) * 3)
    gr = np.abs(np.random.default_rng(32).standard_normal(512)) + 0.5
    g["rms_x"], g["rms_gain"], g["rms_y"] = xr, gr, rmsnorm(xr, gr)
    g["rms_codes"] = mx_encode(g["rms_y"], 32).element_codes

    # -- a whole toy decoder block (toymodel.py:88-124), MXFP4 SERQ via the reference's own
    #    quantize_block + save_bundle; forward_quantized (graph_forward + forward_reconstructed)
    #    is the golden block output for the device block forward
    from serq.toymodel import forward_fp, forward_quantized, quantize_block, random_block

    blk = random_block(256, 512, head_dim=64, seed=51)
    calib = gen_synthetic_activations(SyntheticSpec(rows=64, cols=256, n_outlier_channels=3,
                                                    outlier_magnitude=20, seed=52))
    qb = quantize_block(blk, calib, rank=32, fmt="mxfp4")
    save_bundle(os.path.join(os.path.dirname(OUT), "block_mx"), qb)
    xbk = bf16(gen_synthetic_activations(SyntheticSpec(rows=48, cols=256, n_outlier_channels=3,
                                                       outlier_magnitude=20, seed=53)))
    g["block_x"] = xbk
    g["block_y_quant"] = forward_quantized(blk, xbk, qb)
    g["block_y_fp"] = forward_fp(blk, xbk)
    g["block_head_dim"] = np.array(64)

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT)/1e6:.2f} MB, {len(g)} arrays)")


if __name__ == "__main__":
    main()
