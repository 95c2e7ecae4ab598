"""CPU oracle for the SERQ quantized-linear hot path.  TEST INFRASTRUCTURE ONLY.

This module is the *checker*: a NumPy restatement of the reference
algorithm (``/root/reference/pkg/src/serq``) for the functions on the hot
path.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  The product
package (``paper_2603_08185_b200``) never imports it and has no CPU
fallback.

Pinning.  The restatement is pinned against golden vectors produced by the
reference package itself (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src`` read-only and writes ``tests/golden/*.npz``) and
against the reference's own known-answer tests (hand cases, the exhaustive
E2M1 grid, big-integer accumulator oracles), see ``tests/test_oracle.py``.

Third-party arithmetic.  The reference computes with NumPy (pinned only as
``numpy>=1.24``, ``pkg/pyproject.toml:11``); the operations it relies on are
IEEE float64 division, ``np.rint`` (round half to even), ``np.frexp`` and
BLAS dgemm whose integer results are exact below 2**53
(``mxfmt.py:122-132``).  This restatement uses the same primitives.

Every function cites the reference file:line it follows.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# ---------------------------------------------------------------------------
# integer grid (reference quantcore.py)
# ---------------------------------------------------------------------------


class OracleError(ValueError):
    """Mirror of reference ``ValidationError`` (``_validation.py:14-15``)."""


@dataclass(frozen=True)
class IntCfg:
    """``IntQuantConfig`` (quantcore.py:28-51)."""

    bits: int = 4
    symmetric: bool = True
    group_size: object = "per-row"
    axis: str = "row"

    @property
    def qmax(self) -> int:  # quantcore.py:45-47
        return 2 ** (self.bits - 1) - 1

    @property
    def levels(self) -> int:  # quantcore.py:49-51
        return 2**self.bits - 1


@dataclass
class IntQ:
    """``QuantizedTensor`` (quantcore.py:59-80)."""

    codes: np.ndarray
    scales: np.ndarray
    zero_points: np.ndarray | None
    config: IntCfg
    shape: tuple


def _groups(cfg: IntCfg, shape):
    """quantcore.py:83-94 -- 'per-row' means one column group spanning the row."""
    rows, cols = shape
    if cfg.group_size == "per-row":
        return "col", cols
    gs = int(cfg.group_size)
    dim = rows if cfg.axis == "row" else cols
    if dim % gs:
        raise OracleError(f"group_size {gs} does not divide grouped dimension {dim}")
    return cfg.axis, gs


def _reduce(x, axis, gs, fn):
    r, c = x.shape
    if axis == "row":
        return fn(x.reshape(r // gs, gs, c), axis=1)
    return fn(x.reshape(r, c // gs, gs), axis=2)


def _expand(v, axis, gs):
    return np.repeat(v, gs, axis=0 if axis == "row" else 1)


def quantize_symmetric(x, cfg: IntCfg) -> IntQ:
    """quantcore.py:108-118: s = max|x|/qmax (0 -> 1); codes = clip(rint(x/s))."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    axis, gs = _groups(cfg, x.shape)
    s = _reduce(np.abs(x), axis, gs, np.max) / cfg.qmax
    s = np.where(s == 0.0, 1.0, s)
    q = np.clip(np.rint(x / _expand(s, axis, gs)), -cfg.qmax, cfg.qmax)
    return IntQ(q.astype(np.int32), s, None, cfg, x.shape)


def quantize_asymmetric(x, cfg: IntCfg) -> IntQ:
    """quantcore.py:121-137: s=(hi-lo)/(2^n-1) (0 -> 1); zp=rint(-lo/s);
    codes = clip(rint(x/s)+zp, 0, 2^n-1)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    axis, gs = _groups(cfg, x.shape)
    lo = _reduce(x, axis, gs, np.min)
    hi = _reduce(x, axis, gs, np.max)
    s = (hi - lo) / cfg.levels
    s = np.where(s == 0.0, 1.0, s)
    zp = np.rint(-lo / s).astype(np.int64)
    q = np.rint(x / _expand(s, axis, gs)) + _expand(zp, axis, gs)
    q = np.clip(q, 0, cfg.levels)
    return IntQ(q.astype(np.int32), s, zp.astype(np.int32), cfg, x.shape)


def dequantize(q: IntQ) -> np.ndarray:
    """quantcore.py:144-150."""
    axis, gs = _groups(q.config, q.shape)
    s = _expand(q.scales, axis, gs)
    if q.zero_points is None:
        return s * q.codes
    return s * (q.codes.astype(np.float64) - _expand(q.zero_points, axis, gs))


def gather_columns(q: IntQ, idx) -> IntQ:
    """quantcore.py:158-175: salient slice sharing the per-token scales/zps."""
    axis, gs = _groups(q.config, q.shape)
    if axis != "col" or gs != q.shape[1]:
        raise OracleError("gather_columns requires one scale group per row")
    idx = np.asarray(idx, dtype=np.intp)
    cfg = IntCfg(q.config.bits, q.config.symmetric, "per-row", q.config.axis)
    return IntQ(np.ascontiguousarray(q.codes[:, idx]), q.scales, q.zero_points, cfg,
                (q.shape[0], idx.size))


def exact_int_matmul(a, b) -> np.ndarray:
    """mxfmt.py:122-132: int64-exact product (dgemm when every partial sum < 2^53)."""
    a = np.asarray(a, dtype=np.int64)
    b = np.asarray(b, dtype=np.int64)
    bound = a.shape[1] * float(np.abs(a).max(initial=0)) * float(np.abs(b).max(initial=0))
    if bound < 2.0**53:
        return np.rint(a.astype(np.float64) @ b.astype(np.float64)).astype(np.int64)
    return a @ b


def int_gemm(xq: IntQ, wq: IntQ, return_partials: bool = False):
    """mxfmt.py:135-195 (``int_gemm_reference``).

    Row-grouped W: per refined group, acc = sum (c - zp) * w with int64
    semantics, then out += sx * acc * sw, groups ascending (mxfmt.py:177-195).
    Column-grouped W: sx * ((c - zp) @ dequant(W)) in float64 (mxfmt.py:165-175).
    """
    if xq.shape[1] != wq.shape[0]:
        raise OracleError(f"inner dimensions disagree: {xq.shape} x {wq.shape}")
    xa, xgs = _groups(xq.config, xq.shape)
    if xa != "col":
        raise OracleError("xq must use column groups (per-token scales)")
    wa, wgs = _groups(wq.config, wq.shape)
    k = xq.shape[1]
    xc = xq.codes.astype(np.int64)
    if xq.zero_points is not None:
        xc = xc - np.repeat(xq.zero_points.astype(np.int64), xgs, axis=1)
    if wa == "col":
        w_hat = dequantize(wq)
        if xgs == k:
            out = xq.scales[:, [0]] * (xc.astype(np.float64) @ w_hat)
        else:
            out = (xc.astype(np.float64) * np.repeat(xq.scales, xgs, axis=1)) @ w_hat
        return (out, []) if return_partials else out
    xb = set(range(0, k + 1, xgs))
    wb = set(range(0, k + 1, wgs))
    if not (xb <= wb or wb <= xb):
        raise OracleError("scale group boundaries are misaligned")
    bounds = sorted(xb | wb)
    out = np.zeros((xq.shape[0], wq.shape[1]))
    parts = []
    for a, b in zip(bounds[:-1], bounds[1:]):
        acc = exact_int_matmul(xc[:, a:b], wq.codes[a:b, :])
        out += xq.scales[:, [a // xgs]] * acc * wq.scales[[a // wgs], :]
        if return_partials:
            parts.append(((a, b), acc))
    return (out, parts) if return_partials else out


# ---------------------------------------------------------------------------
# MXFP4 (reference mxfmt.py)
# ---------------------------------------------------------------------------

E2M1_MAG = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])
# decision points between consecutive magnitudes
_E2M1_MID = (E2M1_MAG[:-1] + E2M1_MAG[1:]) / 2.0


@dataclass
class MxT:
    """``MxBlockTensor`` (mxfmt.py:34-49): unpacked uint8 codes + int32 exps."""

    element_codes: np.ndarray
    block_scale_exponents: np.ndarray
    block_size: int
    shape: tuple


def e2m1_nearest(v):
    """mxfmt.py:52-72: nearest E2M1 magnitude, ties to the even mantissa
    index, saturating at 6; values rounding to zero get the +0 code.

    Restated as a threshold search instead of the reference's broadcast
    argmin: magnitude index = number of decision points below |v|, and an
    exact hit on a decision point picks the even neighbour.
    """
    arr = np.asarray(v, dtype=np.float64)
    if arr.size and not np.isfinite(arr).all():
        raise OracleError("e2m1_nearest requires finite input")
    a = np.abs(arr)
    idx = np.searchsorted(_E2M1_MID, a, side="left")
    hit = np.zeros(a.shape, dtype=bool)
    inside = idx < _E2M1_MID.size
    hit[inside] = a[inside] == _E2M1_MID[idx[inside]]
    idx = np.where(hit & (idx % 2 == 1), idx + 1, idx)
    vals = E2M1_MAG[idx]
    neg = (arr < 0) & (idx > 0)
    codes = np.where(neg, idx + 8, idx).astype(np.uint8)
    vals = np.where(neg, -vals, vals)
    if arr.ndim == 0:
        return codes[()], float(vals[()])
    return codes, vals


def e2m1_decode(codes) -> np.ndarray:
    """mxfmt.py:75-79."""
    codes = np.asarray(codes)
    return np.where((codes & 8) != 0, -1.0, 1.0) * E2M1_MAG[codes & 7]


def block_exponents(x, bs: int) -> np.ndarray:
    """mxfmt.py:88-94: e = floor(log2 amax) - 2 via frexp; 0 for an all-zero
    block; clipped to [-127, 127]."""
    r, c = x.shape
    amax = np.abs(x).reshape(r, c // bs, bs).max(axis=2)
    _, ex = np.frexp(amax)
    e = np.where(amax == 0.0, 0, ex - 3)
    return np.clip(e, -127, 127).astype(np.int32)


def mx_encode(x, bs: int = 32) -> MxT:
    """mxfmt.py:97-108."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    r, c = x.shape
    if c % bs:
        raise OracleError(f"row length {c} not divisible by block_size {bs}")
    e = block_exponents(x, bs)
    codes, _ = e2m1_nearest(x / np.ldexp(1.0, np.repeat(e, bs, axis=1)))
    return MxT(codes, e, bs, (r, c))


def mx_decode(t: MxT) -> np.ndarray:
    """mxfmt.py:111-113."""
    return e2m1_decode(t.element_codes) * np.ldexp(
        1.0, np.repeat(t.block_scale_exponents, t.block_size, axis=1))


def mx_gemm(x: MxT, wt: MxT) -> np.ndarray:
    """mxfmt.py:198-225: per aligned 32-block (ascending) a float64 dot of the
    decoded codes, scaled by 2^(ex+ew), accumulated into a float64 output."""
    if x.block_size != wt.block_size:
        raise OracleError("block sizes disagree")
    if x.shape[1] != wt.shape[1]:
        raise OracleError(f"inner dimensions disagree: {x.shape} x {wt.shape} (transposed)")
    bs = x.block_size
    xv = e2m1_decode(x.element_codes)
    wv = e2m1_decode(wt.element_codes)
    out = np.zeros((x.shape[0], wt.shape[0]))
    for b in range(x.shape[1] // bs):
        s = slice(b * bs, (b + 1) * bs)
        out += (xv[:, s] @ wv[:, s].T) * np.ldexp(
            1.0, x.block_scale_exponents[:, [b]] + wt.block_scale_exponents[:, [b]].T)
    return out


def pack_mx_file_bytes(t: MxT) -> bytes:
    """mxfmt.py:228-251 on-disk layout: 16-byte magic, <III rows, cols, bs,
    then per block one biased exponent byte (+127) and bs/2 nibble bytes
    (low nibble = even index)."""
    import struct

    r, c = t.shape
    nb = c // t.block_size
    out = bytearray(b"SERQMXB0" + b"\x00" * 8)
    out += struct.pack("<III", r, c, t.block_size)
    codes = t.element_codes.reshape(r, nb, t.block_size).astype(np.uint8)
    packed = (codes[..., 0::2] & 0xF) | ((codes[..., 1::2] & 0xF) << 4)
    body = np.concatenate(
        [(t.block_scale_exponents.reshape(r, nb, 1) + 127).astype(np.uint8), packed], axis=2)
    out += body.tobytes()
    return bytes(out)


# ---------------------------------------------------------------------------
# the decomposed forward (reference compensate.py)
# ---------------------------------------------------------------------------


@dataclass
class Comp:
    """``Compensator`` (compensate.py:48-69): one matrix R (rtn_residual /
    gptq_swapped) or the SVD baseline's two factors L1 [K, r], L2 [r, N]."""

    rank: int
    salient_idx: np.ndarray | None = None
    r_q: object = None
    r_dense: np.ndarray | None = None
    l1: np.ndarray | None = None
    l2: np.ndarray | None = None


def forward_int(x, main: IntQ, comp: Comp | None, act_cfg: IntCfg, symmetric_act=False):
    """compensate.py:272-316 integer branch.

    The reference requires an asymmetric ``act_cfg`` (compensate.py:298-299);
    ``symmetric_act=True`` composes the same reference primitives with
    ``quantize_symmetric`` for BASELINE config 1."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    if symmetric_act:
        xq = quantize_symmetric(x, act_cfg)
    else:
        if act_cfg is None or act_cfg.symmetric:
            raise OracleError("act_cfg must be asymmetric (per-token)")
        xq = quantize_asymmetric(x, act_cfg)
    y = int_gemm(xq, main)
    if comp is None or comp.rank == 0:
        return y, xq
    if comp.l1 is not None:
        # SVD baseline (compensate.py:304-310): sequential two-factor product over the
        # full dequantized activation
        return y + (dequantize(xq) @ comp.l1) @ comp.l2, xq
    xs = gather_columns(xq, comp.salient_idx)
    if comp.r_dense is not None:
        return y + dequantize(xs) @ comp.r_dense, xq
    return y + int_gemm(xs, comp.r_q), xq


def forward_mx(x, main_t: MxT, comp: Comp | None):
    """compensate.py:319-340: encode X, main MX GEMM, re-encode the gathered
    salient columns, R GEMM (or the SVD baseline's two factors, :326-331)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    bs = main_t.block_size
    xm = mx_encode(x, bs)
    y = mx_gemm(xm, main_t)
    if comp is None or comp.rank == 0:
        return y
    if comp.l1 is not None:
        # SVD baseline over an MX main (compensate.py:326-331): the decoded activation times the
        # two factors, in sequence, no rank restriction
        return y + (mx_decode(xm) @ comp.l1) @ comp.l2
    if comp.rank % bs:
        raise OracleError("MX residual path needs rank divisible by block size")
    xs = mx_encode(np.ascontiguousarray(x[:, comp.salient_idx]), bs)
    if comp.r_dense is not None:
        return y + mx_decode(xs) @ comp.r_dense
    return y + mx_gemm(xs, comp.r_q)


def build_serq_rtn_mx(w, salient_idx, bs: int = 32):
    """compensate.py:343-357: main = mx_encode(W^T); R = exact residual of the
    salient rows, MX-encoded transposed."""
    w = np.ascontiguousarray(w, dtype=np.float64)
    main_t = mx_encode(w.T, bs)
    r = len(salient_idx)
    if r == 0:
        return main_t, Comp(0, np.empty(0, np.intp))
    if r % bs:
        raise OracleError("MX mode needs rank divisible by block size")
    resid = (w - mx_decode(main_t).T)[salient_idx, :]
    return main_t, Comp(r, np.asarray(salient_idx, np.intp),
                        r_q=mx_encode(np.ascontiguousarray(resid.T), bs))


def build_per_channel_int(w, salient_idx, bits=4, r_mode="dense"):
    """Per-output-channel INT artefacts: the reference's
    ``build_serq_rtn`` raises for ``group_size=K`` (compensate.py:102-113), so
    the composition is main = quantize_symmetric(W, (bits,True,K,'row')) and
    R = W[idx] - dequantize(main)[idx], the same exact residual the MX builder
    uses (compensate.py:355).  ``r_mode``: 'dense' keeps bf16(R) as the
    r_dense matrix (BASELINE C1 "L in bf16"); 'int' quantizes R with one
    scale per output column (row groups of size r), the integer layout of
    the reference's acceptance criterion 03 (test_acceptance.py:134-155)."""
    w = np.ascontiguousarray(w, dtype=np.float64)
    k = w.shape[0]
    main = quantize_symmetric(w, IntCfg(bits, True, k, "row"))
    idx = np.asarray(salient_idx, np.intp)
    r = idx.size
    if r == 0:
        return main, Comp(0, idx)
    resid = w[idx] - dequantize(main)[idx]
    if r_mode == "dense":
        return main, Comp(r, idx, r_dense=bf16_round(resid))
    return main, Comp(r, idx, r_q=quantize_symmetric(resid, IntCfg(bits, True, r, "row")))


def default_r_config(cols, bits=4, main_group="per-row") -> IntCfg:
    """compensate.py:80-86: R scales per (salient row x column group)."""
    gs = cols if main_group == "per-row" else min(cols, int(main_group))
    if cols % gs != 0:
        gs = cols
    return IntCfg(bits, True, gs, "col")


def build_grouped_int(w, salient_idx, group, bits=4, r_mode="int"):
    """Group-wise INT artefacts: main = quantize_symmetric(W,
    (bits, True, g, 'row')) -- scales [K/g, N], _weight_config with an integer
    group (pipeline.py:134-137) -- and R = W[idx] - dequantize(main)[idx]
    (build_serq_rtn's R when the salient rows fill the leading group,
    compensate.py:102-113).  ``r_mode``: 'int' (row groups of size r, one
    scale per output column), 'dense' (bf16 residual) or 'col' (the
    reference's default_r_config, compensate.py:80-86)."""
    w = np.ascontiguousarray(w, dtype=np.float64)
    main = quantize_symmetric(w, IntCfg(bits, True, int(group), "row"))
    idx = np.asarray(salient_idx, np.intp)
    r = idx.size
    if r == 0:
        return main, Comp(0, idx)
    resid = w[idx] - dequantize(main)[idx]
    if r_mode == "dense":
        return main, Comp(r, idx, r_dense=bf16_round(resid))
    if r_mode == "col":
        return main, Comp(r, idx, r_q=quantize_symmetric(resid, default_r_config(w.shape[1], bits, group)))
    return main, Comp(r, idx, r_q=quantize_symmetric(resid, IntCfg(bits, True, r, "row")))


# ---------------------------------------------------------------------------
# workload recipe helpers (reference tensorio.py / flatten.py / saliency.py)
# ---------------------------------------------------------------------------


def synthetic_activations(rows, cols, n_outlier=0, magnitude=1.0, seed=0):
    """tensorio.py:157-168: standard normal, then a seeded permutation picks
    the outlier columns, which are scaled by ``magnitude``."""
    g = np.random.default_rng(seed)
    x = g.standard_normal((rows, cols))
    if n_outlier:
        x[:, g.permutation(cols)[:n_outlier]] *= magnitude
    return x


def smoothing_scales(calib, w, alpha=0.5):
    """flatten.py:34-51 with tensorio.py:181-188 stats."""
    amax = np.abs(calib).max(axis=0)
    wmax = np.abs(w).max(axis=1)
    with np.errstate(divide="ignore", invalid="ignore"):
        s = amax**alpha / wmax ** (1.0 - alpha)
    return np.where(np.isfinite(s) & (s > 0), s, 1.0)


def plan_permutation(scores, r):
    """saliency.py:77-92: stable top-r (ties to the lower index), salient rows
    first, the rest ascending."""
    scores = np.asarray(scores, dtype=np.float64)
    order = np.argsort(-scores, kind="stable")
    sal = order[:r].astype(np.intp)
    if r == scores.size:
        return sal, order.astype(np.intp)
    rest = np.setdiff1d(np.arange(scores.size, dtype=np.intp), sal)
    return sal, np.concatenate([sal, rest])


def rmsnorm(x, gain, eps: float = 1e-6) -> np.ndarray:
    """saliency.py:194-196: x / sqrt(mean(x^2) + eps) * gain, in float64."""
    x = np.asarray(x, dtype=np.float64)
    rms = np.sqrt(np.mean(x * x, axis=1, keepdims=True) + eps)
    return x / rms * np.asarray(gain, dtype=np.float64)[None, :]


def silu(x) -> np.ndarray:
    """saliency.py:199-200."""
    return x / (1.0 + np.exp(-x))


def attention_mix(q, k, v, head_dim: int) -> np.ndarray:
    """saliency.py:203-216: per-head softmax(Q K^T / sqrt(d)) V over the token batch."""
    out = np.empty_like(v)
    for h in range(q.shape[1] // head_dim):
        sl = slice(h * head_dim, (h + 1) * head_dim)
        logits = q[:, sl] @ k[:, sl].T / np.sqrt(head_dim)
        logits -= logits.max(axis=1, keepdims=True)
        a = np.exp(logits)
        a /= a.sum(axis=1, keepdims=True)
        out[:, sl] = a @ v[:, sl]
    return out


def forward_block_mx(x, linears: dict, gains: dict, head_dim: int, bf16_linear_out: bool = False) -> np.ndarray:
    """toymodel.forward_quantized (toymodel.py:363-374) on toy_block_graph (toymodel.py:88-124):
    graph_forward's node order with every linear through forward_mx.  ``linears``:
    name -> (main_t, comp).  ``bf16_linear_out`` rounds every linear's output to bf16 --
    the device linears' output contract -- before it feeds the next node."""
    x = np.asarray(x, dtype=np.float64)

    def lin(name, xin):
        main_t, comp = linears[name]
        y = forward_mx(xin, main_t, comp)
        return bf16_round(y) if bf16_linear_out else y

    h1 = rmsnorm(x, gains["ln1"])
    attn = attention_mix(lin("q_proj", h1), lin("k_proj", h1), lin("v_proj", h1), head_dim)
    res1 = x + lin("o_proj", attn)
    h2 = rmsnorm(res1, gains["ln2"])
    mid = silu(lin("gate_proj", h2)) * lin("up_proj", h2)
    return res1 + lin("down_proj", mid)


def bf16_round(x) -> np.ndarray:
    """Round float64 to the nearest bfloat16 (ties to even), returned as f64.

    One rounding step from f64 (no f32 intermediate): scale the value so its
    8 significant bits are integral and ``np.rint`` it."""
    x = np.asarray(x, dtype=np.float64)
    _, e = np.frexp(x)  # x = m * 2^e, |m| in [0.5, 1)
    e = np.maximum(e, -125)  # below 2^-126 the bf16 spacing is fixed at 2^-133
    return np.ldexp(np.rint(np.ldexp(x, 8 - e)), e - 8)


def parity_errors(y, y_oracle):
    """SURVEY 8(d) parity metric against bf16_rne(Y_oracle):
    (max|dY|/max|Yref|, mean|dY|/mean|Yref|)."""
    ref = bf16_round(y_oracle)
    d = np.abs(np.asarray(y, np.float64) - ref)
    return float(d.max() / max(np.abs(ref).max(), 1e-300)), float(d.mean() / max(np.abs(ref).mean(), 1e-300))
