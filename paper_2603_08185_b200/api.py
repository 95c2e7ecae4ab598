"""Reference-facing mirror of the SERQ hot path, backed by the sm_100a kernels.

Same names, argument meaning and error behaviour as the reference package
(``/root/reference/pkg/src/serq``) for the functions on the hot path, so a
caller of the reference can switch import paths:

  IntQuantConfig, QuantizedTensor, per_token_config   quantcore.py:28-80
  quantize_symmetric / quantize_asymmetric            quantcore.py:108-137 (GPU, bit-exact)
  dequantize, gather_columns                          quantcore.py:144-175
  MxBlockTensor, mx_encode, mx_decode                 mxfmt.py:34-113 (encode on GPU, bit-exact)
  Compensator, OpProbe                                compensate.py:48-77
  build_serq_rtn_mx                                   compensate.py:343-357 (encodes on GPU)
  forward_reconstructed                               compensate.py:272-340 (GPU linear)
  SerqLinear / make_linear_fn                         the module-level API used by
                                                      SerqQuantizer.predict (estimators.py:89-97)
                                                      and forward_quantized's linear_fn
                                                      (toymodel.py:363-374)

Artefacts produced by the reference builders (its dataclasses) are accepted
by duck typing.  Layouts that integer tensor cores cannot evaluate exactly
(scales that vary along the reduction dimension) raise
``ValidationError`` naming the layout; there is no CPU fallback.
"""

from __future__ import annotations

import threading
import weakref
from collections import OrderedDict
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import device as D
from .errors import ValidationError

ROW_GROUPS, COL_GROUPS, PER_ROW = "row", "col", "per-row"
RTN_RESIDUAL, GPTQ_SWAPPED, SVD_BASELINE = "rtn_residual", "gptq_swapped", "svd_baseline"

E2M1_MAGNITUDES = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])


# ------------------------------------------------------------------ containers


@dataclass(frozen=True)
class IntQuantConfig:
    bits: int = 4
    symmetric: bool = True
    group_size: int | str = PER_ROW
    axis: str = ROW_GROUPS

    def __post_init__(self):
        if not 2 <= self.bits <= 8:
            raise ValidationError(f"bits must be in [2, 8], got {self.bits}")
        if self.axis not in (ROW_GROUPS, COL_GROUPS):
            raise ValidationError(f"unknown axis {self.axis!r}")
        if self.group_size != PER_ROW and (not isinstance(self.group_size, (int, np.integer)) or self.group_size < 1):
            raise ValidationError(f"invalid group_size {self.group_size!r}")

    @property
    def qmax(self) -> int:
        return 2 ** (self.bits - 1) - 1

    @property
    def levels(self) -> int:
        return 2**self.bits - 1


def per_token_config(bits: int = 8) -> IntQuantConfig:
    return IntQuantConfig(bits=bits, symmetric=False, group_size=PER_ROW)


@dataclass
class QuantizedTensor:
    codes: np.ndarray
    scales: np.ndarray
    zero_points: np.ndarray | None
    config: IntQuantConfig
    shape: tuple

    @property
    def rows(self) -> int:
        return self.shape[0]

    @property
    def cols(self) -> int:
        return self.shape[1]


@dataclass
class MxBlockTensor:
    element_codes: np.ndarray
    block_scale_exponents: np.ndarray
    block_size: int
    shape: tuple

    @property
    def rows(self) -> int:
        return self.shape[0]

    @property
    def cols(self) -> int:
        return self.shape[1]


@dataclass
class Compensator:
    mode: str
    rank: int
    salient_idx: np.ndarray | None = None
    r_q: object = None
    r_dense: np.ndarray | None = None
    l1: np.ndarray | None = None
    l2: np.ndarray | None = None

    def __post_init__(self):
        if self.mode not in (RTN_RESIDUAL, GPTQ_SWAPPED, SVD_BASELINE):
            raise ValidationError(f"unknown compensator mode {self.mode!r}")
        if self.rank and self.mode == SVD_BASELINE:  # compensate.py:59-63
            if self.l1 is None or self.l2 is None:
                raise ValidationError("SVD mode carries two factors")
            if self.r_q is not None or self.r_dense is not None:
                raise ValidationError("SVD mode must not carry a residual matrix")
        if self.rank and self.mode in (RTN_RESIDUAL, GPTQ_SWAPPED):
            if (self.r_q is not None) + (self.r_dense is not None) != 1:
                raise ValidationError("single-matrix modes carry exactly one R")


@dataclass
class OpProbe:
    aux_matmuls: int = 0
    notes: list = field(default_factory=list)


# ------------------------------------------------------------------ helpers


def _as_matrix(a, name="x") -> np.ndarray:
    arr = np.ascontiguousarray(a, dtype=np.float64)
    if arr.ndim != 2:
        raise ValidationError(f"{name} must be 2-D, got shape {arr.shape}")
    if arr.size == 0:
        raise ValidationError(f"{name} must be non-empty")
    if not np.isfinite(arr).all():
        raise ValidationError(f"{name} contains non-finite values")
    return arr


def _groups(cfg, shape):
    rows, cols = shape
    if cfg.group_size == PER_ROW:
        return COL_GROUPS, cols
    gs = int(cfg.group_size)
    dim = rows if cfg.axis == ROW_GROUPS else cols
    if dim % gs:
        raise ValidationError(f"group_size {gs} does not divide grouped dimension {dim}")
    return cfg.axis, gs


def _to_gpu(x: np.ndarray, dtype=torch.float64) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)


# ------------------------------------------------------------------ quantizers


def _quantize(x, cfg: IntQuantConfig, symmetric: bool) -> QuantizedTensor:
    if cfg.symmetric != symmetric:
        raise ValidationError("config is not symmetric" if symmetric else "config is not asymmetric")
    x = _as_matrix(x)
    rows, cols = x.shape
    axis, gs = _groups(cfg, x.shape)
    # every group is a 1-D run of gs elements: lay the groups out as the rows of a
    # [n_groups, gs] matrix and quantize per row on the device (quantcore.py:83-94 layouts)
    if axis == COL_GROUPS:
        src = x.reshape(rows * (cols // gs), gs)  # scale per (row, column group)
    else:
        src = np.ascontiguousarray(x.reshape(rows // gs, gs, cols).transpose(0, 2, 1)).reshape(-1, gs)
    act = D.quantize_int(_to_gpu(np.ascontiguousarray(src)), cfg.bits, symmetric)
    codes = act.codes.cpu().numpy()
    codes = codes.astype(np.int32) if symmetric else codes.view(np.uint8).astype(np.int32)
    scales = act.scale64.cpu().numpy()
    zps = None if symmetric else act.zp.cpu().numpy().astype(np.int32)
    if axis == COL_GROUPS:
        codes = codes.reshape(rows, cols)
        scales = scales.reshape(rows, cols // gs)
        zps = None if zps is None else zps.reshape(rows, cols // gs)
    else:
        codes = np.ascontiguousarray(codes.reshape(rows // gs, cols, gs).transpose(0, 2, 1)).reshape(rows, cols)
        scales = scales.reshape(rows // gs, cols)
        zps = None if zps is None else zps.reshape(rows // gs, cols)
    return QuantizedTensor(codes, scales, zps, cfg, x.shape)


def quantize_symmetric(x, cfg: IntQuantConfig) -> QuantizedTensor:
    """GPU twin of quantcore.quantize_symmetric (quantcore.py:108-118), bit-exact."""
    return _quantize(x, cfg, True)


def quantize_asymmetric(x, cfg: IntQuantConfig) -> QuantizedTensor:
    """GPU twin of quantcore.quantize_asymmetric (quantcore.py:121-137), bit-exact."""
    return _quantize(x, cfg, False)


def dequantize(q) -> np.ndarray:
    """quantcore.py:144-150 (host arithmetic on artefacts; not on the hot path)."""
    axis, gs = _groups(q.config, q.shape)
    s = np.repeat(q.scales, gs, axis=0 if axis == ROW_GROUPS else 1)
    if q.zero_points is None:
        return s * q.codes
    z = np.repeat(q.zero_points, gs, axis=0 if axis == ROW_GROUPS else 1)
    return s * (q.codes.astype(np.float64) - z)


def gather_columns(q, idx) -> QuantizedTensor:
    """quantcore.py:158-175."""
    axis, gs = _groups(q.config, q.shape)
    if axis != COL_GROUPS or gs != q.shape[1]:
        raise ValidationError("gather_columns requires one scale group per row")
    idx = np.asarray(idx, dtype=np.intp)
    return QuantizedTensor(np.ascontiguousarray(q.codes[:, idx]), q.scales, q.zero_points,
                           replace(q.config, group_size=PER_ROW), (q.shape[0], idx.size))


def mx_encode(x, block_size: int = 32) -> MxBlockTensor:
    """GPU twin of mxfmt.mx_encode (mxfmt.py:97-108): exact for float64 input."""
    if block_size != 32:
        raise ValidationError("the device MX format uses 32-element blocks")
    x = _as_matrix(x)
    rows, cols = x.shape
    if cols % block_size:
        raise ValidationError(f"row length {cols} not divisible by block_size {block_size}")
    act = D.quantize_mx(_to_gpu(x))
    c, e = D.unpack_mx(act.codes, act.sf, rows, cols)
    return MxBlockTensor(c.cpu().numpy(), e.cpu().numpy(), block_size, (rows, cols))


def mx_decode(t) -> np.ndarray:
    """mxfmt.py:111-113 (artefact utility, host)."""
    c = np.asarray(t.element_codes)
    v = np.where((c & 8) != 0, -1.0, 1.0) * E2M1_MAGNITUDES[c & 7]
    return v * np.ldexp(1.0, np.repeat(t.block_scale_exponents, t.block_size, axis=1))


def build_serq_rtn_mx(w_folded, plan, block_size: int = 32):
    """compensate.py:343-357 with the encodes on the GPU.  ``plan`` is a
    SaliencyPlan (uses ``.rank`` / ``.salient_idx``) or an index array."""
    w = _as_matrix(w_folded, "w_folded")
    idx = np.asarray(getattr(plan, "salient_idx", plan), dtype=np.intp)
    r = idx.size
    main_t = mx_encode(np.ascontiguousarray(w.T), block_size)
    if r == 0:
        return main_t, Compensator(RTN_RESIDUAL, 0, np.empty(0, np.intp))
    if r % block_size:
        raise ValidationError("MX mode needs rank divisible by block size")
    resid = (w - mx_decode(main_t).T)[idx, :]
    return main_t, Compensator(RTN_RESIDUAL, r, idx.copy(), r_q=mx_encode(np.ascontiguousarray(resid.T), block_size))


def build_per_channel_int(w, salient_idx, bits: int = 4, r_mode: str = "dense"):
    """Per-output-channel integer artefacts: main =
    quantize_symmetric(W, (bits, True, K, 'row')); R = W[idx] -
    dequantize(main)[idx], kept as bf16 (``r_mode='dense'``) or quantized with
    one scale per output column (``'int'``)."""
    w = _as_matrix(w, "w")
    k = w.shape[0]
    main = quantize_symmetric(w, IntQuantConfig(bits, True, k, ROW_GROUPS))
    idx = np.asarray(salient_idx, dtype=np.intp)
    r = idx.size
    if r == 0:
        return main, Compensator(RTN_RESIDUAL, 0, idx)
    resid = w[idx] - dequantize(main)[idx]
    if r_mode == "dense":
        rd = torch.from_numpy(resid).to(torch.bfloat16).to(torch.float64).numpy()
        return main, Compensator(RTN_RESIDUAL, r, idx.copy(), r_dense=rd)
    return main, Compensator(RTN_RESIDUAL, r, idx.copy(),
                             r_q=quantize_symmetric(resid, IntQuantConfig(bits, True, r, ROW_GROUPS)))


# ------------------------------------------------------------------ linear modules


def build_serq_rtn(w_folded, plan, wcfg: IntQuantConfig, rcfg: IntQuantConfig | None):
    """compensate.build_serq_rtn (compensate.py:89-114) with the device quantizers:
    main = quantize_symmetric(W, wcfg); R = Ws - fake_quant(Ws, wcfg) over the
    salient rows, quantized with ``rcfg`` or kept dense (``rcfg=None``).  With
    wcfg row groups of g and r a multiple of g this is the
    group-wise artefact the device consumes."""
    w = _as_matrix(w_folded, "w_folded")
    scores = np.asarray(plan.scores)
    if scores.shape[0] != w.shape[0]:
        raise ValidationError("plan was not built for this weight")
    main = quantize_symmetric(w, wcfg)
    r = int(plan.rank)
    if r == 0:
        return main, Compensator(RTN_RESIDUAL, 0, np.empty(0, np.intp))
    idx = np.asarray(plan.salient_idx, dtype=np.intp)
    ws = w[idx]
    resid = ws - dequantize(quantize_symmetric(ws, wcfg))
    if rcfg is None:
        return main, Compensator(RTN_RESIDUAL, r, idx.copy(), r_dense=resid)
    return main, Compensator(RTN_RESIDUAL, r, idx.copy(), r_q=quantize_symmetric(resid, rcfg))


def _is_mx(t) -> bool:
    return hasattr(t, "element_codes") and hasattr(t, "block_scale_exponents")


class SerqLinear:
    """One SERQ linear resident on the GPU (packed once from the artefacts).

    ``__call__`` takes a CUDA tensor [M, K] (bf16 for the serving path; f32/f64
    accepted) and returns bf16 [M, N].  INT layers quantize activations with
    ``act_cfg`` (asymmetric per-token as the reference requires, or symmetric
    when ``allow_symmetric_act`` -- BASELINE config 1)."""

    def __init__(self, main, comp=None, act_cfg=None, allow_symmetric_act=False, device="cuda"):
        self.fmt = "mx" if _is_mx(main) else "int"
        has_r = comp is not None and getattr(comp, "rank", 0)
        self.svd = None
        if has_r and getattr(comp, "mode", RTN_RESIDUAL) == SVD_BASELINE:
            # SVD baseline (compensate.py:209-224, 304-310, MX 326-331): the two-factor correction
            # (x_hat @ L1) @ L2 spans all K columns.  INT: U = (codes - zp) @ L1 as one bf16 GEMM, then
            # U @ L2 as the fused INT kernel's dense side term (device.SvdIntLinear); MX: x_hat =
            # mx_decode(x_mx) on the device, the correction as an fp32 addend of the MX kernel
            # (device.SvdMxLinear)
            l1 = np.asarray(comp.l1, dtype=np.float64)
            l2 = np.asarray(comp.l2, dtype=np.float64)
            k_in, n_out = (main.shape[1], main.shape[0]) if _is_mx(main) else main.shape
            if l1.shape != (k_in, comp.rank) or l2.shape != (comp.rank, n_out):
                raise ValidationError("SVD factors must be L1 [K, r] and L2 [r, N]")
            self.svd = (l1, l2)
            comp, has_r = None, 0
        idx = None if not has_r else np.asarray(comp.salient_idx, dtype=np.intp)
        if self.fmt == "mx":
            if getattr(main, "block_size", 32) != 32:
                raise ValidationError("the device MX format uses 32-element blocks")
            if has_r and comp.rank % 32:
                raise ValidationError("MX residual path needs rank divisible by block size")
            rq = comp.r_q if has_r else None
            if has_r and comp.r_dense is not None:
                # unquantized R (compensate.py:338-339): the decoded salient slice times R, added in
                # the MX kernel's epilogue (device.MxDenseRLinear)
                self.impl = D.MxDenseRLinear(main.element_codes, main.block_scale_exponents, comp.r_dense, idx,
                                             device=device)
            elif self.svd is not None:
                self.impl = D.SvdMxLinear(main.element_codes, main.block_scale_exponents, *self.svd, device=device)
            else:
                self.impl = D.MxLinear(main.element_codes, main.block_scale_exponents,
                                       None if rq is None else rq.element_codes,
                                       None if rq is None else rq.block_scale_exponents, idx, device)
            self.K, self.N = main.shape[1], main.shape[0]
        else:
            if act_cfg is None or (act_cfg.symmetric and not allow_symmetric_act):
                raise ValidationError("act_cfg must be asymmetric (per-token)")
            a_axis, a_gs = _groups(act_cfg, (1, main.shape[0]))
            if not (a_axis == COL_GROUPS and a_gs == main.shape[0]):
                raise ValidationError("activations must be quantized per token ('per-row')")
            axis, gs = _groups(main.config, main.shape)
            k = main.shape[0]
            if not (axis == ROW_GROUPS and (gs == k or (gs % 128 == 0 and gs <= 8192))) or main.zero_points is not None:
                raise ValidationError(
                    f"integer main layout (group_size={main.config.group_size!r}, axis={main.config.axis!r}) is not "
                    "GPU-native: scales must be symmetric per output column (group_size == K, axis 'row') or per "
                    "(row group, output column) with group_size a multiple of 128 up to 8192 (SURVEY F12)")
            kw = {}
            if has_r:
                if comp.r_dense is not None:
                    # a GPTQ-swapped R holds the salient rows themselves (compensate.py:136-143): hi + lo planes
                    kw = dict(r_dense=np.asarray(comp.r_dense), r_split=comp.mode == GPTQ_SWAPPED)
                else:
                    rq = comp.r_q
                    ax, g = _groups(rq.config, rq.shape)
                    if ax == ROW_GROUPS and g == rq.shape[0] and rq.zero_points is None:
                        kw = dict(r_codes=rq.codes, r_scales=rq.scales)
                    elif ax == COL_GROUPS:
                        # default_r_config (compensate.py:80-86): scales vary along the salient rows, so the
                        # reference runs this term in its float branch (mxfmt.py:165-175) on dequantize(r_q);
                        # the device runs it as a dense R split into bf16 hi + lo planes (a GPTQ-swapped R
                        # is the salient rows themselves, too large a share of Y for one bf16 rounding)
                        kw = dict(r_dense=dequantize(rq), r_split=True)
                    else:
                        raise ValidationError(
                            "integer R must be symmetric with one scale per output column (row groups of size r) or "
                            "column-grouped (default_r_config)")
            if self.svd is not None:
                self.impl = D.SvdIntLinear(main.codes, main.scales, main.config.bits, *self.svd, device=device,
                                           group_size=gs)
            else:
                self.impl = D.IntLinear(main.codes, main.scales, main.config.bits, salient_idx=idx, device=device,
                                        group_size=gs, **kw)
            self.act_bits, self.act_symmetric = act_cfg.bits, act_cfg.symmetric
            self.K, self.N = main.shape
        self.rank = int(comp.rank) if has_r else 0
        self.aux_matmuls = 2 if self.svd is not None else (1 if self.rank else 0)

    def __call__(self, x: torch.Tensor, y: torch.Tensor | None = None) -> torch.Tensor:
        if x.shape[-1] != self.K:
            raise ValidationError("x columns must equal main rows")
        if self.fmt == "mx":
            return self.impl(x, y)
        if self.svd is not None:
            return self.impl.forward(x, self.act_bits, self.act_symmetric, y)
        return self.impl(x, self.act_bits, self.act_symmetric, y)


# Packed device linears per artefact object.  The cache holds the artefacts WEAKLY (an
# entry, and with it the device weights, is dropped when its main or comp artefact is
# garbage collected) and at most CACHE_MAX entries (least recently used evicted); artefacts
# that cannot be weakly referenced are held strongly, under the same bound.
CACHE_MAX = 64
_CACHE: OrderedDict = OrderedDict()
_CACHE_LOCK = threading.Lock()


def clear_cache() -> None:
    with _CACHE_LOCK:
        _CACHE.clear()


def _ref(obj, key, entry_box):
    if obj is None:
        return lambda: None

    def drop(_):
        with _CACHE_LOCK:
            if _CACHE.get(key) is entry_box[0]:
                del _CACHE[key]

    try:
        return weakref.ref(obj, drop)
    except TypeError:
        return lambda: obj


def _linear_for(main, comp, act_cfg, allow_symmetric_act=False) -> SerqLinear:
    key = (id(main), id(comp), act_cfg, allow_symmetric_act)
    with _CACHE_LOCK:
        hit = _CACHE.get(key)
        if hit is not None and hit[0]() is main and hit[1]() is comp:
            _CACHE.move_to_end(key)
            return hit[2]
    lin = SerqLinear(main, comp, act_cfg, allow_symmetric_act)
    box = [None]
    entry = (_ref(main, key, box), _ref(comp, key, box), lin)
    box[0] = entry
    with _CACHE_LOCK:
        _CACHE[key] = entry
        _CACHE.move_to_end(key)
        while len(_CACHE) > CACHE_MAX:
            _CACHE.popitem(last=False)
    return lin


def forward_reconstructed(x, main, comp, act_cfg, probe: OpProbe | None = None) -> np.ndarray:
    """Drop-in for compensate.forward_reconstructed (compensate.py:272-316).

    Activations are sent to the device as float64 and quantized there
    bit-exactly; the main and salient products run in ONE fused kernel; the
    bf16 result is returned as float64.  Weights are packed once per artefact
    object and cached.  ``probe.aux_matmuls`` still counts the one auxiliary
    product of the SERQ path (compensate.py:312-313)."""
    x = _as_matrix(x)
    if isinstance(main, np.ndarray):
        # quantization-disabled mode (compensate.py:288-293): exact product on the device
        xt = _to_gpu(x)
        y = xt @ _to_gpu(main)
        if comp is not None and comp.rank:
            full = np.zeros(main.shape)
            full[np.asarray(comp.salient_idx)] = np.asarray(comp.r_dense if comp.r_dense is not None else dequantize(comp.r_q))
            y = y + xt @ _to_gpu(full)
        return y.cpu().numpy()
    if _is_mx(main):
        if x.shape[1] != main.shape[1]:
            raise ValidationError("x columns must equal weight input dim")
    else:
        if x.shape[1] != main.shape[0]:
            raise ValidationError("x columns must equal main rows")
        if act_cfg is None or act_cfg.symmetric:
            raise ValidationError("act_cfg must be asymmetric (per-token)")
    lin = _linear_for(main, comp, act_cfg)
    y = lin(_to_gpu(x))
    if probe is not None and lin.aux_matmuls:
        probe.aux_matmuls += lin.aux_matmuls
        if lin.svd is not None and lin.fmt == "int":  # (the MX branch adds no note, compensate.py:328-329)
            probe.notes.append("sequential two-factor path")
    return y.float().cpu().numpy().astype(np.float64)


def layer_forward(art, x, probe: OpProbe | None = None) -> np.ndarray:
    """Drop-in for pipeline.layer_forward (pipeline.py:126-131): divide the activation
    columns by the SAF smoothing scales (flatten.py:62-67, host float64 exactly as the
    reference) and run forward_reconstructed on the device.  ``art`` is the reference's
    LayerArtifacts (main, comp, act_cfg, smoothing) or any object with those fields."""
    x = _as_matrix(x)
    smoothing = getattr(art, "smoothing", None)
    if smoothing is not None:
        s = np.asarray(smoothing.s, dtype=np.float64)
        if s.shape[0] != x.shape[1]:
            raise ValidationError("plan length does not match activation columns")
        x = x / s[None, :]
    return forward_reconstructed(x, art.main, art.comp, art.act_cfg, probe)


def predict(estimator, X, probe: OpProbe | None = None) -> np.ndarray:
    """SerqQuantizer.predict (estimators.py:89-97) on the device, for an estimator fitted by
    the reference (its ``artifacts_`` are the LayerArtifacts of quantize_layer): the same
    not-fitted / feature-count ValidationErrors, then layer_forward."""
    if not hasattr(estimator, "artifacts_"):
        raise ValidationError("estimator is not fitted")
    X = _as_matrix(X, "X")
    if X.shape[1] != estimator.n_features_in_:
        raise ValidationError(f"X has {X.shape[1]} features, expected {estimator.n_features_in_}")
    return layer_forward(estimator.artifacts_, X, probe)


def forward_symmetric_act(x, main, comp, act_cfg: IntQuantConfig) -> np.ndarray:
    """BASELINE config 1: symmetric per-token activations.  The reference
    forward rejects symmetric act_cfg (compensate.py:298-299); this is the
    composition int_gemm_reference(quantize_symmetric(x), main) +
    dequantize(gather_columns(xq, idx)) @ r_dense."""
    if not act_cfg.symmetric:
        raise ValidationError("forward_symmetric_act needs a symmetric act_cfg")
    x = _as_matrix(x)
    lin = _linear_for(main, comp, act_cfg, allow_symmetric_act=True)
    return lin(_to_gpu(x)).float().cpu().numpy().astype(np.float64)


def make_linear_fn(bundle, device="cuda"):
    """``linear_fn(name, x)`` for the reference's graph_forward hook
    (saliency.py:256-257; toymodel.forward_quantized, toymodel.py:363-374):
    every linear of a QuantizedBlockBundle runs on the GPU."""
    lins = {}
    for name, lb in bundle.linears.items():
        if isinstance(lb.main, np.ndarray):
            lins[name] = None
        else:
            lins[name] = SerqLinear(lb.main, lb.comp, lb.act_cfg, device=device)

    def linear_fn(name, xin):
        lin = lins[name]
        lb = bundle.linears[name]
        if lin is None:
            return forward_reconstructed(xin, lb.main, lb.comp, lb.act_cfg)
        return lin(_to_gpu(_as_matrix(xin))).float().cpu().numpy().astype(np.float64)

    return linear_fn
