"""Device-resident SERQ operators on torch tensors (torch = memory + streams).

Every operator here is a thin call through the C-ABI (``_lib``) on the
current torch CUDA stream; there is no PyTorch or CPU compute fallback.

Layouts:
  MX activation  codes uint8 [M, K/2] + tiled E8M0 scale factors
  INT activation codes int8 [M, K] + per-token scales f32/f64 + zero points
  MX weight      packed [N, K/2] (+ R [N, r/2]) owned by an ``MxLinear`` handle
  INT weight     int8 [N, K] + f32 scales + column sums (+ R) in an ``IntLinear``
"""

from __future__ import annotations

import ctypes
import threading
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ValidationError


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _dtype_id(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return _lib.SERQ_BF16
    if t.dtype == torch.float32:
        return _lib.SERQ_F32
    if t.dtype == torch.float64:
        return _lib.SERQ_F64
    raise ValidationError(f"unsupported activation dtype {t.dtype}")


def _require_cuda(t: torch.Tensor, name: str) -> None:
    if not (isinstance(t, torch.Tensor) and t.is_cuda):
        raise ValidationError(f"{name} must be a CUDA tensor")


def _check_salient_idx(salient_idx, r: int, K: int) -> np.ndarray | None:
    """The reference indexes x[:, idx] (compensate.py:311, 335) and raises on a bad index; the
    kernels read x[row, idx[j]] for j < r straight from device memory, so a short, out-of-range or
    repeated index must be rejected here, before it can fault the context or read garbage."""
    if salient_idx is None:
        return None
    idx = np.asarray(salient_idx.cpu() if isinstance(salient_idx, torch.Tensor) else salient_idx)
    if idx.ndim != 1:
        raise ValidationError(f"salient_idx must be 1-D, got shape {idx.shape}")
    if idx.size and not np.issubdtype(idx.dtype, np.integer):
        raise ValidationError(f"salient_idx must be integers, got {idx.dtype}")
    idx = idx.astype(np.int64)
    if idx.size != r:
        raise ValidationError(f"salient_idx has {idx.size} entries, the compensator rank is {r}")
    if idx.size and (idx.min() < 0 or idx.max() >= K):
        raise ValidationError(f"salient_idx out of range [0, {K})")
    if np.unique(idx).size != idx.size:
        raise ValidationError("salient_idx repeats a channel")
    return idx


def mx_sizes(rows: int, cols: int) -> tuple[int, int]:
    cb, sb = ctypes.c_int64(), ctypes.c_int64()
    _lib.call("serq_mx_sizes", rows, cols, ctypes.byref(cb), ctypes.byref(sb))
    return cb.value, sb.value


# ---------------------------------------------------------------- activations


@dataclass
class MxActivation:
    """Device MXFP4 activation: packed E2M1 codes + tiled E8M0 scales."""

    codes: torch.Tensor
    sf: torch.Tensor
    M: int
    K: int
    xs_codes: torch.Tensor | None = None
    xs_sf: torch.Tensor | None = None


@dataclass
class IntActivation:
    """Device per-token integer activation (codes int8, u8 bit patterns if asymmetric)."""

    codes: torch.Tensor
    scale64: torch.Tensor
    scale32: torch.Tensor
    zp: torch.Tensor | None
    bits: int
    symmetric: bool
    xs: torch.Tensor | None = None


def quantize_mx(x: torch.Tensor, gather_idx: torch.Tensor | None = None, out: MxActivation | None = None) -> MxActivation:
    """K1-MX.  x: [M, K] bf16/f32/f64 on the GPU.  ``gather_idx`` (int32, length
    r) additionally encodes the salient slice x[:, idx] (compensate.py:335)."""
    _require_cuda(x, "x")
    if x.dim() != 2 or x.stride(1) != 1:
        raise ValidationError("x must be a row-major 2-D tensor")
    M, K = x.shape
    if K % 32:
        raise ValidationError(f"row length {K} not divisible by block_size 32")
    r = 0 if gather_idx is None else int(gather_idx.numel())
    if out is None:
        cb, sb = mx_sizes(M, K)
        out = MxActivation(torch.empty(cb, dtype=torch.uint8, device=x.device),
                           torch.empty(sb, dtype=torch.uint8, device=x.device), M, K)
        if r:
            cbr, sbr = mx_sizes(M, r)
            out.xs_codes = torch.empty(cbr, dtype=torch.uint8, device=x.device)
            out.xs_sf = torch.empty(sbr, dtype=torch.uint8, device=x.device)
    _lib.call("serq_act_quant_mx", x.data_ptr(), _dtype_id(x), M, K, x.stride(0), out.codes.data_ptr(),
              out.sf.data_ptr(), _ptr(gather_idx), r, _ptr(out.xs_codes), _ptr(out.xs_sf), _stream())
    return out


def rmsnorm_quantize_mx(x: torch.Tensor, gain: torch.Tensor, eps: float = 1e-6,
                        out: MxActivation | None = None, gather_idx: torch.Tensor | None = None,
                        r: int = 0) -> MxActivation:
    """Producer fusion: mx_encode(rmsnorm(x, gain, eps)) in ONE kernel
    (saliency.py:194-196 then mxfmt.py:97-108).  x: bf16/f32 [M, K] residual
    stream on the GPU; gain: float64 [K] (the RMSNorm weight with the smoothing
    scales folded in).  ``gather_idx`` (int32 [r]): also encode the normalised
    salient slice rmsnorm(x)[:, idx] (compensate.py:335) into out.xs_codes /
    out.xs_sf -- the gather fallback of q/k/v and gate/up."""
    _require_cuda(x, "x")
    if x.dim() != 2 or x.stride(1) != 1:
        raise ValidationError("x must be a row-major 2-D tensor")
    M, K = x.shape
    if gain.dtype != torch.float64 or gain.numel() != K or not gain.is_cuda:
        raise ValidationError("gain must be a float64 CUDA vector of length K")
    if out is None:
        cb, sb = mx_sizes(M, K)
        out = MxActivation(torch.empty(cb, dtype=torch.uint8, device=x.device),
                           torch.empty(sb, dtype=torch.uint8, device=x.device), M, K)
    if gather_idx is not None and out.xs_codes is None:
        cbr, sbr = mx_sizes(M, r)
        out.xs_codes = torch.empty(cbr, dtype=torch.uint8, device=x.device)
        out.xs_sf = torch.empty(sbr, dtype=torch.uint8, device=x.device)
    gain = gain.contiguous()
    g32 = _gain32(gain)
    _lib.call("serq_rmsnorm_quant_mx_gather", x.data_ptr(), _dtype_id(x), M, K, x.stride(0), gain.data_ptr(),
              g32.data_ptr(), float(eps), _ptr(gather_idx), int(r) if gather_idx is not None else 0,
              out.codes.data_ptr(), out.sf.data_ptr(), _ptr(out.xs_codes if gather_idx is not None else None),
              _ptr(out.xs_sf if gather_idx is not None else None), _stream())
    return out


_G32: dict = {}
_G32_LOCK = threading.Lock()


def _gain32(gain: torch.Tensor) -> torch.Tensor:
    """The f32 rounding of an RMSNorm gain (a layer weight), converted once per tensor version."""
    key = id(gain)
    with _G32_LOCK:
        hit = _G32.get(key)
        if hit is not None and hit[0]() is gain and hit[1] == gain._version:
            return hit[2]
    g32 = gain.float()
    if torch.cuda.is_current_stream_capturing():
        return g32  # a captured conversion: its result only exists once the graph replays
    with _G32_LOCK:
        if len(_G32) >= 64:
            _G32.clear()
        _G32[key] = (weakref.ref(gain), gain._version, g32)
    return g32


def rmsnorm_quantize_int(x: torch.Tensor, gain: torch.Tensor, eps: float, bits: int, symmetric: bool,
                         salient_idx: torch.Tensor | None = None, r: int = 0, xs_kind: int = 0,
                         exact_f64: bool = False) -> IntActivation:
    """Producer fusion for the integer formats: quantize_*(rmsnorm(x, gain, eps)) per token in ONE
    kernel, bit-identical to the reference's float64 (saliency.py:194-196, quantcore.py:108-137;
    NumPy's pairwise row sum replayed): codes / scales / zero points.  ``exact_f64`` forces the
    all-f64 kernel (otherwise used only for rows it alone serves: K % 8 != 0, unaligned rows)."""
    _require_cuda(x, "x")
    if x.dim() != 2 or x.stride(1) != 1:
        raise ValidationError("x must be a row-major 2-D tensor")
    M, K = x.shape
    if gain.dtype != torch.float64 or gain.numel() != K or not gain.is_cuda:
        raise ValidationError("gain must be a float64 CUDA vector of length K")
    act = _int_activation(M, K, bits, symmetric, xs_kind, r, x.device)
    gain = gain.contiguous()
    g32 = _gain32(gain) if exact_f64 is False else None
    _lib.call("serq_rmsnorm_quant_int", x.data_ptr(), _dtype_id(x), M, K, x.stride(0), gain.data_ptr(), _ptr(g32),
              float(eps), bits, int(symmetric), act.codes.data_ptr(), act.scale64.data_ptr(), act.scale32.data_ptr(),
              _ptr(act.zp), _ptr(salient_idx), r, _ptr(act.xs), xs_kind, _stream())
    return act


def unpack_mx(codes: torch.Tensor, sf: torch.Tensor, rows: int, cols: int) -> tuple[torch.Tensor, torch.Tensor]:
    """Device layout -> reference artefact layout (uint8 codes [rows, cols], int32 exps [rows, cols/32])."""
    c = torch.empty((rows, cols), dtype=torch.uint8, device=codes.device)
    e = torch.empty((rows, cols // 32), dtype=torch.int32, device=codes.device)
    _lib.call("serq_unpack_mx", codes.data_ptr(), sf.data_ptr(), rows, cols, c.data_ptr(), e.data_ptr(), _stream())
    return c, e


def _int_activation(M: int, K: int, bits: int, symmetric: bool, xs_kind: int, r: int, dev) -> IntActivation:
    xs = None
    if xs_kind == 1:
        xs = torch.empty((M, r), dtype=torch.bfloat16, device=dev)
    elif xs_kind == 2:
        xs = torch.empty((M, r), dtype=torch.int8, device=dev)
    return IntActivation(torch.empty((M, K), dtype=torch.int8, device=dev), torch.empty(M, dtype=torch.float64, device=dev),
                         torch.empty(M, dtype=torch.float32, device=dev),
                         None if symmetric else torch.empty(M, dtype=torch.int32, device=dev), bits, symmetric, xs)


def quantize_int(x: torch.Tensor, bits: int, symmetric: bool, salient_idx: torch.Tensor | None = None, r: int = 0,
                 xs_kind: int = 0) -> IntActivation:
    """K1-INT per-token quantizer (quantcore.py:108-137), bit-exact codes/scales/zps.

    xs_kind 1: also emit the bf16 (codes - zp) salient slice for a dense R;
    xs_kind 2: emit the gathered int8 salient codes for a non-contiguous int R."""
    _require_cuda(x, "x")
    if x.dim() != 2 or x.stride(1) != 1:
        raise ValidationError("x must be a row-major 2-D tensor")
    M, K = x.shape
    dev = x.device
    codes = torch.empty((M, K), dtype=torch.int8, device=dev)
    s64 = torch.empty(M, dtype=torch.float64, device=dev)
    s32 = torch.empty(M, dtype=torch.float32, device=dev)
    zp = None if symmetric else torch.empty(M, dtype=torch.int32, device=dev)
    xs = None
    if xs_kind == 1:
        xs = torch.empty((M, r), dtype=torch.bfloat16, device=dev)
    elif xs_kind == 2:
        xs = torch.empty((M, r), dtype=torch.int8, device=dev)
    _lib.call("serq_act_quant_int", x.data_ptr(), _dtype_id(x), M, K, x.stride(0), bits, int(symmetric),
              codes.data_ptr(), s64.data_ptr(), s32.data_ptr(), _ptr(zp), _ptr(salient_idx), r, _ptr(xs),
              xs_kind, _stream())
    return IntActivation(codes, s64, s32, zp, bits, symmetric, xs)


def int_token_ranges(x: torch.Tensor) -> torch.Tensor:
    """Per-token (min, max) of a K-slice of the activations: float32 [2, M] (row 0 min, row 1
    max; exact for bf16 input) -- the local half of a K-sharded INT quantization."""
    _require_cuda(x, "x")
    if x.dim() != 2 or x.stride(1) != 1 or x.dtype != torch.bfloat16:
        raise ValidationError("x must be a row-major bf16 2-D tensor")
    M, K = x.shape
    rng = torch.empty((2, M), dtype=torch.float32, device=x.device)
    _lib.call("serq_act_quant_int_range", x.data_ptr(), _lib.SERQ_BF16, M, K, x.stride(0), rng.data_ptr(), _stream())
    return rng


def quantize_int_with_range(x: torch.Tensor, rng: torch.Tensor, bits: int, symmetric: bool,
                            salient_idx: torch.Tensor | None = None, r: int = 0, xs_kind: int = 0) -> IntActivation:
    """K1-INT on a K-slice with the GLOBAL per-token range ``rng`` ([2, M], all-reduced MIN /
    MAX over the slices, tp.int_token_range_allreduce): codes / scales / zero points of the
    unsharded row (quantcore.py:121-137)."""
    _require_cuda(x, "x")
    if x.dim() != 2 or x.stride(1) != 1 or x.dtype != torch.bfloat16:
        raise ValidationError("x must be a row-major bf16 2-D tensor")
    M, K = x.shape
    if rng.dtype != torch.float32 or tuple(rng.shape) != (2, M) or not rng.is_contiguous():
        raise ValidationError("range must be a contiguous float32 [2, M] tensor")
    act = _int_activation(M, K, bits, symmetric, xs_kind, r, x.device)
    _lib.call("serq_act_quant_int_ext", x.data_ptr(), _lib.SERQ_BF16, M, K, x.stride(0), bits, int(symmetric),
              rng.data_ptr(), act.codes.data_ptr(), act.scale64.data_ptr(), act.scale32.data_ptr(), _ptr(act.zp),
              _ptr(salient_idx), r, _ptr(act.xs), xs_kind, _stream())
    return act


# ---------------------------------------------------------------- weights


def _dev(a, dtype, device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dtype).contiguous()


class _Handle:
    def __init__(self, h: ctypes.c_void_p):
        self._h = h

    @property
    def ptr(self):
        return self._h

    def close(self):
        if self._h:
            _lib.load().serq_linear_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _check_host_io(x_host: torch.Tensor, y_host: torch.Tensor, K: int, N: int) -> None:
    """The *_host entry points copy M*K*2 bytes in and M*N*2 bytes out with raw cudaMemcpyAsync:
    the host tensors must be exactly bf16 [M, K] / [M, N], contiguous, on the host."""
    for t, name in ((x_host, "x_host"), (y_host, "y_host")):
        if not isinstance(t, torch.Tensor) or t.is_cuda:
            raise ValidationError(f"{name} must be a host tensor")
        if t.dtype != torch.bfloat16:
            raise ValidationError(f"{name} must be bfloat16, got {t.dtype}")
        if t.dim() != 2 or not t.is_contiguous():
            raise ValidationError(f"{name} must be a contiguous 2-D tensor")
    M = x_host.shape[0]
    if M <= 0:
        raise ValidationError("x must be non-empty")
    if tuple(x_host.shape) != (M, K):
        raise ValidationError(f"x_host must be [M, {K}], got {tuple(x_host.shape)}")
    if tuple(y_host.shape) != (M, N):
        raise ValidationError(f"y_host must be [{M}, {N}], got {tuple(y_host.shape)}")


class MxLinear:
    """Packed MXFP4 SERQ linear (main_t + comp.r_q of build_serq_rtn_mx,
    compensate.py:343-357) resident on one GPU."""

    def __init__(self, codes, exps, r_codes=None, r_exps=None, salient_idx=None, device="cuda"):
        device = torch.device(device)
        if device.type != "cuda":
            raise ValidationError("MxLinear lives on a CUDA device")
        with torch.cuda.device(device):
            self._init(codes, exps, r_codes, r_exps, salient_idx, device)

    def _init(self, codes, exps, r_codes, r_exps, salient_idx, device):
        codes = _dev(codes, torch.uint8, device)
        exps = _dev(exps, torch.int32, device)
        self.N, self.K = codes.shape
        self.r = 0 if r_codes is None else int(r_codes.shape[1])
        if self.r:
            rc = _dev(r_codes, torch.uint8, device)
            re = _dev(r_exps, torch.int32, device)
        else:
            rc = re = None
        if exps.shape != (self.N, self.K // 32):
            raise ValidationError(f"exps must be [N, K/32] = {(self.N, self.K // 32)}, got {tuple(exps.shape)}")
        if self.r and (r_codes.shape[0] != self.N or tuple(r_exps.shape) != (self.N, self.r // 32)):
            raise ValidationError("r_codes / r_exps must be [N, r] / [N, r/32]")
        idx = _check_salient_idx(salient_idx, self.r, self.K) if self.r else None
        self.contiguous = idx is None or np.array_equal(idx, np.arange(self.r))
        self.gather_idx = None if self.contiguous else torch.from_numpy(idx.astype(np.int32)).to(device)
        self.xs_cols = self.r  # columns of the quantizer's salient slice (128 per segment when fused)
        h = ctypes.c_void_p()
        _lib.call("serq_pack_mx", codes.data_ptr(), exps.data_ptr(), self.N, self.K, _ptr(rc), _ptr(re), self.r,
                  int(self.contiguous), ctypes.byref(h), _stream())
        torch.cuda.current_stream().synchronize()  # inputs may be temporaries
        self._h = _Handle(h)
        self.device = device

    def quantize(self, x: torch.Tensor, out: MxActivation | None = None) -> MxActivation:
        return quantize_mx(x, None if self.contiguous else self.gather_idx, out)

    def _activation(self, M: int, dev) -> MxActivation:
        cb, sb = mx_sizes(M, self.K)
        act = MxActivation(torch.empty(cb, dtype=torch.uint8, device=dev), torch.empty(sb, dtype=torch.uint8, device=dev),
                           M, self.K)
        if not self.contiguous:
            cbr, sbr = mx_sizes(M, self.xs_cols)
            act.xs_codes = torch.empty(cbr, dtype=torch.uint8, device=dev)
            act.xs_sf = torch.empty(sbr, dtype=torch.uint8, device=dev)
        return act

    def gemm(self, act: MxActivation, y: torch.Tensor | None = None) -> torch.Tensor:
        if act.K != self.K:
            raise ValidationError("x columns must equal weight input dim")
        if y is None:
            y = torch.empty((act.M, self.N), dtype=torch.bfloat16, device=self.device)
        _lib.call("serq_linear_mx", self._h.ptr, act.codes.data_ptr(), act.sf.data_ptr(), act.M, _ptr(act.xs_codes),
                  _ptr(act.xs_sf), y.data_ptr(), y.stride(0), _stream())
        return y

    def forward(self, x: torch.Tensor, act: MxActivation | None = None, y: torch.Tensor | None = None) -> torch.Tensor:
        """Quantize + linear in ONE C-ABI call (serq_forward_mx): the linear is launched with
        programmatic dependent launch behind the quantizer (M <= 8: the quantizer runs inside
        the decode kernel)."""
        _require_cuda(x, "x")
        if x.dim() != 2 or x.stride(1) != 1:
            raise ValidationError("x must be a row-major 2-D tensor")
        M, K = x.shape
        if K != self.K:
            raise ValidationError("x columns must equal weight input dim")
        if act is None:
            act = self._activation(M, x.device)
        if y is None:
            y = torch.empty((M, self.N), dtype=torch.bfloat16, device=self.device)
        _lib.call("serq_forward_mx", self._h.ptr, x.data_ptr(), _dtype_id(x), M, x.stride(0), _ptr(self.gather_idx),
                  act.codes.data_ptr(), act.sf.data_ptr(), _ptr(act.xs_codes), _ptr(act.xs_sf), y.data_ptr(),
                  y.stride(0), _stream())
        return y

    def __call__(self, x: torch.Tensor, y: torch.Tensor | None = None) -> torch.Tensor:
        return self.forward(x, None, y)

    def forward_rmsnorm(self, x: torch.Tensor, gain: torch.Tensor, eps: float = 1e-6,
                        act: MxActivation | None = None, y: torch.Tensor | None = None) -> torch.Tensor:
        """linear(rmsnorm(x, gain)) with the normalisation fused into the quantizer; for a
        non-contiguous salient set the same kernel also encodes the normalised slice x[:, idx]."""
        act = rmsnorm_quantize_mx(x, gain, eps, act, None if self.contiguous else self.gather_idx, self.r)
        return self.gemm(act, y)

    def forward_host(self, x_host: torch.Tensor, y_host: torch.Tensor) -> None:
        """End to end from (pinned) host bf16 memory through the C-ABI."""
        _check_host_io(x_host, y_host, self.K, self.N)
        with torch.cuda.device(self.device):
            _lib.call("serq_forward_mx_host_gather", self._h.ptr, x_host.data_ptr(), x_host.shape[0],
                      _ptr(self.gather_idx), y_host.data_ptr(), _stream())


class FusedMxLinear:
    """Several MX SERQ linears that read the same activation -- q/k/v, gate/up (SURVEY 7
    hard-part 6) -- packed as ONE handle over their row-concatenated weights, each keeping its
    own salient set (the reference plans them separately, toymodel.py:267-277; every one takes
    the gather fallback).  The quantizer runs once (its salient buffer holds 128 columns per
    part) and, with r = 64, for M <= 16 (and optionally M > 128 with 256-row-aligned parts) ONE
    kernel computes every part (serq_linear_set_segments); other token counts run per-part views
    of the same weights (serq_linear_view, no copy).  ``parts``: (codes [N_j, K], exps, r_codes
    [N_j, r], r_exps, salient_idx [r]) per linear, N_j a multiple of 128, equal K and r."""

    def __init__(self, parts, device="cuda", prefill_one_kernel: bool = False):
        """``prefill_one_kernel``: also run M > 128 as ONE CTA-pair launch over all parts (r = 64,
        256-row-aligned parts); off by default -- per-part launches measured faster in the
        Llama-2-7B block at M = 2048 (558 vs 597 us per block)."""
        device = torch.device(device)
        if not 1 <= len(parts) <= 4:
            raise ValidationError("fuse 1 to 4 linears")
        arrs = [[np.asarray(a.cpu() if isinstance(a, torch.Tensor) else a) for a in p[:4]] for p in parts]
        K = arrs[0][0].shape[1]
        r = arrs[0][2].shape[1]
        self.n_parts = [a[0].shape[0] for a in arrs]
        if any(a[0].shape[1] != K or a[2].shape[1] != r for a in arrs):
            raise ValidationError("fused linears need the same K and rank")
        if any(n % 128 for n in self.n_parts) or not 0 < r <= 128:
            raise ValidationError("fused linears need output dims that are multiples of 128 and 0 < r <= 128")
        idxs = [_check_salient_idx(p[4], r, K) for p in parts]
        pad = np.concatenate([np.concatenate([ix, np.full(128 - r, ix[0], np.int64)]) for ix in idxs])
        cat = [np.ascontiguousarray(np.concatenate([a[j] for a in arrs])) for j in range(4)]
        # any non-contiguous index set puts the packed handle in gather mode; the real list follows
        self.fused = MxLinear(cat[0], cat[1], cat[2], cat[3], np.arange(r)[::-1].copy(), device)
        self.fused.gather_idx = torch.from_numpy(pad.astype(np.int32)).to(device)
        self.fused.xs_cols = 128 * len(parts)
        rows = (ctypes.c_int64 * len(parts))(*self.n_parts)
        _lib.call("serq_linear_set_segments", self.fused._h.ptr, len(parts), rows)
        self.K, self.N, self.r, self.device = K, sum(self.n_parts), r, device
        self.bounds = np.concatenate([[0], np.cumsum(self.n_parts)]).tolist()
        self.views = []
        for j, ix in enumerate(idxs):
            h = ctypes.c_void_p()
            contiguous = bool(np.array_equal(ix, np.arange(r)))
            _lib.call("serq_linear_view", self.fused._h.ptr, self.bounds[j], self.n_parts[j], int(contiguous),
                      ctypes.byref(h))
            v = MxLinear.__new__(MxLinear)
            v._h, v.N, v.K, v.r, v.device, v.contiguous, v.xs_cols = _Handle(h), self.n_parts[j], K, r, device, contiguous, r
            v.gather_idx = None if contiguous else torch.from_numpy(ix.astype(np.int32)).to(device)
            v._parent = self.fused  # the weights belong to the fused handle
            self.views.append(v)
        aligned = all(b % 256 == 0 for b in self.bounds[1:-1])
        # one kernel: the decode kernel (M <= 16) and the CTA-pair kernel (M > 128) take the gathered
        # salient slice as 32-byte rows, i.e. r = 64
        self._one_kernel = lambda m: r == 64 and (m <= 16 or (prefill_one_kernel and m > 128 and aligned))

    def forward(self, x: torch.Tensor, y: torch.Tensor | None = None) -> torch.Tensor:
        """Y [M, sum N_j] (bf16): part j's output in columns [bounds[j], bounds[j+1])."""
        M = x.shape[0]
        if y is None:
            y = torch.empty((M, self.N), dtype=torch.bfloat16, device=self.device)
        if self._one_kernel(M):
            return self.fused.forward(x, None, y)
        for j, v in enumerate(self.views):
            v.forward(x, None, y[:, self.bounds[j]:self.bounds[j + 1]])
        return y

    __call__ = forward

    def forward_parts(self, x: torch.Tensor) -> list:
        """Each part's output as its own tensor: column views of one buffer when one kernel ran
        (small M), separate contiguous buffers from the per-part launches otherwise."""
        if self._one_kernel(x.shape[0]):
            return self.split(self.forward(x))
        return [v.forward(x) for v in self.views]

    def split(self, y: torch.Tensor) -> list:
        return [y[:, self.bounds[j]:self.bounds[j + 1]] for j in range(len(self.n_parts))]


class IntLinear:
    """Packed integer SERQ linear: INT weights with per-output-channel scales
    (QuantizedTensor with group_size == K, quantcore.py:59-80; ``scales`` [N])
    or group-wise along K (row groups of ``group_size`` a multiple of 128,
    gptq.py:98-146 / pipeline.py:134-137; ``scales`` [K/group_size, N]) plus the
    compensator R as bf16 (r_dense) or integer codes with one scale per
    output column (r_q, row groups of size r)."""

    def __init__(self, codes, scales, bits=4, r_dense=None, r_codes=None, r_scales=None, salient_idx=None,
                 device="cuda", group_size=None, r_split=False, weight_format="int8"):
        """``r_split``: consume the dense R as bf16 hi + lo planes (relative error 2^-17) instead
        of one bf16 plane -- for R matrices that carry a large share of the output (a GPTQ-swapped
        R holds the salient rows themselves); served by the group-wise kernel (K <= 8192).
        ``weight_format``: "int8" (weights int8 in HBM, TMA'd into the operand; the default) or
        "int4" (packed INT4 in HBM, 0.5 B / weight, widened in the SM; serq_pack_int4)."""
        if weight_format not in ("int8", "int4"):
            raise ValidationError(f"weight_format must be 'int8' or 'int4', got {weight_format!r}")
        self.weight_format = weight_format
        device = torch.device(device)
        if device.type != "cuda":
            raise ValidationError("IntLinear lives on a CUDA device")
        with torch.cuda.device(device):
            self._init(codes, scales, bits, r_dense, r_codes, r_scales, salient_idx, device, group_size, r_split)

    def _init(self, codes, scales, bits, r_dense, r_codes, r_scales, salient_idx, device, group_size, r_split):
        codes = _dev(codes, torch.int32, device)
        self.K, self.N = codes.shape
        scales = _dev(np.asarray(scales, dtype=np.float64) if not isinstance(scales, torch.Tensor) else scales,
                      torch.float64, device)
        self.group_size = self.K if group_size is None else int(group_size)
        if self.group_size <= 0 or self.K % self.group_size:
            raise ValidationError(f"group_size {self.group_size} does not divide K = {self.K}")
        if scales.numel() != (self.K // self.group_size) * self.N:
            raise ValidationError("integer main path needs scales [K/group_size, N] (one per output column and group)")
        scales = scales.reshape(-1).contiguous()
        if r_dense is not None:
            self.r_mode = _lib.SERQ_R_DENSE_SPLIT if r_split else _lib.SERQ_R_DENSE
            rd = _dev(r_dense, torch.float64, device)
            self.r = rd.shape[0]
            rdata, rs = rd, None
        elif r_codes is not None:
            self.r_mode = _lib.SERQ_R_INT
            rdata = _dev(r_codes, torch.int32, device)
            self.r = rdata.shape[0]
            rs = _dev(np.asarray(r_scales, dtype=np.float64).reshape(-1) if not isinstance(r_scales, torch.Tensor)
                      else r_scales.reshape(-1), torch.float64, device)
            if rs.numel() != self.N:
                raise ValidationError("integer R needs one scale per output column (row groups of size r)")
        else:
            self.r_mode, self.r, rdata, rs = _lib.SERQ_R_NONE, 0, None, None
        if self.r and rdata.shape[1] != self.N:
            raise ValidationError(f"R must be [r, N] with N = {self.N}")
        idx = _check_salient_idx(salient_idx, self.r, self.K) if self.r else None
        self.contiguous = idx is None or np.array_equal(idx, np.arange(self.r))
        self.salient_idx = None if idx is None or self.contiguous else torch.from_numpy(idx.astype(np.int32)).to(device)
        h = ctypes.c_void_p()
        if self.weight_format == "int4":
            if self.group_size != self.K or self.r_mode == _lib.SERQ_R_DENSE_SPLIT:
                raise ValidationError("packed INT4 weights need per-output-channel scales and a plain R")
            _lib.call("serq_pack_int4", codes.data_ptr(), scales.data_ptr(), self.K, self.N, bits, self.r_mode,
                      _ptr(rdata), _ptr(rs), self.r, int(self.contiguous), ctypes.byref(h), _stream())
        else:
            _lib.call("serq_pack_int_grouped", codes.data_ptr(), scales.data_ptr(), self.group_size, self.K, self.N,
                      bits, self.r_mode, _ptr(rdata), _ptr(rs), self.r, int(self.contiguous), ctypes.byref(h),
                      _stream())
        torch.cuda.current_stream().synchronize()
        self._h = _Handle(h)
        self.device = device

    def forward_rmsnorm(self, x: torch.Tensor, gain: torch.Tensor, eps: float, bits: int, symmetric: bool,
                        y: torch.Tensor | None = None) -> torch.Tensor:
        """linear(rmsnorm(x, gain)) with the normalisation fused into the per-token quantizer."""
        return self.gemm(rmsnorm_quantize_int(x, gain, eps, bits, symmetric, self.salient_idx, self.r,
                                              self.xs_kind()), y)

    def weight_bytes(self) -> tuple[int, bool]:
        """(bytes of the resident main weights, held as packed INT4?)"""
        b, w4 = ctypes.c_int64(), ctypes.c_int()
        _lib.call("serq_linear_weight_bytes", self._h.ptr, ctypes.byref(b), ctypes.byref(w4))
        return b.value, bool(w4.value)

    def xs_kind(self) -> int:
        if self.r_mode in (_lib.SERQ_R_DENSE, _lib.SERQ_R_DENSE_SPLIT):
            return 1
        if self.r_mode == _lib.SERQ_R_INT and not self.contiguous:
            return 2
        return 0

    def quantize(self, x: torch.Tensor, bits: int, symmetric: bool) -> IntActivation:
        return quantize_int(x, bits, symmetric, self.salient_idx, self.r, self.xs_kind())

    def gemm(self, act: IntActivation, y=None, acc_dump=None, accr_dump=None,
             addend: torch.Tensor | None = None) -> torch.Tensor:
        M, K = act.codes.shape
        if K != self.K:
            raise ValidationError("x columns must equal main rows")
        if y is None:
            y = torch.empty((M, self.N), dtype=torch.bfloat16, device=self.device)
        if addend is not None:
            if addend.dtype != torch.float32 or tuple(addend.shape) != (M, self.N) or not addend.is_contiguous():
                raise ValidationError("addend must be a contiguous float32 [M, N] tensor")
            _lib.call("serq_linear_int_addend", self._h.ptr, act.codes.data_ptr(), act.scale32.data_ptr(),
                      _ptr(act.zp), M, _ptr(act.xs), addend.data_ptr(), y.data_ptr(), y.stride(0), _stream())
            return y
        _lib.call("serq_linear_int", self._h.ptr, act.codes.data_ptr(), act.scale32.data_ptr(), _ptr(act.zp), M,
                  _ptr(act.xs), y.data_ptr(), y.stride(0), _ptr(acc_dump), _ptr(accr_dump), _stream())
        return y

    @staticmethod
    def dequantize(act: IntActivation) -> torch.Tensor:
        """x_hat = s * (codes - zp) in float32 (quantcore.py:144-150) on the device."""
        c = act.codes.view(torch.uint8).float() if not act.symmetric else act.codes.float()
        if act.zp is not None:
            c = c - act.zp.float()[:, None]
        return c * act.scale32[:, None]

    def forward(self, x: torch.Tensor, bits: int, symmetric: bool, act: IntActivation | None = None,
                y: torch.Tensor | None = None) -> torch.Tensor:
        """Quantize + linear in ONE C-ABI call (serq_forward_int, the int branch of
        forward_reconstructed, compensate.py:296-316); ``act`` (optional) receives the codes,
        scales and zero points."""
        _require_cuda(x, "x")
        if x.dim() != 2 or x.stride(1) != 1:
            raise ValidationError("x must be a row-major 2-D tensor")
        M, K = x.shape
        if K != self.K:
            raise ValidationError("x columns must equal main rows")
        if act is None:
            act = _int_activation(M, K, bits, symmetric, self.xs_kind(), self.r, x.device)
        if y is None:
            y = torch.empty((M, self.N), dtype=torch.bfloat16, device=self.device)
        _lib.call("serq_forward_int", self._h.ptr, x.data_ptr(), _dtype_id(x), M, x.stride(0), bits, int(symmetric),
                  _ptr(self.salient_idx), act.codes.data_ptr(), act.scale64.data_ptr(), act.scale32.data_ptr(),
                  _ptr(act.zp), _ptr(act.xs), y.data_ptr(), y.stride(0), _stream())
        return y

    def forward_host(self, x_host: torch.Tensor, y_host: torch.Tensor, bits: int, symmetric: bool) -> None:
        """End to end from (pinned) host bf16 memory through the C-ABI (serq_forward_int_host)."""
        _check_host_io(x_host, y_host, self.K, self.N)
        with torch.cuda.device(self.device):
            _lib.call("serq_forward_int_host", self._h.ptr, x_host.data_ptr(), x_host.shape[0], bits, int(symmetric),
                      _ptr(self.salient_idx), y_host.data_ptr(), _stream())

    def __call__(self, x: torch.Tensor, bits: int, symmetric: bool, y=None) -> torch.Tensor:
        return self.forward(x, bits, symmetric, None, y)



class SvdIntLinear:
    """The SVD baseline (build_svd_baseline, compensate.py:209-224; forward_reconstructed,
    compensate.py:304-310): Y = x_hat W + (x_hat L1) L2 with x_hat = s (codes - zp).

    B200 path: the quantizer also emits the exact bf16 (codes - zp) of every column, one plain
    bf16 GEMM (cuBLAS, fp32 accumulation) forms U = (codes - zp) L1 [M, r], and the fused INT
    kernel runs U L2 as its dense side term -- tcgen05 kind::f16 into the second TMEM
    accumulator, scaled by s in the epilogue -- so the second factor product and the add never
    leave the SM (no [M, N] fp32 correction in HBM).  L1 / L2 / U are bf16 (2^-9 relative on the
    correction term)."""

    def __init__(self, codes, scales, bits, l1, l2, device="cuda", group_size=None):
        l1 = np.asarray(l1, dtype=np.float64)
        l2 = np.asarray(l2, dtype=np.float64)
        K, r = l1.shape
        if l2.shape[0] != r:
            raise ValidationError("SVD factors must be L1 [K, r] and L2 [r, N]")
        rp = -(-r // 8) * 8  # dense R rows in multiples of 8 (zero factors add nothing)
        l1p = np.zeros((K, rp))
        l1p[:, :r] = l1
        l2p = np.zeros((rp, l2.shape[1]))
        l2p[:r] = l2
        self.K, self.r = K, rp
        self.lin = IntLinear(codes, scales, bits, r_dense=l2p, salient_idx=np.arange(rp), device=device,
                             group_size=group_size)
        self.N = self.lin.N
        self.l1 = torch.from_numpy(l1p).to(self.lin.device, torch.bfloat16)

    def quantize(self, x: torch.Tensor, bits: int, symmetric: bool) -> IntActivation:
        """Codes / scales / zero points and U = (codes - zp) L1 as the activation's side slice."""
        act = quantize_int(x, bits, symmetric, None, self.K, 1)  # xs: bf16 (codes - zp) of all K columns
        prev = torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction
        torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
        try:
            act.xs = (act.xs @ self.l1).contiguous()
        finally:
            torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = prev
        return act

    def forward(self, x: torch.Tensor, bits: int, symmetric: bool, y: torch.Tensor | None = None) -> torch.Tensor:
        return self.lin.gemm(self.quantize(x, bits, symmetric), y)

    __call__ = forward

class SvdMxLinear:
    """The SVD baseline over an MX main (_forward_mx, compensate.py:326-331):
    Y = mx_gemm_reference(x_mx, main_t) + (mx_decode(x_mx) L1) L2, any rank.

    B200 path: K1-MX encodes X; ``serq_mx_decode_bf16`` writes x_hat = mx_decode(x_mx) (exact in
    bf16); U = x_hat L1 and C = U L2 are two plain cuBLAS GEMMs (bf16 operands, fp32
    accumulation, U rounded to bf16 between them -- 2^-9 relative on the correction term, as in
    SvdIntLinear -- and C kept in fp32); the MX kernel adds C to its fp32 accumulator before the
    one bf16 rounding of Y (``serq_linear_mx_addend``: the CTA-pair kernel for M > 16).  A
    comparison baseline, not the SERQ hot path: the salient-term fusion of MxLinear does not
    apply, because the correction spans all K columns."""

    def __init__(self, codes, exps, l1, l2, device="cuda"):
        l1 = np.asarray(l1, dtype=np.float64)
        l2 = np.asarray(l2, dtype=np.float64)
        self.lin = MxLinear(codes, exps, device=device)
        self.K, self.N, self.device = self.lin.K, self.lin.N, self.lin.device
        if l1.ndim != 2 or l2.ndim != 2 or l1.shape[0] != self.K or l2.shape != (l1.shape[1], self.N):
            raise ValidationError("SVD factors must be L1 [K, r] and L2 [r, N]")
        self.r = l1.shape[1]
        self.l1 = torch.from_numpy(l1).to(self.device, torch.bfloat16)
        self.l2 = torch.from_numpy(l2).to(self.device, torch.bfloat16)

    def forward(self, x: torch.Tensor, y: torch.Tensor | None = None) -> torch.Tensor:
        _require_cuda(x, "x")
        if x.dim() != 2 or x.stride(1) != 1 or x.shape[1] != self.K:
            raise ValidationError("x must be a row-major [M, K] tensor")
        M = x.shape[0]
        act = self.lin.quantize(x)
        xhat = torch.empty((M, self.K), dtype=torch.bfloat16, device=self.device)
        _lib.call("serq_mx_decode_bf16", act.codes.data_ptr(), act.sf.data_ptr(), M, self.K, xhat.data_ptr(),
                  _stream())
        prev = torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction
        torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
        try:
            u = xhat @ self.l1
            c = torch.mm(u, self.l2, out_dtype=torch.float32)
        finally:
            torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = prev
        if y is None:
            y = torch.empty((M, self.N), dtype=torch.bfloat16, device=self.device)
        _lib.call("serq_linear_mx_addend", self.lin._h.ptr, act.codes.data_ptr(), act.sf.data_ptr(), M, c.data_ptr(),
                  y.data_ptr(), y.stride(0), _stream())
        return y

    __call__ = forward


class MxDenseRLinear:
    """An MX main with an UNQUANTIZED salient R (the reference's "test mode" r_dense,
    compensate.py:54, :338-339): Y = mx_gemm_reference(x_mx, main_t) + mx_decode(mx_encode(x[:, idx])) @ R.

    K1-MX encodes X and the gathered slice x[:, idx] in one launch; ``serq_mx_decode_bf16`` turns
    the slice's codes into its exact bf16 values; one cuBLAS GEMM forms C = x_s_hat @ R with R as
    bf16 hi + lo planes (relative 2^-17; the rows of R may carry a large share of Y) and fp32
    accumulation / output; the MX kernel adds C before Y's one bf16 rounding
    (``serq_linear_mx_addend``)."""

    def __init__(self, codes, exps, r_dense, salient_idx, device="cuda"):
        r_dense = np.asarray(r_dense, dtype=np.float64)
        self.lin = MxLinear(codes, exps, device=device)
        self.K, self.N, self.device = self.lin.K, self.lin.N, self.lin.device
        self.r = r_dense.shape[0]
        if r_dense.ndim != 2 or r_dense.shape[1] != self.N:
            raise ValidationError(f"r_dense must be [r, N] with N = {self.N}")
        if self.r % 32:
            raise ValidationError("MX residual path needs rank divisible by block size")
        idx = _check_salient_idx(salient_idx, self.r, self.K)
        self.gather_idx = torch.from_numpy(idx.astype(np.int32)).to(self.device)
        rt = torch.from_numpy(r_dense).to(self.device)
        hi = rt.to(torch.bfloat16)
        lo = (rt - hi.double()).to(torch.bfloat16)
        self.r_hilo = torch.cat([hi, lo], 0).contiguous()  # [2r, N]

    def forward(self, x: torch.Tensor, y: torch.Tensor | None = None) -> torch.Tensor:
        _require_cuda(x, "x")
        if x.dim() != 2 or x.stride(1) != 1 or x.shape[1] != self.K:
            raise ValidationError("x must be a row-major [M, K] tensor")
        M = x.shape[0]
        act = quantize_mx(x, self.gather_idx)
        xs = mx_decode_bf16(MxActivation(act.xs_codes, act.xs_sf, M, self.r))
        prev = torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction
        torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
        try:
            c = torch.mm(torch.cat([xs, xs], 1), self.r_hilo, out_dtype=torch.float32)
        finally:
            torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = prev
        if y is None:
            y = torch.empty((M, self.N), dtype=torch.bfloat16, device=self.device)
        _lib.call("serq_linear_mx_addend", self.lin._h.ptr, act.codes.data_ptr(), act.sf.data_ptr(), M, c.data_ptr(),
                  y.data_ptr(), y.stride(0), _stream())
        return y

    __call__ = forward


def mx_decode_bf16(act: MxActivation) -> torch.Tensor:
    """mx_decode (mxfmt.py:111-113) of a device MX activation, bf16 [M, K] (exact)."""
    out = torch.empty((act.M, act.K), dtype=torch.bfloat16, device=act.codes.device)
    _lib.call("serq_mx_decode_bf16", act.codes.data_ptr(), act.sf.data_ptr(), act.M, act.K, out.data_ptr(), _stream())
    return out


def device_info() -> dict:
    sm, ma, mi = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _lib.call("serq_device_info", ctypes.byref(sm), ctypes.byref(ma), ctypes.byref(mi))
    return {"sm_count": sm.value, "cc": (ma.value, mi.value)}


def last_launch_count() -> int:
    return int(_lib.load().serq_last_launch_count())


def last_kernel() -> str:
    """Name of the last kernel the C-ABI launched on this thread (which instantiation a
    configuration takes, e.g. ``serq_i8_pair_kernel<256>``)."""
    return _lib.load().serq_last_kernel().decode()
