"""Offline artefacts on disk -> resident device linears.

Reads the reference's bundle directory (``bundle.json`` + ``.npy`` sections +
packed MX containers; writer: bundleio.py:73-126, reader: bundleio.py:129-172)
and builds one :class:`api.SerqLinear` per linear without ever materialising
the MX tensors on the host: each container's 17-byte block records are copied
to the GPU as raw bytes and decoded there (``serq_mx_container_decode``, the
replacement for load_mx's per-block Python loop, mxfmt.py:254-280), then
packed into the device layout (``serq_pack_mx``).  Integer sections are
``.npy`` arrays exactly as the reference writes them.

The result drops into the reference's block path through ``linear_fn``
(saliency.py:256-257; toymodel.forward_quantized, toymodel.py:363-374).
"""

from __future__ import annotations

import json
import os
import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from . import api
from .errors import ValidationError

MAGIC_MX = b"SERQMXB0" + b"\x00" * 8  # mxfmt.py:31
_HEADER = len(MAGIC_MX) + 12  # magic, <III rows, cols, block_size


def read_mx_container(path: str) -> tuple[int, int, int, np.ndarray]:
    """Header check and raw body of a packed MX file (mxfmt.py:254-268)."""
    raw = np.fromfile(path, dtype=np.uint8)
    if raw.size < _HEADER or raw[: len(MAGIC_MX)].tobytes() != MAGIC_MX:
        raise ValidationError(f"{path}: bad magic, not an MX file")
    rows, cols, bs = struct.unpack_from("<III", raw[len(MAGIC_MX):_HEADER].tobytes())
    if bs <= 0 or cols % bs:
        raise ValidationError(f"{path}: cols {cols} not divisible by block size {bs}")
    per_block = 1 + bs // 2
    if raw.size != _HEADER + rows * (cols // bs) * per_block:
        raise ValidationError(f"{path}: payload length mismatch")
    return rows, cols, bs, raw[_HEADER:]


def load_mx_device(path: str, device="cuda") -> api.MxBlockTensor:
    """A packed MX file as an MxBlockTensor whose codes [rows, cols] (uint8) and
    exponents [rows, cols/32] (int32) live on the device."""
    rows, cols, bs, body = read_mx_container(path)
    if bs != 32:
        raise ValidationError(f"{path}: the device MX format uses 32-element blocks, file has {bs}")
    dev = torch.device(device)
    body_d = torch.from_numpy(body).to(dev)
    codes = torch.empty((rows, cols), dtype=torch.uint8, device=dev)
    exps = torch.empty((rows, cols // 32), dtype=torch.int32, device=dev)
    _lib.call("serq_mx_container_decode", body_d.data_ptr(), rows, cols, codes.data_ptr(), exps.data_ptr(),
              torch.cuda.current_stream(dev).cuda_stream)
    return api.MxBlockTensor(codes, exps, 32, (rows, cols))


def _npy(dirpath, fname, dtype):
    return np.load(os.path.join(dirpath, fname)).astype(dtype)


def _qt(dirpath, rec) -> api.QuantizedTensor:
    zps = _npy(dirpath, rec["zero_points"], np.int32) if "zero_points" in rec else None
    return api.QuantizedTensor(_npy(dirpath, rec["codes"], np.int32), _npy(dirpath, rec["scales"], np.float64), zps,
                               api.IntQuantConfig(**rec["config"]), tuple(rec["shape"]))


@dataclass
class DeviceLinear:
    main: object
    comp: api.Compensator | None
    act_cfg: api.IntQuantConfig | None
    linear: api.SerqLinear | None  # None: unquantized passthrough section


@dataclass
class DeviceBundle:
    """``QuantizedBlockBundle`` (toymodel.py:192-201) with resident linears."""

    linears: dict = field(default_factory=dict)
    nl_weights: dict = field(default_factory=dict)
    source_hash: int = 0
    rank: int = 0
    fmt: str = "int"

    def linear_fn(self):
        """``linear_fn(name, x)`` for graph_forward: float64 in / float64 out, like
        the reference's quantized linears."""

        def fn(name, xin):
            dl = self.linears[name]
            x = api._as_matrix(xin)
            y = dl.linear(api._to_gpu(x))
            return y.float().cpu().numpy().astype(np.float64)

        return fn


def load_bundle_device(dirpath: str, device="cuda") -> DeviceBundle:
    """Mirror of bundleio.load_bundle (bundleio.py:129-172) that returns
    device-resident SERQ linears; raises ValidationError on the same
    malformed inputs (missing sections, bad MX magic or length)."""
    with open(os.path.join(dirpath, "bundle.json")) as f:
        doc = json.load(f)
    gains = {name: _npy(dirpath, fname, np.float64) for name, fname in doc.get("gains", {}).items()}
    out = DeviceBundle(nl_weights=gains, source_hash=int(doc.get("source_hash", 0)), rank=int(doc.get("rank", 0)),
                       fmt=doc.get("fmt", "int"))
    for name, rec in doc.get("linears", {}).items():
        mrec = rec["main"]
        main = load_mx_device(os.path.join(dirpath, mrec["file"]), device) if mrec["kind"] == "mx" else _qt(dirpath, mrec)
        act_cfg = api.IntQuantConfig(**rec["act_cfg"]) if rec.get("act_cfg") else None
        comp = None
        crec = rec.get("comp")
        if crec:
            kw = {}
            if "salient_idx" in crec:
                kw["salient_idx"] = _npy(dirpath, crec["salient_idx"], np.intp)
            if "l1" in crec:
                kw["l1"] = _npy(dirpath, crec["l1"], np.float64)
                kw["l2"] = _npy(dirpath, crec["l2"], np.float64)
            elif "r_mx" in crec:
                kw["r_q"] = load_mx_device(os.path.join(dirpath, crec["r_mx"]["file"]), device)
            elif "r_q" in crec:
                kw["r_q"] = _qt(dirpath, crec["r_q"])
            elif "r_dense" in crec:
                kw["r_dense"] = _npy(dirpath, crec["r_dense"], np.float64)
            comp = api.Compensator(mode=crec["mode"], rank=int(crec["rank"]), **kw)
        out.linears[name] = DeviceLinear(main, comp, act_cfg, api.SerqLinear(main, comp, act_cfg, device=device))
    if not out.linears:
        raise ValidationError(f"{dirpath}: bundle has no linear sections")
    return out
