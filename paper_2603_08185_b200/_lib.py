"""ctypes binding of the C-ABI library ``libserq_b200.so`` (include/serq_b200.h).

There is no fallback: if the library is missing or fails to load, every
product entry point raises.  Status codes map to ``ValidationError``
(SERQ_EINVAL) or ``RuntimeError`` (SERQ_ECUDA), mirroring the reference's
error convention (``_validation.py:14-15``).
"""

from __future__ import annotations

import ctypes
import os

from .errors import ValidationError

LIB_NAME = "libserq_b200.so"
# SERQ_B200_LIB: load another build of the same library (A/B timing of compile-time variants)
LIB_PATH = os.environ.get("SERQ_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

SERQ_OK, SERQ_EINVAL, SERQ_ECUDA = 0, 1, 2
SERQ_BF16, SERQ_F32, SERQ_F64 = 0, 1, 2
SERQ_R_NONE, SERQ_R_DENSE, SERQ_R_INT, SERQ_R_DENSE_SPLIT = 0, 1, 2, 3

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int

# name -> (restype, argtypes); every symbol declared in include/serq_b200.h
SIGNATURES = {
    "serq_last_error": (ctypes.c_char_p, []),
    "serq_version": (ctypes.c_char_p, []),
    "serq_device_info": (_I, [_P, _P, _P]),
    "serq_mx_sizes": (_I, [_I64, _I64, _P, _P]),
    "serq_act_quant_mx": (_I, [_P, _I, _I64, _I64, _I64, _P, _P, _P, _I, _P, _P, _P]),
    "serq_act_quant_int": (_I, [_P, _I, _I64, _I64, _I64, _I, _I, _P, _P, _P, _P, _P, _I, _P, _I, _P]),
    "serq_act_quant_int_range": (_I, [_P, _I, _I64, _I64, _I64, _P, _P]),
    "serq_act_quant_int_ext": (_I, [_P, _I, _I64, _I64, _I64, _I, _I, _P, _P, _P, _P, _P, _P, _I, _P, _I, _P]),
    "serq_pack_mx": (_I, [_P, _P, _I64, _I64, _P, _P, _I, _I, _P, _P]),
    "serq_unpack_mx": (_I, [_P, _P, _I64, _I64, _P, _P, _P]),
    "serq_mx_decode_bf16": (_I, [_P, _P, _I64, _I64, _P, _P]),
    "serq_linear_mx_addend": (_I, [_P, _P, _P, _I64, _P, _P, _I64, _P]),
    "serq_block_add_rmsnorm": (_I, [_P, _P, _I64, _I64, _I64, _P, ctypes.c_float, _P, _P, _P]),
    "serq_block_silu_mul": (_I, [_P, _I64, _P, _I64, _I64, _I64, _P, _P]),
    "serq_block_attention": (_I, [_P, _I64, _P, _I64, _P, _I64, _I64, _I64, _I64, ctypes.c_float, _P, _I64, _P]),
    "serq_rmsnorm_quant_int": (_I, [_P, _I, _I64, _I64, _I64, _P, _P, ctypes.c_double, _I, _I, _P, _P, _P, _P, _P, _I,
                                    _P, _I, _P]),
    "serq_mx_container_decode": (_I, [_P, _I64, _I64, _P, _P, _P]),
    "serq_rmsnorm_quant_mx": (_I, [_P, _I, _I64, _I64, _I64, _P, _P, ctypes.c_double, _P, _P, _P]),
    "serq_rmsnorm_quant_mx_gather": (_I, [_P, _I, _I64, _I64, _I64, _P, _P, ctypes.c_double, _P, _I, _P, _P, _P, _P,
                                          _P]),
    "serq_pack_int": (_I, [_P, _P, _I64, _I64, _I, _I, _P, _P, _I, _I, _P, _P]),
    "serq_pack_int4": (_I, [_P, _P, _I64, _I64, _I, _I, _P, _P, _I, _I, _P, _P]),
    "serq_pack_int_grouped": (_I, [_P, _P, _I64, _I64, _I64, _I, _I, _P, _P, _I, _I, _P, _P]),
    "serq_linear_destroy": (_I, [_P]),
    "serq_linear_set_segments": (_I, [_P, _I, _P]),
    "serq_linear_view": (_I, [_P, _I64, _I64, _I, _P]),
    "serq_linear_info": (_I, [_P, _P, _P, _P, _P, _P]),
    "serq_linear_weight_bytes": (_I, [_P, _P, _P]),
    "serq_linear_mx": (_I, [_P, _P, _P, _I64, _P, _P, _P, _I64, _P]),
    "serq_linear_int": (_I, [_P, _P, _P, _P, _I64, _P, _P, _I64, _P, _P, _P]),
    "serq_linear_int_addend": (_I, [_P, _P, _P, _P, _I64, _P, _P, _P, _I64, _P]),
    "serq_forward_mx": (_I, [_P, _P, _I, _I64, _I64, _P, _P, _P, _P, _P, _P, _I64, _P]),
    "serq_forward_mx_host_gather": (_I, [_P, _P, _I64, _P, _P, _P]),
    "serq_forward_mx_host": (_I, [_P, _P, _I64, _P, _P]),
    "serq_forward_int": (_I, [_P, _P, _I, _I64, _I64, _I, _I, _P, _P, _P, _P, _P, _P, _P, _I64, _P]),
    "serq_forward_int_host": (_I, [_P, _P, _I64, _I, _I, _P, _P, _P]),
    "serq_last_launch_count": (_I, []),
    "serq_last_kernel": (ctypes.c_char_p, []),
    "serq_set_debug_flags": (_I, [_I]),
    "serq_set_debug_timestamps": (_I, [_P]),
}

_lib = None


def load(path: str | None = None) -> ctypes.CDLL:
    """Load (once) and type the C-ABI library; raise loudly if it is absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError(
            f"{p} not found: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = ctypes.CDLL(p)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == SERQ_OK:
        return
    msg = load().serq_last_error().decode(errors="replace")
    if rc == SERQ_EINVAL:
        raise ValidationError(msg)
    raise RuntimeError(f"serq CUDA error: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))
