"""CPU checks of the C-ABI boundary: the library builds/loads and exports every
symbol include/serq_b200.h declares (no compute calls without a GPU)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "serq_b200.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(serq_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2603_08185_b200 import _lib, build

    build.build()
    return _lib.load()


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("serq_act_quant_mx", "serq_act_quant_int", "serq_pack_mx", "serq_pack_int", "serq_linear_mx",
                 "serq_linear_int", "serq_forward_mx_host", "serq_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2603_08185_b200 import _lib

    for name in _declared():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} missing from the ctypes signature table"


def test_version_and_sizes_without_gpu(lib):
    assert b"sm_100a" in lib.serq_version()
    cb, sb = ctypes.c_int64(), ctypes.c_int64()
    assert lib.serq_mx_sizes(4096, 4096, ctypes.byref(cb), ctypes.byref(sb)) == 0
    assert cb.value == 4096 * 2048
    assert sb.value == 32 * 32 * 512  # 128-row blocks x 128-col chunks x 512-B atoms
    # precondition failures return SERQ_EINVAL with a message, no GPU needed
    assert lib.serq_mx_sizes(4, 33, None, None) == 1
    assert b"32" in lib.serq_last_error()


def test_validation_errors_map_to_ValidationError(lib):
    from paper_2603_08185_b200 import _lib
    from paper_2603_08185_b200.errors import ValidationError

    with pytest.raises(ValidationError, match="divisible"):
        _lib.call("serq_act_quant_mx", None, 0, 4, 33, 33, None, None, None, 0, None, None, None)
    with pytest.raises(ValidationError, match="bits"):
        _lib.call("serq_act_quant_int", None, 0, 4, 32, 32, 9, 1, None, None, None, None, None, 0, None, 0, None)
    h = ctypes.c_void_p()
    with pytest.raises(ValidationError, match="rank divisible"):
        _lib.call("serq_pack_mx", None, None, 64, 64, None, None, 20, 1, ctypes.byref(h), None)


def test_sass_contains_tcgen05_and_tma(lib):
    import shutil
    import subprocess

    from paper_2603_08185_b200 import build

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([exe, "-sass", build.OUT], capture_output=True, text=True).stdout
    for mnem in ("UTCOMMA", "UTCIMMA", "UTCHMMA", "UTCCP", "UTMALDG", "UTMASTG", "LDTM"):
        assert mnem in sass, mnem
