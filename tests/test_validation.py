"""Host-side validation and the drop-in's artefact cache (no GPU needed).

The kernels read salient indices and host buffers through raw pointers, so the
Python mirror rejects what the reference would reject (compensate.py:296-311 raises
on shape / index errors) before anything reaches the C-ABI."""

import gc

import numpy as np
import pytest
import torch

from paper_2603_08185_b200 import api
from paper_2603_08185_b200 import device as D
from paper_2603_08185_b200.errors import ValidationError


@pytest.mark.parametrize("idx,msg", [
    (np.arange(31), "rank"),
    (np.arange(32).reshape(4, 8), "1-D"),
    (np.r_[np.arange(31), 4096], "range"),
    (np.r_[np.arange(31), -1], "range"),
    (np.r_[np.arange(31), 3], "repeats"),
    (np.linspace(0, 1, 32), "integers"),
])
def test_salient_idx_rejected(idx, msg):
    with pytest.raises(ValidationError, match=msg):
        D._check_salient_idx(idx, 32, 4096)


def test_salient_idx_accepted():
    idx = np.random.default_rng(0).permutation(4096)[:64]
    assert np.array_equal(D._check_salient_idx(idx, 64, 4096), idx)
    assert np.array_equal(D._check_salient_idx(torch.arange(32), 32, 64), np.arange(32))


def test_host_io_checked():
    K, N, M = 64, 32, 8
    x = torch.zeros((M, K), dtype=torch.bfloat16)
    y = torch.zeros((M, N), dtype=torch.bfloat16)
    D._check_host_io(x, y, K, N)
    with pytest.raises(ValidationError, match="bfloat16"):
        D._check_host_io(x.float(), y, K, N)
    with pytest.raises(ValidationError, match="y_host"):
        D._check_host_io(x, y[:4], K, N)
    with pytest.raises(ValidationError, match="x_host"):
        D._check_host_io(x[:, :32].contiguous(), y, K, N)
    with pytest.raises(ValidationError, match="contiguous"):
        D._check_host_io(torch.zeros((K, M), dtype=torch.bfloat16).t(), y, K, N)
    with pytest.raises(ValidationError, match="non-empty"):
        D._check_host_io(x[:0], y[:0], K, N)


class _Art:
    """Stands in for a reference artefact dataclass (weak-referenceable)."""


class _FakeLinear:
    built = 0

    def __init__(self, main, comp, act_cfg, allow_symmetric_act=False):
        _FakeLinear.built += 1


def test_cache_reuses_and_releases(monkeypatch):
    monkeypatch.setattr(api, "SerqLinear", _FakeLinear)
    api.clear_cache()
    main, comp = _Art(), _Art()
    a = api._linear_for(main, comp, None)
    assert api._linear_for(main, comp, None) is a  # packed once per artefact pair
    assert len(api._CACHE) == 1
    del main
    gc.collect()
    assert len(api._CACHE) == 0  # the device weights go with the artefact


def test_cache_is_bounded(monkeypatch):
    monkeypatch.setattr(api, "SerqLinear", _FakeLinear)
    api.clear_cache()
    keep = [(_Art(), _Art()) for _ in range(api.CACHE_MAX + 10)]
    for m, c in keep:
        api._linear_for(m, c, None)
    assert len(api._CACHE) == api.CACHE_MAX
    api.clear_cache()
