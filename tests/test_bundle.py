"""Bundle directory (written by the reference's save_bundle, tests/golden/bundle)
-> device-resident linears (paper_2603_08185_b200.bundle)."""

import os
import shutil

import numpy as np
import pytest

from oracle import serq_oracle as O
from paper_2603_08185_b200 import bundle as BD
from paper_2603_08185_b200.errors import ValidationError

HERE = os.path.dirname(os.path.abspath(__file__))
BUNDLE = os.path.join(HERE, "golden", "bundle")
TOL_MAX, TOL_MEAN = 1e-2, 1e-3


def test_container_header_and_length_checks(tmp_path):
    rows, cols, bs, body = BD.read_mx_container(os.path.join(BUNDLE, "up_proj.main.mx"))
    assert (rows, cols, bs) == (128, 256, 32) and body.size == rows * (cols // bs) * 17
    bad = tmp_path / "bad.mx"
    raw = open(os.path.join(BUNDLE, "up_proj.main.mx"), "rb").read()
    bad.write_bytes(b"X" + raw[1:])
    with pytest.raises(ValidationError, match="magic"):
        BD.read_mx_container(str(bad))
    bad.write_bytes(raw[:-1])
    with pytest.raises(ValidationError, match="length"):
        BD.read_mx_container(str(bad))


def test_oracle_container_bytes_match_reference_file(golden):
    # the oracle's restatement of save_mx (mxfmt.py:228-251) reproduces the reference-written file
    t = O.MxT(golden["bundle_up_codes"], golden["bundle_up_exps"], 32, golden["bundle_up_codes"].shape)
    assert O.pack_mx_file_bytes(t) == open(os.path.join(BUNDLE, "up_proj.main.mx"), "rb").read()


def test_empty_bundle_rejected(tmp_path):
    d = tmp_path / "b"
    d.mkdir()
    (d / "bundle.json").write_text('{"linears": {}, "gains": {}}')
    with pytest.raises(ValidationError, match="no linear"):
        BD.load_bundle_device(str(d), device="cpu")


@pytest.mark.gpu
def test_device_bundle_matches_reference(golden):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_08185_b200 import device as D

    b = BD.load_bundle_device(BUNDLE)
    assert set(b.linears) == {"up_proj", "down_proj", "o_proj"} and b.rank == 32
    np.testing.assert_array_equal(b.nl_weights["ln1"], np.load(os.path.join(BUNDLE, "gain.ln1.npy")))
    # MX sections decoded on the device equal the reference's load_mx tensors bit for bit
    up = b.linears["up_proj"]
    assert np.array_equal(up.main.element_codes.cpu().numpy(), golden["bundle_up_codes"])
    assert np.array_equal(up.main.block_scale_exponents.cpu().numpy(), golden["bundle_up_exps"])
    assert np.array_equal(up.comp.r_q.element_codes.cpu().numpy(), golden["bundle_up_rcodes"])
    assert np.array_equal(up.comp.r_q.block_scale_exponents.cpu().numpy(), golden["bundle_up_rexps"])
    # every section's forward vs the reference's forward_reconstructed on the same input
    fn = b.linear_fn()
    for name in ("up_proj", "down_proj", "o_proj"):
        y = fn(name, golden["bundle_x"])
        mx, mean = O.parity_errors(y, golden[f"bundle_y_{name}"])
        assert mx <= TOL_MAX and mean <= TOL_MEAN, (name, mx, mean)
    assert D is not None
