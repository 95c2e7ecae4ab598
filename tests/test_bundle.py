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


@pytest.mark.gpu
def test_device_block_matches_forward_quantized(golden):
    # a whole toy decoder block quantized by the reference (quantize_block, MXFP4, r=32; gather
    # fallback on every linear) and saved with save_bundle, run on the device.  The device
    # linears store bf16 (the BASELINE output contract); the block's attention turns a 2^-9
    # change of q or k into an e^(2^-9 |logit|) change of its weights (the outlier channels give
    # |logits| in the hundreds), so the bit-level reference for the device block is the
    # reference's forward_quantized with every linear output rounded to bf16 (the oracle
    # restatement, pinned to the reference above): 1e-2 max / 1e-3 mean of |y|.
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_08185_b200.block import DeviceBlock

    bdir = os.path.join(HERE, "golden", "block_mx")
    hd = int(golden["block_head_dim"])
    b = BD.load_bundle_device(bdir)
    blk = DeviceBlock.from_bundle(b, hd)
    x = torch.from_numpy(golden["block_x"]).to("cuda", torch.float32)
    y = blk(x).double().cpu().numpy()
    lins, gains = _oracle_block_linears(bdir)
    ref = O.forward_block_mx(golden["block_x"], lins, gains, hd, bf16_linear_out=True)
    err = np.abs(y - ref)
    assert err.max() <= 1e-2 * np.abs(ref).max() and err.mean() <= 1e-3 * np.abs(ref).mean(), (
        err.max() / np.abs(ref).max(), err.mean() / np.abs(ref).mean())
    # the CUDA-graph replay reproduces the eager forward exactly
    xs = x.clone()
    replay, out = blk.graphed(xs)
    replay()
    torch.cuda.synchronize()
    assert np.array_equal(out.double().cpu().numpy(), y)


def _oracle_block_linears(b_dir):
    # the bundle's MX sections through the oracle's container reader (host, for the oracle only)
    import json

    doc = json.load(open(os.path.join(b_dir, "bundle.json")))
    out = {}
    for name, rec in doc["linears"].items():
        def mx(fname):
            rows, cols, bs, body = BD.read_mx_container(os.path.join(b_dir, fname))
            recs = body.reshape(rows, cols // bs, 1 + bs // 2)
            exps = recs[:, :, 0].astype(np.int32) - 127
            nib = recs[:, :, 1:]
            codes = np.empty((rows, cols // bs, bs), np.uint8)
            codes[:, :, 0::2] = nib & 0xF
            codes[:, :, 1::2] = nib >> 4
            return O.MxT(codes.reshape(rows, cols), exps, bs, (rows, cols))

        main = mx(rec["main"]["file"])
        c = rec["comp"]
        comp = O.Comp(int(c["rank"]), np.load(os.path.join(b_dir, c["salient_idx"])), r_q=mx(c["r_mx"]["file"]))
        out[name] = (main, comp)
    gains = {k: np.load(os.path.join(b_dir, f)) for k, f in doc["gains"].items()}
    return out, gains


def test_oracle_block_matches_reference_forward_quantized(golden):
    # the oracle's restatement of forward_quantized on the reference-written block bundle
    lins, gains = _oracle_block_linears(os.path.join(HERE, "golden", "block_mx"))
    y = O.forward_block_mx(golden["block_x"], lins, gains, int(golden["block_head_dim"]))
    np.testing.assert_allclose(y, golden["block_y_quant"], rtol=1e-12, atol=1e-12)
