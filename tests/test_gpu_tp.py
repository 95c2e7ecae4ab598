"""The pipelined tensor-parallel block on the GPU (one rank: every collective is still
issued through NCCL, so the stream / event / graph-capture path is the multi-GPU one).

Only one GPU is reachable here; the multi-rank sums are covered by the gloo tests in
test_tp.py and by the single-GPU shard emulation in test_gpu_parity.py."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist

    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    if dist.is_initialized():
        dist.destroy_process_group()


def _block(r=64):
    from paper_2603_08185_b200 import benchmarks as B, tp

    specs = tp.block_specs(1024, 2048, 256)
    lins = {s.name: B.device_mx_linear(s.k, s.n, r, seed=5 + i) for i, s in enumerate(specs)}
    return specs, lins


def test_pipelined_block_chunks_graph_and_nccl(nccl):
    from paper_2603_08185_b200 import benchmarks as B, tp

    specs, lins = _block()
    M = 1024
    x = B.outlier_x(M, 1024, seed=1)
    feeds = {"o_proj": B.outlier_x(M, 1024, seed=2), "down_proj": B.outlier_x(M, 2048, seed=3)}
    ref = tp.PipelinedTPBlock(specs, tp.DeviceBackend(lins), chunks=1).forward(x, feeds)
    ref = {k: v.clone() for k, v in ref.items()}
    be = tp.DeviceBackend(lins, force_collective=True)  # NCCL all-reduces on the comm stream
    blk = tp.PipelinedTPBlock(specs, be, chunks=4)
    out = blk.forward(x, feeds)
    torch.cuda.synchronize()
    for k in ref:  # row chunks take the same kernels: identical bits
        assert torch.equal(out[k], ref[k]), k
    assert be.launches_per_forward == 4 * 4 * 2  # quantizer + fused linear per linear and chunk
    g = B.graph_of(lambda: blk.forward(x, feeds))  # the whole step incl. NCCL in one graph
    for v in out.values():
        v.zero_()
    g.replay()
    torch.cuda.synchronize()
    for k in ref:
        assert torch.equal(out[k], ref[k]), k
