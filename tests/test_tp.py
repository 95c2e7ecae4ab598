"""Tensor-parallel host logic on CPU: gloo, world_size 2.

The per-rank linear here is the ORACLE (test-only); on the GPU the same
driver runs the sm_100a kernels over NCCL.  What is checked: shard plans,
that K-sharded SERQ MX layers with per-rank salient shares sum (one
all-reduce) to the single-device reference on the union salient set, that
N-sharded layers concatenate to it, and that the block driver reduces only
after o_proj / down_proj.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from oracle import serq_oracle as O  # noqa: E402
from paper_2603_08185_b200 import tp  # noqa: E402
from paper_2603_08185_b200.errors import ValidationError  # noqa: E402

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(fn, *args):
    port = _free_port()
    mp.spawn(_entry, args=(fn, port, args), nprocs=WORLD, join=True)


def _entry(rank, fn, port, args):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        fn(rank, *args)
    finally:
        dist.destroy_process_group()


# ------------------------------------------------------------------ plans


def test_shard_plans_cover_and_align():
    for n, world in [(4096, 8), (1024, 8), (11008, 4), (28672, 8), (96, 2)]:
        spans = [tp.column_shard(n, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert all((b - a) % 8 == 0 for a, b in spans)
    spans = [tp.row_shard(28672, 8, r) for r in range(8)]
    assert all((b - a) % 32 == 0 and b - a == 3584 for a, b in spans)
    with pytest.raises(ValidationError):
        tp.row_shard(100, 2, 0)
    assert tp.salient_per_rank(128, 8) == 32 and tp.salient_per_rank(64, 2) == 32


def test_row_parallel_salient_layout():
    scores = np.random.default_rng(0).random(256)
    perm, idx = tp.row_parallel_salient_layout(scores, 2, 32)
    assert sorted(perm.tolist()) == list(range(256))
    for rank in range(2):
        k0, k1 = tp.row_shard(256, 2, rank)
        local = perm[k0:k1]
        assert (local >= k0).all() and (local < k1).all()  # permutation stays inside the slice
        top = np.argsort(-scores[k0:k1], kind="stable")[:32] + k0
        assert np.array_equal(local[:32], top)


# ------------------------------------------------------------------ row parallel (one all-reduce)


def _row_parallel_worker(rank, k, n, m, r_rank, seed):
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((k, n)) * 0.02
    x = O.bf16_round(O.synthetic_activations(m, k, 4, 50.0, seed + 1))
    scores = np.abs(w).max(axis=1)
    perm, _ = tp.row_parallel_salient_layout(scores, WORLD, r_rank)
    wp, xp = w[perm], x[:, perm]
    k0, k1 = tp.row_shard(k, WORLD, rank)
    main_t, comp = O.build_serq_rtn_mx(wp[k0:k1], np.arange(r_rank), 32)
    y_local = O.forward_mx(np.ascontiguousarray(xp[:, k0:k1]), main_t, comp)
    t = torch.from_numpy(y_local)
    tp.allreduce_sum_(t)
    # single-device reference on the union salient set
    union = np.concatenate([tp.row_shard(k, WORLD, rk)[0] + np.arange(r_rank) for rk in range(WORLD)])
    main_g, comp_g = O.build_serq_rtn_mx(wp, union, 32)
    y_ref = O.forward_mx(xp, main_g, comp_g)
    assert np.abs(t.numpy() - y_ref).max() <= 1e-9 * np.abs(y_ref).max()


def test_row_parallel_mx_sum_equals_single_device():
    _spawn(_row_parallel_worker, 256, 64, 16, 32, 3)


# ------------------------------------------------------------------ column parallel (no exchange)


def _column_parallel_worker(rank, k, n, m, r, seed):
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((k, n)) * 0.02
    x = O.bf16_round(O.synthetic_activations(m, k, 3, 50.0, seed + 1))
    main_t, comp = O.build_serq_rtn_mx(w, np.arange(r), 32)
    n0, n1 = tp.column_shard(n, WORLD, rank)
    c, e, rc, re_ = tp.shard_columns_mx(main_t.element_codes, main_t.block_scale_exponents, comp.r_q.element_codes,
                                        comp.r_q.block_scale_exponents, n0, n1)
    main_s = O.MxT(c, e, 32, c.shape)
    comp_s = O.Comp(r, np.arange(r), r_q=O.MxT(rc, re_, 32, rc.shape))
    y_local = torch.from_numpy(np.ascontiguousarray(O.forward_mx(x, main_s, comp_s)))
    parts = [torch.zeros_like(y_local) for _ in range(WORLD)]
    dist.all_gather(parts, y_local)
    y = torch.cat(parts, dim=1).numpy()
    assert np.array_equal(y, O.forward_mx(x, main_t, comp))


def test_column_parallel_mx_concat_equals_single_device():
    _spawn(_column_parallel_worker, 128, 96, 8, 32, 5)


# ------------------------------------------------------------------ block driver


def _block_worker(rank, hidden, ffn, kv, m):
    specs = tp.block_specs(hidden, ffn, kv)
    rng = np.random.default_rng(11)
    weights = {s.name: rng.standard_normal((s.k, s.n)) for s in specs}
    calls = []

    def make(spec):
        w = weights[spec.name]
        if spec.kind == "column":
            n0, n1 = tp.column_shard(spec.n, WORLD, rank)
            return lambda x: (calls.append(spec.name), torch.from_numpy(x.numpy() @ w[:, n0:n1]))[1]
        k0, k1 = tp.row_shard(spec.k, WORLD, rank)
        return lambda x: (calls.append(spec.name), torch.from_numpy(x.numpy() @ w[k0:k1]))[1]

    drv = tp.TPBlockLinears(specs, {s.name: make(s) for s in specs}, WORLD, rank)
    x = torch.from_numpy(np.random.default_rng(12).standard_normal((m, hidden)))
    attn = np.random.default_rng(13).standard_normal((m, hidden))
    act = np.random.default_rng(14).standard_normal((m, ffn))
    k0, k1 = tp.row_shard(hidden, WORLD, rank)
    f0, f1 = tp.row_shard(ffn, WORLD, rank)
    out = drv.forward(x, feeds={"o_proj": torch.from_numpy(attn[:, k0:k1]),
                                "down_proj": torch.from_numpy(act[:, f0:f1])})
    assert calls == ["qkv_proj", "o_proj", "gate_up_proj", "down_proj"]
    np.testing.assert_allclose(out["o_proj"].numpy(), attn @ weights["o_proj"], rtol=1e-10, atol=1e-9)
    np.testing.assert_allclose(out["down_proj"].numpy(), act @ weights["down_proj"], rtol=1e-10, atol=1e-9)
    n0, n1 = tp.column_shard(specs[0].n, WORLD, rank)
    np.testing.assert_allclose(out["qkv_proj"].numpy(), x.numpy() @ weights["qkv_proj"][:, n0:n1], rtol=1e-12)


def test_block_driver_reduces_after_o_and_down_only():
    _spawn(_block_worker, 64, 128, 16, 4)


# ------------------------------------------------------------------ pipelined block (token chunks)


def test_pipeline_schedule_overlaps_and_orders():
    for n in (1, 2, 4, 7):
        order = tp.pipeline_schedule(n)
        assert sorted(order) == sorted([("A", c) for c in range(n)] + [("B", c) for c in range(n)])
        pos = {op: i for i, op in enumerate(order)}
        for c in range(n):
            assert pos[("A", c)] < pos[("B", c)]  # gate/up needs the reduced o_proj output
            if c + 1 < n:  # the o_proj all-reduce of chunk c has chunk c + 1's GEMMs to hide under
                assert pos[("A", c + 1)] < pos[("B", c)]
    for m, n in [(8192, 4), (300, 4), (1000, 4), (4096, 3)]:
        b = tp.chunk_bounds(m, n)
        assert b[0][0] == 0 and b[-1][1] == m and all(x[1] == y[0] for x, y in zip(b, b[1:]))
        assert all(r0 % 256 == 0 for r0, _ in b)


class _CpuBackend:
    """Synchronous gloo backend: records the issue order of linears and all-reduces."""

    def __init__(self, fns):
        self.fns, self.log, self._outs = fns, [], {}

    def out(self, name, m, n):
        return self._outs.setdefault(name, torch.zeros((m, self.fns[name][1]), dtype=torch.float64))

    def linear(self, name, c, x_rows, y_rows):
        self.log.append(("lin", name, c))
        y_rows.copy_(self.fns[name][0](x_rows))

    def reduce(self, name, c, y_rows):
        self.log.append(("ar", name, c))
        tp.allreduce_sum_(y_rows)

    def wait(self, name, c):
        assert ("ar", name, c) in self.log

    def join(self):
        pass


def _pipelined_worker(rank, hidden, ffn, kv, m, chunks):
    specs = tp.block_specs(hidden, ffn, kv)
    rng = np.random.default_rng(21)
    weights = {s.name: rng.standard_normal((s.k, s.n)) for s in specs}
    fns = {}
    for s in specs:
        w = weights[s.name]
        if s.kind == "column":
            n0, n1 = tp.column_shard(s.n, WORLD, rank)
            fns[s.name] = ((lambda w=w, n0=n0, n1=n1: lambda x: x @ torch.from_numpy(w[:, n0:n1]))(), n1 - n0)
        else:
            k0, k1 = tp.row_shard(s.k, WORLD, rank)
            fns[s.name] = ((lambda w=w, k0=k0, k1=k1: lambda x: x @ torch.from_numpy(w[k0:k1]))(), s.n)
    be = _CpuBackend(fns)
    blk = tp.PipelinedTPBlock(specs, be, chunks=chunks)
    x = torch.from_numpy(np.random.default_rng(22).standard_normal((m, hidden)))
    attn = np.random.default_rng(23).standard_normal((m, hidden))
    act = np.random.default_rng(24).standard_normal((m, ffn))
    k0, k1 = tp.row_shard(hidden, WORLD, rank)
    f0, f1 = tp.row_shard(ffn, WORLD, rank)
    out = blk.forward(x, {"o_proj": torch.from_numpy(attn[:, k0:k1]), "down_proj": torch.from_numpy(act[:, f0:f1])})
    # exactly one all-reduce per chunk, after o_proj and down_proj only
    ars = [e for e in be.log if e[0] == "ar"]
    n_chunks = len(tp.chunk_bounds(m, chunks))
    assert sorted(ars) == sorted([("ar", "o_proj", c) for c in range(n_chunks)] +
                                 [("ar", "down_proj", c) for c in range(n_chunks)])
    o_full = attn @ weights["o_proj"]
    np.testing.assert_allclose(out["o_proj"].numpy(), o_full, rtol=1e-10, atol=1e-9)
    n0, n1 = tp.column_shard(specs[2].n, WORLD, rank)
    np.testing.assert_allclose(out["gate_up_proj"].numpy(), o_full @ weights["gate_up_proj"][:, n0:n1],
                               rtol=1e-9, atol=1e-8)
    np.testing.assert_allclose(out["down_proj"].numpy(), act @ weights["down_proj"], rtol=1e-10, atol=1e-9)


@pytest.mark.parametrize("m,chunks", [(1024, 4), (600, 4), (256, 2)])
def test_pipelined_block_matches_unchunked(m, chunks):
    _spawn(_pipelined_worker, 64, 128, 16, m, chunks)
