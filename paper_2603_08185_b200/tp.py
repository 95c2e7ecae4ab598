"""Tensor parallelism for SERQ decoder-block linears.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch on B200;
gloo in the CPU tests).  Column-parallel linears (q/k/v, gate/up) shard the
output dim N: every rank quantizes the same replicated activation, so there is
no exchange.  Row-parallel linears (o_proj, down_proj) shard the reduction
dim K in multiples of the 32-element MX block; each rank computes
Y_k = X_k W_k + X_{s,k} R_k and ONE all-reduce (sum) produces Y.  Those are
the only collectives of the block (BASELINE.json: "NCCL all-reduce ... after
o_proj/down_proj only").

Exactness of the sharded salient term.  The reference re-encodes the gathered
salient columns x[:, idx] in 32-column MX blocks (compensate.py:335).  If each
rank's K-slice starts with its own salient share of a multiple of 32 channels
(the offline permutation puts them there), the global gathered slice is the
concatenation of the per-rank slices with block boundaries on rank
boundaries, so  sum_k forward(X_k; W_k, R_k) == forward(X; W, R)  term by term
(the per-block products are identical; only the fp32/f64 summation order of
the blocks differs).  For integer per-token activations the token scale spans
the full K, so a K-sharded INT layer needs the [M,2] min/max all-reduce before
quantizing (``int_token_range_allreduce``); MX needs nothing.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from .errors import ValidationError

MX_BLOCK = 32


# ------------------------------------------------------------------ sharding plans


def column_shard(n: int, world: int, rank: int, align: int = 8) -> tuple[int, int]:
    """[n0, n1) output columns of ``rank`` (balanced, ``align``-aligned)."""
    if n % align:
        raise ValidationError(f"output dim {n} not a multiple of {align}")
    units = n // align
    base, extra = divmod(units, world)
    n0 = (rank * base + min(rank, extra)) * align
    return n0, n0 + (base + (1 if rank < extra else 0)) * align


def row_shard(k: int, world: int, rank: int, align: int = MX_BLOCK) -> tuple[int, int]:
    """[k0, k1) reduction rows of ``rank``, aligned to the MX block."""
    if k % align:
        raise ValidationError(f"reduction dim {k} not a multiple of {align}")
    return column_shard(k, world, rank, align)


def salient_per_rank(r: int, world: int, align: int = MX_BLOCK) -> int:
    """Salient channels each rank owns in a row-parallel layer (multiple of the
    MX block; BASELINE C5 r=128 at tp=8 -> 32 per rank, i.e. padded to 256)."""
    per = -(-r // world)
    return -(-per // align) * align


def shard_columns_mx(main_codes, main_exps, r_codes, r_exps, n0: int, n1: int):
    """Column-parallel shard of MX artefacts stored [N, K] (main_t) and [N, r]
    (comp.r_q): rows n0..n1 of both."""
    sl = slice(n0, n1)
    return (main_codes[sl], main_exps[sl], None if r_codes is None else r_codes[sl],
            None if r_exps is None else r_exps[sl])


def shard_rows_weight(w: np.ndarray, k0: int, k1: int) -> np.ndarray:
    """Row-parallel shard of a [K, N] (in, out) weight."""
    return np.ascontiguousarray(w[k0:k1])


def row_parallel_salient_layout(scores: np.ndarray, world: int, r_rank: int) -> tuple[np.ndarray, list]:
    """Offline permutation for a row-parallel layer: split K into ``world``
    aligned slices and, inside every slice, move that slice's top-``r_rank``
    channels (by saliency score, ties to the lower index, saliency.py:77-92)
    to the front.  Returns the global permutation and each rank's salient
    indices (local to its slice, always arange(r_rank))."""
    k = scores.shape[0]
    perm = []
    for rank in range(world):
        k0, k1 = row_shard(k, world, rank)
        local = np.asarray(scores[k0:k1], dtype=np.float64)
        order = np.argsort(-local, kind="stable")
        sal = order[:r_rank]
        rest = np.setdiff1d(np.arange(k1 - k0), sal)
        perm.append(k0 + np.concatenate([sal, rest]))
    return np.concatenate(perm).astype(np.intp), [np.arange(r_rank)] * world


# ------------------------------------------------------------------ collectives


def allreduce_sum_(t, group=None):
    """In-place sum across ranks (bf16 on NCCL / any dtype on gloo)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def int_token_range_allreduce(lo, hi, group=None):
    """Per-token (min, max) over a K-sharded activation: the INT quantizer's
    scale spans the full K (quantcore.py:127-129)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    return lo, hi


# ------------------------------------------------------------------ block driver


@dataclass
class TPLinearSpec:
    name: str
    k: int
    n: int
    kind: str  # "column" | "row"


# Llama-style decoder block with q/k/v and gate/up fused (one joint salient plan each)
def block_specs(hidden: int, ffn: int, kv_dim: int) -> list[TPLinearSpec]:
    return [
        TPLinearSpec("qkv_proj", hidden, hidden + 2 * kv_dim, "column"),
        TPLinearSpec("o_proj", hidden, hidden, "row"),
        TPLinearSpec("gate_up_proj", hidden, 2 * ffn, "column"),
        TPLinearSpec("down_proj", ffn, hidden, "row"),
    ]


class TPBlockLinears:
    """Runs the linears of one decoder block on this rank.

    ``linears[name]`` is a callable ``f(x_local) -> y_local`` (the device
    SERQ linear on the GPU, or an injected implementation in CPU tests).
    Column-parallel outputs stay sharded; row-parallel outputs are summed with
    one all-reduce.  Non-linear ops (attention mix, RMSNorm, SiLU) are out of
    scope for this path (SURVEY 2.1 toymodel row); ``feeds`` supplies the
    inputs of o_proj / down_proj (the attention output and SiLU(gate)*up
    shards) so the linear path can be driven and timed on its own."""

    def __init__(self, specs: list[TPLinearSpec], linears: dict[str, Callable], world: int, rank: int, group=None):
        self.specs = specs
        self.linears = linears
        self.world, self.rank, self.group = world, rank, group

    def forward(self, x, feeds: dict | None = None) -> dict:
        feeds = feeds or {}
        out = {}
        h = x
        for spec in self.specs:
            xin = feeds.get(spec.name, h)
            y = self.linears[spec.name](xin)
            if spec.kind == "row":
                y = allreduce_sum_(y, self.group)
                h = y
            out[spec.name] = y
        return out
