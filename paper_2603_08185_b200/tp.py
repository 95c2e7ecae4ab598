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


def allreduce_sum_(t, group=None, force: bool = False):
    """In-place sum across ranks (bf16 on NCCL / any dtype on gloo).  ``force``: issue the
    collective even for a single rank (exercises the NCCL / graph-capture path on one GPU)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and (force or dist.get_world_size(group) > 1):
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


def quantize_int_k_sharded(x_shard, bits: int, symmetric: bool, group=None, salient_idx=None, r: int = 0,
                           xs_kind: int = 0):
    """K1-INT for a row-parallel INT layer: this rank's K-slice of the activations quantized
    with the per-token range of the WHOLE row -- local (min, max) on the device
    (serq_act_quant_int_range), one [2, M] MIN / MAX all-reduce, then the quantizer on the
    global range (serq_act_quant_int_ext).  Codes, scales and zero points equal the
    unsharded quantizer's, so the sharded integer accumulators sum exactly."""
    from . import device as D

    rng = D.int_token_ranges(x_shard)
    int_token_range_allreduce(rng[0], rng[1], group)
    return D.quantize_int_with_range(x_shard, rng, bits, symmetric, salient_idx, r, xs_kind)


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


# ------------------------------------------------------------------ pipelined device driver


def pipeline_schedule(n_chunks: int) -> list[tuple[str, int]]:
    """Issue order of the token-chunk pipeline (SURVEY 7 hard-part 5).

    ``("A", c)``: q/k/v and o_proj of chunk c, then o_proj's all-reduce of chunk c on the
    communication stream.  ``("B", c)``: gate/up (on the reduced o output of chunk c) and
    down_proj, then down_proj's all-reduce.  A(c + 1) is issued before B(c), so the o_proj
    all-reduce of chunk c runs under chunk c + 1's q/k/v and o_proj GEMMs, and the
    down_proj all-reduce of chunk c under B(c + 1).  Every chunk appears once in each
    phase and B(c) always follows A(c)."""
    if n_chunks < 1:
        raise ValidationError("need at least one token chunk")
    order = [("A", 0)]
    for c in range(n_chunks):
        if c + 1 < n_chunks:
            order.append(("A", c + 1))
        order.append(("B", c))
    return order


def chunk_bounds(m: int, n_chunks: int, align: int = 256) -> list[tuple[int, int]]:
    """Row ranges of the token chunks: ``align``-row multiples (whole CTA-pair tiles), the
    last chunk absorbing the remainder."""
    n = max(1, min(n_chunks, m // align if m >= align else 1))
    step = -(-m // n)
    step = -(-step // align) * align
    out, r0 = [], 0
    while r0 < m:
        out.append((r0, min(m, r0 + step)))
        r0 += step
    return out


class PipelinedTPBlock:
    """The C5 block linears of one rank with the two all-reduces pipelined under the GEMMs
    (``pipeline_schedule`` over ``chunk_bounds`` token chunks).

    The schedule is backend-independent; ``backend`` provides
      ``out(name, m, n)``                   the [m, n] output buffer of a linear (allocated once),
      ``linear(name, c, x_rows, y_rows)``   linear ``name`` on token chunk c,
      ``reduce(name, c, y_rows)``           start the all-reduce (sum) of chunk c's output,
      ``wait(name, c)``                     make later work wait for that all-reduce,
      ``join()``                            wait for every outstanding all-reduce.
    ``DeviceBackend`` issues the kernels on the current CUDA stream and the NCCL
    collectives on a dedicated stream (events in between), so one ``forward`` -- quantizers,
    fused SERQ GEMMs and collectives -- captures into ONE CUDA graph; the CPU tests drive the
    same schedule over gloo."""

    def __init__(self, specs: list[TPLinearSpec], backend, chunks: int = 4):
        self.specs = {s.name: s for s in specs}
        col = [s.name for s in specs if s.kind == "column"]
        row = [s.name for s in specs if s.kind == "row"]
        if len(col) != 2 or len(row) != 2:
            raise ValidationError("the pipelined block expects qkv, o, gate_up, down")
        (self.qkv, self.gate_up), (self.o_proj, self.down) = col, row
        self.backend = backend
        self.chunks = chunks

    def forward(self, x, feeds: dict) -> dict:
        """x [M, hidden] (replicated); feeds: this rank's K-slices of the o_proj input
        (attention output) and of the down_proj input (SiLU(gate) * up).  gate/up consumes
        the all-reduced o_proj output (the residual stream in the real block)."""
        be = self.backend
        m = x.shape[0]
        bounds = chunk_bounds(m, self.chunks)
        outs = {n: be.out(n, m, self.specs[n].n) for n in self.specs}

        def rows(t, c):
            r0, r1 = bounds[c]
            return t[r0:r1]

        for phase, c in pipeline_schedule(len(bounds)):
            if phase == "A":
                be.linear(self.qkv, c, rows(x, c), rows(outs[self.qkv], c))
                be.linear(self.o_proj, c, rows(feeds[self.o_proj], c), rows(outs[self.o_proj], c))
                be.reduce(self.o_proj, c, rows(outs[self.o_proj], c))
            else:
                be.wait(self.o_proj, c)
                be.linear(self.gate_up, c, rows(outs[self.o_proj], c), rows(outs[self.gate_up], c))
                be.linear(self.down, c, rows(feeds[self.down], c), rows(outs[self.down], c))
                be.reduce(self.down, c, rows(outs[self.down], c))
        be.join()
        return outs


class DeviceBackend:
    """CUDA backend of ``PipelinedTPBlock``: per-shard device linears (``MxLinear``; their
    N is this rank's shard), per-(linear, chunk) activation buffers, NCCL all-reduces on a
    communication stream ordered by events."""

    def __init__(self, lins: dict, group=None, force_collective: bool = False, collectives: bool = True):
        """``collectives=False``: a single-GPU (tp = 1) run inside a multi-rank job -- no
        collective may be issued from one rank alone."""
        import torch

        self.lins = lins
        self.group = group
        self.force = force_collective
        self.collectives = collectives
        self.comm = torch.cuda.Stream()
        self._outs = {}
        self._acts = {}
        self._ev = {}
        self._started = False
        self.launches_per_forward = 0  # kernels of ours one forward issues (not counting NCCL's)
        self._launches = 0

    def out(self, name, m, n):
        import torch

        lin = self.lins[name]
        key = (name, m)
        if key not in self._outs:
            self._outs[key] = torch.empty((m, lin.N), dtype=torch.bfloat16, device="cuda")
        return self._outs[key]

    def _act(self, name, c, m):
        import torch

        from . import device as D

        key = (name, c, m)
        if key not in self._acts:
            lin = self.lins[name]
            cb, sb = D.mx_sizes(m, lin.K)
            a = D.MxActivation(torch.empty(cb, dtype=torch.uint8, device="cuda"),
                               torch.empty(sb, dtype=torch.uint8, device="cuda"), m, lin.K)
            if not lin.contiguous:
                cbr, sbr = D.mx_sizes(m, lin.r)
                a.xs_codes = torch.empty(cbr, dtype=torch.uint8, device="cuda")
                a.xs_sf = torch.empty(sbr, dtype=torch.uint8, device="cuda")
            self._acts[key] = a
        return self._acts[key]

    def _event(self, *key):
        import torch

        if key not in self._ev:
            self._ev[key] = torch.cuda.Event()
        return self._ev[key]

    def linear(self, name, c, x_rows, y_rows):
        import torch

        if not self._started:  # the comm stream must follow earlier work on the caller's stream
            self.comm.wait_stream(torch.cuda.current_stream())
            self._started = True
        from . import device as D

        self.lins[name].forward(x_rows, self._act(name, c, x_rows.shape[0]), y_rows)
        self._launches += D.last_launch_count()

    def reduce(self, name, c, y_rows):
        import torch

        ready, done = self._event(name, c, "ready"), self._event(name, c, "done")
        ready.record(torch.cuda.current_stream())
        self.comm.wait_event(ready)
        with torch.cuda.stream(self.comm):
            if self.collectives:
                allreduce_sum_(y_rows, self.group, self.force)
            done.record(self.comm)

    def wait(self, name, c):
        import torch

        torch.cuda.current_stream().wait_event(self._event(name, c, "done"))

    def join(self):
        import torch

        torch.cuda.current_stream().wait_stream(self.comm)
        self._started = False
        self.launches_per_forward, self._launches = self._launches, 0
