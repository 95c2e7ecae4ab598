"""Whole decoder block on the device.

The reference evaluates its block graph node by node in float64 NumPy
(`toy_block_graph`, toymodel.py:88-124; `graph_forward`, saliency.py:222-290)
and its quantized forward swaps every linear for `forward_reconstructed`
(`forward_quantized`, toymodel.py:363-374).  `DeviceBlock` runs the same graph
with every activation resident on the GPU: the seven SERQ linears go through
the sm_100a kernels (quantizer + fused linear, one C-ABI call each), the
non-linear nodes -- RMSNorm (saliency.py:194-196), the per-head token-batch
attention (`attention_mix`, saliency.py:203-216), SiLU (saliency.py:199-200),
the gating product and the residual adds -- are float32 PyTorch ops (they stay
in full precision in the reference; SERQ quantizes only the linears).  The
whole forward captures into one CUDA graph for a fixed token count.

Activations between nodes are float32 (the linears quantize their f32 input
exactly like mx_encode of the reference's f64 value, up to E2M1 ties), each
linear's output is bf16 (the kernel's store), promoted to f32 for the
residual stream.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from .errors import ValidationError

LINEAR_NAMES = ("q_proj", "k_proj", "v_proj", "o_proj", "up_proj", "gate_proj", "down_proj")  # toymodel.py:54


def rmsnorm(x: torch.Tensor, gain: torch.Tensor, eps: float = 1e-6) -> torch.Tensor:
    """saliency.py:194-196 in float32 (one fused kernel)."""
    return torch.nn.functional.rms_norm(x, (x.shape[-1],), gain, eps)


def attention_mix(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, head_dim: int, fast: bool = False) -> torch.Tensor:
    """saliency.py:203-216: per-head softmax(Q K^T / sqrt(d)) V over the token batch (no mask).
    float32 by default (the parity mode: with outlier channels the logits reach the hundreds, so a
    bf16 rounding of q or k moves the softmax weights by e^(2^-9 |logit|)); ``fast`` runs bf16
    flash attention -- the non-SERQ part of a serving block."""
    m, hidden = q.shape
    if hidden % head_dim:
        raise ValidationError("hidden dim not divisible by head_dim")
    h = hidden // head_dim
    dt = torch.bfloat16 if fast else torch.float32
    qh, kh, vh = (t.to(dt).view(m, h, head_dim).transpose(0, 1) for t in (q, k, v))
    if fast:
        out = torch.nn.functional.scaled_dot_product_attention(
            qh.unsqueeze(0), kh.unsqueeze(0), vh.unsqueeze(0), scale=1.0 / math.sqrt(head_dim))[0]
    else:
        out = torch.softmax(qh @ kh.transpose(1, 2) * (1.0 / math.sqrt(head_dim)), dim=-1) @ vh
    return out.transpose(0, 1).reshape(m, hidden).float()


class DeviceBlock:
    """The reference's toy decoder block with SERQ linears on the GPU.

    ``linears``: name -> callable (x f32/bf16 [M, in] cuda -> bf16 [M, out]), e.g. the
    ``SerqLinear`` objects of a ``bundle.DeviceBundle``; ``gains``: 'ln1', 'ln2'
    (the folded RMSNorm gains of the quantized bundle, toymodel.py:203-217)."""

    def __init__(self, linears: dict, gains: dict, head_dim: int, eps: float = 1e-6, device="cuda",
                 fast_attention: bool = False, glue_kernels: bool = True):
        """``linears`` may hold "qkv_proj" (q, k, v) and / or "up_gate_proj" (up, gate) as one
        ``device.FusedMxLinear`` (one quantizer + one kernel for the parts) instead of the parts."""
        self.qkv = linears.get("qkv_proj")
        self.up_gate = linears.get("up_gate_proj")
        need = [n for n in LINEAR_NAMES
                if not (self.qkv is not None and n in ("q_proj", "k_proj", "v_proj"))
                and not (self.up_gate is not None and n in ("up_proj", "gate_proj"))]
        missing = [n for n in need if n not in linears]
        if missing:
            raise ValidationError(f"block needs linears {missing}")
        self.lin = {n: linears[n] for n in need}
        self.g1 = torch.as_tensor(np.asarray(gains["ln1"]), dtype=torch.float32, device=device)
        self.g2 = torch.as_tensor(np.asarray(gains["ln2"]), dtype=torch.float32, device=device)
        self.head_dim = int(head_dim)
        self.eps = eps
        self.fast_attention = fast_attention
        self.glue_kernels = glue_kernels  # M <= 16: the fused f32 glue kernels (csrc/serq_block.cuh)

    @classmethod
    def from_bundle(cls, bundle, head_dim: int, **kw) -> "DeviceBlock":
        return cls({n: bundle.linears[n].linear for n in LINEAR_NAMES}, bundle.nl_weights, head_dim, **kw)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        """x [M, hidden] on the GPU -> block output float32 [M, hidden].  At M <= 16 (decode) the
        non-SERQ glue runs as 4 fused f32 kernels (csrc/serq_block.cuh) instead of ~9 PyTorch
        micro-kernels; larger batches use the PyTorch ops."""
        x = x.float().contiguous()
        m, hidden = x.shape
        if self.glue_kernels and m <= 16 and self.head_dim == 128:
            return self._forward_small(x)
        h1 = rmsnorm(x, self.g1, self.eps)
        if self.qkv is not None:
            q, k, v = (t.contiguous() for t in self.qkv.forward_parts(h1))
        else:
            q = self.lin["q_proj"](h1)
            k = self.lin["k_proj"](h1)
            v = self.lin["v_proj"](h1)
        attn = attention_mix(q, k, v, self.head_dim, self.fast_attention)
        res1 = x + self.lin["o_proj"](attn.contiguous())  # bf16 + f32 -> f32
        h2 = rmsnorm(res1, self.g2, self.eps)
        if self.up_gate is not None:
            up, gate = self.up_gate.forward_parts(h2)
            gate = gate.float()
        else:
            up = self.lin["up_proj"](h2)
            gate = self.lin["gate_proj"](h2).float()
        mid = torch.nn.functional.silu(gate) * up
        return res1 + self.lin["down_proj"](mid)

    def _forward_small(self, x: torch.Tensor) -> torch.Tensor:
        from . import _lib
        from .device import _stream

        m, hidden = x.shape
        st = _stream()
        h1 = torch.empty_like(x)
        _lib.call("serq_block_add_rmsnorm", x.data_ptr(), None, 0, m, hidden, self.g1.data_ptr(), self.eps, None,
                  h1.data_ptr(), st)
        if self.qkv is not None:
            q, k, v = self.qkv.forward_parts(h1)  # column views of one buffer (read in place)
        else:
            q, k, v = (self.lin[n](h1) for n in ("q_proj", "k_proj", "v_proj"))
        attn = torch.empty_like(x)
        _lib.call("serq_block_attention", q.data_ptr(), q.stride(0), k.data_ptr(), k.stride(0), v.data_ptr(),
                  v.stride(0), m, hidden // self.head_dim, self.head_dim, 1.0 / math.sqrt(self.head_dim),
                  attn.data_ptr(), hidden, st)
        o = self.lin["o_proj"](attn)
        res1, h2 = torch.empty_like(x), torch.empty_like(x)
        _lib.call("serq_block_add_rmsnorm", x.data_ptr(), o.data_ptr(), o.stride(0), m, hidden, self.g2.data_ptr(),
                  self.eps, res1.data_ptr(), h2.data_ptr(), st)
        if self.up_gate is not None:
            up, gate = self.up_gate.forward_parts(h2)
        else:
            up, gate = self.lin["up_proj"](h2), self.lin["gate_proj"](h2)
        ffn = up.shape[1]
        mid = torch.empty((m, ffn), dtype=torch.float32, device=x.device)
        _lib.call("serq_block_silu_mul", gate.data_ptr(), gate.stride(0), up.data_ptr(), up.stride(0), m, ffn,
                  mid.data_ptr(), st)
        down = self.lin["down_proj"](mid)
        out = torch.empty_like(x)  # res1 + down, PDL-chained like the rest of the glue
        _lib.call("serq_block_add_rmsnorm", res1.data_ptr(), down.data_ptr(), down.stride(0), m, hidden, None,
                  self.eps, out.data_ptr(), None, st)
        return out

    __call__ = forward

    def graphed(self, x_static: torch.Tensor):
        """Capture forward(x_static) into a CUDA graph; returns (replay, output tensor)."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.forward(x_static)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                out = self.forward(x_static)
        torch.cuda.synchronize()
        return g.replay, out
