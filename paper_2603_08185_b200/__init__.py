"""B200-native SERQ quantized-linear forward (arxiv 2603.08185 hot path).

The product is the C-ABI library ``libserq_b200.so`` (hand-written sm_100a
kernels, include/serq_b200.h).  ``device`` wraps it for torch tensors; the
reference-facing mirror (``forward_reconstructed`` and friends) lives in
``api``.  There is no CPU fallback.
"""

from .errors import ValidationError

__all__ = ["ValidationError"]
__version__ = "0.1.0"
