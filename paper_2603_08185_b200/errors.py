"""Error type mirroring the reference (``serq._validation.ValidationError``,
``_validation.py:14-15``): a ``ValueError`` raised on any violated
precondition."""


class ValidationError(ValueError):
    """Raised when an input violates a documented precondition."""
