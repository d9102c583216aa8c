"""Exception hierarchy of the drop-in API (mirrors b2sr/errors.py:4-13).

ValueError / TypeError / RuntimeError / MemoryError are used exactly where
the reference uses them; FormatError marks structural invariant violations.
"""


class B2srError(Exception):
    """Root of this package's own exception types."""


class FormatError(B2srError):
    """Matrix, vector or container breaks a structural invariant."""


class MatrixMarketError(B2srError):
    """Matrix Market input problem (kept for API compatibility)."""
