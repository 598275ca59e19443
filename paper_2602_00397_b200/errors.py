"""Exception types of the hot path, same names and bases as the reference.

``ValidationError(ValueError)`` for malformed shapes, k, index sets or plans and
``NumericError(RuntimeError)`` for non-finite results (reference ``errors.py:9-14``).
Non-zero C-ABI status codes map onto these (see ``_lib.check``).
"""


class ValidationError(ValueError):
    """Inputs, shapes, or configuration violate a documented precondition."""


class NumericError(RuntimeError):
    """A computation produced NaN/inf or otherwise diverged."""


class UnsupportedError(ValidationError):
    """A shape or device the sm_100a kernels do not cover (e.g. d_model % 64 != 0)."""
