"""Exception types of the drop-in API.

Same names and base classes as the reference (`pkg/src/spectralstokes/errors.py:4-13`) so that
callers catching ``MeshError``/``ConfigError``/``ConvergenceError`` keep working.  The C-ABI never
throws; it returns status codes that :mod:`._lib` maps onto these types.
"""


class MeshError(ValueError):
    """Invalid mesh content: dangling indices, inverted or degenerate elements, bad patches."""


class ConfigError(ValueError):
    """Invalid or inconsistent configuration."""


class ConvergenceError(RuntimeError):
    """Iterative solve failed to reach its tolerance."""


class DeviceError(RuntimeError):
    """CUDA/driver failure reported by the native library (no CPU fallback exists)."""
