"""Error types with machine-readable codes.

Mirrors the reference's error convention (`pkg/src/ipcsim/errors.py:8-42`):
every failure carries a short ``code`` string; the native library returns an
integer status that maps 1:1 onto these codes (see ``include/maspncg.h``).
"""


class SimError(Exception):
    code = "sim-error"

    def __init__(self, message: str = ""):
        super().__init__(message or self.code)


class DegeneratePrimitiveError(SimError):
    code = "degenerate-primitive"


class PenetrationError(SimError):
    code = "penetration-detected"


class NotSpdError(SimError):
    code = "not-spd"

    def __init__(self, code: str, message: str = ""):
        self.code = code
        super().__init__(message or code)


class ConfigError(SimError):
    code = "config-error"


class CapacityError(SimError):
    """A device buffer could not be grown to hold a dynamic set."""

    code = "capacity-overflow"


class CudaError(SimError):
    """A CUDA runtime/library call failed inside the native backend."""

    code = "cuda-error"
