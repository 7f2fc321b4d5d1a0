"""Exception taxonomy mirroring fusim::Error (/root/reference/proj/include/fusim/errors.hpp:8-25).

The C ABI returns an ``mlora_status``; the Python host layer maps it onto these
classes so callers see the same error types, raised at the same preconditions,
as users of the reference C++ API.
"""


class Error(RuntimeError):
    """fusim::Error"""


class ConfigError(Error):
    """bad configuration / input files"""


class UsageError(Error):
    """caller violated a precondition"""


class StateError(Error):
    """operation not valid in the object's current state"""


class ShapeError(Error):
    """matrix dimension mismatch"""


class NumericError(Error):
    """non-finite values where finite ones are required"""


class RoutingError(Error):
    """fused batch routed to a job without an adapter"""


class FitError(Error):
    """least-squares fit cannot proceed"""


class CudaError(Error):
    """device/runtime failure (no reference analogue)"""


# mlora_status -> exception class (include/mlora.h)
STATUS_TO_ERROR = {
    1: UsageError,
    2: ShapeError,
    3: RoutingError,
    4: NumericError,
    5: StateError,
    6: CudaError,
}
