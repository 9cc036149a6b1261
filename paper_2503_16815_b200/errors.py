"""Error hierarchy of the DeFT hot path (mirrors deftsim/errors.py:7-60).

The names and the subclass tree are the reference's, so code written against
``deftsim`` catches the same exceptions.  The C-ABI library reports failures as
negative ``deft_status_t`` codes (include/deft_b200.h); ``raise_for_status``
turns them back into the matching Python class.
"""
from __future__ import annotations


class DeftError(Exception):
    """Root of every error raised by this package (errors.py:7)."""


class ValidationError(DeftError):
    """Bad user input: profile, cluster, config (errors.py:11)."""


class ProfileValidationError(ValidationError):
    """A bucket / link / model profile breaks an invariant (errors.py:15)."""


class SchemaError(ValidationError):
    """A JSON document is missing fields or has the wrong shape (errors.py:19)."""


class MalformedTraceError(ValidationError):
    """Structurally broken operator trace (errors.py:23)."""


class ReconstructionError(DeftError):
    """Bucket reconstruction from a trace failed (errors.py:27)."""

    def __init__(self, message, bucket_id=None):
        super().__init__(message)
        self.bucket_id = bucket_id


class InfeasiblePartitionError(DeftError):
    """A bucket cannot be split below the capacity bound (errors.py:35)."""

    def __init__(self, message, bucket_id=None):
        super().__init__(message)
        self.bucket_id = bucket_id


class ScheduleMismatchError(DeftError):
    """A plan names buckets or links the executor does not know (errors.py:43)."""


class InternalInvariantError(DeftError):
    """The delayed-update state machine reached an impossible state (errors.py:47)."""


class NonSteadyStateError(DeftError):
    """The update stream never becomes periodic (errors.py:51)."""


class DegenerateDistributionError(DeftError):
    """sigma_t == 0 makes the walk step degenerate (errors.py:55)."""


class ComparisonError(DeftError):
    """Reports that cannot be compared (errors.py:59)."""


class DeviceError(DeftError):
    """A CUDA call inside the native library failed (no reference equivalent:
    the reference never touches a device)."""


# deft_status_t values returned by the C-ABI (include/deft_b200.h)
STATUS_OK = 0
STATUS_INVALID_ARGUMENT = -1
STATUS_CUDA = -2
STATUS_WORKSPACE = -3
STATUS_UNSUPPORTED = -4
STATUS_PEER = -5

_STATUS_CLASS = {
    STATUS_INVALID_ARGUMENT: DeftError,
    STATUS_CUDA: DeviceError,
    STATUS_WORKSPACE: DeviceError,
    STATUS_UNSUPPORTED: DeviceError,
    STATUS_PEER: DeviceError,
}


def raise_for_status(status: int, what: str, detail: str = "") -> None:
    """Re-raise a negative deft_status_t as the matching DeftError subclass."""
    if status == STATUS_OK:
        return
    cls = _STATUS_CLASS.get(status, DeviceError)
    msg = f"{what} failed with deft_status {status}"
    if detail:
        msg += f": {detail}"
    raise cls(msg)


def check_rules(rules, error: type = ValueError) -> None:
    """Validate in order: every rule is (ok, message) or (ok, message, exception
    class); the first failing rule raises (``error`` unless the rule names one)."""
    for rule in rules:
        if not rule[0]:
            raise (rule[2] if len(rule) > 2 else error)(rule[1])
