"""Exception types of the reference (errors.hpp:9-21) and the ABI code map."""
from __future__ import annotations


class InvalidInputError(ValueError):
    """gmt::InvalidInputError (errors.hpp:9-11): bad arguments to a call."""


class InfeasibleSamplingError(RuntimeError):
    """gmt::InfeasibleSamplingError (errors.hpp:14-16): rejection budget spent."""


class GoalBlockedError(RuntimeError):
    """gmt::GoalBlockedError (errors.hpp:19-21): no free goal sample."""


class CudaError(RuntimeError):
    """CUDA runtime failure inside the B200 library."""


class NoDeviceError(RuntimeError):
    """No usable B200 (sm_100) device: the library never falls back to the CPU."""


_CODES = {
    1: InvalidInputError,
    2: InfeasibleSamplingError,
    3: GoalBlockedError,
    4: CudaError,
    5: NoDeviceError,
    7: OSError,
}


def raise_for(code: int, message: str) -> None:
    if code == 0:
        return
    raise _CODES.get(code, RuntimeError)(message)
