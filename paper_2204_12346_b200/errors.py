"""Exception taxonomy of the reference (include/sirdfit/errors.hpp:8-50).

The C-ABI reports sg_status codes (include/sirdgpu.h); `raise_for_status`
turns them back into these classes so callers catch the same types the
reference throws.
"""


class Error(RuntimeError):
    """sirdfit::Error (errors.hpp:8-10)."""


class SchemeError(Error):
    """sirdfit::SchemeError (errors.hpp:24-26)."""


class DegenerateRatesError(Error):
    """sirdfit::DegenerateRatesError (errors.hpp:32-34)."""

    def __init__(self, msg: str = "gamma + mu must be positive"):
        super().__init__(msg)


class ConstantObservedError(Error):
    """sirdfit::ConstantObservedError (errors.hpp:36-38)."""

    def __init__(self, msg: str = "observed series is constant; R^2 undefined"):
        super().__init__(msg)


class AllInfeasibleError(Error):
    """sirdfit::AllInfeasibleError (errors.hpp:40-42)."""

    def __init__(self, msg: str = "no particle produced a finite cost"):
        super().__init__(msg)


class InsufficientPopulationError(Error):
    """sirdfit::InsufficientPopulationError (errors.hpp:44-46)."""


class NonFiniteError(Error):
    """sirdfit::NonFiniteError (errors.hpp:48-50)."""

    def __init__(self, msg: str = "trajectory left the finite range"):
        super().__init__(msg)


class DeviceError(Error):
    """CUDA failure inside the engine (no reference counterpart)."""


class NoDeviceError(DeviceError):
    """No sm_100 device is visible, so the engine cannot run."""


SG_OK = 0
_BY_CODE = {
    1: Error,
    2: SchemeError,
    3: InsufficientPopulationError,
    4: AllInfeasibleError,
    5: NonFiniteError,
    6: DeviceError,
    7: NoDeviceError,
    8: DeviceError,
}


def raise_for_status(code: int, message: str = "") -> None:
    if code == SG_OK:
        return
    cls = _BY_CODE.get(code, Error)
    if cls in (AllInfeasibleError, NonFiniteError) and not message:
        raise cls()
    raise cls(message or f"sg_status {code}")
