"""Exception taxonomy mirroring /root/reference/proj/include/rray/core/error.hpp:9-55.

The integer ``code`` of each class is the reference CLI exit code
(tools/rray_main.cpp:185-194) and the C-ABI status (include/rray_cuda.h).
"""


class Error(RuntimeError):
    code = 4


class NumericError(Error):          # error.hpp:13-16, exit code 2
    code = 2


class SingularMatrix(NumericError):
    pass


class SingularJacobian(NumericError):
    pass


class DegenerateBasis(NumericError):
    pass


class ConfigError(Error):           # error.hpp:29-32, exit code 1
    code = 1


class ParseError(ConfigError):
    pass


class ValidationError(ConfigError):
    pass


class IoError(Error):               # error.hpp:47-50, exit code 3
    code = 3


class DeviceError(Error):           # extension: CUDA/runtime failure, status 4
    code = 4


def raise_for_status(code: int, msg: str) -> None:
    if code == 0:
        return
    cls = {1: ValidationError, 2: NumericError, 3: IoError}.get(code, DeviceError)
    raise cls(msg)
