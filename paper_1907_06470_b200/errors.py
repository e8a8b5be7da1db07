"""Exception taxonomy mirroring the reference's (src/errors.py:1-58).

The C ABI returns an xb_status; `raise_for_status` maps it onto these
classes exactly as include/xsvd_b200.h documents:
XB_ESHAPE -> ShapeError, XB_EVALUE -> ValueError, XB_ENOMEM -> BudgetError,
XB_ECONV -> ConvergenceError, anything else -> XsvdError.
"""


class XsvdError(Exception):
    """Base class for all errors raised by this package (errors.py:4)."""


class ShapeError(XsvdError):
    """Operand dimensions are incompatible (errors.py:8)."""


class BudgetError(XsvdError):
    """The memory budget (here: device memory) cannot fit the operation (errors.py:38)."""


class ConvergenceError(XsvdError):
    """An iterative kernel exceeded its sweep limit (errors.py:42)."""

    def __init__(self, message, residual=None):
        super().__init__(message)
        self.residual = residual


class ParseError(XsvdError):
    """A text input (Matrix Market header or body) is malformed; carries the
    1-based line where the problem was found (errors.py:12-23)."""

    def __init__(self, message, line=None):
        if line is not None:
            message = f"line {line}: {message}"
        super().__init__(message)
        self.line = line


class FormatError(XsvdError):
    """A block file or descriptor is not in the expected format (errors.py:26)."""


class BlockAbsentError(XsvdError):
    """A block or descriptor is missing from the store (errors.py:30)."""


class BlockCorruptError(XsvdError):
    """A stored block fails its header or checksum checks (errors.py:34)."""


class PlanNotFoundError(XsvdError):
    """No resumable plan under the workdir (errors.py:53)."""


class ConfigMismatchError(XsvdError):
    """A resume was asked under settings other than the plan's (errors.py:57)."""


XB_ESHAPE, XB_EVALUE, XB_ENOMEM, XB_ECONV, XB_ECUDA, XB_ENCCL, XB_EUNSUPPORTED = 1, 2, 3, 4, 5, 6, 7
XB_EPARSE = 8


def raise_for_status(status: int, message: str, line=None):
    if status == XB_EPARSE:
        raise ParseError(message, line)
    if status == XB_ESHAPE:
        raise ShapeError(message)
    if status == XB_EVALUE:
        raise ValueError(message)
    if status == XB_ENOMEM:
        raise BudgetError(message)
    if status == XB_ECONV:
        raise ConvergenceError(message)
    raise XsvdError(f"[xb status {status}] {message}")
