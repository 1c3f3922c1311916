"""Exception taxonomy of the reference (include/lcnn/errors.hpp:8-56).

The C ABI returns an lcnn_status code; ``raise_for_status`` rethrows the
matching class with the library's message, so callers catch the same types
the reference's tests expect (PlanError for bad transform plans, LayoutError
for NCHW into pool_coarsened, DomainError for non-finite softmax input...).
"""


class Error(RuntimeError):
    """Common base (errors.hpp:8)."""


class ShapeError(Error):
    pass


class IndexError_(Error):  # noqa: N801 -- avoid shadowing the builtin
    pass


class LayoutError(Error):
    pass


class PlanError(Error):
    pass


class FormatError(Error):
    pass


class DomainError(Error):
    pass


class UnsupportedError(Error):
    pass


class ValidationError(Error):
    pass


class CalibrationError(Error):
    pass


class CudaError(Error):
    """CUDA runtime failure inside the library (LCNN_ECUDA)."""


_BY_STATUS = {
    1: ShapeError, 2: IndexError_, 3: LayoutError, 4: PlanError, 5: FormatError,
    6: DomainError, 7: UnsupportedError, 8: ValidationError, 9: CalibrationError,
    10: CudaError, 11: ValueError,
}


def raise_for_status(status: int, message: str) -> None:
    if status == 0:
        return
    raise _BY_STATUS.get(status, Error)(message)
