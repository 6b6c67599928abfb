"""Exception hierarchy mirroring exsim's (proj/core/include/exsim/errors.hpp:9-84).

Every C-ABI status code maps 1:1 onto one class, so callers catch the same
types they catch around the reference's functions.
"""
from __future__ import annotations


class Error(RuntimeError):
    """exsim::Error"""


class ContractError(Error):
    """exsim::ContractError — broken precondition."""


class NonFiniteError(Error):
    """exsim::NonFiniteError"""


class SingularMatrixError(Error):
    """exsim::SingularMatrixError"""

    def __init__(self, what: str, pivot_index: int = -1):
        super().__init__(what)
        self.pivot_index = pivot_index


class ZeroStartVectorError(Error):
    """exsim::ZeroStartVectorError"""


class NoConvergenceError(Error):
    """exsim::NoConvergenceError — Krylov dimension cap reached."""

    def __init__(self, what: str, last_residual: float = float("nan")):
        super().__init__(what)
        self.last_residual = last_residual


class SingularReducedMatrixError(Error):
    """exsim::SingularReducedMatrixError"""


class NoDcConvergenceError(Error):
    """exsim::NoDcConvergenceError"""


class StepFailureError(Error):
    """exsim::StepFailureError"""


class CudaError(Error):
    """CUDA runtime failure inside the device library (no reference analogue)."""


_BY_CODE = {
    1: ContractError,
    2: NonFiniteError,
    3: SingularMatrixError,
    4: ZeroStartVectorError,
    5: NoConvergenceError,
    6: SingularReducedMatrixError,
    7: NoDcConvergenceError,
    8: StepFailureError,
    100: CudaError,
    101: MemoryError,
}


def raise_for(status: int, message: str, value: float | None = None):
    cls = _BY_CODE.get(status, Error)
    if cls is NoConvergenceError:
        raise NoConvergenceError(message, float("nan") if value is None else value)
    if cls is SingularMatrixError:
        raise SingularMatrixError(message, -1 if value is None else int(value))
    raise cls(message)
