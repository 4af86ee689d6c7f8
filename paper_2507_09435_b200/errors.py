"""Exception hierarchy of the reference (/root/reference/proj/include/impm/errors.hpp:9-50),
mapped from the C ABI's impm_status codes."""


class Error(RuntimeError):
    """impm::Error"""


class ConfigError(Error):
    """impm::ConfigError: invalid or inconsistent configuration."""


class DomainError(Error):
    """impm::DomainError: inverted element, lp past h/2, ..."""


class UnsupportedOperation(Error):
    pass


class NonConvergenceError(Error):
    """impm::NonConvergenceError, carries residual_history (errors.hpp:36-40)."""

    def __init__(self, what, residual_history=()):
        super().__init__(what)
        self.residual_history = list(residual_history)


class LinearSolverError(Error):
    pass


class OutOfDomainError(Error):
    """impm::OutOfDomainError: a particle's support left the grid."""


class SeedingFault(Error):
    pass


class CudaError(Error):
    """Device-side failure (no reference counterpart)."""


class NcclError(Error):
    pass


_BY_CODE = {
    1: ConfigError,
    2: DomainError,
    3: OutOfDomainError,
    4: NonConvergenceError,
    5: LinearSolverError,
    6: CudaError,
    7: NcclError,
    8: SeedingFault,
    9: UnsupportedOperation,
}


def raise_for(code, message, history=()):
    cls = _BY_CODE.get(code, Error)
    if cls is NonConvergenceError:
        raise NonConvergenceError(message, history)
    raise cls(message)
