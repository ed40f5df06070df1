"""Exception hierarchy of the solver API.

Same class names, bases and meaning as the reference's error module
(reference: pkg/src/qsocp/errors.py:4-45) so that code written against the
reference's ``qsocp.errors`` catches the same things here.
"""


class QsocpError(Exception):
    """Root of every error this package raises on purpose."""


def _err(name, base, doc):
    return type(name, (QsocpError, base), {"__doc__": doc, "__module__": __name__})


DimensionMismatch = _err("DimensionMismatch", ValueError, "vector/matrix sizes disagree with (n, m, p)")
ConeMismatch = _err("ConeMismatch", ValueError, "cone sizes do not sum to m")
BadSparseStructure = _err("BadSparseStructure", ValueError, "CSC invariant broken")
EmptyCone = _err("EmptyCone", ValueError, "m == 0: no conic rows")
IndexOutOfRange = _err("IndexOutOfRange", IndexError, "triplet index outside the matrix shape")
BadPermutation = _err("BadPermutation", ValueError, "not a bijection on 0..n-1")
NotInterior = _err("NotInterior", ValueError, "point not strictly inside the cone")
NumericalError = _err("NumericalError", ArithmeticError, "non-finite value / unrecoverable numerical failure")
NotSetUp = _err("NotSetUp", RuntimeError, "solve() before setup()")
EmptyInput = _err("EmptyInput", ValueError, "aggregate over an empty collection")


class CudaUnavailable(QsocpError, RuntimeError):
    """The CUDA shared library is missing or no CUDA device is usable.

    There is deliberately no CPU fallback behind the ``cuda`` algebra; this is
    what the product path raises instead.
    """
