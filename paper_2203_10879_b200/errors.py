"""Exception classes of the reference API, same names and meaning.

  SeparationError, NonFiniteError  /root/reference/pkg/src/ddschur/trisolve.py:50-55
  NormTooLarge                     /root/reference/pkg/src/ddschur/orthogonal.py:38-39
  NotSymmetric                     /root/reference/pkg/src/ddschur/refine.py:35-36
"""


class SeparationError(Exception):
    """Diagonal entries of T coincide exactly; the equation is singular."""


class NonFiniteError(Exception):
    """An overflow or NaN appeared in the solution."""


class NormTooLarge(Exception):
    """Spectral norm at or above sqrt(3); Newton-Schulz would diverge."""


class NotSymmetric(Exception):
    """Input to the Hermitian driver is not Hermitian within tolerance."""
