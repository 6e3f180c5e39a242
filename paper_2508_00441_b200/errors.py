"""Exception classes with the reference's names and base classes.

ozdgemm declares them across modules; callers catch them by these bases:
  RangeError(ArithmeticError)      fp64emu.py:50
  SlicingInfeasible(Exception)     slicing.py:41
  DimensionError(ValueError)       ozgemm.py:43
  RepresentabilityError(Exception) lpgemm.py:23
"""


class RangeError(ArithmeticError):
    """Operand or result outside the supported normal FP64 range."""


class SlicingInfeasible(Exception):
    """The target format cannot retain the information of a slice."""


class DimensionError(ValueError):
    """Operand shapes do not conform."""


class RepresentabilityError(Exception):
    """An operand entry is not representable in the operand format."""
