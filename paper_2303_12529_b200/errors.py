"""Error taxonomy of the drop-in.

The three names and their base classes must match the reference
(errors.py:4-13) so callers' `except` clauses keep working; the C ABI status
codes map onto them in `_native.check`.
"""


class FormatError(ValueError):
    """Raised by the file readers on a malformed DVLK1/DVLF1/PGM/layout file."""


class DegenerateInputError(ValueError):
    """Raised when an input has no boundary to work with (uniform mask/target)."""


class NumericalError(RuntimeError):
    """Raised when a loss, update or field turns NaN/Inf."""
