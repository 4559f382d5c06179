"""Exception classes kept at the drop-in boundary.

The class names and the inheritance tree are the ones the reference exposes
(reference pkg/src/hybir/errors.py:4-29) so that callers written against
``hybir`` keep catching the same exceptions.  ``EngineError`` is new: it is
raised when the CUDA library is missing or a CUDA call fails -- the product
path never falls back to a CPU implementation.
"""


class HybirError(Exception):
    """Root of every exception this package raises on purpose."""


class InputError(HybirError):
    """Bad user input (flags, malformed graph data, out-of-range sources)."""


class ParseError(InputError):
    def __init__(self, message, line_number=None):
        self.line_number = line_number
        if line_number is not None:
            message = "line %d: %s" % (line_number, message)
        super().__init__(message)


class FormatError(InputError):
    """Structurally invalid data (vertex id out of range, wrong length)."""


class DomainError(InputError):
    """A value outside the algorithm's domain (non-positive weight ...)."""


class ContractViolation(HybirError):
    """An internal precondition was broken (e.g. a seed outside its partition)."""


class EngineError(HybirError):
    """The CUDA engine is unavailable or reported a CUDA / NCCL failure."""
