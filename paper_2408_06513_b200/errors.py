"""Exception hierarchy of the reference package (uncrowd errors.py:4-77), so callers
catching the reference's exceptions keep working against the drop-in.

Raised on the hot path: ZeroBackground (density.py:67-68), SingularMass
(mapping.py:88-89, 183-184), InvalidParams (model.py:115-132), OutOfRangeLevel
(model.py:166-167, regularize.py:86-87); the rest are kept for import compatibility.
"""


class UncrowdError(Exception):
    """Base class of every package-specific error."""


def _err(name: str, doc: str, *bases):
    return type(name, (UncrowdError,) + (bases or (ValueError,)), {"__doc__": doc})


NonFiniteCoordinate = _err("NonFiniteCoordinate", "A sample coordinate is NaN or infinite.")
CoordinateOutOfRange = _err("CoordinateOutOfRange", "A coordinate lies outside [0,1]^2 with normalization off.")
LabelLengthMismatch = _err("LabelLengthMismatch", "Number of labels differs from the number of samples.")
ZeroBackground = _err("ZeroBackground", "Explicit background density is not strictly positive.")
SingularMass = _err("SingularMass", "Total texture mass is not strictly positive.")
EmptyDataset = _err("EmptyDataset", "The operation needs at least one sample.")
TooFewSamples = _err("TooFewSamples", "The operation needs more samples than the neighbourhood size.")
OutOfRangeLevel = _err("OutOfRangeLevel", "Transition level outside [0, iterations].")
LevelOutOfRange = _err("LevelOutOfRange", "Contour level outside the open density range.")
DegeneratePolygon = _err("DegeneratePolygon", "Lasso polygon without interior.")
InvalidSpec = _err("InvalidSpec", "Inconsistent dataset generator spec.")
FormatError = _err("FormatError", "Binary field file with a bad magic or header.")
UnknownSession = _err("UnknownSession", "Session id absent (never created or evicted).", KeyError)
UnknownKind = _err("UnknownKind", "Unsupported encoding kind.")
PayloadTooLarge = _err("PayloadTooLarge", "Dataset exceeds the session sample cap.")
InvalidParams = _err("InvalidParams", "Regularization parameters fail validation.")


class ParseError(UncrowdError, ValueError):
    """A CSV row could not be parsed."""

    def __init__(self, line: int, message: str):
        super().__init__(f"line {line}: {message}")
        self.line = line
