"""Exception classes of the reference, mapped from C-ABI status codes.

Same names, base classes and attributes as the reference's (model.py:32-46,
split.py:28-33, pack.py:26-27, sample.py:40-41, stats.py:17-22); each module
of this package re-exports the ones its reference counterpart defines.
"""

from __future__ import annotations

AK_OK = 0
AK_ERR_EMPTY_INPUT = 1
AK_ERR_INVALID_WEIGHT = 2
AK_ERR_SIZE_MISMATCH = 3
AK_ERR_INVALID_SECTION_COUNT = 4
AK_ERR_UNSORTED_INPUT = 5
AK_ERR_PLAN_INCONSISTENT = 6
AK_ERR_INVALID_SECTION_SIZE = 7
AK_ERR_VALUE = 8
AK_ERR_CUDA = 9
AK_ERR_WORKSPACE = 10
AK_ERR_INDEX_OUT_OF_RANGE = 11


class EmptyInput(ValueError):
    pass


class InvalidWeight(ValueError):
    """A weight is non-positive or non-finite; carries the 1-based index."""

    def __init__(self, index: int, value: float):
        self.index = int(index)
        self.value = float(value)
        super().__init__(f"weight {index} is invalid: {value!r}")


class SizeMismatch(ValueError):
    pass


class InvalidSectionCount(ValueError):
    pass


class UnsortedInput(ValueError):
    pass


class PlanInconsistent(ValueError):
    pass


class InvalidSectionSize(ValueError):
    pass


class IndexOutOfRange(ValueError):
    pass


class DegenerateBins(ValueError):
    pass


def from_status(status: int, msg: str = "", index=None, value=None) -> Exception:
    if status == AK_ERR_EMPTY_INPUT:
        return EmptyInput(msg or "at least one weight is required")
    if status == AK_ERR_INVALID_WEIGHT:
        return InvalidWeight(index if index is not None else 0, value if value is not None else float("nan"))
    if status == AK_ERR_SIZE_MISMATCH:
        return SizeMismatch(msg)
    if status == AK_ERR_INVALID_SECTION_COUNT:
        return InvalidSectionCount(msg)
    if status == AK_ERR_UNSORTED_INPUT:
        return UnsortedInput(msg)
    if status == AK_ERR_PLAN_INCONSISTENT:
        return PlanInconsistent(msg)
    if status == AK_ERR_INVALID_SECTION_SIZE:
        return InvalidSectionSize(msg)
    if status == AK_ERR_VALUE:
        return ValueError(msg)
    if status == AK_ERR_INDEX_OUT_OF_RANGE:
        return IndexOutOfRange(msg)
    return RuntimeError(f"aliaskit_b200 status {status}: {msg}")
