"""Exception classes of the reference surface (re-used when `capfields` is importable).

OutOfSupportError      capfields/edgraph.py:27
DegenerateWeightsError capfields/transforms.py:15
RecordFormatError      capfields/records.py:24
InsufficientOverlapError capfields/tracking.py:33
"""
from __future__ import annotations

try:  # same classes as the reference, so its tests catch our errors unchanged
    from capfields.edgraph import OutOfSupportError  # type: ignore
    from capfields.transforms import DegenerateWeightsError  # type: ignore
except Exception:  # the reference is not installed on the GPU box

    class OutOfSupportError(ValueError):
        """Query point is outside the influence of every graph node."""

    class DegenerateWeightsError(ValueError):
        """A blend received no positive weight."""

try:
    from capfields.tracking import InsufficientOverlapError  # type: ignore
except Exception:

    class InsufficientOverlapError(ValueError):
        """Too few valid depth pixels to constrain a pose."""

try:
    from capfields.records import RecordFormatError  # type: ignore
except Exception:

    class RecordFormatError(ValueError):
        """A record file with a bad magic, version or payload."""


__all__ = ["OutOfSupportError", "DegenerateWeightsError", "RecordFormatError", "InsufficientOverlapError"]
