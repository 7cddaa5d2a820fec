"""Exception types of the segmentation path.

Same names and hierarchy as the reference (ref errors.py:4-50) so callers can
catch either; only the types the hot path raises are defined here.
"""


class ClonetrackError(Exception):
    """Base class for all pipeline errors (ref errors.py:4)."""


class ManifestError(ClonetrackError):
    """Raised by VoxelSpacing validation (ref errors.py:8, imaging.py:33-36)."""


class ParameterError(ClonetrackError):
    """A processing parameter is outside its valid range (ref errors.py:16)."""


class DegenerateHistogramError(ClonetrackError):
    """Fewer than two non-empty histogram bins (ref errors.py:20)."""


class EmptyDistanceMapError(ClonetrackError):
    """Distance map has no foreground (ref errors.py:36)."""
