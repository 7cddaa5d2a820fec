"""Exception types of the segmentation path.

Drop-in identity (ref errors.py:4-50): when the reference package
``clonetrack`` is importable, its exception classes are used AS these names,
so the reference's own handlers -- ``except ClonetrackError`` (ref
cli.py:57, :83, :126), ``except (EditError, ParameterError)`` (ref
server.py:224) -- catch the errors this package raises, and vice versa.
Without the reference, classes with the same names and hierarchy are defined
here.  ``REFERENCE_BOUND`` says which case applies.
"""

from __future__ import annotations

import importlib
import sys

# the types the segmentation path raises (the reference's other exception
# types belong to subsystems outside this path)
_NAMES = ("ClonetrackError", "ManifestError", "ParameterError", "DegenerateHistogramError", "EmptyDistanceMapError")


def _reference_errors():
    """The reference's errors module, if the reference is importable."""
    mod = sys.modules.get("clonetrack.errors")
    if mod is None:
        try:
            mod = importlib.import_module("clonetrack.errors")
        except Exception:
            # the package body may fail on an optional dependency after its
            # errors submodule loaded (ref __init__.py imports it first)
            mod = sys.modules.get("clonetrack.errors")
    if mod is not None and all(hasattr(mod, n) for n in _NAMES):
        return mod
    return None


_ref = _reference_errors()
REFERENCE_BOUND = _ref is not None

if REFERENCE_BOUND:
    ClonetrackError = _ref.ClonetrackError
    ManifestError = _ref.ManifestError
    ParameterError = _ref.ParameterError
    DegenerateHistogramError = _ref.DegenerateHistogramError
    EmptyDistanceMapError = _ref.EmptyDistanceMapError
else:

    class ClonetrackError(Exception):
        """Root of the pipeline's exception tree (ref errors.py:4)."""

    class ManifestError(ClonetrackError):
        """Unreadable image input or bad spacing (ref errors.py:8; imaging.py:33-36, :213-216)."""

    class ParameterError(ClonetrackError):
        """Invalid processing parameter for the given grid (ref errors.py:16)."""

    class DegenerateHistogramError(ClonetrackError):
        """No threshold separates the histogram (ref errors.py:20)."""

    class EmptyDistanceMapError(ClonetrackError):
        """Distance lookup on a map without foreground (ref errors.py:36)."""
