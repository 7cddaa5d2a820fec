"""Import the live reference (read-only) for oracle pinning -- test helper.

Only usable in the build container, where /root/reference exists.  The
reference imports ``tifffile`` at module top (ref imaging.py:16) but the hot
path never touches TIFF, so a module stub is enough.
"""

from __future__ import annotations

import os
import sys
import types

REF_SRC = "/root/reference/pkg/src"


def available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "clonetrack"))


def clonetrack():
    if not available():
        raise ImportError("reference not present")
    if "tifffile" not in sys.modules:
        try:
            import tifffile  # noqa: F401
        except ImportError:
            stub = types.ModuleType("tifffile")

            def _missing(*a, **k):
                raise RuntimeError("tifffile stub: TIFF I/O is off the hot path")

            stub.imread = stub.imwrite = _missing
            stub.TiffFile = _missing
            sys.modules["tifffile"] = stub
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import clonetrack  # noqa: F401
    import clonetrack.denoise
    import clonetrack.segment

    return clonetrack
