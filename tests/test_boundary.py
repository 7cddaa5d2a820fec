"""Drop-in boundary checks that need no GPU: exception identity with the
reference (ref errors.py:4-50, caught at ref cli.py:57/:83/:126 and
server.py:224) and the ct_cell row layout (include/ct.h)."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.join(ROOT, "tests")


def _run(code: str):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ROOT, TESTS]))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    return r.stdout


def test_errors_alias_reference_when_importable():
    import _refimport

    if not _refimport.available():
        pytest.skip("reference not present (GPU box)")
    out = _run(
        "import _refimport; ct = _refimport.clonetrack()\n"
        "import clonetrack.errors as R\n"
        "import paper_1407_2089_b200.errors as E\n"
        "assert E.REFERENCE_BOUND\n"
        "for n in ('ClonetrackError','ManifestError','ParameterError','DegenerateHistogramError',"
        "'EmptyDistanceMapError'):\n"
        "    assert getattr(E, n) is getattr(R, n), n\n"
        "from paper_1407_2089_b200 import SegmentationConfig\n"
        "try:\n"
        "    SegmentationConfig(min_volume_um3=-1)\n"
        "except (R.EditError, R.ParameterError) as e:\n"  # the reference server's handler (server.py:224)
        "    print('caught', type(e).__name__)\n"
    )
    assert "caught ParameterError" in out


def test_errors_standalone_without_reference():
    out = _run(
        "import sys; sys.modules['clonetrack'] = None\n"  # makes `import clonetrack` fail
        "import paper_1407_2089_b200.errors as E\n"
        "assert not E.REFERENCE_BOUND\n"
        "assert issubclass(E.ParameterError, E.ClonetrackError)\n"
        "assert issubclass(E.DegenerateHistogramError, E.ClonetrackError)\n"
        "assert issubclass(E.EmptyDistanceMapError, E.ClonetrackError)\n"
        "assert issubclass(E.ManifestError, E.ClonetrackError)\n"
        "print('ok')\n"
    )
    assert "ok" in out


def test_cell_row_layout_matches_header():
    """CELL_DTYPE (Python view of ct_cell) follows include/ct.h field for field."""
    import re

    from paper_1407_2089_b200._lib import CELL_DTYPE

    hdr = open(os.path.join(ROOT, "include", "ct.h")).read()
    body = hdr[hdr.index("typedef struct ct_cell {"):hdr.index("} ct_cell;")]
    fields = re.findall(r"^\s+(int64_t|double)\s+(\w+)(?:\[(\d)\])?;", body, re.M)
    assert [f[1] for f in fields] == list(CELL_DTYPE.names)
    for typ, name, n in fields:
        dt, shape = CELL_DTYPE.fields[name][0].base, CELL_DTYPE.fields[name][0].shape
        assert dt.kind == ("f" if typ == "double" else "i") and dt.itemsize == 8
        assert shape == ((int(n),) if n else ())
    assert CELL_DTYPE.itemsize == 128
