"""The C-ABI library loads and exports every symbol include/ct.h declares
(no kernel launches: runs without a GPU)."""

import os
import re
import subprocess

from conftest import ROOT


def header_functions():
    src = open(os.path.join(ROOT, "include", "ct.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ct_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_binding():
    from paper_1407_2089_b200 import _lib

    assert header_functions() == sorted(_lib.exported_symbols())


def test_library_exports_every_header_symbol():
    from paper_1407_2089_b200 import _lib

    L = _lib.lib()
    for name in header_functions():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (ct_[a-z0-9_]+)$", out, flags=re.M))
    assert set(header_functions()) <= exported
    assert L.ct_version().startswith(b"libct")


def test_workspace_sizes_are_sane():
    from paper_1407_2089_b200 import _lib

    n = 1024 * 1024 * 64
    assert _lib.workspace_bytes(0, 1024, 1024, 64) == 2 * n * 8
    assert _lib.workspace_bytes(2, 1024, 1024, 64, 1 << 20) > n * 4
    assert _lib.workspace_bytes(3, 1024, 1024, 64) >= 5 * n


def test_library_is_sm100a():
    from paper_1407_2089_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
