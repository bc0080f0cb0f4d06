"""The C-ABI library loads and exports exactly what include/bfq.h declares."""

import os
import re

from conftest import ROOT
from paper_2605_28475_b200 import _lib


def header_functions():
    text = open(os.path.join(ROOT, "include", "bfq.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(bfq_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = _lib.lib()
    names = header_functions()
    assert names, "no functions parsed from bfq.h"
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(_lib.EXPORTED_SYMBOLS) == names


def test_strerror_codes():
    lib = _lib.lib()
    for code in range(0, -10, -1):
        assert lib.bfq_strerror(code)
    assert lib.bfq_strerror(-1234) == b"unknown error"


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    try:
        _lib.lib()
    except _lib.EngineUnavailable:
        pass
    else:  # pragma: no cover
        raise AssertionError("missing engine must raise")
