"""The C-ABI library loads and exports exactly what include/bfq.h and bfr.h declare."""

import os
import re

from conftest import ROOT
from paper_2605_28475_b200 import _lib


def header_functions(header="bfq.h", prefix="bfq"):
    text = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(rf"^\s*(?:int|const char\*)\s+({prefix}_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = _lib.lib()
    names = header_functions()
    assert names, "no functions parsed from bfq.h"
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(_lib.EXPORTED_SYMBOLS) == names
    bfr = header_functions("bfr.h", "bfr")
    assert bfr, "no functions parsed from bfr.h"
    for name in bfr:
        assert hasattr(lib, name), name
    assert sorted(_lib.EXPORTED_SYMBOLS_BFR) == bfr


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
