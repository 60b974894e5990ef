"""The C ABI library loads and exports every symbol include/hpeel_b200.h
declares (no compute calls that need a GPU)."""
import ctypes
import os
import re

import paper_2205_03406_b200 as hp
from paper_2205_03406_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols(path=os.path.join(ROOT, "include", "hpeel_b200.h")):
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hp_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert set(declared_symbols()) == set(_lib.exported_symbols())


def test_probe_entry_points_are_not_in_the_public_header():
    """The K2 switches and parity probes live in the internal probe header
    (csrc/hpeel_probe.h), not in the drop-in boundary."""
    probe = declared_symbols(os.path.join(ROOT, "paper_2205_03406_b200", "csrc", "hpeel_probe.h"))
    public = declared_symbols()
    assert probe and not set(probe) & set(public)
    assert not [n for n in public if n.startswith("hp_debug")]
    assert set(probe) == set(_lib.probe_symbols())
    lib = ctypes.CDLL(_lib.LIB_PATH)
    assert all(hasattr(lib, n) for n in probe)


def test_library_is_sm100a():
    """The fat binary carries sm_100a SASS (cuobjdump lists the arch)."""
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_missing_library_fails_loudly(monkeypatch):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/libhpeel_b200.so")
    try:
        _lib.lib()
        raise AssertionError("expected RuntimeError")
    except RuntimeError as e:
        assert "no CPU fallback" in str(e)
