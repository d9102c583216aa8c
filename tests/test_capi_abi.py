"""CPU checks of the drop-in boundary: the C-ABI library loads and exports
every entry point include/b2sr_sm100.h declares, and the ctypes binding
covers them all.  No compute calls (no GPU here)."""

import re
import subprocess
from pathlib import Path

import pytest

from paper_2201_08560_b200 import _build, _capi

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "b2sr_sm100.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(b2sr_\w+)\s*\(", text, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return _capi.lib()


def test_header_parses():
    names = declared()
    assert "b2sr_from_csr" in names and "b2sr_bfs" in names and len(names) >= 30


def test_every_declared_symbol_is_exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", str(_capi.library_path())],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (b2sr_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    for n in declared():
        assert hasattr(lib, n)


def test_binding_covers_header():
    assert sorted(_capi.SIGNATURES) == declared()


def test_error_mapping(lib):
    assert lib.b2sr_version() >= 100
    assert isinstance(_capi.launch_count(), int)
    # a call that fails validation before touching the device
    out = __import__("ctypes").c_void_p()
    with pytest.raises(ValueError):
        _capi.call("b2sr_from_csr", 4, 5, None, None, 0, None, __import__("ctypes").byref(out))
    assert "tile dim" in lib.b2sr_last_error().decode()


def test_sm100a_cubin():
    """The library carries sm_100a SASS (not PTX-only, not another arch)."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_capi.library_path())],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
