"""The C-ABI library builds for sm_100a, loads, and exports every symbol of
include/trmcr.h (no compute calls: no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "trmcr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(trmcr_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1009_2768_b200 import build
    return build.build()


def test_header_declares_the_boundary():
    names = _declared()
    for f in ("trmcr_init", "trmcr_step", "trmcr_moments", "trmcr_stats", "trmcr_destroy"):
        assert f in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for name in _declared():
        assert hasattr(lib, name), name
    lib.trmcr_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.trmcr_version()


def test_sass_is_sm100a(libpath):
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump missing")
    out = subprocess.run([exe, "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_in_product_path():
    """The product package never imports, links or loads the oracle."""
    pkg = os.path.join(ROOT, "paper_1009_2768_b200")
    bad = re.compile(r"(import\s+oracle|from\s+oracle|trmcr_oracle|liborc|orc_[a-z])")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not bad.search(txt), f
