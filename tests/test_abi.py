"""The C-ABI library builds, loads and exports every symbol include/fsfem.h declares (no GPU needed)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fsfem.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fsfem_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2001_08849_b200 import build
    so = build.build()
    return ctypes.CDLL(so)


def test_header_declares_the_north_star_entry_points():
    syms = declared_symbols()
    for s in ("fsfem_build_faces", "fsfem_assemble_csr", "fsfem_apply_bc", "fsfem_pcg_solve"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib._name]).decode()
    exported = set(re.findall(r" T (fsfem_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    from paper_2001_08849_b200.fsfem import EXPORTS
    assert sorted(EXPORTS) == declared_symbols()


def test_library_is_sm100a_only(lib):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib._name]).decode()
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_status_strings(lib):
    lib.fsfem_status_string.restype = ctypes.c_char_p
    assert lib.fsfem_status_string(0) == b"ok"
    assert lib.fsfem_status_string(2) == b"topology error"


def test_binding_fails_loudly_without_library(tmp_path):
    from paper_2001_08849_b200 import fsfem as B
    saved = B._lib
    try:
        B._lib = None
        with pytest.raises(OSError):
            B.load_library(str(tmp_path / "missing.so"))
    finally:
        B._lib = saved


def test_oracle_not_imported_by_product():
    pkg = os.path.join(ROOT, "paper_2001_08849_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).lower() or f == "build.py", f
