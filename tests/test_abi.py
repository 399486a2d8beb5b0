"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/dialsort.h
declares (no compute calls: this runs on the CPU-only build host)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dialsort.h")


@pytest.fixture(scope="module")
def libpath():
    import __graft_entry__
    return __graft_entry__.build_lib()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dialsort_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for must in ("dialsort_histogram", "dialsort_reconstruct", "dialsort_sort", "dialsort_sort_int32"):
        assert must in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    for n in declared_functions():
        assert re.search(r"\bT %s$" % n, out, flags=re.M), n


def test_binding_names_match_header(libpath):
    from paper_2605_16667_b200 import _lib
    assert sorted(_lib.EXPORTS) == declared_functions()


def test_status_strings_without_gpu(libpath):
    lib = ctypes.CDLL(libpath)
    lib.dialsort_status_string.restype = ctypes.c_char_p
    assert lib.dialsort_status_string(0) == b"ok"
    assert b"key" in lib.dialsort_status_string(2)
    assert lib.dialsort_version() >= 100


def test_kernels_are_sm100a(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
