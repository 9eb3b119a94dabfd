"""CPU-only checks of the boundary: libaa builds for sm_100a, loads, and exports every
symbol include/*.h declares; argument errors are reported without a GPU."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2110_09667_b200 import build
    build.build()
    from paper_2110_09667_b200 import aa
    return aa


def _declared():
    names = set()
    for h in ("aa.h", "aa_testing.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(aa_[a-z_0-9]+)\s*\(", src))
    return names


def test_headers_declare_the_north_star_calls():
    d = _declared()
    for name in ("aa_create", "aa_init", "aa_step", "aa_delete_oldest", "aa_stats"):
        assert name in d


def test_every_declared_symbol_is_exported(lib):
    so = ctypes.CDLL(lib.LIB_PATH)
    for name in _declared():
        assert hasattr(so, name), name
    assert set(lib.EXPORTS) == _declared()
    out = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True, text=True).stdout
    for name in _declared():
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib.LIB_PATH],
                          capture_output=True, text=True).stdout
    assert "UBLKCP" in sass or "UTMALDG" in sass      # TMA bulk copies (cp.async.bulk)
    assert "DMMA" in sass                             # fp64 tensor-core Gram blocks


def test_argument_errors_without_gpu(lib):
    assert lib.aa_status_string(0) == "ok"
    assert "argument" in lib.aa_status_string(1)
    h = ctypes.c_void_p()
    # invalid sizes are rejected before touching the device
    assert lib._lib.aa_create(ctypes.byref(h), 0, 5, 0, 0, 1, None, None) == 1
    assert lib._lib.aa_create(ctypes.byref(h), 100, 65, 0, 0, 1, None, None) == 1
    assert lib._lib.aa_create(ctypes.byref(h), 100, 5, 7, 0, 1, None, None) == 1
    assert lib._lib.aa_create(ctypes.byref(h), 100, 5, 0, 0, 2, None, None) == 1   # p>1 needs an id
    assert lib._lib.aa_step(None, None, None, None) == 1
    assert lib._lib.aa_stats(None, None, 0) == 1
    info = lib.aa_build_info()
    assert "sm_100a" in info


def test_product_path_does_not_use_the_oracle():
    """The CUDA path and the oracle share no code; the package never imports oracle/."""
    pkg = os.path.join(ROOT, "paper_2110_09667_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).replace("oracle/", ""), f
