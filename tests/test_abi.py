"""Host-side checks of the C-ABI library (no compute calls without a GPU)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "mmsb.h")).read()
    return sorted(set(re.findall(r"\b(mmsb_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2302_07992_b200 import build

    path = build.build()
    return C.CDLL(path)


def test_exports_every_declared_symbol(lib):
    syms = _declared_symbols()
    assert len(syms) >= 9
    for s in syms:
        assert hasattr(lib, s), s


def test_workspace_and_validation(lib):
    from paper_2302_07992_b200.mmsb import _Shape

    lib.mmsb_workspace_bytes.restype = C.c_size_t
    ok = _Shape(0, 1000, 512, 512, 7)
    assert lib.mmsb_workspace_bytes(C.byref(ok)) > 0
    for bad in [_Shape(0, 1, 500, 512, 7), _Shape(0, 1, 8, 8, 7), _Shape(2, 1, 64, 64, 7), _Shape(1, 1, 64, 64, 8),
                _Shape(0, 0, 64, 64, 7), _Shape(0, 1, 64, 64, 7, 0, 9), _Shape(1, 1, 64, 64, 7, 0, 16)]:
        assert lib.mmsb_workspace_bytes(C.byref(bad)) == 0
    # null pointers are rejected synchronously, before any CUDA call
    lib.mmsb_content_owner_encode.restype = C.c_int
    assert lib.mmsb_content_owner_encode(C.byref(ok), None, None, None, None, None, None, None, C.c_size_t(0),
                                         None) == 2


def test_der_psnr_host(lib):
    import math

    import numpy as np

    from paper_2302_07992_b200 import mmsb as G

    der, psnr = G.der_psnr(512, 512, [1000, 7], [65025, 0])
    assert der[0] == 1000 / 262144 and psnr[1] == math.inf
    assert abs(psnr[0] - 54.1854) < 5e-5
    import oracle as O

    d, p = O.der_psnr(512, 512, 1000, 65025)
    assert d == der[0] and abs(p - psnr[0]) < 1e-12


def test_status_strings(lib):
    lib.mmsb_status_string.restype = C.c_char_p
    for code in (0, 2, 3, 4, 5, 6, 7, 8):
        assert lib.mmsb_status_string(code)


def test_product_path_has_no_oracle_import():
    pkg = os.path.join(ROOT, "paper_2302_07992_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "mmsb_oracle" not in txt and "orc_" not in txt, f


def test_header_is_clean_c():
    """include/mmsb.h compiles as plain C with every warning an error (no torch / C++ types)."""
    import shutil
    import subprocess

    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    hdr = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "mmsb.h")
    r = subprocess.run([gcc, "-fsyntax-only", "-Wall", "-Wextra", "-Werror", "-x", "c", hdr], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr
