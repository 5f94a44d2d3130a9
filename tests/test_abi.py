"""The C-ABI library loads and exports every entry point include/qt.h declares
(no GPU needed: nothing here calls into the device)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qt.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qt_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1501_07800_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_boundary():
    names = _declared()
    for must in ["qt_ctx_create", "qt_create", "qt_multiply", "qt_truncate", "qt_read_back",
                 "qt_destroy", "qt_last_error", "qt_info"]:
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_wraps_every_declared_symbol():
    from paper_1501_07800_b200 import build
    build.build()
    from paper_1501_07800_b200 import qtmm
    assert sorted(qtmm.EXPORTED) == _declared()


def test_last_error_callable_without_gpu(lib):
    lib.qt_last_error.restype = ctypes.c_char_p
    assert lib.qt_last_error() == b""


def test_oracle_and_product_share_no_code():
    # the oracle never imports the product package and vice versa
    imp = re.compile(r"^\s*(import|from)\s+paper_1501_07800_b200|#include\s+[<\"].*(qt\.h|csrc)", re.M)
    for path in [os.path.join(ROOT, "oracle", "__init__.py"), os.path.join(ROOT, "oracle", "qt_oracle.c")]:
        assert not imp.search(open(path).read()), path
    pkg = os.path.join(ROOT, "paper_1501_07800_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
