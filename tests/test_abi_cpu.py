"""CPU-side checks of the boundary: the C-ABI library builds, loads and exports every
entry point include/lc.h declares; host-side argument errors are reported without a GPU."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "lc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lc_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2603_17201_b200 import build, _lib
    build.build()
    return _lib.load()


def test_header_declares_the_four_entry_points():
    d = _declared()
    for fn in ("lc_upload_map", "lc_correct_sim3", "lc_search_by_projection", "lc_fuse"):
        assert fn in d


def test_library_exports_every_declared_symbol(lib):
    from paper_2603_17201_b200 import _lib
    so = _lib.LIB_PATH
    out = subprocess.check_output(["nm", "-D", "--defined-only", so], text=True)
    exported = set(re.findall(r"\bT\s+(lc_[a-z_0-9]+)", out))
    for fn in _declared():
        assert fn in exported, fn
        assert hasattr(lib, fn)
    assert set(_lib.exported_symbols()) == set(_declared())


def test_sm100a_code_in_library(lib):
    from paper_2603_17201_b200 import _lib
    out = subprocess.check_output(["cuobjdump", "--list-elf", _lib.LIB_PATH], text=True)
    assert "sm_100a" in out


def test_null_and_no_device_errors(lib):
    from paper_2603_17201_b200 import _lib
    h = C.c_void_p()
    assert lib.lc_create(None, 0) == _lib.LC_EINVAL
    st = lib.lc_create(C.byref(h), 0)
    import torch
    if not torch.cuda.is_available():
        assert st == _lib.LC_ECUDA
        assert len(lib.lc_last_error(None)) > 0
    else:
        assert st == 0
        lib.lc_destroy(h)
    assert lib.lc_destroy(None) == _lib.LC_EINVAL
    assert lib.lc_fuse(None, 3, 0, 0, 0, None, None, None, None, 0, None, -1, None, None, None, None,
                       None, None, None) == _lib.LC_EINVAL
    assert lib.lc_correct_sim3(None, 1, 1, None, None, None, None, None, None, None, None, None, 0, None,
                               None) == _lib.LC_EINVAL


def test_binding_fails_loudly_without_library(monkeypatch, tmp_path):
    from paper_2603_17201_b200 import _lib
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.load()


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2603_17201_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "lc_oracle" not in txt and "liboracle" not in txt, f
