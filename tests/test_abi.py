"""CPU-only checks of the C-ABI boundary: the library loads, exports exactly what
include/ptycho.h declares, and validates arguments before touching a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "ptycho.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ptycho_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2205_06327_b200 import ptycho
    declared = header_functions()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(ptycho.lib, name), name
    assert sorted(ptycho.EXPORTED) == declared


def test_create_rejects_bad_config_without_gpu():
    from paper_2205_06327_b200 import ptycho
    cfg = ptycho.ptycho_config(100, 2, 64, 64, 0.1, 3.1, 1.0, 1.0, 1e-4, 0, 0)
    h = ctypes.c_void_p()
    st = ptycho.ptycho_create(ctypes.byref(cfg), 0, None, ctypes.byref(h))
    assert st == 1  # EARG, checked before any device call
    assert b"64, 256, 1024" in ptycho.ptycho_last_error(None)
    cfg = ptycho.ptycho_config(64, 2, 64, 64, 0.1, 3.1, 1.0, 1.0, 1e-4, -1, 0)
    assert ptycho.ptycho_create(ctypes.byref(cfg), 0, None, ctypes.byref(h)) == 1


def test_header_documents_every_call():
    src = open(os.path.join(ROOT, "include", "ptycho.h")).read()
    for name in header_functions():
        i = src.index(name + "(")
        assert "/*" in src[max(0, i - 1200):i], f"{name} lacks a comment"


def test_binding_fails_loudly_without_the_library(tmp_path):
    """No CPU or PyTorch fallback: with the shared library missing, importing the binding raises."""
    import subprocess
    import sys
    code = "import paper_2205_06327_b200.ptycho"
    env = dict(os.environ, PTYCHO_LIB=str(tmp_path / "missing.so"))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=ROOT)
    assert out.returncode != 0
    assert "ImportError" in out.stderr or "OSError" in out.stderr
