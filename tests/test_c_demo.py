"""The C boundary without Python: examples/ptycho_demo.c (plain C, cudaMalloc'd workspace,
built by __graft_entry__.build()) runs a small synthetic reconstruction through
include/ptycho.h and must see F(V) decrease."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_demo_reconstructs():
    from paper_2205_06327_b200 import build
    exe = build.DEMO if os.path.exists(build.DEMO) else build.build_demo(verbose=False)
    out = subprocess.run([exe, "64", "4", "256", "256", "12", "2", "2", "5"], capture_output=True, text=True,
                         timeout=300)
    print(out.stdout, out.stderr)
    assert out.returncode == 0 and "DEMO OK" in out.stdout
