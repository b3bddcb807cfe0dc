"""Ordering / race evidence for the hand-rolled protocols.  compute-sanitizer
is closed on this pool, so two checks of our own:

1. The PTYCHO_DEBUG_CHECKS library (lib/libptycho_debug.so, same arithmetic) re-reads, after
   griddepcontrol.wait, every V / AccBuf / stash word a pass prefetched (TMA / bulk copies) BEFORE
   its grid dependency resolved; any mismatch = a stale read of data the protocol claims was
   written >= 2 kernels earlier.  Covered: CUDA-graph + PDL chains of 4 concurrent tiles, the
   device cursor advance, the batched schedule, the stash-free adjoint's ring, HVE, N = 64 / 256 /
   1024.  The bits must be 0 and the results bit-identical to the product library.
2. Launch-mode invariance of the product library: graph + PDL (default), PDL off
   (PTYCHO_NO_PDL=1: every pass fully serialised after the previous one), graphs off
   (PTYCHO_NO_GRAPH=1), and for N <= 256 the opt-in cluster-resident chain (PTYCHO_CLUSTER=1:
   wavefield exchanged over DSMEM, cluster barriers instead of kernel boundaries) -- a race in the
   pre-wait prefetch or in the DSMEM exchange would make these differ.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEBUG_LIB = os.path.join(ROOT, "paper_2205_06327_b200", "lib", "libptycho_debug.so")
CASES = ["tiny_2x2", "tiny_2x2_batched", "tiny_2x2_stash_free", "tiny_hve", "small_1x1", "small_2x2", "lt_2x4"]


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ordering_run.py")] + CASES, env=env,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    return {d["case"]: d for d in (json.loads(l) for l in out.stdout.splitlines() if l.startswith("{"))}


@pytest.fixture(scope="module")
def product():
    return _run({})


def test_debug_checks_see_no_stale_prefetch(product):
    assert os.path.exists(DEBUG_LIB), "build() makes lib/libptycho_debug.so"
    dbg = _run({"PTYCHO_LIB": DEBUG_LIB})
    for name in CASES:
        print(name, dbg[name]["bits"], dbg[name]["losses"])
        assert dbg[name]["checks_built"]
        assert dbg[name]["bits"] == 0, (name, dbg[name]["bits"])
        assert dbg[name]["sha"] == product[name]["sha"], name  # the checks only read


@pytest.mark.parametrize("mode", [{"PTYCHO_NO_PDL": "1"}, {"PTYCHO_NO_GRAPH": "1"}, {"PTYCHO_CLUSTER": "1"}])
def test_launch_mode_invariance(product, mode):
    other = _run(mode)
    for name in CASES:
        assert other[name]["sha"] == product[name]["sha"], (name, mode)
        assert other[name]["losses"] == product[name]["losses"], (name, mode)
