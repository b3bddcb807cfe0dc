"""Runs the hot path on small cases and prints, as JSON, the stitched V (hash + values) and the
debug error bits -- executed by tests/test_gpu_ordering.py under the product library and under the
PTYCHO_DEBUG_CHECKS library (PTYCHO_LIB) and with different launch modes (PTYCHO_NO_PDL,
PTYCHO_NO_GRAPH).  Not part of the product."""
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2205_06327_b200.ptycho import Ptycho, PTYCHO_F_STASH_FREE  # noqa: E402

CASES = {
    "tiny_2x2": dict(n=64, s=4, h=128, scan=(4, 4), grid=(2, 2), halo=32),
    "tiny_2x2_batched": dict(n=64, s=4, h=128, scan=(4, 4), grid=(2, 2), halo=32, batched=4),
    "tiny_2x2_stash_free": dict(n=64, s=4, h=128, scan=(4, 4), grid=(2, 2), halo=32, flags=PTYCHO_F_STASH_FREE),
    "tiny_hve": dict(n=64, s=4, h=128, scan=(4, 4), grid=(2, 2), halo=32, hve=32),
    "small_1x1": dict(n=256, s=6, h=512, scan=(8, 8), grid=(1, 1), halo=128),
    "small_2x2": dict(n=256, s=6, h=512, scan=(8, 8), grid=(2, 2), halo=128, period=5),
    "lt_2x4": dict(n=1024, s=4, h=1536, scan=(5, 6), grid=(2, 4), halo=512),
}


def run(name):
    c = CASES[name]
    n, s, h = c["n"], c["s"], c["h"]
    p = Ptycho(n, s, h, h, 0.1, 3.135, alpha=1024.0, flags=c.get("flags", 0), pass_period=c.get("period", 0))
    if "hve" in c:
        p.set_tiles_hve(*c["grid"], c["halo"], c["hve"])
    else:
        p.set_tiles(*c["grid"], c["halo"])
    p.set_scan(synth.scan_centers(h, h, *c["scan"]))
    if c.get("batched"):
        p.set_schedule(True, c["batched"])
    p.allocate_workspace()
    p.set_probe(synth.probe(n, 25.0 if n > 64 else 8.0).astype(np.complex64))
    vt = synth.volume(0, s, h, h)
    p.set_volume(vt)
    p.simulate_measurements()
    p.set_volume(0.5 * vt)
    losses = [p.iterate(want_loss=True) for _ in range(2)]
    v = p.stitch()
    bits, built = p.debug_errors()
    p.close()
    return {"case": name, "sha": hashlib.sha256(v.tobytes()).hexdigest(), "losses": losses, "bits": bits,
            "checks_built": built}


if __name__ == "__main__":
    for name in sys.argv[1:] or CASES:
        print(json.dumps(run(name)), flush=True)
