"""Small workload for compute-sanitizer ("tested by data-race
detectors"): the tiny config's hot path through the C ABI, exercising the PDL pre-wait prefetch
(TMA / cp.async issued before griddepcontrol.wait), the device cursor advance by the last CTA, the
CUDA-graph chains of 4 concurrent tiles, the batched schedule, the stash-free adjoint, the HVE
exchange, the APPP local hops and the accumulated step.

  compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_tiny.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2205_06327_b200.ptycho import Ptycho, PTYCHO_F_STASH_FREE  # noqa: E402

c = synth.CONFIGS["tiny"]
centers = synth.scan_centers(c.height, c.width, c.scan_ny, c.scan_nx)
probe = synth.probe(c.n, c.defocus_nm).astype(np.complex64)
vt = synth.volume(0, c.slices, c.height, c.width)


def run(grid, flags=0, batched=False, hve=False, iters=2):
    p = Ptycho(c.n, c.slices, c.height, c.width, c.sigma, c.prop_c, alpha=1.0, flags=flags, pass_period=5)
    if hve:
        p.set_tiles_hve(grid[0], grid[1], 32, 32)
    else:
        p.set_tiles(grid[0], grid[1], c.n // 2)
    p.set_scan(centers)
    if batched:
        p.set_schedule(True, 4)
    p.allocate_workspace()
    p.set_probe(probe)
    p.set_volume(vt)
    p.simulate_measurements()
    p.set_volume(0.5 * vt)
    losses = [p.iterate(want_loss=True) for _ in range(iters)]
    out = p.stitch()
    p.close()
    print(grid, "flags", flags, "batched", batched, "hve", hve, "losses", losses, "V", float(np.abs(out).sum()))


run((2, 2))
run((1, 1))
run((2, 2), batched=True)
run((2, 2), flags=PTYCHO_F_STASH_FREE)
run((2, 2), hve=True)
print("sanitize_tiny done")
