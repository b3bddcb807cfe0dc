"""Where does the e2e step lose time against the device-only step?  LT-small, 2x4 virtual tiles,
one B200: times (CUDA events on the context stream) iterate alone, async load + iterate, sync
load + iterate, and stitch to pinned host memory."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2205_06327_b200.ptycho import Ptycho, PTYCHO_AMP_ASYNC  # noqa: E402

c = synth.CONFIGS["lt_small"]
stream = torch.cuda.Stream(0)
p = Ptycho(c.n, c.slices, c.height, c.width, c.sigma, c.prop_c, alpha=0.5, stream=stream.cuda_stream)
p.set_tiles(2, 4, c.n // 2)
p.set_scan(synth.scan_centers(c.height, c.width, c.scan_ny, c.scan_nx))
p.allocate_workspace()
p.set_probe(synth.probe(c.n, c.defocus_nm).astype(np.complex64))
p.set_volume(synth.volume(0, c.slices, c.height, c.width))
p.simulate_measurements()
p.set_volume(None)
nloc = len(p.local_probes())
host = torch.empty((nloc, c.n, c.n), dtype=torch.float32, pin_memory=True)
p.read_measurements(0, nloc, host)
hv = torch.empty((c.slices, c.height, c.width), dtype=torch.float32, pin_memory=True)
p.iterate()
p.synchronize()


def timed(fn, label):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    fn()
    e1.record(stream)
    p.synchronize()
    print(f"{label}: {e0.elapsed_time(e1):.1f} ms (host wall {1e3 * (time.perf_counter() - t0):.1f} ms)", flush=True)


for rep in range(2):
    timed(lambda: (p.load_measurements(host), p.iterate()), "sync load + iterate")
    timed(lambda: (p.load_measurements(host, flags=PTYCHO_AMP_ASYNC), p.iterate()),
          f"async load (chunk {os.environ.get('PTYCHO_AMP_CHUNK', 8)}) + iterate")
    timed(lambda: p.iterate(), "iterate")
