"""Does the overlapped measurement upload slow the chains?  N = 1, bench.py's lt_small setup:
iterate alone vs async load + iterate vs staged load + iterate (device-event timed, 2 reps each)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2205_06327_b200.ptycho import Ptycho, PTYCHO_AMP_ASYNC  # noqa: E402

cfg = synth.CONFIGS["lt_small"]
n, S, H, W = cfg.n, cfg.slices, cfg.height, cfg.width
stream = torch.cuda.Stream(0)
p = Ptycho(n, S, H, W, cfg.sigma, cfg.prop_c, alpha=0.5, device=0, stream=stream.cuda_stream)
p.set_tiles(*cfg.grid, n // 2)
p.set_scan(synth.scan_centers(H, W, cfg.scan_ny, cfg.scan_nx))
p.allocate_workspace()
p.set_probe(synth.probe(n, cfg.defocus_nm).astype(np.complex64))
p.set_volume(None)
nloc = len(p.local_probes())
host_amp = torch.empty((nloc, n, n), dtype=torch.float32, pin_memory=True)
host_amp.uniform_()


def timed(fn, reps=2):
    out = []
    for _ in range(reps):
        p.synchronize()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        p.synchronize()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return out


p.load_measurements(host_amp)
p.iterate()
res = {"chunk": os.environ.get("PTYCHO_AMP_CHUNK", "8")}
res["iterate_ms"] = timed(lambda: p.iterate())
res["async_load_iterate_ms"] = timed(lambda: (p.load_measurements(host_amp, flags=PTYCHO_AMP_ASYNC), p.iterate()))
res["staged_load_iterate_ms"] = timed(lambda: (p.load_measurements(host_amp), p.iterate()))
scratch = torch.empty_like(host_amp, device="cuda")
side = torch.cuda.Stream(0)


def raw_copy_then_iterate():
    ev = torch.cuda.Event()
    ev.record(stream)
    with torch.cuda.stream(side):
        side.wait_event(ev)
        scratch.copy_(host_amp, non_blocking=True)
    p.iterate()
    stream.wait_stream(side)


res["raw_dma_concurrent_iterate_ms"] = timed(raw_copy_then_iterate)
evs = [torch.cuda.Event() for _ in range(len(host_amp) // 8 + 1)]


def raw_chunked_then_iterate():
    ev = torch.cuda.Event()
    ev.record(stream)
    with torch.cuda.stream(side):
        side.wait_event(ev)
        for i, c in enumerate(range(0, len(host_amp), 8)):
            scratch[c:c + 8].copy_(host_amp[c:c + 8], non_blocking=True)
            evs[i].record(side)
    p.iterate()
    stream.wait_stream(side)


res["raw_chunked_dma_concurrent_iterate_ms"] = timed(raw_chunked_then_iterate)
import time  # noqa: E402
hs = []
for _ in range(2):
    p.synchronize()
    t0 = time.perf_counter()
    p.load_measurements(host_amp, flags=PTYCHO_AMP_ASYNC)
    hs.append(time.perf_counter() - t0)
    p.synchronize()
res["async_load_call_host_s"] = hs
res["iterate_ms_2"] = timed(lambda: p.iterate())
print(json.dumps(res), flush=True)
p.close()
