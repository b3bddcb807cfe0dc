"""Where the e2e leg's extra time goes at N ranks (bench.py's lt_small setup, torchrun): raw pinned
H2D bandwidth (all ranks at once and one rank at a time), load_measurements (staged and async),
stitch to pinned host memory on rank 0, one iterate().  Wall-clock around synchronised phases,
max over ranks.  Prints one JSON line on rank 0."""
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2205_06327_b200.ptycho import Ptycho, PTYCHO_AMP_ASYNC  # noqa: E402


def main():
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = synth.CONFIGS["lt_small"]
    R, C = cfg.grid
    nt = R * C
    owner = [k * world // nt for k in range(nt)]
    nid = None
    if world > 1:
        obj = [Ptycho.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    n, S, H, W = cfg.n, cfg.slices, cfg.height, cfg.width
    p = Ptycho(n, S, H, W, cfg.sigma, cfg.prop_c, alpha=0.5, device=local)
    p.set_tiles(R, C, n // 2, owner, nid, rank, world)
    p.set_scan(synth.scan_centers(H, W, cfg.scan_ny, cfg.scan_nx))
    p.allocate_workspace()
    p.set_probe(synth.probe(n, cfg.defocus_nm).astype(np.complex64))
    p.set_volume(None)
    nloc = len(p.local_probes())
    host_amp = torch.empty((nloc, n, n), dtype=torch.float32, pin_memory=True)
    host_amp.uniform_()
    host_v = torch.empty((S, H, W), dtype=torch.float32, pin_memory=True) if rank == 0 else None
    dev = torch.empty((nloc, n, n), dtype=torch.float32, device="cuda")

    def sync():
        torch.cuda.synchronize()
        p.synchronize()
        if world > 1:
            dist.barrier()

    def timed(fn):
        sync()
        t0 = time.perf_counter()
        fn()
        p.synchronize()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        return dt

    out = {"world": world, "bytes_per_rank": host_amp.numel() * 4}
    p.load_measurements(host_amp)  # warm
    p.iterate()
    out["raw_h2d_all_s"] = timed(lambda: dev.copy_(host_amp, non_blocking=True))
    alone = []
    for r in range(world):
        def f(r=r):
            if rank == r:
                dev.copy_(host_amp, non_blocking=True)
        alone.append(timed(f))
    out["raw_h2d_one_at_a_time_s"] = alone
    out["load_staged_s"] = timed(lambda: p.load_measurements(host_amp))
    out["load_async_s"] = timed(lambda: p.load_measurements(host_amp, flags=PTYCHO_AMP_ASYNC))
    out["stitch_host_s"] = timed(lambda: p.stitch(host_v, root=0, rank=rank))
    out["iterate_s"] = timed(lambda: p.iterate())
    out["e2e_step_serial_s"] = timed(lambda: (p.load_measurements(host_amp), p.iterate(),
                                              p.stitch(host_v, root=0, rank=rank)))
    out["e2e_step_async_s"] = timed(lambda: (p.load_measurements(host_amp, flags=PTYCHO_AMP_ASYNC), p.iterate(),
                                             p.stitch(host_v, root=0, rank=rank)))
    gb = out["bytes_per_rank"] / 1e9
    out["raw_h2d_all_gbs_per_rank"] = gb / out["raw_h2d_all_s"]
    out["raw_h2d_alone_gbs"] = [gb / t for t in alone]
    if rank == 0:
        print(json.dumps(out), flush=True)
    p.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
