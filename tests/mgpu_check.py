"""torchrun driver for tests/test_multigpu.py: the same reconstruction on N GPUs (tiles spread
over ranks, APPP hops over NCCL) and on one GPU (all tiles virtual) must be bit-identical; the
APPP integer check must equal the oracle's global sum on every tile."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ptycho_oracle as O  # noqa: E402
import synth  # noqa: E402
from paper_2205_06327_b200.ptycho import Ptycho  # noqa: E402


def problem():
    n, s, h, w = 64, 3, 150, 131
    rng = np.random.default_rng(3)
    probe = synth.probe(n, 8.0)
    vt = rng.random((s, h, w)).astype(np.float32)
    centers = synth.scan_centers(h, w, 5, 6)
    sigma, c = 0.3, 3.135
    full = (0, 0, h, w)
    amps = np.stack([O.farfield_magnitude(probe, O.window(vt.astype(np.float64), full, tuple(cc), n), sigma, c)
                     for cc in centers]).astype(np.float32)
    return n, s, h, w, sigma, c, probe, vt, centers, amps


def run(grid, owner, nid, rank, world, device, iters=2, period=0, hve=False):
    n, s, h, w, sigma, c, probe, vt, centers, amps = problem()
    p = Ptycho(n, s, h, w, sigma, c, alpha=1.0, alpha_acc=0.0 if hve else None, pass_period=period, device=device)
    if hve:  # Halo Voxel Exchange baseline: V copy-paste messages between ranks (NCCL)
        p.set_tiles_hve(grid[0], grid[1], 24, 25, owner, nid, rank, world)
    else:
        p.set_tiles(grid[0], grid[1], n // 2, owner, nid, rank, world)
    p.set_scan(centers)
    p.allocate_workspace()
    p.set_probe(probe.astype(np.complex64))
    p.load_measurements(amps[p.local_probes()])
    p.set_volume(0.5 * vt)
    losses = [p.iterate(want_loss=True) for _ in range(iters)]
    out = p.stitch(root=0, rank=rank)
    transport = p.appp_transport()
    p.close()
    return out, losses, transport


def main():
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ok = True
    for grid, period in [((2, 3), 0), ((2, 3), 4), ((3, 2), 0), ((2, 4), 0)]:
        nt = grid[0] * grid[1]
        owner = [k * world // nt for k in range(nt)]
        obj = [Ptycho.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        multi, lm, tr = run(grid, owner, obj[0], rank, world, local, period=period)
        want = os.environ.get("PTYCHO_APPP_TRANSPORT")
        if want in ("nccl", "p2p") and tr != want:
            print(f"rank {rank}: APPP transport {tr}, requested {want}", flush=True)
            ok = False
        if rank == 0:
            single, ls, _ = run(grid, None, None, 0, 1, local, period=period)
            same = np.array_equal(multi, single) and lm == ls
            print(f"grid {grid} T={period} transport {tr}: multi-GPU == single-GPU virtual tiles: {same}; "
                  f"losses {lm} {ls}", flush=True)
            ok &= same
        dist.barrier()
    for grid in [(2, 3), (2, 2)]:
        nt = grid[0] * grid[1]
        owner = [k * world // nt for k in range(nt)]
        obj = [Ptycho.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        multi, lm, _ = run(grid, owner, obj[0], rank, world, local, hve=True)
        if rank == 0:
            single, ls, _ = run(grid, None, None, 0, 1, local, hve=True)
            same = np.array_equal(multi, single) and lm == ls
            print(f"HVE grid {grid}: multi-GPU == single-GPU virtual tiles: {same}; losses {lm} {ls}", flush=True)
            ok &= same
        dist.barrier()
    # APPP integer bit-exactness across ranks
    shape, grid, halo, slices = (192, 192), (2, 4), 64, 5
    nt = grid[0] * grid[1]
    owner = [k * world // nt for k in range(nt)]
    obj = [Ptycho.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    p = Ptycho(64, slices, shape[0], shape[1], 0.1, 3.1, device=local)
    p.set_tiles(grid[0], grid[1], halo, owner, obj[0], rank, world)
    p.set_scan(synth.scan_centers(shape[0], shape[1], 2, 2))
    p.allocate_workspace()
    tiles = O.tile_geometry(shape[0], shape[1], grid[0], grid[1], halo)
    rng = np.random.default_rng(2)
    init = [rng.integers(0, 2 ** 16, (slices, t["ext"][2] - t["ext"][0], t["ext"][3] - t["ext"][1])).astype(np.float32)
            for t in tiles]
    for k in range(nt):
        if owner[k] == rank:
            p.debug_write_tile(k, 1, init[k])
    p.appp_passes()
    p.synchronize()
    if os.environ.get("PTYCHO_APPP_TRANSPORT") in ("nccl", "p2p"):
        ok &= p.appp_transport() == os.environ["PTYCHO_APPP_TRANSPORT"]
    total = O.global_sum([b.astype(np.float64) for b in init], tiles, slices, *shape)
    mine = all(np.array_equal(p.debug_read_tile(k, 1).astype(np.float64),
                              total[:, tiles[k]["ext"][0]:tiles[k]["ext"][2], tiles[k]["ext"][1]:tiles[k]["ext"][3]])
               for k in range(nt) if owner[k] == rank)
    flags = [None] * world
    dist.all_gather_object(flags, mine and ok)
    if rank == 0:
        print(f"APPP integer check over {world} ranks: {flags}", flush=True)
        ok &= all(flags)
    p.close()
    if rank == 0:
        print("MGPU OK" if ok else "MGPU FAIL", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
