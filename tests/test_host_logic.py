"""CPU tests of the library's host logic (geometry, APPP hop schedule) and of the N>1 exchange
protocol: world_size 2 and 4 gloo process groups execute the library's hop list with blocking
P2P send/recv, in the global order every rank follows (no barrier), and must reproduce the
oracle's global sum bit-exactly on every extended rect (north_star APPP invariant)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import ptycho_oracle as O

GRIDS = [((96, 96), (3, 3), 8), ((96, 96), (3, 3), 40), ((60, 90), (4, 3), 7), ((192, 192), (2, 4), 64),
         ((101, 77), (2, 3), 33), ((1536, 1536), (2, 4), 512), ((50, 70), (1, 3), 11), ((70, 50), (3, 1), 11)]


@pytest.mark.parametrize("shape,grid,halo", GRIDS)
def test_library_geometry_matches_oracle(shape, grid, halo):
    from paper_2205_06327_b200.ptycho import tile_geometry
    lib = tile_geometry(shape[0], shape[1], grid[0], grid[1], halo)
    ora = O.tile_geometry(shape[0], shape[1], grid[0], grid[1], halo)
    assert [(e, i) for e, i in lib] == [(t["ext"], t["interior"]) for t in ora]


@pytest.mark.parametrize("shape,grid,halo", GRIDS)
def test_schedule_message_budget(shape, grid, halo):
    from paper_2205_06327_b200.ptycho import appp_schedule
    hops = appp_schedule(shape[0], shape[1], grid[0], grid[1], halo)
    r, c = grid
    assert len(hops) == 2 * (r - 1) * c + 2 * (c - 1) * r
    # vertical hops first (forward then backward), then horizontal
    nv = 2 * (r - 1) * c
    assert all(abs(h[0] - h[1]) == c for h in hops[:nv])
    assert all(abs(h[0] - h[1]) == 1 for h in hops[nv:])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, shape, grid, halo, slices, q):
    import torch
    import torch.distributed as dist
    from paper_2205_06327_b200.ptycho import appp_schedule, tile_geometry
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tiles = tile_geometry(shape[0], shape[1], grid[0], grid[1], halo)
    nt = len(tiles)
    owner = [k * world // nt for k in range(nt)]  # bench.py's mapping
    rng = np.random.default_rng(7)
    init = [rng.integers(0, 2 ** 16, (slices, e[2] - e[0], e[3] - e[1])).astype(np.float32) for e, _ in tiles]
    bufs = {k: init[k].copy() for k in range(nt) if owner[k] == rank}
    for (src, dst, y0, y1, x0, x1, add) in appp_schedule(shape[0], shape[1], grid[0], grid[1], halo):
        if y1 <= y0 or x1 <= x0:
            continue
        es, ed = tiles[src][0], tiles[dst][0]
        if owner[src] == rank:
            payload = bufs[src][:, y0 - es[0]:y1 - es[0], x0 - es[1]:x1 - es[1]].copy()  # snapshot
        if owner[src] == rank and owner[dst] != rank:
            dist.send(torch.from_numpy(payload), dst=owner[dst])
        if owner[dst] == rank:
            if owner[src] != rank:
                t = torch.empty((slices, y1 - y0, x1 - x0), dtype=torch.float32)
                dist.recv(t, src=owner[src])
                payload = t.numpy()
            view = bufs[dst][:, y0 - ed[0]:y1 - ed[0], x0 - ed[1]:x1 - ed[1]]
            if add:
                view += payload
            else:
                view[...] = payload
    total = O.global_sum([b.astype(np.float64) for b in init],
                         [dict(ext=e, interior=i) for e, i in tiles], slices, *shape)
    ok = all(np.array_equal(b.astype(np.float64), total[:, tiles[k][0][0]:tiles[k][0][2], tiles[k][0][1]:tiles[k][0][3]])
             for k, b in bufs.items())
    q.put((rank, ok, sorted(bufs)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("shape,grid,halo", [((192, 192), (2, 4), 64), ((101, 77), (2, 3), 33),
                                             ((96, 96), (3, 3), 40)])
def test_gloo_appp_protocol(world, shape, grid, halo):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, grid, halo, 3, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res
    owned = sorted(k for _, _, ks in res for k in ks)
    assert owned == list(range(grid[0] * grid[1]))
