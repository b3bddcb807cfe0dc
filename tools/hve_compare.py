"""Gradient Decomposition vs the Halo Voxel Exchange baseline on the same B200 (
PAPER.md §Results, Tables II/III memory rows, Fig. artifact).

  python tools/hve_compare.py perf   # LT-small shape, 2x4 virtual tiles on one GPU: s/iteration,
                                     # probe-locations/s, per-GPU workspace, per-tile voxels/probes
  python tools/hve_compare.py seam   # lattice phantom, 2x2 tiles: seam score of GD, HVE, 1x1

Paper settings: GD halo 600 pm = 60 px; HVE halo 890 pm = 89 px and two extra rows of
probe locations (margin = 2 scan steps).  Prints one JSON line per measurement."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402


def make(c, method, grid, halo, margin, alpha, alpha_acc=None):
    from paper_2205_06327_b200.ptycho import Ptycho
    p = Ptycho(c.n, c.slices, c.height, c.width, c.sigma, c.prop_c, alpha=alpha,
               alpha_acc=(0.0 if method == "hve" else alpha) if alpha_acc is None else alpha_acc)
    if method == "hve":
        p.set_tiles_hve(grid[0], grid[1], halo, margin)
    else:
        p.set_tiles(grid[0], grid[1], halo)
    p.set_scan(synth.scan_centers(c.height, c.width, c.scan_ny, c.scan_nx))
    ws = p.allocate_workspace()
    p.set_probe(synth.probe(c.n, c.defocus_nm).astype(np.complex64))
    return p, ws


def tile_report(p, c):
    rows = []
    for k in range(p.rows * p.cols):
        (y0, x0, y1, x1), _ = p.tile_rect(k)
        rows.append({"tile": k, "voxels": (y1 - y0) * (x1 - x0) * c.slices, "probes": p.tile_probe_count(k)})
    return rows


def perf(steps=2):
    import torch
    c = synth.CONFIGS["lt_small"]
    step = c.height / c.scan_ny
    for method, halo, margin in [("gd", 60, 0), ("hve", 89, int(round(2 * step))), ("gd", 512, 0)]:
        p, ws = make(c, method, c.grid, halo, margin, alpha=0.5)
        p.set_volume(synth.volume(0, c.slices, c.height, c.width))
        p.simulate_measurements()
        p.set_volume(None)
        p.iterate()
        p.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            p.iterate()
        e1.record()
        p.synchronize()
        sec = e0.elapsed_time(e1) / steps / 1e3
        tiles = tile_report(p, c)
        print(json.dumps({"study": "hve_vs_gd_perf", "method": method, "workload": "lt_small 2x4 virtual tiles, 1 GPU",
                          "halo": halo, "margin": margin, "sec_per_iteration": sec,
                          "probe_locations_per_s": c.n_probes / sec,
                          "probe_chains_per_iteration": sum(t["probes"] for t in tiles),
                          "workspace_gb": ws / 1e9,
                          "max_tile_voxels": max(t["voxels"] for t in tiles),
                          "max_tile_measurement_gb": max(t["probes"] for t in tiles) * c.n * c.n * 4 / 1e9,
                          "per_gpu_8way_gb_model": (max(t["voxels"] for t in tiles) * (4 if method == "hve" else 8)
                                                    + max(t["probes"] for t in tiles) * c.n * c.n * 4) / 1e9,
                          "tiles": tiles}), flush=True)
        p.close()


def seam_score(err, height, width, rows, cols):
    """mean |jump| of err across tile borders / mean |jump| elsewhere (SPEC SeamScore)."""
    ys = [height // rows * r for r in range(1, rows)]
    xs = [width // cols * q for q in range(1, cols)]
    dy, dx = np.abs(np.diff(err, axis=1)), np.abs(np.diff(err, axis=2))
    by, bx = np.zeros(dy.shape[1], bool), np.zeros(dx.shape[2], bool)
    by[[y - 1 for y in ys]] = True
    bx[[x - 1 for x in xs]] = True
    border = np.concatenate([dy[:, by, :].ravel(), dx[:, :, bx].ravel()])
    inner = np.concatenate([dy[:, ~by, :].ravel(), dx[:, :, ~bx].ravel()])
    return float(border.mean() / inner.mean())


def seam(iters=20):
    base = synth.CONFIGS["small"]
    c = synth.Config("seam", 256, 8, 512, 512, 16, 16, (2, 2), 128)
    vt = synth.lattice_phantom(0, c.slices, c.height, c.width, amplitude=1.0)
    step = c.height / c.scan_ny
    out = {}
    for name, method, grid, halo, margin in [("single_tile", "gd", (1, 1), 0, 0), ("gd_halo60", "gd", (2, 2), 60, 0),
                                             ("gd_exact", "gd", (2, 2), 128, 0),
                                             ("hve_halo89", "hve", (2, 2), 89, int(round(2 * step)))]:
        p, _ = make(c, method, grid, halo, margin, alpha=256.0)
        p.set_volume(vt)
        p.simulate_measurements()
        p.set_volume(None)
        losses = [p.iterate(want_loss=True) for _ in range(iters)]
        v = p.stitch()
        p.close()
        err = v.astype(np.float64) - vt
        out[name] = {"seam": seam_score(err, c.height, c.width, 2, 2), "rel_err": float(np.linalg.norm(err) / np.linalg.norm(vt)),
                     "loss_first": losses[0], "loss_last": losses[-1]}
        print(json.dumps({"study": "seam", "run": name, "halo": halo, "margin": margin, "iterations": iters,
                          **out[name]}), flush=True)
    return out


if __name__ == "__main__":
    t0 = time.time()
    if sys.argv[1] == "seam" and len(sys.argv) > 2:
        seam(int(sys.argv[2]))
    else:
        {"perf": perf, "seam": seam}[sys.argv[1]]()
    print(json.dumps({"elapsed_s": time.time() - t0}))
