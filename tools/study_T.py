"""Pass-frequency (T) and halo study on synthetic data (PAPER.md P:446-456,
Fig. convergence: "once or twice per iteration converges slightly faster than every probe").

F(V) (Eq. 1, summed over the sweep) per iteration for T in {every probe, twice per iteration,
once per iteration}, in exact-window mode (halo N/2) and the paper's circle-halo mode (small halo,
zero-extended windows, reading #13), on a 2x2 tile grid.  Writes profiles/round1_T_study.json;
CONFIG=appp runs the BASELINE "APPP check" shape instead (N = 256, S = 20, 1024^2 object, 64 x 64
probes, circle halo 60 px = the paper's 600 pm) and writes profiles/round1_T_study_appp.json."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2205_06327_b200.ptycho import Ptycho  # noqa: E402

CONFIG = os.environ.get("CONFIG", "")
if CONFIG:
    _c = synth.CONFIGS[CONFIG]
    n, s, h, w, ny, nx, sigma, prop_c = _c.n, _c.slices, _c.height, _c.width, _c.scan_ny, _c.scan_nx, _c.sigma, _c.prop_c
    defocus, circle_halo = _c.defocus_nm, 60
else:
    n, s, h, w = 64, 4, 256, 256
    ny = nx = 12
    sigma, prop_c, defocus, circle_halo = 0.1, 3.135, 8.0, 12
iters = int(os.environ.get("ITERS", 40))
alpha = float(os.environ.get("ALPHA", 0.5))
probe = synth.probe(n, defocus).astype(np.complex64)
vt = synth.volume(1, s, h, w)
centers = synth.scan_centers(h, w, ny, nx)


def run(period, halo, grid=(2, 2)):
    p = Ptycho(n, s, h, w, sigma, prop_c, alpha=alpha, pass_period=period)
    p.set_tiles(grid[0], grid[1], halo)
    p.set_scan(centers)
    p.allocate_workspace()
    p.set_probe(probe)
    p.set_volume(vt)
    p.simulate_measurements()
    p.set_volume(None)
    nmax = max(p.tile_probe_count(k) for k in range(grid[0] * grid[1]))
    losses = [p.iterate(want_loss=True) for _ in range(iters)]
    v = p.stitch()
    # the per-slice mean of V is a gauge (a constant phase over the object leaves |Psi| unchanged,
    # App. A.6): compare mean-free volumes
    dv = v - v.mean(axis=(1, 2), keepdims=True)
    dt = vt - vt.mean(axis=(1, 2), keepdims=True)
    err = float(np.linalg.norm(dv - dt) / np.linalg.norm(dt))
    p.close()
    return nmax, losses, err


# alpha: the largest of 2^0..2^12 whose F decreases monotonically over 10 iterations
if "ALPHA" not in os.environ:
    best = None
    for e in range(0, 17):
        alpha = float(2 ** e)
        iters_save, iters = iters, 10
        _, ls, _ = run(0, n // 2)
        iters = iters_save
        ok = all(b < a for a, b in zip(ls, ls[1:])) and np.isfinite(ls).all()
        print(f"alpha sweep 2^{e}: F[0]={ls[0]:.4e} F[9]={ls[-1]:.4e} monotone={ok}", flush=True)
        if ok:
            best = alpha
    alpha = best
print("alpha =", alpha, flush=True)
out = {"config": dict(n=n, slices=s, object=[h, w], probes=ny * nx, grid="2x2", alpha=alpha, iterations=iters,
                      v0="0", measurements="simulated |G(p, V_true)| (noise-free)"), "runs": []}
nmax = None
for halo, mode in [(n // 2, "exact-window"), (circle_halo, "circle-halo")]:
    base = run(0, halo)
    nmax = base[0]
    for name, period in [("every probe (T=1)", 1), ("twice per iteration", -(-nmax // 2)), ("once per iteration", 0)]:
        _, losses, err = base if period == 0 else run(period, halo)
        out["runs"].append(dict(mode=mode, halo=halo, T=name, period=period, F=losses, rel_err_V=err))
        print(f"{mode:13s} {name:22s} F[0]={losses[0]:.4e} F[9]={losses[9]:.4e} F[-1]={losses[-1]:.4e} "
              f"|V-Vtrue|/|Vtrue|={err:.4f}", flush=True)
single = run(0, n // 2, grid=(1, 1))
out["runs"].append(dict(mode="single tile", halo=0, T="once per iteration", period=0, F=single[1], rel_err_V=single[2]))
print(f"{'single tile':13s} {'once per iteration':22s} F[-1]={single[1][-1]:.4e} |V-Vtrue|/|Vtrue|={single[2]:.4f}")
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
name = f"round1_T_study_{CONFIG}.json" if CONFIG else "round1_T_study.json"
json.dump(out, open(os.path.join(ROOT, "profiles", name), "w"), indent=1)
