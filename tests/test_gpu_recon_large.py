"""Reconstruction parity beyond N = 64: multi-probe,
multi-segment Alg. 1 iterations (steps 5-16) through the C ABI at N = 256 and N = 1024
against oracle.reconstruct running the same schedule, and the N = 1024 / S = 100 exit wave.

Inputs: BASELINE.json's small / LT-small shapes with a subsampled raster (the oracle is float64
numpy: ~0.3 s per N = 256 probe, ~8 s per N = 1024 / S = 20 probe), V0 = 0.5 V_true,
measurements |G(p, V_true)| from the oracle.  Bars (north_star): V rel L2 <= 1e-4 after the
iterations; the update dV = V - V0 <= 1e-3 (it is small next to V, so this is the stricter view).
"""
import numpy as np
import pytest

from oracle import ptycho_oracle as O
import synth

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def _run(c, slices, scan, grid, halo, period, iters, alpha, seed=0):
    from paper_2205_06327_b200.ptycho import Ptycho
    n, h, w = c.n, c.height, c.width
    probe = synth.probe(n, c.defocus_nm)
    vt = synth.volume(seed, slices, h, w)
    v0 = (0.5 * vt).astype(np.float32)
    centers = synth.scan_centers(h, w, *scan)
    full = (0, 0, h, w)
    amps = np.stack([O.farfield_magnitude(probe, O.window(vt.astype(np.float64), full, tuple(cc), n), c.sigma,
                                          c.prop_c) for cc in centers]).astype(np.float32)
    d = dict(n=n, slices=slices, height=h, width=w, sigma=c.sigma, prop_c=c.prop_c)
    ref, losses, _, _ = O.reconstruct(v0.astype(np.float64), probe, amps.astype(np.float64), centers, d, grid[0],
                                      grid[1], halo, iters, alpha=alpha, period=period)
    p = Ptycho(n, slices, h, w, c.sigma, c.prop_c, alpha=alpha, pass_period=period)
    p.set_tiles(grid[0], grid[1], halo)
    p.set_scan(centers)
    p.allocate_workspace()
    p.set_probe(probe.astype(np.complex64))
    p.load_measurements(amps[p.local_probes()])
    p.set_volume(v0)
    got_losses = [p.iterate(want_loss=True) for _ in range(iters)]
    out = p.stitch()
    p.close()
    err, derr = rel(out, ref), rel(out - v0, ref - v0)
    print(f"{c.name} S={slices} scan {scan} grid {grid} halo {halo} T={period} x{iters}: V rel {err:.2e}, "
          f"dV rel {derr:.2e} (|dV|/|V| {np.linalg.norm(ref - v0) / np.linalg.norm(ref):.1e}); "
          f"losses {got_losses} vs {losses}")
    assert err <= 1e-4
    assert derr <= 1e-3
    for a, b in zip(got_losses, losses):
        assert abs(a - b) <= 1e-4 * b


@pytest.mark.parametrize("grid,period", [((1, 1), 0), ((1, 1), 16), ((2, 2), 0), ((2, 2), 5)])
def test_small_reconstruction_n256(grid, period):
    """N = 256, S = 20, 512^2 object (BASELINE small), 8 x 8 raster (64 probes; 16 per tile on
    2 x 2 with the exact-window halo 128), 2 iterations, passes once per iteration or every T
    local probes (several segments plus the end-of-iteration flush, reading #17)."""
    _run(synth.CONFIGS["small"], 20, (8, 8), grid, 128, period, 2, alpha=1024.0)


def test_lt_geometry_segment_n1024():
    """N = 1024 on the LT-small geometry (1536^2, 2 x 4 tiles, halo 512 > interior width 384),
    S = 20 (oracle time), 4 x 4 raster (two probes per tile), one iteration, passes once: the
    EngFour<32> engine across an accumulating segment, the APPP at the LT geometry, the step."""
    _run(synth.CONFIGS["lt_small"], 20, (4, 4), (2, 4), 512, 0, 1, alpha=1024.0)


def test_exit_wave_n1024_s100():
    """psi_S of one LT-small probe at full depth (N = 1024, S = 100): 200 chained 1-D transform
    passes; bar max(1e-5, 2 x the float32 floor of the same oracle arithmetic)."""
    from paper_2205_06327_b200.ptycho import Ptycho
    c = synth.CONFIGS["lt_small"]
    n, s, h, w = c.n, c.slices, c.height, c.width
    probe = synth.probe(n, c.defocus_nm)
    v0 = (0.5 * synth.volume(0, s, h, w)).astype(np.float32)
    centers = synth.scan_centers(h, w, c.scan_ny, c.scan_nx)
    gid = 2000
    vwin = O.window(v0.astype(np.float64), (0, 0, h, w), tuple(centers[gid]), n)
    psi_ref, _, _ = O.forward(probe, vwin, c.sigma, c.prop_c)
    psi32, _, _ = O.forward(probe, vwin, c.sigma, c.prop_c, dtype=np.float32)
    floor = rel(psi32, psi_ref)
    p = Ptycho(n, s, h, w, c.sigma, c.prop_c, alpha=0.0)
    p.set_tiles(*c.grid, n // 2)
    p.set_scan(centers)
    p.allocate_workspace()
    p.set_probe(probe.astype(np.complex64))
    p.set_volume(v0)
    psi = p.probe_exitwave(gid)
    p.close()
    err = rel(psi, psi_ref)
    print(f"exit wave N=1024 S=100 probe {gid}: rel {err:.2e} (fp32 floor {floor:.2e})")
    assert err <= max(1e-5, 2 * floor)
