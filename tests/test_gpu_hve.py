"""Halo Voxel Exchange baseline on the GPU through the C ABI
(ptycho_set_tiles_hve) against oracle.hve_reconstruct: duplicated neighbour probes, independent
per-tile SGD sweeps on the same pass kernels (AccBuf off), halo copy-paste.  Bars as for GD
reconstructions (north_star): V rel L2 <= 1e-4, dV <= 1e-3; the exchange is bit-exact."""
import numpy as np
import pytest

from oracle import ptycho_oracle as O
import synth

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def _problem(n, s, h, w, scan, seed=3, defocus=8.0, sigma=0.3):
    rng = np.random.default_rng(seed)
    probe = synth.probe(n, defocus)
    vt = rng.random((s, h, w)).astype(np.float32)
    centers = synth.scan_centers(h, w, *scan)
    d = dict(n=n, slices=s, height=h, width=w, sigma=sigma, prop_c=3.135)
    full = (0, 0, h, w)
    amps = np.stack([O.farfield_magnitude(probe, O.window(vt.astype(np.float64), full, tuple(cc), n), sigma, 3.135)
                     for cc in centers]).astype(np.float32)
    return d, probe, vt, centers, amps


def _gpu(d, probe, v0, centers, amps, grid, halo, margin, alpha, iters, hve=True):
    from paper_2205_06327_b200.ptycho import Ptycho
    p = Ptycho(d["n"], d["slices"], d["height"], d["width"], d["sigma"], d["prop_c"], alpha=alpha,
               alpha_acc=0.0)
    if hve:
        p.set_tiles_hve(grid[0], grid[1], halo, margin)
    else:
        p.set_tiles(grid[0], grid[1], halo)
    p.set_scan(centers)
    p.allocate_workspace()
    p.set_probe(probe.astype(np.complex64))
    p.load_measurements(amps[p.local_probes()])
    p.set_volume(v0)
    losses = [p.iterate(want_loss=True) for _ in range(iters)]
    return p, p.stitch(), losses


@pytest.mark.parametrize("grid,halo,margin,iters", [((2, 3), 32, 25, 2), ((3, 2), 12, 50, 2), ((1, 1), 0, 0, 1)])
def test_hve_matches_oracle_n64(grid, halo, margin, iters):
    d, probe, vt, centers, amps = _problem(64, 3, 150, 131, (5, 6))
    v0 = (0.5 * vt).astype(np.float32)
    alpha = 1.0
    ref, ref_losses, _ = O.hve_reconstruct(v0.astype(np.float64), probe, amps.astype(np.float64), centers, d,
                                           grid[0], grid[1], margin, halo, iters, alpha=alpha)
    p, out, losses = _gpu(d, probe, v0, centers, amps, grid, halo, margin, alpha, iters)
    # the exchange: every tile's halo equals the owner's interior, bitwise
    for k in range(grid[0] * grid[1]):
        (y0, x0, y1, x1), _ = p.tile_rect(k)
        assert np.array_equal(p.debug_read_tile(k, 0), out[:, y0:y1, x0:x1]), k
    p.close()
    err, derr = rel(out, ref), rel(out - v0, ref - v0)
    print(f"HVE {grid} halo {halo} margin {margin}: V {err:.2e} dV {derr:.2e}; losses {losses} vs {ref_losses}")
    assert err <= 1e-4 and derr <= 1e-3
    for a, b in zip(losses, ref_losses):
        assert abs(a - b) <= 1e-4 * b


def test_hve_matches_oracle_n256():
    """BASELINE small shape (N = 256, S = 20, 512^2), 8 x 8 raster (step 64), 2 x 2 mesh, two extra
    rows of probe locations (margin 128), halo 128, one iteration."""
    c = synth.CONFIGS["small"]
    d, probe, vt, centers, amps = _problem(256, 20, 512, 512, (8, 8), seed=0, defocus=25.0, sigma=c.sigma)
    v0 = (0.5 * vt).astype(np.float32)
    ref, _, _ = O.hve_reconstruct(v0.astype(np.float64), probe, amps.astype(np.float64), centers, d, 2, 2, 128, 128,
                                  1, alpha=1024.0)
    p, out, _ = _gpu(d, probe, v0, centers, amps, (2, 2), 128, 128, 1024.0, 1)
    p.close()
    err, derr = rel(out, ref), rel(out - v0, ref - v0)
    print(f"HVE small 2x2: V {err:.2e} dV {derr:.2e}")
    assert err <= 1e-4 and derr <= 1e-3


def test_hve_one_tile_equals_gd_without_accumulated_step():
    d, probe, vt, centers, amps = _problem(64, 3, 150, 131, (5, 6))
    v0 = (0.5 * vt).astype(np.float32)
    p1, a, _ = _gpu(d, probe, v0, centers, amps, (1, 1), 0, 0, 1.0, 2, hve=True)
    p2, b, _ = _gpu(d, probe, v0, centers, amps, (1, 1), 0, 0, 1.0, 2, hve=False)
    p1.close()
    p2.close()
    assert np.array_equal(a, b)


def test_hve_tile_too_small_and_no_step():
    from paper_2205_06327_b200.ptycho import Ptycho, PtychoError
    p = Ptycho(64, 2, 96, 96, alpha=1.0)
    with pytest.raises(PtychoError, match="EHALO"):
        p.set_tiles_hve(6, 6, 24, 16)  # interiors 16 < halo 24
    p.close()
    p = Ptycho(64, 2, 96, 96, alpha=1.0)
    p.set_tiles_hve(3, 3, 16, 16)
    p.set_scan(synth.scan_centers(96, 96, 3, 3))
    p.allocate_workspace()
    p.set_probe(synth.probe(64, 8.0).astype(np.complex64))
    with pytest.raises(PtychoError, match="ESTATE"):
        p.step()
    p.close()
