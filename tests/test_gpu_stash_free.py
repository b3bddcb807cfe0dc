"""Stash-free adjoint (PTYCHO_F_STASH_FREE) against the float64 oracle.

The CUDA path keeps only phi_{S-1} and rebuilds phi_s = P^H(conj(t_{s+1}) phi_{s+1}) in a second
adjoint chain.  The gradient is the same quantity as with the stash, so it is compared with
oracle.probe_grad (float64); the rounding floor is that of the recomputation,
oracle.probe_grad_recompute run in float32 (the phi chain adds S-1 propagations).
Tolerance: max(1e-5, 2 x that floor) rel L2 per probe; reconstructions 1e-4 (north_star)."""
import numpy as np
import pytest

from oracle import ptycho_oracle as O
import synth

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def _ptycho(c, flags, rows=1, cols=1, halo=None, alpha=0.0, period=0, **kw):
    from paper_2205_06327_b200.ptycho import Ptycho
    p = Ptycho(c["n"], c["slices"], c["height"], c["width"], c["sigma"], c["prop_c"], alpha=alpha,
               pass_period=period, flags=flags, device=0, **kw)
    p.set_tiles(rows, cols, c["n"] // 2 if halo is None else halo)
    return p


@pytest.mark.parametrize("name,probe_idx", [("tiny", 0), ("tiny", 5), ("small", 0), ("small", 530)])
def test_stash_free_gradient(name, probe_idx):
    from paper_2205_06327_b200.ptycho import PTYCHO_F_STASH_FREE
    c = synth.CONFIGS[name]
    probe = synth.probe(c.n, c.defocus_nm)
    vt = synth.volume(0, c.slices, c.height, c.width)
    centers = synth.scan_centers(c.height, c.width, c.scan_ny, c.scan_nx)
    full = (0, 0, c.height, c.width)
    v0 = 0.5 * vt
    amp = O.farfield_magnitude(probe, O.window(vt.astype(np.float64), full, tuple(centers[probe_idx]), c.n),
                               c.sigma, c.prop_c)
    vwin = O.window(v0.astype(np.float64), full, tuple(centers[probe_idx]), c.n)
    g_ref, f_ref = O.probe_grad(probe, vwin, amp, c.sigma, c.prop_c)
    g32, _ = O.probe_grad_recompute(probe, vwin, amp, c.sigma, c.prop_c, dtype=np.float32)
    floor = rel(g32, g_ref)
    d = dict(n=c.n, slices=c.slices, height=c.height, width=c.width, sigma=c.sigma, prop_c=c.prop_c)
    got = {}
    for flags in (0, PTYCHO_F_STASH_FREE):
        p = _ptycho(d, flags)
        p.set_scan(centers)
        got[flags, "ws"] = p.workspace_bytes()
        p.allocate_workspace()
        p.set_probe(probe.astype(np.complex64))
        p.load_measurements(amp[None].astype(np.float32), first_local=probe_idx)
        p.set_volume(v0.astype(np.float32))
        got[flags] = p.debug_probe_grad(0, probe_idx)
        p.close()
    g, f = got[PTYCHO_F_STASH_FREE]
    err = rel(g, g_ref)
    print(f"{name} probe {probe_idx} stash-free: grad rel L2 {err:.2e} (recompute fp32 floor {floor:.2e}), "
          f"stash {rel(got[0][0], g_ref):.2e}; workspace {got[PTYCHO_F_STASH_FREE, 'ws'] / 2**20:.1f} MiB vs "
          f"{got[0, 'ws'] / 2**20:.1f} MiB")
    assert err <= max(1e-5, 2 * floor)
    assert f == got[0][1]  # the loss comes from the (unchanged) forward
    stash_bytes = (c.slices - 2) * c.n * c.n * 8
    assert got[0, "ws"] - got[PTYCHO_F_STASH_FREE, "ws"] >= stash_bytes - 2 * c.n * c.n * 8 - 4096


def _recon_case(s, seed=3):
    n, h, w = 64, 200, 180
    rng = np.random.default_rng(seed)
    probe = synth.probe(n, 8.0)
    vt = rng.random((s, h, w)).astype(np.float32)
    centers = synth.scan_centers(h, w, 6, 5)
    d = dict(n=n, slices=s, height=h, width=w, sigma=0.3, prop_c=3.135)
    amps = np.stack([O.farfield_magnitude(probe, O.window(vt.astype(np.float64), (0, 0, h, w), tuple(cc), n),
                                          d["sigma"], d["prop_c"]) for cc in centers]).astype(np.float32)
    return d, probe, vt, centers, amps


@pytest.mark.parametrize("s,grid,period,batch", [(1, (1, 1), 0, 0), (2, (2, 2), 0, 0), (3, (2, 3), 3, 0),
                                                 (6, (1, 1), 0, 0), (4, (2, 2), 0, 4)])
def test_stash_free_reconstruction(s, grid, period, batch):
    """S = 1 (flag is a no-op), 2 (RECON_FIRST -> RECON_END), 3 and more (RECON_MID), multi-tile
    APPP, and the batched schedule (stash ring per batch slot) against the oracle."""
    from paper_2205_06327_b200.ptycho import PTYCHO_F_STASH_FREE
    d, probe, vt, centers, amps = _recon_case(s)
    v0 = (0.5 * vt).astype(np.float32)
    ref, losses, _, _ = O.reconstruct(v0.astype(np.float64), probe, amps.astype(np.float64), centers, d, grid[0],
                                      grid[1], d["n"] // 2, 2, alpha=1.0, period=period, batch=batch)
    outs = []
    for flags in (0, PTYCHO_F_STASH_FREE):
        p = _ptycho(d, flags, rows=grid[0], cols=grid[1], alpha=1.0, period=period)
        p.set_scan(centers)
        if batch:
            p.set_schedule(True, batch)
        p.allocate_workspace()
        p.set_probe(probe.astype(np.complex64))
        p.load_measurements(amps[p.local_probes()])
        p.set_volume(v0)
        got = [p.iterate(want_loss=True) for _ in range(2)]
        outs.append(p.stitch())
        p.close()
        for a, b in zip(got, losses):
            assert abs(a - b) <= 1e-4 * b
    out = outs[1]
    print(f"S={s} grid {grid} T={period} batch {batch}: stash-free V rel {rel(out, ref):.2e}, dV rel "
          f"{rel(out - v0, ref - v0):.2e} (stash dV rel {rel(outs[0] - v0, ref - v0):.2e})")
    assert rel(out, ref) <= 1e-4 and rel(out - v0, ref - v0) <= 1e-3
    if s == 1:
        assert np.array_equal(outs[0], outs[1])  # nothing to recompute: same kernels


def test_stash_free_launch_count():
    """S more passes per probe (RECON_FIRST + (S-2) RECON_MID + RECON_END), counted by the library."""
    from paper_2205_06327_b200.ptycho import PTYCHO_F_STASH_FREE
    d, probe, vt, centers, amps = _recon_case(5)
    counts = []
    for flags in (0, PTYCHO_F_STASH_FREE):
        p = _ptycho(d, flags)
        p.set_scan(centers)
        p.allocate_workspace()
        p.set_probe(probe.astype(np.complex64))
        p.load_measurements(amps)
        p.set_volume(vt)
        before = p.kernel_launches()
        p.forward_grad(0, 3)
        p.synchronize()
        counts.append(p.kernel_launches() - before)
        p.close()
    assert counts[1] - counts[0] == 3 * 5
