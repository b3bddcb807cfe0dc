"""Parity of the CUDA path (through the C ABI) against the float64 oracle.

Tolerances:
  * per-probe exit wave and gradient: rel L2 <= max(1e-5, 2 x fp32 floor), the floor being the
    same oracle run in float32 on the same input; tiny (N=64) must meet 1e-5.
  * reconstruction after N iterations: rel L2 <= 1e-4 (north_star).
  * APPP region indexing with integer data, stitch, set_volume: bit-exact.
"""
import numpy as np
import pytest

from oracle import ptycho_oracle as O
import synth

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def make(cfgd, rows=1, cols=1, halo=None, alpha=0.0, alpha_acc=None, period=0, flags=0, tau=1e-4):
    from paper_2205_06327_b200.ptycho import Ptycho
    p = Ptycho(cfgd["n"], cfgd["slices"], cfgd["height"], cfgd["width"], cfgd["sigma"], cfgd["prop_c"],
               alpha=alpha, alpha_acc=alpha_acc, tau=tau, pass_period=period, flags=flags, device=0)
    p.set_tiles(rows, cols, cfgd["n"] // 2 if halo is None else halo)
    return p


def cfg_dict(c):
    return dict(n=c.n, slices=c.slices, height=c.height, width=c.width, sigma=c.sigma, prop_c=c.prop_c)


def problem(name, seed=0):
    c = synth.CONFIGS[name]
    probe = synth.probe(c.n, c.defocus_nm)
    vt = synth.volume(seed, c.slices, c.height, c.width)
    centers = synth.scan_centers(c.height, c.width, c.scan_ny, c.scan_nx)
    return c, probe, vt, centers


def oracle_amp(probe, vt, center, c):
    full = (0, 0, c.height, c.width)
    return O.farfield_magnitude(probe, O.window(vt.astype(np.float64), full, tuple(center), c.n), c.sigma, c.prop_c)


# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("probe_idx", [0, 5, 15])
def test_tiny_gradient_and_loss(probe_idx):
    c, probe, vt, centers = problem("tiny")
    v0 = 0.5 * vt
    amp = oracle_amp(probe, vt, centers[probe_idx], c)
    full = (0, 0, c.height, c.width)
    vwin = O.window(v0.astype(np.float64), full, tuple(centers[probe_idx]), c.n)
    g_ref, f_ref = O.probe_grad(probe, vwin, amp, c.sigma, c.prop_c)
    g32, _ = O.probe_grad(probe, vwin, amp, c.sigma, c.prop_c, dtype=np.float32)
    floor = rel(g32, g_ref)

    p = make(cfg_dict(c))
    p.set_scan(centers)
    p.allocate_workspace()
    p.set_probe(probe.astype(np.complex64))
    amps = np.zeros((len(centers), c.n, c.n), np.float32)
    amps[probe_idx] = amp
    p.load_measurements(amps)
    p.set_volume(v0)
    g, f = p.debug_probe_grad(0, probe_idx)
    err = rel(g, g_ref)
    print(f"tiny probe {probe_idx}: grad rel L2 {err:.2e} (fp32 floor {floor:.2e}); loss {f:.8e} vs {f_ref:.8e}")
    assert err <= 1e-5
    assert abs(f - f_ref) <= 1e-5 * f_ref


@pytest.mark.parametrize("name,probe_idx", [("tiny", 5), ("tiny", 0), ("small", 0), ("small", 530)])
def test_exit_wave(name, probe_idx):
    c, probe, vt, centers = problem(name)
    full = (0, 0, c.height, c.width)
    vwin = O.window(vt.astype(np.float64), full, tuple(centers[probe_idx]), c.n)
    psi_ref = O.forward(probe, vwin, c.sigma, c.prop_c)[0]
    psi32 = O.forward(probe, vwin, c.sigma, c.prop_c, dtype=np.float32)[0]
    floor = rel(psi32, psi_ref)
    p = make(cfg_dict(c))
    p.set_scan(centers)
    p.allocate_workspace()
    p.set_probe(probe.astype(np.complex64))
    p.set_volume(vt)
    psi = p.debug_exit_wave(0, probe_idx)
    err = rel(psi, psi_ref)
    print(f"{name} exit wave probe {probe_idx}: rel L2 {err:.2e} (fp32 floor {floor:.2e})")
    assert err <= max(1e-5, 2 * floor)


@pytest.mark.parametrize("probe_idx", [0, 530, 1023])
def test_small_gradient(probe_idx):
    c, probe, vt, centers = problem("small")
    v0 = 0.5 * vt
    amp = oracle_amp(probe, vt, centers[probe_idx], c)
    full = (0, 0, c.height, c.width)
    vwin = O.window(v0.astype(np.float64), full, tuple(centers[probe_idx]), c.n)
    g_ref, f_ref = O.probe_grad(probe, vwin, amp, c.sigma, c.prop_c)
    g32, _ = O.probe_grad(probe, vwin, amp, c.sigma, c.prop_c, dtype=np.float32)
    floor = rel(g32, g_ref)
    p = make(cfg_dict(c))
    p.set_scan(centers)
    p.allocate_workspace()
    p.set_probe(probe.astype(np.complex64))
    amps = np.zeros((1, c.n, c.n), np.float32)
    amps[0] = amp
    p.load_measurements(amps, first_local=probe_idx)
    p.set_volume(v0)
    g, f = p.debug_probe_grad(0, probe_idx)
    err = rel(g, g_ref)
    print(f"small probe {probe_idx}: grad rel L2 {err:.2e} (fp32 floor {floor:.2e}); loss rel {abs(f-f_ref)/f_ref:.2e}")
    assert err <= max(1e-5, 2 * floor)
    assert abs(f - f_ref) <= 1e-5 * f_ref


def test_simulated_measurements_match_oracle():
    c, probe, vt, centers = problem("tiny")
    p = make(cfg_dict(c))
    p.set_scan(centers)
    p.allocate_workspace()
    p.set_probe(probe.astype(np.complex64))
    p.set_volume(vt)
    p.simulate_measurements()
    # read back through the loss: with V = V_true every probe's loss must vanish
    p.set_volume(vt)
    loss = p.forward_grad(0, len(centers), want_loss=True)
    assert loss < 1e-9, loss


def test_set_volume_stitch_round_trip_bit_exact():
    c = synth.CONFIGS["tiny"]
    rng = np.random.default_rng(1)
    v = rng.random((5, 150, 131), dtype=np.float32)
    d = dict(n=64, slices=5, height=150, width=131, sigma=0.1, prop_c=3.1)
    p = make(d, rows=3, cols=2, halo=20)
    p.set_scan(synth.scan_centers(150, 131, 3, 3))
    p.allocate_workspace()
    p.set_volume(v)
    out = p.stitch()
    assert np.array_equal(out, v)
    tiles = O.tile_geometry(150, 131, 3, 2, 20)
    for k, t in enumerate(tiles):
        got = p.debug_read_tile(k, 0)
        y0, x0, y1, x1 = t["ext"]
        assert np.array_equal(got, v[:, y0:y1, x0:x1])


@pytest.mark.parametrize("shape,grid,halo,slices", [((96, 96), (3, 3), 8, 3), ((96, 96), (3, 3), 40, 2),
                                                     ((60, 90), (4, 3), 7, 3), ((192, 192), (2, 4), 64, 5),
                                                     ((101, 77), (2, 3), 33, 4)])
def test_appp_integer_bit_exact(shape, grid, halo, slices):
    rng = np.random.default_rng(2)
    d = dict(n=64, slices=slices, height=shape[0], width=shape[1], sigma=0.1, prop_c=3.1)
    p = make(d, rows=grid[0], cols=grid[1], halo=halo)
    p.set_scan(synth.scan_centers(shape[0], shape[1], 2, 2))
    p.allocate_workspace()
    tiles = O.tile_geometry(shape[0], shape[1], grid[0], grid[1], halo)
    bufs = []
    for k, t in enumerate(tiles):
        ext, _ = p.tile_rect(k)
        assert ext == t["ext"]
        b = rng.integers(0, 2 ** 16, (slices, ext[2] - ext[0], ext[3] - ext[1])).astype(np.float32)
        p.debug_write_tile(k, 1, b)
        bufs.append(b.astype(np.float64))
    total = O.global_sum(bufs, tiles, slices, *shape)
    p.appp_passes()
    for k, t in enumerate(tiles):
        y0, x0, y1, x1 = t["ext"]
        got = p.debug_read_tile(k, 1)
        assert np.array_equal(got.astype(np.float64), total[:, y0:y1, x0:x1]), k


def _recon_problem():
    # ragged object, several tiles, windows overhanging the object edge, tail segment
    n, s, h, w = 64, 3, 150, 131
    rng = np.random.default_rng(3)
    probe = synth.probe(n, 8.0)
    vt = rng.random((s, h, w)).astype(np.float32)
    centers = synth.scan_centers(h, w, 5, 6)
    d = dict(n=n, slices=s, height=h, width=w, sigma=0.3, prop_c=3.135)
    full = (0, 0, h, w)
    amps = np.stack([O.farfield_magnitude(probe, O.window(vt.astype(np.float64), full, tuple(cc), n), d["sigma"],
                                          d["prop_c"]) for cc in centers]).astype(np.float32)
    return d, probe, vt, centers, amps


@pytest.mark.parametrize("grid,period,iters,halo", [((1, 1), 0, 2, 32), ((2, 3), 0, 2, 32), ((2, 3), 3, 1, 32),
                                                    ((3, 2), 4, 2, 32), ((2, 3), 0, 2, 12), ((3, 2), 1, 1, 7)])
def test_reconstruction_matches_oracle(grid, period, iters, halo):
    """halo 32 = N/2 (exact window); halo 12 / 7 = the paper's circle-halo mode (reading #13:
    windows are zero-extended past R_k, an approximation both sides implement identically)."""
    d, probe, vt, centers, amps = _recon_problem()
    v0 = (0.5 * vt).astype(np.float32)
    alpha = 1.0
    ref, losses, _, _ = O.reconstruct(v0.astype(np.float64), probe, amps.astype(np.float64), centers, d, grid[0],
                                      grid[1], halo, iters, alpha=alpha, period=period)
    p = make(d, rows=grid[0], cols=grid[1], halo=halo, alpha=alpha, period=period)
    p.set_scan(centers)
    p.allocate_workspace()
    p.set_probe(probe.astype(np.complex64))
    ids = p.local_probes()
    p.load_measurements(amps[ids])
    p.set_volume(v0)
    got_losses = [p.iterate(want_loss=True) for _ in range(iters)]
    out = p.stitch()
    err = rel(out, ref)
    derr = rel(out - v0, ref - v0)
    print(f"grid {grid} T={period} halo {halo}: V rel {err:.2e}, dV rel {derr:.2e}, losses {got_losses} vs {losses}")
    assert err <= 1e-4
    assert derr <= 1e-3
    for a, b in zip(got_losses, losses):
        assert abs(a - b) <= 1e-4 * b


def test_frozen_multi_tile_equals_single_tile():
    """alpha = 0: after the four passes every tile's AccBuf equals the single-tile AccBuf on R_k."""
    d, probe, vt, centers, amps = _recon_problem()
    v0 = (0.5 * vt).astype(np.float32)
    accs = {}
    for grid in [(1, 1), (2, 3)]:
        p = make(d, rows=grid[0], cols=grid[1], alpha=0.0, alpha_acc=0.0)
        p.set_scan(centers)
        p.allocate_workspace()
        p.set_probe(probe.astype(np.complex64))
        p.load_measurements(amps[p.local_probes()])
        p.set_volume(v0)
        p.forward_grad(0, 10 ** 6)
        p.appp_passes()
        accs[grid] = [(p.tile_rect(k)[0], p.debug_read_tile(k, 1)) for k in range(grid[0] * grid[1])]
    single = accs[(1, 1)][0][1]
    for ext, a in accs[(2, 3)]:
        y0, x0, y1, x1 = ext
        e = rel(a, single[:, y0:y1, x0:x1])
        assert e < 2e-6, e


def test_deterministic_bitwise():
    d, probe, vt, centers, amps = _recon_problem()
    outs = []
    for _ in range(2):
        p = make(d, rows=2, cols=3, alpha=1.0)
        p.set_scan(centers)
        p.allocate_workspace()
        p.set_probe(probe.astype(np.complex64))
        p.load_measurements(amps[p.local_probes()])
        p.set_volume(0.5 * vt)
        p.iterate()
        outs.append(p.stitch())
    assert np.array_equal(outs[0], outs[1])


def test_error_codes():
    from paper_2205_06327_b200.ptycho import Ptycho, PtychoError, PTYCHO_F_EXACT_WINDOW
    with pytest.raises(PtychoError) as e:
        Ptycho(100, 2, 64, 64)
    assert e.value.status == 1
    p = Ptycho(64, 2, 128, 128, flags=PTYCHO_F_EXACT_WINDOW)
    with pytest.raises(PtychoError) as e:
        p.forward_grad(0, 1)
    assert e.value.status == 3
    p.set_tiles(2, 2, 8)
    with pytest.raises(PtychoError) as e:
        p.set_scan(synth.scan_centers(128, 128, 4, 4))
    assert e.value.status == 4
    q = Ptycho(64, 2, 128, 128)
    q.set_tiles(1, 1, 0)
    with pytest.raises(PtychoError) as e:
        q.set_scan(np.array([[200, 5]], np.int32))
    assert e.value.status == 1


@pytest.mark.parametrize("s", [1, 2])
def test_degenerate_slices_and_empty_tile(s):
    """S = 1 and 2 (the chain's special first/last passes) and a tile with no probes at all."""
    n, h, w = 64, 140, 120
    rng = np.random.default_rng(4)
    probe = synth.probe(n, 8.0)
    vt = rng.random((s, h, w)).astype(np.float32)
    centers = synth.scan_centers(h // 2, w, 3, 4)  # only the upper half: tiles of the lower row are empty
    d = dict(n=n, slices=s, height=h, width=w, sigma=0.3, prop_c=3.135)
    amps = np.stack([O.farfield_magnitude(probe, O.window(vt.astype(np.float64), (0, 0, h, w), tuple(cc), n),
                                          d["sigma"], d["prop_c"]) for cc in centers]).astype(np.float32)
    v0 = (0.5 * vt).astype(np.float32)
    ref, losses, _, _ = O.reconstruct(v0.astype(np.float64), probe, amps.astype(np.float64), centers, d, 2, 2,
                                      n // 2, 2, alpha=1.0, period=2)
    p = make(d, rows=2, cols=2, alpha=1.0, period=2)
    p.set_scan(centers)
    assert p.tile_probe_count(2) == 0 and p.tile_probe_count(3) == 0
    p.allocate_workspace()
    p.set_probe(probe.astype(np.complex64))
    p.load_measurements(amps[p.local_probes()])
    p.set_volume(v0)
    got = [p.iterate(want_loss=True) for _ in range(2)]
    out = p.stitch()
    assert rel(out, ref) <= 1e-4 and rel(out - v0, ref - v0) <= 1e-3
    for a, b in zip(got, losses):
        assert abs(a - b) <= 1e-4 * b


@pytest.mark.parametrize("grid,period,batch", [((1, 1), 0, 4), ((2, 3), 3, 2), ((2, 2), 0, 8)])
def test_batched_schedule_bit_identical(grid, period, batch):
    """opt-in batched schedule == sequential, bitwise (V, AccBuf); and vs the oracle running it."""
    n, s, h, w = 64, 3, 220, 200
    rng = np.random.default_rng(5)
    probe = synth.probe(n, 8.0)
    vt = rng.random((s, h, w)).astype(np.float32)
    centers = synth.scan_centers(h, w, 7, 6)
    d = dict(n=n, slices=s, height=h, width=w, sigma=0.3, prop_c=3.135)
    amps = np.stack([O.farfield_magnitude(probe, O.window(vt.astype(np.float64), (0, 0, h, w), tuple(cc), n),
                                          d["sigma"], d["prop_c"]) for cc in centers]).astype(np.float32)
    v0 = (0.5 * vt).astype(np.float32)
    outs, accs = [], []
    for batched in (False, True):
        p = make(d, rows=grid[0], cols=grid[1], alpha=1.0, period=period)
        p.set_scan(centers)
        if batched:
            p.set_schedule(True, batch)
        p.allocate_workspace()
        p.set_probe(probe.astype(np.complex64))
        p.load_measurements(amps[p.local_probes()])
        p.set_volume(v0)
        p.iterate()
        outs.append(p.stitch())
        p.forward_grad(0, 10 ** 6)  # AccBuf after one more sweep (no passes)
        accs.append([p.debug_read_tile(k, 1) for k in range(grid[0] * grid[1])])
        p.close()
    assert np.array_equal(outs[0], outs[1])
    for a, b in zip(*accs):
        assert np.array_equal(a, b)
    ref, _, _, _ = O.reconstruct(v0.astype(np.float64), probe, amps.astype(np.float64), centers, d, grid[0], grid[1],
                                 n // 2, 1, alpha=1.0, period=period, batch=batch)
    assert rel(outs[1], ref) <= 1e-4 and rel(outs[1] - v0, ref - v0) <= 1e-3


def test_measurement_layout_flags_and_round_trip():
    """load_measurements: DC-centred intensities (reading #6: ifftshift once + sqrt at load) give
    the same store as DC-at-origin amplitudes; read_measurements inverts the load (bit-exact)."""
    from paper_2205_06327_b200.ptycho import PTYCHO_AMP_DC_CENTERED, PTYCHO_AMP_INTENSITY
    for s in (3, 4):  # odd S stores the turnaround layout transposed
        d = dict(n=64, slices=s, height=128, width=128, sigma=0.1, prop_c=3.1)
        p = make(d)
        p.set_scan(synth.scan_centers(128, 128, 2, 3))
        p.allocate_workspace()
        amp = synth.random_amplitudes(3, 6, 64)
        p.load_measurements(amp)
        assert np.array_equal(p.read_measurements(), amp)
        inten = np.fft.fftshift(amp.astype(np.float64) ** 2, axes=(1, 2)).astype(np.float32)
        p.load_measurements(inten, flags=PTYCHO_AMP_DC_CENTERED | PTYCHO_AMP_INTENSITY)
        got = p.read_measurements()
        assert np.abs(got - amp).max() <= 2e-7 * np.abs(amp).max()
        p.close()


def test_stitch_to_device_and_tile_rects():
    import torch
    d = dict(n=64, slices=3, height=150, width=131, sigma=0.1, prop_c=3.1)
    p = make(d, rows=2, cols=3, halo=20)
    p.set_scan(synth.scan_centers(150, 131, 3, 3))
    p.allocate_workspace()
    v = np.random.default_rng(6).random((3, 150, 131), dtype=np.float32)
    p.set_volume(torch.from_numpy(v).cuda())
    out = torch.zeros((3, 150, 131), dtype=torch.float32, device="cuda")
    p.stitch(out)
    assert np.array_equal(out.cpu().numpy(), v)
    for k, t in enumerate(O.tile_geometry(150, 131, 2, 3, 20)):
        assert p.tile_rect(k) == (t["ext"], t["interior"])


@pytest.mark.parametrize("batched", [False, True])
def test_async_measurement_load_bit_identical(batched):
    """PTYCHO_AMP_ASYNC (copies straight into the stores, overlapping the chains; each chain waits
    for its own chunk) == the synchronous load, bitwise -- including a second load with different
    data issued while the previous iteration's chains may still read the stores."""
    import torch
    from paper_2205_06327_b200.ptycho import PTYCHO_AMP_ASYNC
    n, s, h, w = 64, 4, 150, 131  # S even: the store needs no transposition
    rng = np.random.default_rng(8)
    probe = synth.probe(n, 8.0)
    vt = rng.random((s, h, w)).astype(np.float32)
    centers = synth.scan_centers(h, w, 5, 6)
    d = dict(n=n, slices=s, height=h, width=w, sigma=0.3, prop_c=3.135)
    full = (0, 0, h, w)
    amps = np.stack([O.farfield_magnitude(probe, O.window(vt.astype(np.float64), full, tuple(cc), n), d["sigma"],
                                          d["prop_c"]) for cc in centers]).astype(np.float32)
    amps2 = (amps * 1.01).astype(np.float32)
    outs = []
    for flags in (0, PTYCHO_AMP_ASYNC):
        p = make(d, rows=2, cols=3, alpha=1.0, period=3)
        p.set_scan(centers)
        if batched:
            p.set_schedule(True, 4)
        p.allocate_workspace()
        p.set_probe(probe.astype(np.complex64))
        ids = p.local_probes()
        h1 = torch.from_numpy(amps[ids]).pin_memory()
        h2 = torch.from_numpy(amps2[ids]).pin_memory()
        p.set_volume(0.5 * vt)
        losses = []
        for hb in (h1, h2, h1):
            p.load_measurements(hb, flags=flags)
            losses.append(p.iterate(want_loss=True))
        # loads of different data with NO synchronisation in between (iterate without
        # the loss returns with the chains still queued), so a load is enqueued while the previous
        # iteration's chains may still read the stores it overwrites
        for hb in (h2, h1, h2):
            p.load_measurements(hb, flags=flags)
            p.iterate()
        p.synchronize()
        back = np.zeros_like(amps[ids])
        p.read_measurements(0, len(ids), back)
        outs.append((p.stitch(), losses, back))
        p.close()
    assert np.array_equal(outs[0][0], outs[1][0]) and outs[0][1] == outs[1][1]
    assert np.array_equal(outs[1][2], amps2[ids])


def test_global_probe_exports_match_tile_exports():
    """ptycho_probe_grad / ptycho_probe_exitwave (SURVEY §8(b) names, global probe id, host or
    device output) == the per-tile debug exports, bitwise; a probe of another rank is EARG."""
    import torch
    from paper_2205_06327_b200.ptycho import PtychoError
    d, probe, vt, centers, amps = _recon_problem()
    p = make(d, rows=2, cols=3)
    p.set_scan(centers)
    p.allocate_workspace()
    p.set_probe(probe.astype(np.complex64))
    p.load_measurements(amps[p.local_probes()])
    p.set_volume(0.5 * vt)
    ids = list(p.local_probes())
    for gid in (ids[0], ids[len(ids) // 2], ids[-1]):
        tile = next(k for k in range(6) if gid in set(_tile_probes(p, k)))
        j = _tile_probes(p, tile).index(gid)
        g0, f0 = p.debug_probe_grad(tile, j)
        g1, f1 = p.probe_grad(gid)
        gd = torch.zeros((d["slices"], d["n"], d["n"]), dtype=torch.float32, device="cuda:0")
        _, f2 = p.probe_grad(gid, out=gd)
        assert np.array_equal(g0, g1) and np.array_equal(g0, gd.cpu().numpy()) and f0 == f1 == f2
        assert np.array_equal(p.debug_exit_wave(tile, j), p.probe_exitwave(gid))
    with pytest.raises(PtychoError) as e:
        p.probe_grad(10 ** 6)
    assert e.value.status == 1
    p.close()


def _tile_probes(p, k):
    """Global ids of tile k's probes (ascending) = local_probes() restricted to the tile."""
    lp = list(p.local_probes())
    start = sum(p.tile_probe_count(t) for t in range(k))
    return lp[start:start + p.tile_probe_count(k)]


def test_appp_transport_api_states():
    """set_appp_transport: EARG for an unknown mode, ESTATE once the first APPP call fixed the
    transport; a single rank reports NCCL (no cross-rank hops) after that call."""
    from paper_2205_06327_b200.ptycho import PtychoError, PTYCHO_APPP_P2P
    d, probe, vt, centers, amps = _recon_problem()
    p = make(d, rows=2, cols=3)
    p.set_scan(centers)
    p.allocate_workspace()
    assert p.appp_transport() == "auto"
    with pytest.raises(PtychoError) as e:
        p.set_appp_transport(7)
    assert e.value.status == 1
    p.set_appp_transport(PTYCHO_APPP_P2P)  # allowed before the first APPP call; moot on one rank
    p.appp_passes()
    assert p.appp_transport() == "nccl"
    with pytest.raises(PtychoError) as e:
        p.set_appp_transport(PTYCHO_APPP_P2P)
    assert e.value.status == 3
    p.close()


def test_stitch_pinned_zero_copy_equals_staged():
    """ptycho_stitch into pinned host memory (gather kernels write through the mapped alias, one
    launch per tile and slice parity, the bench's e2e path) == the staged per-slice copy into
    pageable memory == the device output, bitwise."""
    import torch
    c = synth.CONFIGS["tiny"]
    rng = np.random.default_rng(4)
    v = rng.random((5, 150, 131), dtype=np.float32)
    d = dict(n=64, slices=5, height=150, width=131, sigma=0.1, prop_c=3.135)
    p = make(d, rows=2, cols=3)
    p.set_scan(synth.scan_centers(150, 131, 3, 3))
    p.allocate_workspace()
    p.set_volume(v)
    staged = p.stitch()
    pinned = torch.empty((5, 150, 131), dtype=torch.float32).pin_memory()
    p.stitch(pinned)
    dev = torch.empty((5, 150, 131), dtype=torch.float32, device="cuda")
    p.stitch(dev)
    p.close()
    assert np.array_equal(staged, v)
    assert np.array_equal(pinned.numpy(), v)
    assert np.array_equal(dev.cpu().numpy(), v)


def test_profile_iteration_is_a_real_iteration():
    """ptycho_profile_iteration runs one real iteration (phases serial): the result equals
    ptycho_iterate's bitwise, and the phase times add up."""
    d, probe, vt, centers, amps = _recon_problem()
    v0 = (0.5 * vt).astype(np.float32)
    outs = []
    for prof in (False, True):
        p = make(d, rows=2, cols=3, alpha=1.0, period=4)
        p.set_scan(centers)
        p.allocate_workspace()
        p.set_probe(probe.astype(np.complex64))
        p.load_measurements(amps[p.local_probes()])
        p.set_volume(v0)
        if prof:
            bd = p.profile_iteration()
            assert bd["compute_ms"] > 0 and bd["acc_step_ms"] > 0 and bd["comm_ms"] >= 0
            assert bd["compute_ms"] + bd["comm_ms"] + bd["acc_step_ms"] <= bd["total_ms"] * 1.01
            assert bd["wait_ms"] == 0 and bd["nvlink_copy_bytes"] == 0  # one rank: no peers
        else:
            p.iterate()
        outs.append(p.stitch())
        p.close()
    assert np.array_equal(outs[0], outs[1])
