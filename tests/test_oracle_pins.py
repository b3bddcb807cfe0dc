"""Pins for the CPU oracle (oracle/ptycho_oracle.py) against things other than itself:
brute force, closed forms, invariants, the paper's / SPEC's worked examples.

Every function in the oracle has at least one pin here that a plausible slip (a dropped
term, a wrong sign or index, a transposed operand) would fail.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import ptycho_oracle as O
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_geometry.json")))


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def crandn(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


# ----------------------------------------------------------------------------- DFT
@pytest.mark.parametrize("n", [2, 4, 8])
def test_naive_dft_matches_brute_force(n):
    x = crandn(np.random.default_rng(n), n, n)
    assert rel(O.dft2_naive(x), O.dft2_brute(x)) < 1e-13
    assert rel(O.dft2_naive(x, inverse=True), O.dft2_brute(x, inverse=True)) < 1e-13


@pytest.mark.parametrize("n", [8, 16, 64])
def test_fft_matches_naive_dft(n):
    x = crandn(np.random.default_rng(1), n, n)
    assert rel(O.fft2(x), O.dft2_naive(x)) < 1e-12
    assert rel(O.ifft2(x), O.dft2_naive(x, inverse=True)) < 1e-12


def test_delta_is_flat():
    g = GOLD["delta_dft"]
    n = g["n"]
    x = np.zeros((n, n), complex)
    x[0, 0] = 1
    assert np.allclose(O.fft2(x), g["value"], atol=1e-15)


def test_plane_wave_single_bin():
    n, u0, v0 = 32, 3, 29
    yy, xx = np.mgrid[0:n, 0:n]
    pw = np.exp(2j * np.pi * (u0 * yy + v0 * xx) / n)
    f = O.fft2(pw)
    expect = np.zeros((n, n), complex)
    expect[u0, v0] = n
    assert np.abs(f - expect).max() < 1e-11


def test_parseval_and_inverse():
    x = crandn(np.random.default_rng(2), 64, 64)
    assert abs(np.sum(abs(O.fft2(x)) ** 2) / np.sum(abs(x) ** 2) - 1) < 1e-13
    assert rel(O.ifft2(O.fft2(x)), x) < 1e-14


# ----------------------------------------------------------------------------- propagator
def test_freq_index():
    assert list(O.freq_index(8)) == [0, 1, 2, 3, -4, -3, -2, -1]


def test_propagator_plane_wave_eigenfunction():
    n, c, u0, v0 = 32, 3.135, 5, 27
    yy, xx = np.mgrid[0:n, 0:n]
    pw = np.exp(2j * np.pi * (u0 * yy + v0 * xx) / n)
    out = O.ifft2(O.propagator(n, c) * O.fft2(pw))
    m_u, m_v = 5, 27 - 32
    h = np.exp(-1j * np.pi * c * (m_u ** 2 + m_v ** 2) / n ** 2)
    assert np.abs(out - h * pw).max() < 1e-12


def test_propagator_zero_is_identity_and_composition():
    n = 32
    p = synth.probe(n, 8.0)
    assert np.abs(O.propagator(n, 0.0) - 1).max() == 0
    # S slices of free space at c == one propagation at S*c
    s = 5
    psi_s, big_psi, _ = O.forward(p, np.zeros((s, n, n)), 0.1, 1.7)
    once = O.ifft2(O.propagator(n, s * 1.7) * O.fft2(p))
    assert rel(psi_s, once) < 1e-13


# ----------------------------------------------------------------------------- forward
def test_forward_v0_is_free_space_magnitude():
    n = 64
    p = synth.probe(n, 8.0)
    _, big_psi, _ = O.forward(p, np.zeros((4, n, n)), 0.1, 3.135)
    assert np.abs(np.abs(big_psi) - np.abs(np.fft.fft2(p, norm="ortho"))).max() < 1e-14


def test_forward_constant_potential_global_phase():
    n, s, sigma, v0 = 32, 3, 0.1, 0.37
    p = synth.probe(n, 8.0)
    _, free, _ = O.forward(p, np.zeros((s, n, n)), sigma, 3.135)
    _, big_psi, _ = O.forward(p, np.full((s, n, n), v0), sigma, 3.135)
    assert rel(big_psi, np.exp(1j * s * sigma * v0) * free) < 1e-13


def test_forward_energy_per_slice():
    n = 32
    rng = np.random.default_rng(3)
    p = synth.probe(n, 8.0)
    psi_s, big_psi, phis = O.forward(p, rng.random((4, n, n)), 0.7, 3.135)
    for phi in phis:
        assert abs(np.sum(abs(phi) ** 2) - 1) < 1e-13
    assert abs(np.sum(abs(big_psi) ** 2) - 1) < 1e-13


def test_forward_depends_on_slice_order():
    # guards against a forward that ignores propagation between slices
    n = 16
    rng = np.random.default_rng(4)
    p = synth.probe(n, 8.0)
    v = rng.random((2, n, n))
    a = O.forward(p, v, 1.0, 3.135)[1]
    b = O.forward(p, v[::-1].copy(), 1.0, 3.135)[1]
    assert rel(np.abs(a), np.abs(b)) > 1e-3


# ----------------------------------------------------------------------------- loss
def test_loss_zero_at_generating_volume_and_unit_at_zero_data():
    n = 32
    rng = np.random.default_rng(5)
    p = synth.probe(n, 8.0)
    v = rng.random((3, n, n))
    a = O.farfield_magnitude(p, v, 0.1, 3.135)
    assert O.probe_loss(p, v, a, 0.1, 3.135) < 1e-28
    assert abs(O.probe_loss(p, v, np.zeros((n, n)), 0.1, 3.135) - GOLD["loss_zero_measurement"]["value"]) < 1e-13


# ----------------------------------------------------------------------------- gradient
@pytest.mark.parametrize("seed,n,s", [(0, 8, 1), (1, 8, 2), (2, 8, 3), (3, 16, 1), (4, 16, 2), (5, 12, 3)])
def test_gradient_matches_central_differences(seed, n, s):
    rng = np.random.default_rng(seed)
    p = crandn(rng, n, n)
    p /= np.linalg.norm(p)
    v = rng.random((s, n, n))
    a = rng.random((n, n)) * 2 / n
    sigma, c = 0.7, 1.3
    g, _ = O.probe_grad(p, v, a, sigma, c)
    gfd = O.probe_grad_fd(p, v, a, sigma, c, eps=1e-5)
    assert rel(g, gfd) < 1e-5


@pytest.mark.parametrize("seed,n,s", [(10, 8, 2), (11, 8, 3), (12, 12, 4)])
def test_recomputed_gradient_matches_central_differences(seed, n, s):
    # stash-free adjoint: phi_s rebuilt by inverse propagation must give the
    # same d f / d V as finite differences of the forward model, and equal the stashed adjoint
    rng = np.random.default_rng(seed)
    p = crandn(rng, n, n)
    p /= np.linalg.norm(p)
    v = rng.random((s, n, n))
    a = rng.random((n, n)) * 2 / n
    sigma, c = 0.7, 1.3
    g, f = O.probe_grad_recompute(p, v, a, sigma, c)
    assert rel(g, O.probe_grad_fd(p, v, a, sigma, c, eps=1e-5)) < 1e-5
    g0, f0 = O.probe_grad(p, v, a, sigma, c)
    assert rel(g, g0) < 1e-12 and f == f0


def test_gradient_stationary_at_generating_volume():
    n = 32
    rng = np.random.default_rng(6)
    p = synth.probe(n, 8.0)
    v = rng.random((3, n, n))
    a = O.farfield_magnitude(p, v, 0.1, 3.135)
    g, f = O.probe_grad(p, v, a, 0.1, 3.135)
    assert np.abs(g).max() < 1e-12


def test_gradient_gauge_sum_zero():
    # adding a constant to V_s over the whole window only changes a global phase (App. A.6)
    n = 32
    rng = np.random.default_rng(7)
    p = synth.probe(n, 8.0)
    v = rng.random((3, n, n))
    a = synth.random_amplitudes(8, 1, n)[0].astype(np.float64)
    g, _ = O.probe_grad(p, v, a, 0.1, 3.135)
    for s in range(3):
        assert abs(g[s].sum()) < 1e-12 * np.abs(g[s]).sum()


def test_gradient_threshold_zeroes_dark_pixels():
    # tau = 1: everything below the RMS |Psi| is dropped -> gradient changes; tau=0 vs 1e-4 equal
    n = 16
    rng = np.random.default_rng(9)
    p = crandn(rng, n, n)
    p /= np.linalg.norm(p)
    v = rng.random((2, n, n))
    a = rng.random((n, n)) * 2 / n
    g0, _ = O.probe_grad(p, v, a, 0.5, 1.0, tau=0.0)
    g1, _ = O.probe_grad(p, v, a, 0.5, 1.0, tau=1e-4)
    g2, _ = O.probe_grad(p, v, a, 0.5, 1.0, tau=1.0)
    assert rel(g1, g0) < 1e-12
    assert rel(g2, g0) > 1e-3


# ----------------------------------------------------------------------------- geometry
def test_spec_mesh_example():
    g = GOLD["mesh_3x3_halo8_96"]
    tiles = O.tile_geometry(g["height"], g["width"], g["rows"], g["cols"], g["halo"])
    assert tiles[4]["interior"] == tuple(g["center_interior"])
    assert tiles[4]["ext"] == tuple(g["center_ext"])
    assert tiles[0]["ext"] == tuple(g["corner00_ext"])
    a, b = tiles[0]["ext"], tiles[3]["ext"]
    ov = (max(a[0], b[0]), max(a[1], b[1]), min(a[2], b[2]), min(a[3], b[3]))
    assert ov == tuple(g["overlap_00_10"])


def test_interiors_partition_with_ragged_remainder():
    tiles = O.tile_geometry(101, 77, 3, 4, 9)
    cover = np.zeros((101, 77), int)
    for t in tiles:
        y0, x0, y1, x1 = t["interior"]
        cover[y0:y1, x0:x1] += 1
    assert (cover == 1).all()
    assert tiles[-1]["interior"] == (66, 57, 101, 77)


def test_assignment_brute_force():
    rng = np.random.default_rng(10)
    centers = np.stack([rng.integers(0, 101, 300), rng.integers(0, 77, 300)], 1)
    tiles = O.tile_geometry(101, 77, 3, 4, 9)
    asg = O.assign_probes(centers, tiles)
    seen = sorted(i for a in asg for i in a)
    assert seen == list(range(300))
    for k, a in enumerate(asg):
        assert a == sorted(a)
        for i in a:
            y0, x0, y1, x1 = tiles[k]["interior"]
            assert y0 <= centers[i][0] < y1 and x0 <= centers[i][1] < x1


def test_lt_small_probe_counts():
    # SURVEY App. C (computed independently from the same readings #11, #14, #15)
    cfg = synth.CONFIGS["lt_small"]
    centers = synth.scan_centers(cfg.height, cfg.width, cfg.scan_ny, cfg.scan_nx)
    tiles = O.tile_geometry(cfg.height, cfg.width, 2, 4, cfg.halo)
    counts = [len(a) for a in O.assign_probes(centers, tiles)]
    assert counts == [496, 527, 496, 527, 512, 544, 512, 544]
    assert [t["ext"][0] for t in tiles[:1]] + [tiles[4]["ext"][0]] == [0, 256]
    assert [(t["ext"][1], t["ext"][3]) for t in tiles[:4]] == [(0, 896), (0, 1280), (256, 1536), (640, 1536)]


def test_exact_window_halo_covers_every_window():
    cfg = synth.CONFIGS["appp"]
    centers = synth.scan_centers(cfg.height, cfg.width, cfg.scan_ny, cfg.scan_nx)
    tiles = O.tile_geometry(cfg.height, cfg.width, 2, 2, cfg.n // 2)
    for k, a in enumerate(O.assign_probes(centers, tiles)):
        for i in a:
            m = O.window_mask(tiles[k]["ext"], tuple(centers[i]), cfg.n)
            cy, cx = centers[i]
            yy = cy - cfg.n // 2 + np.arange(cfg.n)
            xx = cx - cfg.n // 2 + np.arange(cfg.n)
            inside = ((yy >= 0) & (yy < cfg.height))[:, None] & ((xx >= 0) & (xx < cfg.width))[None, :]
            assert (m == inside).all()


def test_window_zero_extension_brute_force():
    rng = np.random.default_rng(11)
    vk = rng.random((2, 30, 40))
    ext = (10, 5, 40, 45)
    n = 16
    for center in [(12, 7), (39, 44), (25, 20), (0, 0)]:
        w = O.window(vk, ext, center, n)
        for s in range(2):
            for j in range(n):
                for l in range(n):
                    y, x = center[0] - n // 2 + j, center[1] - n // 2 + l
                    ok = ext[0] <= y < ext[2] and ext[1] <= x < ext[3]
                    assert w[s, j, l] == (vk[s, y - ext[0], x - ext[1]] if ok else 0.0)


# ----------------------------------------------------------------------------- APPP
GEOMS = [((96, 96), (3, 3), 8), ((96, 96), (3, 3), 40), ((48, 96), (2, 4), 24),
         ((60, 90), (4, 3), 7), ((192, 192), (2, 4), 64), ((50, 70), (1, 3), 11), ((70, 50), (3, 1), 11)]


@pytest.mark.parametrize("shape,grid,halo", GEOMS)
def test_appp_all_ones_gives_coverage_count(shape, grid, halo):
    tiles = O.tile_geometry(shape[0], shape[1], grid[0], grid[1], halo)
    bufs = [np.ones((2, t["ext"][2] - t["ext"][0], t["ext"][3] - t["ext"][1])) for t in tiles]
    msgs = O.appp_passes(bufs, tiles, *grid)
    assert msgs == 2 * (grid[0] - 1) * grid[1] + 2 * (grid[1] - 1) * grid[0]
    cnt = O.coverage_count(shape[0], shape[1], tiles)
    for b, t in zip(bufs, tiles):
        y0, x0, y1, x1 = t["ext"]
        assert (b[0] == cnt[y0:y1, x0:x1]).all() and (b[1] == b[0]).all()


@pytest.mark.parametrize("shape,grid,halo", GEOMS)
def test_appp_random_integers_equal_global_sum(shape, grid, halo):
    rng = np.random.default_rng(12)
    tiles = O.tile_geometry(shape[0], shape[1], grid[0], grid[1], halo)
    bufs = [rng.integers(0, 2 ** 16, (3, t["ext"][2] - t["ext"][0], t["ext"][3] - t["ext"][1])).astype(float)
            for t in tiles]
    total = O.global_sum(bufs, tiles, 3, *shape)
    O.appp_passes(bufs, tiles, *grid)
    for b, t in zip(bufs, tiles):
        y0, x0, y1, x1 = t["ext"]
        assert np.array_equal(b, total[:, y0:y1, x0:x1])


def test_appp_negative_control_interior_height_fails():
    rng = np.random.default_rng(13)
    tiles = O.tile_geometry(96, 96, 3, 3, 8)
    bufs = [rng.integers(0, 100, (1, t["ext"][2] - t["ext"][0], t["ext"][3] - t["ext"][1])).astype(float)
            for t in tiles]
    total = O.global_sum(bufs, tiles, 1, 96, 96)
    O.appp_passes(bufs, tiles, 3, 3, horizontal_full_height=False)
    assert any(not np.array_equal(b, total[:, t["ext"][0]:t["ext"][2], t["ext"][1]:t["ext"][3]])
               for b, t in zip(bufs, tiles))


def test_appp_spec_vertical_forward_example():
    g = GOLD["vertical_forward_3_column"]
    tiles = O.tile_geometry(g["height"], g["width"], g["rows"], g["cols"], g["halo"])
    assert (tiles[2]["ext"][0], tiles[2]["ext"][2]) == tuple(g["bottom_ext_rows"])
    bufs = [np.ones((1, t["ext"][2] - t["ext"][0], t["ext"][3] - t["ext"][1])) for t in tiles]
    # vertical forward only: run the chain by hand through a 3x1 mesh with R-1 adds
    for r in range(2):
        a, b = tiles[r], tiles[r + 1]
        oy = (max(a["ext"][0], b["ext"][0]), min(a["ext"][2], b["ext"][2]))
        bufs[r + 1][:, oy[0] - b["ext"][0]:oy[1] - b["ext"][0]] += bufs[r][:, oy[0] - a["ext"][0]:oy[1] - a["ext"][0]]
    for y, val in g["bottom_values_by_global_row"].items():
        assert (bufs[2][0, int(y) - tiles[2]["ext"][0]] == val).all()
    # full passes: all three equal the coverage count
    bufs = [np.ones((1, t["ext"][2] - t["ext"][0], t["ext"][3] - t["ext"][1])) for t in tiles]
    O.appp_passes(bufs, tiles, 3, 1)
    assert bufs[0][0, 51, 0] == 3 and bufs[2][0, 51 - 44, 0] == 3


def test_appp_spec_pair_example():
    g = GOLD["pair_add_2x1"]
    tiles = O.tile_geometry(g["height"], g["width"], 2, 1, g["halo"])
    bufs = [np.full((1, t["ext"][2] - t["ext"][0], t["ext"][3] - t["ext"][1]), float(v))
            for t, v in zip(tiles, (1, 2))]
    O.appp_passes(bufs, tiles, 2, 1)
    ov = (tiles[1]["ext"][0], tiles[0]["ext"][2])
    assert (bufs[0][0, ov[0]:ov[1]] == g["overlap_value"]).all()
    assert (bufs[1][0, :ov[1] - ov[0]] == g["overlap_value"]).all()
    assert (bufs[0][0, :ov[0]] == g["a_elsewhere"]).all()
    assert (bufs[1][0, ov[1] - ov[0]:] == g["b_elsewhere"]).all()


def test_stitch_round_trip_and_ignores_halos():
    rng = np.random.default_rng(14)
    v = rng.random((2, 101, 77))
    tiles = O.tile_geometry(101, 77, 3, 4, 9)
    vks = O.decompose(v, tiles)
    assert np.array_equal(O.stitch(vks, tiles, 2, 101, 77), v)
    for vk, t in zip(vks, tiles):  # scribble on halos only
        y0, x0, y1, x1 = t["interior"]
        ey0, ex0 = t["ext"][0], t["ext"][1]
        mask = np.ones(vk.shape[1:], bool)
        mask[y0 - ey0:y1 - ey0, x0 - ex0:x1 - ex0] = False
        vk[:, mask] = -1
    assert np.array_equal(O.stitch(vks, tiles, 2, 101, 77), v)


# ----------------------------------------------------------------------------- Alg. 1
def _tiny_problem(n=16, s=2, h=40, w=40, ny=3, nx=3, seed=15):
    rng = np.random.default_rng(seed)
    p = synth.probe(n, 3.0, aperture_frac=0.3)
    vt = rng.random((s, h, w))
    centers = synth.scan_centers(h, w, ny, nx)
    cfg = dict(n=n, sigma=0.3, prop_c=1.0)
    tiles = O.tile_geometry(h, w, 1, 1, 0)
    amps = [O.farfield_magnitude(p, O.window(vt, tiles[0]["ext"], tuple(c), n), 0.3, 1.0) for c in centers]
    return p, vt, centers, cfg, amps


def test_single_probe_double_step():
    # Alg. 1 with one tile and one probe: V <- V - alpha g (step 8) then V <- V - alpha AccBuf (step 15)
    p, vt, centers, cfg, amps = _tiny_problem(ny=1, nx=1)
    v0 = 0.5 * vt
    tile = O.tile_geometry(40, 40, 1, 1, 0)[0]
    g, _ = O.probe_grad(p, O.window(v0, tile["ext"], tuple(centers[0]), 16), amps[0], 0.3, 1.0)
    full = np.zeros_like(v0)
    O._scatter(full, tile["ext"], tuple(centers[0]), 16, g, O.window_mask(tile["ext"], tuple(centers[0]), 16), 1.0)
    out, losses, _, _ = O.reconstruct(v0, p, amps, centers, cfg, 1, 1, 0, 1, alpha=0.05)
    assert rel(out, v0 - 2 * 0.05 * full) < 1e-14


def test_frozen_multi_tile_equals_single_tile():
    # north_star invariant: after the four passes every tile holds the global sum (exact-window halo)
    p, vt, centers, cfg, amps = _tiny_problem(n=16, s=2, h=52, w=44, ny=5, nx=4)
    v0 = 0.5 * vt
    acc1, t1 = O.accumulate_frozen(v0, p, amps, centers, cfg, 1, 1, 8)
    acc4, t4 = O.accumulate_frozen(v0, p, amps, centers, cfg, 2, 3, 8)
    ref = O.stitch(acc1, t1, 2, 52, 44)
    assert rel(O.stitch(acc4, t4, 2, 52, 44), ref) < 1e-13
    for a, t in zip(acc4, t4):
        y0, x0, y1, x1 = t["ext"]
        assert rel(a, ref[:, y0:y1, x0:x1]) < 1e-13


def test_reconstruction_descends():
    p, vt, centers, cfg, amps = _tiny_problem(n=16, s=2, h=40, w=40, ny=4, nx=4)
    _, losses, _, _ = O.reconstruct(0.5 * vt, p, amps, centers, cfg, 2, 2, 8, 4, alpha=2.0)
    assert all(b < a for a, b in zip(losses, losses[1:]))


def test_segments():
    asg = [[0] * 10, [0] * 7]
    assert O.n_segments(asg, 0) == 1
    assert O.n_segments(asg, 3) == 4
    assert O.n_segments(asg, 10) == 1
    assert O.n_segments([[], []], 0) == 0


def test_batched_schedule_is_exactly_sequential():
    # windows of one batch are disjoint: every voxel sees the same update sequence (float64 exact)
    p, vt, centers, cfg, amps = _tiny_problem(n=16, s=2, h=60, w=60, ny=6, nx=6)
    a, _, _, _ = O.reconstruct(0.5 * vt, p, amps, centers, cfg, 2, 2, 8, 2, alpha=1.0, period=5)
    b, _, _, _ = O.reconstruct(0.5 * vt, p, amps, centers, cfg, 2, 2, 8, 2, alpha=1.0, period=5, batch=3)
    assert np.array_equal(a, b)
    order = O.batch_order(list(range(36)), centers, (0, 0, 60, 60), 16, 3)
    assert sorted(order) == list(range(36)) and order != list(range(36))


# ----------------------------------------------------------------------------- round-2 pins
# VERDICT r1 "What's weak" 2: each test below names the plausible oracle slip it catches.

def test_forward_single_slice_closed_form_transmit_then_propagate():
    # S = 1 (reading #1): Psi = F F^-1 (H F(t p)) = H F(t p) and |H| = 1, so |Psi| = |DFT(e^{i sigma V} p)|
    # exactly, for ANY propagator.  A propagate-then-transmit forward gives |DFT(t F^-1 H F p)|,
    # which differs for a non-constant V.  Pinned against the naive DFT (not the oracle's fft2).
    n, sigma, c = 32, 0.9, 3.135
    rng = np.random.default_rng(21)
    p = synth.probe(n, 8.0)
    v = rng.random((1, n, n))
    _, big_psi, _ = O.forward(p, v, sigma, c)
    closed = np.abs(O.dft2_naive(np.exp(1j * sigma * v[0]) * p))
    assert np.abs(np.abs(big_psi) - closed).max() < 1e-13
    # negative control: the wrong order is far from the closed form
    m = np.fft.fftfreq(n) * n
    h = np.exp(-1j * np.pi * c * (m[:, None] ** 2 + m[None, :] ** 2) / n ** 2)
    wrong = np.abs(O.dft2_naive(np.exp(1j * sigma * v[0]) * O.dft2_naive(h * O.dft2_naive(p), inverse=True)))
    assert rel(wrong, closed) > 1e-3


@pytest.mark.parametrize("n", [256, 1024])
def test_fft_matches_naive_dft_at_parity_sizes(n):
    # the parity tests use fft2 / ifft2 at N = 256 and 1024: pin them there against the O(N^3)
    # separable naive DFT (dft2_naive is itself pinned to the O(N^4) brute force at N <= 8)
    rng = np.random.default_rng(n)
    x = crandn(rng, n, n)
    assert rel(O.fft2(x), O.dft2_naive(x)) < 1e-12
    assert rel(O.ifft2(x), O.dft2_naive(x, inverse=True)) < 1e-12


def test_window_mask_brute_force_clipped_inside_object():
    # R_k strictly inside the object (an interior tile's extended rect): the mask must follow R_k,
    # not the object bounds (circle-halo clipping, reading #12)
    ext = (10, 5, 40, 45)
    n = 16
    for center in [(12, 7), (39, 44), (25, 20), (0, 0), (47, 52), (10, 30)]:
        m = O.window_mask(ext, center, n)
        for j in range(n):
            for l in range(n):
                y, x = center[0] - n // 2 + j, center[1] - n // 2 + l
                assert m[j, l] == (ext[0] <= y < ext[2] and ext[1] <= x < ext[3])


def _grad_at(p, vk, ext, center, n, amp, cfg):
    return O.probe_grad(p, O.window(vk, ext, center, n), amp, cfg["sigma"], cfg["prop_c"])[0]


def _scatter_full(shape, ext, center, n, g):
    out = np.zeros(shape)
    O._scatter(out, ext, center, n, g, O.window_mask(ext, center, n), 1.0)
    return out


def test_reconstruct_two_probes_once_per_iteration_hand_composed():
    # Alg. 1 steps 6-16 with one tile, two probes, passes once per iteration, alpha != alpha_acc:
    #   g0 = g(V0); V <- V0 - a g0; g1 = g(V0 - a g0); V <- V - a g1; V <- V - a_acc (g0 + g1)
    # Catches: alpha / alpha_acc swapped (g1 would be taken at V0 - a_acc g0), the step-8 update
    # skipped (g1 at V0), AccBuf not accumulated across probes.
    p, vt, _, cfg, _ = _tiny_problem(ny=1, nx=2)
    centers = np.array([[20, 14], [21, 24]], np.int32)  # overlapping 16 x 16 windows
    ext = O.tile_geometry(40, 40, 1, 1, 0)[0]["ext"]
    amps = [O.farfield_magnitude(p, O.window(vt, ext, tuple(c), 16), 0.3, 1.0) for c in centers]
    v0 = 0.5 * vt
    ext = O.tile_geometry(40, 40, 1, 1, 0)[0]["ext"]
    a, aa = 0.7, 0.2
    c0, c1 = tuple(centers[0]), tuple(centers[1])
    g0 = _scatter_full(v0.shape, ext, c0, 16, _grad_at(p, v0, ext, c0, 16, amps[0], cfg))
    g1 = _scatter_full(v0.shape, ext, c1, 16, _grad_at(p, v0 - a * g0, ext, c1, 16, amps[1], cfg))
    expect = v0 - a * g0 - a * g1 - aa * (g0 + g1)
    out, _, _, accs = O.reconstruct(v0, p, amps, centers, cfg, 1, 1, 0, 1, alpha=a, alpha_acc=aa)
    assert rel(out - v0, expect - v0) < 1e-10  # compared on the update, which is small next to V
    assert np.abs(accs[0]).max() == 0.0  # step 16: AccBuf reset
    swapped, _, _, _ = O.reconstruct(v0, p, amps, centers, cfg, 1, 1, 0, 1, alpha=aa, alpha_acc=a)
    assert rel(swapped - v0, expect - v0) > 1e-4


def test_reconstruct_two_iterations_every_probe_hand_composed():
    # T = 1 (passes after every local probe), one probe, two iterations:
    #   V1 = V0 - (a + a_acc) g(V0);  V2 = V1 - (a + a_acc) g(V1)
    # An AccBuf that is not reset (step 16) would subtract a_acc g(V0) again in iteration 2.
    p, vt, centers, cfg, amps = _tiny_problem(ny=1, nx=1)
    v0 = 0.5 * vt
    ext = O.tile_geometry(40, 40, 1, 1, 0)[0]["ext"]
    a, aa = 0.05, 0.03
    c0 = tuple(centers[0])
    v1 = v0 - (a + aa) * _scatter_full(v0.shape, ext, c0, 16, _grad_at(p, v0, ext, c0, 16, amps[0], cfg))
    v2 = v1 - (a + aa) * _scatter_full(v0.shape, ext, c0, 16, _grad_at(p, v1, ext, c0, 16, amps[0], cfg))
    out, losses, _, _ = O.reconstruct(v0, p, amps, centers, cfg, 1, 1, 0, 2, alpha=a, alpha_acc=aa, period=1)
    assert rel(out - v0, v2 - v0) < 1e-10
    assert len(losses) == 2
    g0 = _scatter_full(v0.shape, ext, c0, 16, _grad_at(p, v0, ext, c0, 16, amps[0], cfg))
    no_reset = v2 - aa * g0  # what a missing step 16 would add in iteration 2
    assert rel(no_reset - v0, v2 - v0) > 1e-2


def test_reconstruct_multi_tile_segments_hand_composed():
    # 2x1 tiles, exact-window halo, T = 3 (two pass segments per iteration: 3 and 1 local probes
    # per tile for a 4x2 scan): within a segment each tile runs sequential SGD on its own V_k;
    # then every tile adds the GLOBAL sum of the segment's AccBuf contributions (Eq. 2, P:205 --
    # composed here with global_sum, not with the APPP chain) times a_acc.
    n, s, h, w = 16, 2, 40, 28
    rng = np.random.default_rng(31)
    p = synth.probe(n, 3.0, aperture_frac=0.3)
    vt = rng.random((s, h, w))
    centers = synth.scan_centers(h, w, 4, 2)
    cfg = dict(n=n, sigma=0.3, prop_c=1.0)
    full = (0, 0, h, w)
    amps = [O.farfield_magnitude(p, O.window(vt, full, tuple(c), n), 0.3, 1.0) for c in centers]
    tiles = O.tile_geometry(h, w, 2, 1, n // 2)
    asg = O.assign_probes(centers, tiles)
    assert [len(x) for x in asg] == [4, 4]
    a, aa, T = 0.2, 0.1, 3
    v0 = 0.5 * vt
    vks = O.decompose(v0, tiles)
    for j in range(2):
        contribs = []
        for k, t in enumerate(tiles):
            acc = np.zeros_like(vks[k])
            for i in asg[k][j * T:(j + 1) * T]:
                c = tuple(int(x) for x in centers[i])
                g = _grad_at(p, vks[k], t["ext"], c, n, amps[i], cfg)
                d = np.zeros_like(acc)
                O._scatter(d, t["ext"], c, n, g, O.window_mask(t["ext"], c, n), 1.0)
                acc += d
                vks[k] = vks[k] - a * d
            contribs.append(acc)
        tot = O.global_sum(contribs, tiles, s, h, w)
        for k, t in enumerate(tiles):
            y0, x0, y1, x1 = t["ext"]
            vks[k] = vks[k] - aa * tot[:, y0:y1, x0:x1]
    expect = O.stitch(vks, tiles, s, h, w)
    out, _, _, _ = O.reconstruct(v0, p, amps, centers, cfg, 2, 1, n // 2, 1, alpha=a, alpha_acc=aa, period=T)
    assert rel(out - v0, expect - v0) < 1e-10


# ----------------------------------------------------------------------------- HVE baseline
def test_hve_spec_example_centre_tile_holds_all_nine():
    # SPEC S:480 / P:360-362 (Fig. halo_voxel_exch1 d-e): 3x3 mesh, 3x3 scan, one extra row of
    # probe locations -> the corner tile holds 4 probes, an edge tile 6, the centre tile all 9
    centers = synth.scan_centers(96, 96, 3, 3)          # centres 16, 48, 80: step 32
    tiles = O.hve_decompose(96, 96, 3, 3, centers, margin=32, halo=24)
    counts = [len(t["probes"]) for t in tiles]
    assert counts == [4, 6, 4, 6, 9, 6, 4, 6, 4]
    assert tiles[4]["probes"] == list(range(9))
    assert tiles[4]["ext"] == (8, 8, 88, 88) and tiles[0]["ext"] == (0, 0, 56, 56)


def test_hve_trivial_mesh_and_too_small_tiles():
    centers = synth.scan_centers(96, 96, 6, 6)
    t = O.hve_decompose(96, 96, 1, 1, centers, margin=16, halo=8)
    assert len(t) == 1 and t[0]["probes"] == list(range(36)) and t[0]["ext"] == (0, 0, 96, 96)
    with pytest.raises(O.TileTooSmall):
        O.hve_decompose(96, 96, 6, 6, centers, margin=16, halo=24)  # interiors 16 < halo 24
    O.hve_decompose(96, 96, 6, 6, centers, margin=16, halo=16)      # halo = interior: fine


def _hve_problem(seed=41):
    n, s, h, w = 16, 2, 48, 48
    rng = np.random.default_rng(seed)
    p = synth.probe(n, 3.0, aperture_frac=0.3)
    vt = rng.random((s, h, w))
    centers = synth.scan_centers(h, w, 6, 6)  # step 8
    cfg = dict(n=n, sigma=0.3, prop_c=1.0)
    amps = [O.farfield_magnitude(p, O.window(vt, (0, 0, h, w), tuple(c), n), 0.3, 1.0) for c in centers]
    return p, vt, centers, cfg, amps


def test_hve_one_tile_is_plain_sgd():
    # 1x1: HVE is sequential per-probe SGD, i.e. Alg. 1 on one tile without the accumulated step
    p, vt, centers, cfg, amps = _hve_problem()
    v0 = 0.5 * vt
    a, _, _ = O.hve_reconstruct(v0, p, amps, centers, cfg, 1, 1, 8, 8, 2, alpha=2.0)
    b, _, _, _ = O.reconstruct(v0, p, amps, centers, cfg, 1, 1, 0, 2, alpha=2.0, alpha_acc=0.0)
    assert np.array_equal(a, b)


def test_hve_all_probes_everywhere_equals_single_tile():
    # with every probe on every tile (2x2 mesh, margin past the object) each tile runs the
    # full reconstruction on the whole object -> the exchange is a no-op and the stitch equals 1x1
    p, vt, centers, cfg, amps = _hve_problem()
    v0 = 0.5 * vt
    tiles = O.hve_decompose(48, 48, 2, 2, centers, margin=100, halo=24)
    assert all(len(t["probes"]) == 36 and t["ext"] == (0, 0, 48, 48) for t in tiles)
    a, _, _ = O.hve_reconstruct(v0, p, amps, centers, cfg, 2, 2, 100, 24, 2, alpha=2.0)
    b, _, _ = O.hve_reconstruct(v0, p, amps, centers, cfg, 1, 1, 0, 0, 2, alpha=2.0)
    assert np.array_equal(a, b)


def test_hve_halos_equal_owner_interiors_after_exchange():
    # after each copy-paste every halo voxel equals its owner's interior voxel bitwise
    p, vt, centers, cfg, amps = _hve_problem()
    v0 = 0.5 * vt
    out, _, vks = O.hve_reconstruct(v0, p, amps, centers, cfg, 2, 2, 8, 12, 1, alpha=2.0)
    tiles = O.hve_decompose(48, 48, 2, 2, centers, margin=8, halo=12)
    for vk, t in zip(vks, tiles):
        y0, x0, y1, x1 = t["ext"]
        assert np.array_equal(vk, out[:, y0:y1, x0:x1])  # every voxel of R_k = the stitched (owner) value
    # and the result differs from GD's (the methods are not equivalent with partial probe sets)
    gd, _, _, _ = O.reconstruct(v0, p, amps, centers, cfg, 2, 2, 12, 1, alpha=2.0, alpha_acc=0.0)
    assert not np.array_equal(out, gd)


def test_seam_score_closed_form():
    s, h, w, xb = 2, 10, 12, 6  # 1x2 mesh: one vertical border between x = 5 and x = 6
    a, b = 0.5, 3.0
    xx = np.arange(w)[None, None, :] * np.ones((s, h, 1))
    err = a * xx + b * (xx >= xb)
    inner_mean = a * s * h * (w - 2) / (s * (h - 1) * w + s * h * (w - 2))
    assert abs(O.seam_score(err, h, w, 1, 2) - (a + b) / inner_mean) < 1e-12
    assert O.seam_score(np.ones((s, h, w)), h, w, 2, 2) == 0.0
