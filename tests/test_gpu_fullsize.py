"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (the config's
tile grid as virtual tiles on one GPU, halo N/2, CUDA-graph + PDL chains, occupancy-selected
kernels), on sampled outputs the float64 oracle computes one by one: the AccBuf / V update of one
probe of one tile after a real forward_grad, and the per-probe gradient and loss.

Tolerance: max(1e-5, 2 x fp32 floor) rel L2 (the floor = the same oracle run in float32,
SURVEY §8(c.5)); a few minutes of oracle time per config."""
import numpy as np
import pytest

from oracle import ptycho_oracle as O
import synth

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


@pytest.mark.parametrize("name,tile,local", [("lt_small", 5, 200), ("appp", 3, 500), ("lt_small", 0, 0),
                                             ("lt_large", 6, 1500)])
def test_fullsize_sampled_update(name, tile, local):
    from paper_2205_06327_b200.ptycho import Ptycho
    c = synth.CONFIGS[name]
    n, s, h, w = c.n, c.slices, c.height, c.width
    rows, cols = c.grid
    probe = synth.probe(n, c.defocus_nm)
    vt = synth.volume(0, s, h, w)
    v0 = (0.5 * vt).astype(np.float32)
    centers = synth.scan_centers(h, w, c.scan_ny, c.scan_nx)
    tiles = O.tile_geometry(h, w, rows, cols, n // 2)
    asg = O.assign_probes(centers, tiles)
    gid = asg[tile][local]
    ext = tiles[tile]["ext"]
    center = tuple(int(v) for v in centers[gid])

    amp = O.farfield_magnitude(probe, O.window(vt.astype(np.float64), (0, 0, h, w), center, n), c.sigma, c.prop_c)
    vwin = O.window(v0.astype(np.float64), (0, 0, h, w), center, n)
    g_ref, f_ref = O.probe_grad(probe, vwin, amp, c.sigma, c.prop_c)
    g32, f32 = O.probe_grad(probe, vwin, amp, c.sigma, c.prop_c, dtype=np.float32)
    floor = rel(g32, g_ref)
    tol = max(1e-5, 2 * floor)
    ftol = max(1e-5, 2 * abs(f32 - f_ref) / f_ref)

    # alpha large enough that the step-8 update alpha g reaches ~|V| on the window (at alpha = 0.5
    # it sat below one float32 ulp of V and a skipped or sign-flipped update passed)
    alpha = float(np.abs(v0).mean() / np.abs(g_ref).max())
    p = Ptycho(n, s, h, w, c.sigma, c.prop_c, alpha=alpha)
    p.set_tiles(rows, cols, n // 2)
    p.set_scan(centers)
    p.allocate_workspace()
    p.set_probe(probe.astype(np.complex64))
    first_local = sum(len(a) for a in asg[:tile]) + local  # local order: tiles ascending
    p.load_measurements(amp[None].astype(np.float32), first_local=first_local)
    p.set_volume(v0)

    g, f = p.debug_probe_grad(tile, local)
    e_grad = rel(g, g_ref)

    # the real hot path: every tile processes its local probe `local` (graphs + PDL)
    p.forward_grad(local, 1)
    acc = p.debug_read_tile(tile, 1)
    vk = p.debug_read_tile(tile, 0)
    mask = O.window_mask(ext, center, n)
    full_g = np.zeros((s, ext[2] - ext[0], ext[3] - ext[1]))
    O._scatter(full_g, ext, center, n, g_ref, mask, 1.0)
    e_acc = rel(acc, full_g)
    v0k = v0[:, ext[0]:ext[2], ext[1]:ext[3]].astype(np.float64)
    # the step itself, dV / alpha = (V0 - V) / alpha vs the oracle's g (Alg. 1 step 8); the float32
    # store of V - alpha g rounds each voxel by <= 2^-24 |V|, which bounds the extra error
    dv = (v0k - vk.astype(np.float64)) / alpha
    e_dv = rel(dv, full_g)
    round_bound = float(np.linalg.norm(2.0 ** -24 * np.abs(v0k) * (full_g != 0)) / alpha / np.linalg.norm(full_g))
    print(f"{name} tile {tile} probe {local} (global {gid}): grad {e_grad:.2e}, AccBuf {e_acc:.2e}, "
          f"dV/alpha {e_dv:.2e} (alpha {alpha:.3g}, V-rounding bound {round_bound:.1e}, fp32 floor {floor:.2e}); "
          f"loss rel {abs(f - f_ref) / f_ref:.2e}")
    assert e_grad <= tol and e_acc <= tol
    assert e_dv <= tol + 2 * round_bound
    assert np.array_equal(vk[full_g == 0], v0[:, ext[0]:ext[2], ext[1]:ext[3]][full_g == 0])  # outside win ^ R_k
    assert abs(f - f_ref) <= ftol * f_ref
    p.close()


def test_fullsize_stash_free_gradient():
    """LT-small (N = 1024, S = 100) sampled probe through the stash-free adjoint (2-slice stash
    ring + phi recomputation) in the bench launch configuration; tolerance from the float32 floor
    of the same recurrence (oracle.probe_grad_recompute)."""
    from paper_2205_06327_b200.ptycho import Ptycho, PTYCHO_F_STASH_FREE
    c = synth.CONFIGS["lt_small"]
    n, s, h, w = c.n, c.slices, c.height, c.width
    rows, cols = c.grid
    tile, local = 5, 200
    probe = synth.probe(n, c.defocus_nm)
    vt = synth.volume(0, s, h, w)
    v0 = (0.5 * vt).astype(np.float32)
    centers = synth.scan_centers(h, w, c.scan_ny, c.scan_nx)
    tiles = O.tile_geometry(h, w, rows, cols, n // 2)
    asg = O.assign_probes(centers, tiles)
    gid = asg[tile][local]
    center = tuple(int(v) for v in centers[gid])
    amp = O.farfield_magnitude(probe, O.window(vt.astype(np.float64), (0, 0, h, w), center, n), c.sigma, c.prop_c)
    vwin = O.window(v0.astype(np.float64), (0, 0, h, w), center, n)
    g_ref, f_ref = O.probe_grad(probe, vwin, amp, c.sigma, c.prop_c)
    g32, _ = O.probe_grad_recompute(probe, vwin, amp, c.sigma, c.prop_c, dtype=np.float32)
    floor = rel(g32, g_ref)
    p = Ptycho(n, s, h, w, c.sigma, c.prop_c, alpha=0.5, flags=PTYCHO_F_STASH_FREE)
    p.set_tiles(rows, cols, n // 2)
    p.set_scan(centers)
    p.allocate_workspace()
    p.set_probe(probe.astype(np.complex64))
    p.load_measurements(amp[None].astype(np.float32), first_local=sum(len(a) for a in asg[:tile]) + local)
    p.set_volume(v0)
    g, f = p.probe_grad(gid)
    err = rel(g, g_ref)
    print(f"lt_small stash-free tile {tile} probe {local}: grad {err:.2e} (recompute fp32 floor {floor:.2e}); "
          f"loss rel {abs(f - f_ref) / f_ref:.2e}")
    assert err <= max(1e-5, 2 * floor)
    p.close()
