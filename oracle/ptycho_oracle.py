"""CPU oracle for the gradient-decomposition hot path of arXiv 2205.06327.

TEST INFRASTRUCTURE -- NOT PART OF THE PRODUCT.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import this module.  It
shares no code with the CUDA path (paper_2205_06327_b200/) and imports nothing
from it.

Plain float64 / complex128 numpy, written to be checked against the paper by eye.
Library primitive used as a step: numpy.fft (unitary, norm="ortho"); it is pinned
against a naive DFT in tests/test_oracle_pins.py.  Citations: P:n = PAPER.md line
n, S:n = SPEC.md line n (the "readings" #k are listed in DESIGN.md §Readings).

Parity status of each function (all pinned; see tests/test_oracle_pins.py):
  dft2_naive ........... brute force O(N^4) on N<=8, closed forms (delta, plane wave)
  fft2 / ifft2 ......... naive DFT, Parseval, inverse o forward = I
  propagator ........... plane-wave eigenfunction, composition, c=0 identity
  window ............... brute-force loops
  forward .............. V=0 closed form, constant-V phase, per-slice energy
  probe_loss ........... a=|G| -> 0, a=0 -> 1
  probe_grad ........... central finite differences, stationarity, gauge sum
  geometry ............. brute-force assignment / coverage, SPEC worked examples (tests/golden)
  appp_passes .......... coverage count (all ones), random-int global sum, negative control
  reconstruct .......... K=1 literal SGD, alpha=0 frozen equivalence (north_star invariant)
  stitch ............... round trip
  hve_decompose ........ SPEC worked example (3x3 mesh, 3x3 scan, one extra row -> centre tile holds all 9),
                         1x1 trivial case, TileTooSmall on a fine mesh
  hve_reconstruct ...... 1x1 == plain per-probe SGD, all-probes-everywhere == single tile, halos == owners'
                         interiors bitwise after every exchange
  seam_score ........... closed forms (constant field -> 0 jumps; a step placed on a tile border)
The paper's Tables II/III cannot be reproduced (no dataset, no Summit): parity unpinned
for those, and they are not computed here.
"""
from __future__ import annotations

import math
import numpy as np

TAU = 1e-4  # reading #30: chi = 0 where |Psi| <= TAU * ||p||_2 / N


# ---------------------------------------------------------------------------------
# Discrete Fourier transforms (reading #4: unitary normalisation)
# ---------------------------------------------------------------------------------
def dft_matrix(n: int, inverse: bool = False) -> np.ndarray:
    """Unitary 1-D DFT matrix  F[u, y] = exp(-+2 pi i u y / n) / sqrt(n)."""
    u = np.arange(n)
    sign = 1.0 if inverse else -1.0
    return np.exp(sign * 2j * np.pi * np.outer(u, u) / n) / math.sqrt(n)


def dft2_naive(x: np.ndarray, inverse: bool = False) -> np.ndarray:
    """Separable naive 2-D DFT, O(N^3): (F x)[u,v] = (1/N) sum_{y,x} x[y,x] e^{-2 pi i (uy+vx)/N}."""
    n = x.shape[-1]
    f = dft_matrix(n, inverse)
    return f @ x @ f.T


def dft2_brute(x: np.ndarray, inverse: bool = False) -> np.ndarray:
    """Brute-force O(N^4) 2-D DFT straight from the definition (self-check for N <= 8)."""
    n = x.shape[0]
    sign = 1.0 if inverse else -1.0
    out = np.zeros((n, n), dtype=np.complex128)
    for u in range(n):
        for v in range(n):
            acc = 0j
            for yy in range(n):
                for xx in range(n):
                    acc += x[yy, xx] * np.exp(sign * 2j * np.pi * (u * yy + v * xx) / n)
            out[u, v] = acc / n
    return out


def fft2(x: np.ndarray) -> np.ndarray:
    return np.fft.fft2(x, norm="ortho")


def ifft2(x: np.ndarray) -> np.ndarray:
    return np.fft.ifft2(x, norm="ortho")


# ---------------------------------------------------------------------------------
# Fresnel propagator (reading #3):  H[u,v] = exp(-i pi c (m_u^2 + m_v^2) / N^2)
# ---------------------------------------------------------------------------------
def freq_index(n: int) -> np.ndarray:
    """m_u = u for u < N/2, u - N otherwise (fftfreq in pixels of the N-point grid)."""
    u = np.arange(n)
    return np.where(u < n // 2, u, u - n).astype(np.float64)


def propagator(n: int, c: float) -> np.ndarray:
    m = freq_index(n)
    return np.exp(-1j * np.pi * c * (m[:, None] ** 2 + m[None, :] ** 2) / float(n * n))


# ---------------------------------------------------------------------------------
# Probe window with zero-extension (readings #10, #12)
# ---------------------------------------------------------------------------------
def window(vk: np.ndarray, ext: tuple, center: tuple, n: int) -> np.ndarray:
    """V~_s[j,l] = V_k[s][cy-N/2+j][cx-N/2+l] if that voxel lies in R_k = ext, else 0.

    vk is the extended tile [S][ey1-ey0][ex1-ex0] in global coordinates offset by ext=(ey0,ex0,ey1,ex1).
    """
    ey0, ex0, ey1, ex1 = ext
    cy, cx = center
    wy0, wx0 = cy - n // 2, cx - n // 2
    out = np.zeros((vk.shape[0], n, n), dtype=np.float64)
    y0, y1 = max(wy0, ey0), min(wy0 + n, ey1)
    x0, x1 = max(wx0, ex0), min(wx0 + n, ex1)
    if y0 < y1 and x0 < x1:
        out[:, y0 - wy0:y1 - wy0, x0 - wx0:x1 - wx0] = vk[:, y0 - ey0:y1 - ey0, x0 - ex0:x1 - ex0]
    return out


def window_mask(ext: tuple, center: tuple, n: int) -> np.ndarray:
    """Boolean [N][N]: which window pixels lie inside R_k (gradient is kept only there)."""
    ey0, ex0, ey1, ex1 = ext
    cy, cx = center
    yy = cy - n // 2 + np.arange(n)
    xx = cx - n // 2 + np.arange(n)
    return ((yy >= ey0) & (yy < ey1))[:, None] & ((xx >= ex0) & (xx < ex1))[None, :]


# ---------------------------------------------------------------------------------
# Multislice forward model G (reading #1) and loss f_i (Eq. 1; Eq. 2)
# ---------------------------------------------------------------------------------
def forward(probe: np.ndarray, vwin: np.ndarray, sigma: float, c: float, dtype=np.float64):
    """psi_0 = p;  phi_s = exp(i sigma V_s) psi_s;  psi_{s+1} = F^-1(H F phi_s);  Psi = F psi_S.

    Returns (psi_S, Psi, [phi_0 .. phi_{S-1}]).  The propagation after the last slice
    is applied literally (reading #5).  dtype=np.float32 runs the same arithmetic in
    single precision (only to measure the fp32 floor); the oracle is float64.
    """
    n = probe.shape[0]
    cdt = np.complex64 if dtype == np.float32 else np.complex128
    h = propagator(n, c).astype(cdt)
    psi = probe.astype(cdt)
    vwin = vwin.astype(dtype)
    sigma = dtype(sigma)
    phis = []
    for s in range(vwin.shape[0]):
        phi = np.exp(1j * sigma * vwin[s]).astype(cdt) * psi
        phis.append(phi)
        psi = ifft2(h * fft2(phi))
    return psi, fft2(psi), phis


def probe_loss(probe, vwin, amp, sigma, c) -> float:
    """f_i = sum_px (|y_i| - |G(p_i, V)|)^2, plain sum (reading #7)."""
    _, big_psi, _ = forward(probe, vwin, sigma, c)
    return float(np.sum((np.abs(big_psi) - amp) ** 2))


def probe_grad(probe, vwin, amp, sigma, c, tau: float = TAU, dtype=np.float64):
    """Individual image gradient d f_i / d V over the full window (Alg. 1 step 6; Eq. 2).

    Adjoint of the forward chain (Wirtinger chi = d f / d conj z):
      chi_Psi   = (|Psi| - a) Psi / |Psi|       (0 where |Psi| <= tau ||p|| / N, reading #30)
      chi       = F^-1 chi_Psi                  (chi_{psi_S})
      for s = S-1 .. 0:
          chi   = F^-1 (conj(H) F chi)          (chi_{phi_s})
          g_s   = 2 sigma Im(chi conj(phi_s))
          chi   = conj(exp(i sigma V_s)) chi    (chi_{psi_s})
    Returns (g [S][N][N], f_i).  dtype as in forward().
    """
    n = probe.shape[0]
    cdt = np.complex64 if dtype == np.float32 else np.complex128
    h = propagator(n, c).astype(cdt)
    vwin = vwin.astype(dtype)
    _, big_psi, phis = forward(probe, vwin, sigma, c, dtype)
    mag = np.abs(big_psi)
    resid = mag - amp.astype(dtype)
    f = float(np.sum(resid ** 2))
    thr = tau * math.sqrt(float(np.sum(np.abs(probe) ** 2))) / n
    keep = mag > thr
    chi_big = np.zeros_like(big_psi)
    chi_big[keep] = resid[keep] * big_psi[keep] / mag[keep]
    chi = ifft2(chi_big)
    g = np.zeros(vwin.shape, dtype=dtype)
    for s in range(vwin.shape[0] - 1, -1, -1):
        chi = ifft2(np.conj(h) * fft2(chi))
        g[s] = 2.0 * sigma * np.imag(chi * np.conj(phis[s]))
        chi = np.conj(np.exp(1j * dtype(sigma) * vwin[s])).astype(cdt) * chi
    return g, f


def probe_grad_recompute(probe, vwin, amp, sigma, c, tau: float = TAU, dtype=np.float64):
    """The same gradient with phi_s recomputed backwards instead of stashed (SURVEY §8(f) #4,
    derived from App. A: the propagator is unitary and |t_s| = 1, so
      psi_{s+1} = F^-1 H F phi_s   =>   phi_s = F^-1 conj(H) F psi_{s+1},   psi_s = conj(t_s) phi_s).
    Keeps only phi_{S-1} from the forward and runs, for s = S-1 .. 0, the chi recursion of
    probe_grad next to the phi recursion
      g_s = 2 sigma Im(chi conj(phi_s)) ; chi <- conj(t_s) chi ; phi <- conj(t_s) phi ;
      chi <- F^-1 conj(H) F chi ; phi <- F^-1 conj(H) F phi.
    In float64 it equals probe_grad to rounding; in float32 it gives the rounding floor of the
    recomputation (the phi chain adds S-1 propagations).  Returns (g, f_i)."""
    n = probe.shape[0]
    cdt = np.complex64 if dtype == np.float32 else np.complex128
    h = propagator(n, c).astype(cdt)
    vwin = vwin.astype(dtype)
    _, big_psi, phis = forward(probe, vwin, sigma, c, dtype)
    phi = phis[-1]
    mag = np.abs(big_psi)
    resid = mag - amp.astype(dtype)
    f = float(np.sum(resid ** 2))
    thr = tau * math.sqrt(float(np.sum(np.abs(probe) ** 2))) / n
    keep = mag > thr
    chi_big = np.zeros_like(big_psi)
    chi_big[keep] = resid[keep] * big_psi[keep] / mag[keep]
    chi = ifft2(chi_big)
    g = np.zeros(vwin.shape, dtype=dtype)
    s_last = vwin.shape[0] - 1
    for s in range(s_last, -1, -1):
        chi = ifft2(np.conj(h) * fft2(chi))
        if s < s_last:
            phi = ifft2(np.conj(h) * fft2(phi))
        g[s] = 2.0 * sigma * np.imag(chi * np.conj(phi))
        t_conj = np.conj(np.exp(1j * dtype(sigma) * vwin[s])).astype(cdt)
        chi = t_conj * chi
        phi = t_conj * phi
    return g, f


def probe_grad_fd(probe, vwin, amp, sigma, c, eps: float = 1e-5) -> np.ndarray:
    """Central finite differences (f(V+e) - f(V-e)) / (2 eps) for every window voxel."""
    g = np.zeros(vwin.shape, dtype=np.float64)
    for idx in np.ndindex(*vwin.shape):
        vp = vwin.copy()
        vm = vwin.copy()
        vp[idx] += eps
        vm[idx] -= eps
        g[idx] = (probe_loss(probe, vp, amp, sigma, c) - probe_loss(probe, vm, amp, sigma, c)) / (2 * eps)
    return g


def farfield_magnitude(probe, vwin, sigma, c) -> np.ndarray:
    """|G(p, V)| -- the simulated measurement amplitude."""
    return np.abs(forward(probe, vwin, sigma, c)[1])


# ---------------------------------------------------------------------------------
# Geometry: lateral tiles + halos, probe assignment (readings #13-#16)
# ---------------------------------------------------------------------------------
def split_extent(extent: int, parts: int):
    """Uniform split, remainder to the last part (reading #14). Returns [(a, b)] half-open."""
    base = extent // parts
    return [(p * base, extent if p == parts - 1 else (p + 1) * base) for p in range(parts)]


def tile_geometry(height: int, width: int, rows: int, cols: int, halo: int):
    """Interiors and extended rects R_k (interior dilated by halo, clipped).  Tile k = r*C + c.

    Returns list of dicts {r, c, interior:(y0,x0,y1,x1), ext:(y0,x0,y1,x1)}.
    """
    ys = split_extent(height, rows)
    xs = split_extent(width, cols)
    tiles = []
    for r in range(rows):
        for c in range(cols):
            y0, y1 = ys[r]
            x0, x1 = xs[c]
            tiles.append(dict(r=r, c=c, interior=(y0, x0, y1, x1),
                              ext=(max(0, y0 - halo), max(0, x0 - halo),
                                   min(height, y1 + halo), min(width, x1 + halo))))
    return tiles


def assign_probes(centers: np.ndarray, tiles) -> list:
    """Probe -> tile by centre containment in the half-open interior (reading #15);
    each tile's probes in ascending global index (reading #16)."""
    out = [[] for _ in tiles]
    for i, (cy, cx) in enumerate(centers):
        for k, t in enumerate(tiles):
            y0, x0, y1, x1 = t["interior"]
            if y0 <= cy < y1 and x0 <= cx < x1:
                out[k].append(i)
                break
    return out


def coverage_count(height: int, width: int, tiles) -> np.ndarray:
    """Number of extended rects covering each pixel (brute force)."""
    cnt = np.zeros((height, width), dtype=np.int64)
    for t in tiles:
        y0, x0, y1, x1 = t["ext"]
        cnt[y0:y1, x0:x1] += 1
    return cnt


# ---------------------------------------------------------------------------------
# Gradient accumulation passes (Fig. forward_backward; reading #21)
# ---------------------------------------------------------------------------------
def _isect(a, b):
    return (max(a[0], b[0]), min(a[1], b[1]))


def _region_views(buf, ext, y, x):
    """View of buf (tile array in coords offset by ext) over the global y/x intervals."""
    return buf[:, y[0] - ext[0]:y[1] - ext[0], x[0] - ext[1]:x[1] - ext[1]]


def appp_passes(bufs, tiles, rows: int, cols: int, horizontal_full_height: bool = True) -> int:
    """Vertical forward (ADD), vertical backward (REPLACE), horizontal forward (ADD),
    horizontal backward (REPLACE), in Alg. 1's order.  In place on bufs
    (list of [S][eh][ew] arrays indexed by tile k = r*C + c).

    The horizontal overlap spans the full extended height Y_r (reading #21);
    horizontal_full_height=False gives the interior-height variant used as a negative control.
    Returns the number of messages (2(R-1)C + 2(C-1)R).
    """
    msgs = 0
    yint = lambda t: (t["ext"][0], t["ext"][2])
    xint = lambda t: (t["ext"][1], t["ext"][3])
    # vertical forward: chain down each tile column, buffer[r+1] += buffer[r] on the overlap
    for c in range(cols):
        for r in range(rows - 1):
            a, b = tiles[r * cols + c], tiles[(r + 1) * cols + c]
            oy = _isect(yint(a), yint(b))
            ox = xint(a)
            if oy[0] < oy[1]:
                _region_views(bufs[(r + 1) * cols + c], b["ext"], oy, ox)[...] += \
                    _region_views(bufs[r * cols + c], a["ext"], oy, ox)
            msgs += 1
    # vertical backward: chain up, buffer[r-1] := buffer[r] on the overlap ("replaces")
    for c in range(cols):
        for r in range(rows - 1, 0, -1):
            a, b = tiles[r * cols + c], tiles[(r - 1) * cols + c]
            oy = _isect(yint(a), yint(b))
            ox = xint(a)
            if oy[0] < oy[1]:
                _region_views(bufs[(r - 1) * cols + c], b["ext"], oy, ox)[...] = \
                    _region_views(bufs[r * cols + c], a["ext"], oy, ox)
            msgs += 1
    # horizontal forward / backward over the full extended height Y_r
    for r in range(rows):
        for c in range(cols - 1):
            a, b = tiles[r * cols + c], tiles[r * cols + c + 1]
            oy = yint(a) if horizontal_full_height else (a["interior"][0], a["interior"][2])
            ox = _isect(xint(a), xint(b))
            if ox[0] < ox[1]:
                _region_views(bufs[r * cols + c + 1], b["ext"], oy, ox)[...] += \
                    _region_views(bufs[r * cols + c], a["ext"], oy, ox)
            msgs += 1
    for r in range(rows):
        for c in range(cols - 1, 0, -1):
            a, b = tiles[r * cols + c], tiles[r * cols + c - 1]
            oy = yint(a) if horizontal_full_height else (a["interior"][0], a["interior"][2])
            ox = _isect(xint(a), xint(b))
            if ox[0] < ox[1]:
                _region_views(bufs[r * cols + c - 1], b["ext"], oy, ox)[...] = \
                    _region_views(bufs[r * cols + c], a["ext"], oy, ox)
            msgs += 1
    return msgs


def global_sum(contribs, tiles, slices: int, height: int, width: int) -> np.ndarray:
    """Eq. 2: scatter-add every tile's contribution into a zero full-volume array."""
    out = np.zeros((slices, height, width), dtype=np.float64)
    for buf, t in zip(contribs, tiles):
        y0, x0, y1, x1 = t["ext"]
        out[:, y0:y1, x0:x1] += buf
    return out


def stitch(vks, tiles, slices: int, height: int, width: int) -> np.ndarray:
    """Alg. 1 step 20: keep each tile's interior, abandon halos."""
    out = np.zeros((slices, height, width), dtype=np.float64)
    for vk, t in zip(vks, tiles):
        y0, x0, y1, x1 = t["interior"]
        ey0, ex0 = t["ext"][0], t["ext"][1]
        out[:, y0:y1, x0:x1] = vk[:, y0 - ey0:y1 - ey0, x0 - ex0:x1 - ex0]
    return out


def decompose(volume: np.ndarray, tiles):
    """Alg. 1 step 3: each tile receives V on its extended rect R_k."""
    return [np.array(volume[:, t["ext"][0]:t["ext"][2], t["ext"][1]:t["ext"][3]], dtype=np.float64)
            for t in tiles]


# ---------------------------------------------------------------------------------
# Alg. 1 with the fixed schedule of readings #16-#18, #20
# ---------------------------------------------------------------------------------
def n_segments(assignment, period: int) -> int:
    """Pass segments per iteration: passes after local probes T, 2T, ... plus an
    end-of-iteration flush (reading #17); T = 0 means once per iteration."""
    nmax = max((len(a) for a in assignment), default=0)
    if nmax == 0:
        return 0
    t = nmax if period <= 0 else period
    return -(-nmax // t)


def batch_order(seg, centers, ext, n, max_batch):
    """Batched schedule (north_star item 3): the probes `seg` (ascending) regrouped into batches of
    pairwise non-overlapping windows (clipped to R_k): round(i) = 1 + max round of an earlier
    overlapping probe; each round (ascending) split into batches of max_batch.  Returns the probe
    order the batches imply."""
    rects, rounds = [], []
    for i in seg:
        cy, cx = int(centers[i][0]), int(centers[i][1])
        r = (max(cy - n // 2, ext[0]), min(cy - n // 2 + n, ext[2]), max(cx - n // 2, ext[1]), min(cx - n // 2 + n, ext[3]))
        k = 0
        for rj, kj in zip(rects, rounds):
            if rj[0] < r[1] and r[0] < rj[1] and rj[2] < r[3] and r[2] < rj[3]:
                k = max(k, kj + 1)
        rects.append(r)
        rounds.append(k)
    order = []
    for k in range(max(rounds, default=-1) + 1):
        order += [i for i, kk in zip(seg, rounds) if kk == k]
    return order


def reconstruct(v0, probe, amps, centers, cfg, rows, cols, halo, iterations, alpha,
                alpha_acc=None, period=0, tau=TAU, on_segment=None, batch=0):
    """Run Alg. 1 literally.

    For each iteration, for each pass segment j, for each tile k (independent between passes):
      for its local probes of segment j in ascending global index:
          g = d f_i / d V_k                       (step 6)
          AccBuf_k[win ^ R_k] += g                (step 7)
          V_k[win ^ R_k] -= alpha g               (step 8)
      vertical fwd, vertical bwd, horizontal fwd, horizontal bwd on AccBuf  (steps 10-13)
      V_k -= alpha_acc AccBuf_k ; AccBuf_k = 0   (steps 14-16)
    Finally stitch the interiors (step 20).  Returns (V [S][H][W], [F per iteration], vks, accs).
    """
    n, sigma, c = cfg["n"], cfg["sigma"], cfg["prop_c"]
    slices, height, width = v0.shape
    alpha_acc = alpha if alpha_acc is None else alpha_acc
    tiles = tile_geometry(height, width, rows, cols, halo)
    assignment = assign_probes(centers, tiles)
    vks = decompose(v0, tiles)
    accs = [np.zeros_like(v) for v in vks]
    nseg = n_segments(assignment, period)
    t_per = max((len(a) for a in assignment), default=0) if period <= 0 else period
    losses = []
    for _ in range(iterations):
        total = 0.0
        for j in range(nseg):
            for k, t in enumerate(tiles):
                seg = assignment[k][j * t_per:(j + 1) * t_per]
                if batch:  # batched schedule: same per-voxel update order (batch_order)
                    seg = batch_order(seg, centers, t["ext"], n, batch)
                for i in seg:
                    cy, cx = int(centers[i][0]), int(centers[i][1])
                    vwin = window(vks[k], t["ext"], (cy, cx), n)
                    g, f = probe_grad(probe, vwin, amps[i], sigma, c, tau)
                    total += f
                    mask = window_mask(t["ext"], (cy, cx), n)
                    _scatter(accs[k], t["ext"], (cy, cx), n, g, mask, +1.0)
                    _scatter(vks[k], t["ext"], (cy, cx), n, g, mask, -alpha)
            appp_passes(accs, tiles, rows, cols)
            for k in range(len(tiles)):
                vks[k] -= alpha_acc * accs[k]
                accs[k][...] = 0.0
            if on_segment is not None:
                on_segment(j, vks, accs)
        losses.append(total)
    return stitch(vks, tiles, slices, height, width), losses, vks, accs


def _scatter(dst, ext, center, n, g, mask, scale):
    """dst[s][win ^ R_k] += scale * g_s (pixels outside R_k are discarded, reading #12)."""
    ey0, ex0 = ext[0], ext[1]
    wy0, wx0 = center[0] - n // 2, center[1] - n // 2
    ys, xs = np.nonzero(mask)
    if ys.size == 0:
        return
    dst[:, ys + wy0 - ey0, xs + wx0 - ex0] += scale * g[:, ys, xs]


def accumulate_frozen(v0, probe, amps, centers, cfg, rows, cols, halo, tau=TAU):
    """alpha = 0: every tile's AccBuf after one segment and the four passes (no step)."""
    n, sigma, c = cfg["n"], cfg["sigma"], cfg["prop_c"]
    slices, height, width = v0.shape
    tiles = tile_geometry(height, width, rows, cols, halo)
    assignment = assign_probes(centers, tiles)
    vks = decompose(v0, tiles)
    accs = [np.zeros_like(v) for v in vks]
    for k, t in enumerate(tiles):
        for i in assignment[k]:
            cy, cx = int(centers[i][0]), int(centers[i][1])
            g, _ = probe_grad(probe, window(vks[k], t["ext"], (cy, cx), n), amps[i], sigma, c, tau)
            _scatter(accs[k], t["ext"], (cy, cx), n, g, window_mask(t["ext"], (cy, cx), n), 1.0)
    appp_passes(accs, tiles, rows, cols)
    return accs, tiles


# ---------------------------------------------------------------------------------
# Halo Voxel Exchange (HVE) baseline -- the paper's comparison system
#   P:344-369 (§Related Work): tiles get "additional probe locations that are neighbors",
#   halos "augmented accordingly to cover all the additional circles", independent tile
#   reconstructions, then "the voxels in each tile are pasted to the halos in neighboring GPUs",
#   repeated until convergence; "two extra rows of probe locations for each tile".
#   Readings (DESIGN.md §2 #33-#35): extra rows = a margin of (rows x scan step) pixels around the
#   interior for the probe assignment; the augmented halo is a width parameter like GD's (the paper:
#   890 pm for HVE vs 600 pm for GD, "to cover all probe locations"), windows zero-extended past it
#   (reading #12); one sweep of per-probe SGD per tile per iteration, then the copy-paste.
# ---------------------------------------------------------------------------------
class TileTooSmall(ValueError):
    """a tile's augmented halo reaches past its adjacent tiles' interiors (the paper's
    'NA' entries: each tile must be large enough to hold its neighbours' halos)."""


def hve_decompose(height: int, width: int, rows: int, cols: int, centers, margin: int, halo: int):
    """Tiles with interior (uniform split, reading #14), augmented rect = interior dilated by `halo`
    and clipped (as tile_geometry), and probes = every probe whose centre lies in the interior
    dilated by `margin` pixels (own + extra rows; ascending global index; a probe may sit on
    several tiles).  Raises TileTooSmall if an augmented rect extends past the interiors of the
    tile's row / column neighbours (copy-paste could not fill that halo from an adjacent tile)."""
    ys = split_extent(height, rows)
    xs = split_extent(width, cols)
    tiles = tile_geometry(height, width, rows, cols, halo)
    for t in tiles:
        r, c = t["r"], t["c"]
        y0, x0, y1, x1 = t["interior"]
        t["probes"] = [i for i, (cy, cx) in enumerate(centers)
                       if y0 - margin <= cy < y1 + margin and x0 - margin <= cx < x1 + margin]
        lo_y = ys[r - 1][0] if r > 0 else 0
        hi_y = ys[r + 1][1] if r + 1 < rows else height
        lo_x = xs[c - 1][0] if c > 0 else 0
        hi_x = xs[c + 1][1] if c + 1 < cols else width
        a = t["ext"]
        if a[0] < lo_y or a[2] > hi_y or a[1] < lo_x or a[3] > hi_x:
            raise TileTooSmall(f"tile ({r},{c}): augmented rect {a} reaches past its neighbours' interiors")
    return tiles


def hve_exchange(vks, tiles):
    """Copy-paste (REPLACE): every tile's halo voxels take the value of the tile whose interior
    holds them ("the voxels in each tile are pasted to the halos in neighboring GPUs").
    Interiors partition the object, so each halo voxel has exactly one writer.  Returns the number
    of (source, destination) messages."""
    msgs = 0
    snap = [v.copy() for v in vks]  # interiors as they were after the sweep (synchronous exchange)
    for j, tj in enumerate(tiles):
        for k, tk in enumerate(tiles):
            if k == j:
                continue
            y0 = max(tj["ext"][0], tk["interior"][0])
            y1 = min(tj["ext"][2], tk["interior"][2])
            x0 = max(tj["ext"][1], tk["interior"][1])
            x1 = min(tj["ext"][3], tk["interior"][3])
            if y0 < y1 and x0 < x1:
                _region_views(vks[j], tj["ext"], (y0, y1), (x0, x1))[...] = \
                    _region_views(snap[k], tk["ext"], (y0, y1), (x0, x1))
                msgs += 1
    return msgs


def hve_reconstruct(v0, probe, amps, centers, cfg, rows, cols, margin, halo, iterations, alpha, tau=TAU):
    """HVE: per iteration, every tile independently runs one sweep of per-probe SGD
    (g = d f_i / d V, V[win ^ aug] -= alpha g, probes ascending) over its own + extra probes on its
    augmented tile, then the synchronous copy-paste exchange; finally stitch the interiors.
    Returns (V [S][H][W], [F per iteration: sum over every tile's probes, duplicates included], vks)."""
    n, sigma, c = cfg["n"], cfg["sigma"], cfg["prop_c"]
    slices, height, width = v0.shape
    tiles = hve_decompose(height, width, rows, cols, centers, margin, halo)
    vks = decompose(v0, tiles)
    losses = []
    for _ in range(iterations):
        total = 0.0
        for k, t in enumerate(tiles):
            for i in t["probes"]:
                cy, cx = int(centers[i][0]), int(centers[i][1])
                g, f = probe_grad(probe, window(vks[k], t["ext"], (cy, cx), n), amps[i], sigma, c, tau)
                total += f
                _scatter(vks[k], t["ext"], (cy, cx), n, g, window_mask(t["ext"], (cy, cx), n), -alpha)
        hve_exchange(vks, tiles)
        losses.append(total)
    return stitch(vks, tiles, slices, height, width), losses, vks


def seam_score(err, height: int, width: int, rows: int, cols: int) -> float:
    """Seam artifacts (Fig. artifact; SPEC SeamScore): mean |jump| of the error field
    err = V_rec - V_true across tile borders, divided by its mean |jump| between neighbouring voxels
    elsewhere.  ~1: no seam; > 1: discontinuities at the borders."""
    ys = [a for a, _ in split_extent(height, rows)][1:]
    xs = [a for a, _ in split_extent(width, cols)][1:]
    dy = np.abs(np.diff(err, axis=1))  # jump between rows y-1 and y at index y-1
    dx = np.abs(np.diff(err, axis=2))
    by = np.zeros(dy.shape[1], bool)
    bx = np.zeros(dx.shape[2], bool)
    for y in ys:
        by[y - 1] = True
    for x in xs:
        bx[x - 1] = True
    border = np.concatenate([dy[:, by, :].ravel(), dx[:, :, bx].ravel()])
    inner = np.concatenate([dy[:, ~by, :].ravel(), dx[:, :, ~bx].ravel()])
    if border.size == 0 or inner.mean() == 0:
        return 0.0
    return float(border.mean() / inner.mean())


def memory_report(tiles, slices: int, n: int):
    """Analytic per-tile storage (SPEC memory_report): voxels of the (extended / augmented) rect x S
    and measurement values (assigned probes x N^2)."""
    out = []
    for t in tiles:
        y0, x0, y1, x1 = t["ext"]
        nprobe = len(t["probes"]) if "probes" in t else None
        out.append(dict(voxels=(y1 - y0) * (x1 - x0) * slices,
                        measurements=None if nprobe is None else nprobe * n * n))
    return out
