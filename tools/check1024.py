# quick N=1024 parity: lt_small-shaped probe (S=100 slow in oracle) -> use S=6 on a 1536 object
import sys, os, time, numpy as np
sys.path.insert(0, os.getcwd())
from oracle import ptycho_oracle as O
import synth
from paper_2205_06327_b200.ptycho import Ptycho
n, s, h, w = 1024, 6, 1536, 1536
probe = synth.probe(n, 25.0)
vt = synth.volume(0, s, h, w)
centers = synth.scan_centers(h, w, 63, 66)
for idx in [2079, 0]:
    full = (0, 0, h, w)
    amp = O.farfield_magnitude(probe, O.window(vt.astype(np.float64), full, tuple(centers[idx]), n), 0.1, 3.135)
    vwin = O.window((0.5 * vt).astype(np.float64), full, tuple(centers[idx]), n)
    g_ref, f_ref = O.probe_grad(probe, vwin, amp, 0.1, 3.135)
    g32, _ = O.probe_grad(probe, vwin, amp, 0.1, 3.135, dtype=np.float32)
    p = Ptycho(n, s, h, w, 0.1, 3.135, alpha=0.1)
    p.set_tiles(1, 1, 512)
    p.set_scan(centers)
    p.allocate_workspace()
    p.set_probe(probe.astype(np.complex64))
    p.load_measurements(amp[None].astype(np.float32), first_local=idx)
    p.set_volume(0.5 * vt)
    g, f = p.debug_probe_grad(0, idx)
    psi = p.debug_exit_wave(0, idx)
    psi_ref = O.forward(probe, O.window(vt.astype(np.float64)*0.5, full, tuple(centers[idx]), n), 0.1, 3.135)[0]
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    print(f"N=1024 S={s} probe {idx}: grad rel {rel(g, g_ref):.2e} (fp32 floor {rel(g32, g_ref):.2e}) loss rel {abs(f-f_ref)/f_ref:.2e} exit rel {rel(psi, psi_ref):.2e}", flush=True)
    p.close()
