"""Small driver for ncu: the LT-small 2x4 workload, `--probes` probes per tile through forward_grad.
Chain order per probe (pass_kernel launches): 0 fwd_first, 1..S-2 fwd_mid, S-1 fwd_last, S turn,
S+1 bwd_last_prop, S+2..2S-1 bwd_mid, 2S bwd_end."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa
from paper_2205_06327_b200.ptycho import Ptycho  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="lt_small")
ap.add_argument("--probes", type=int, default=1)
ap.add_argument("--grid", default="2x4")
args = ap.parse_args()
c = synth.CONFIGS[args.config]
R, C = (int(v) for v in args.grid.split("x"))
p = Ptycho(c.n, c.slices, c.height, c.width, c.sigma, c.prop_c, alpha=0.5)
p.set_tiles(R, C, c.n // 2)
p.set_scan(synth.scan_centers(c.height, c.width, c.scan_ny, c.scan_nx))
p.allocate_workspace()
p.set_probe(synth.probe(c.n, c.defocus_nm).astype(np.complex64))
rng = np.random.default_rng(0)
p.set_volume(rng.random((c.slices, c.height, c.width), dtype=np.float32))
# probes in the middle of each tile's list (windows inside the object)
p.forward_grad(200, args.probes)
p.synchronize()
print("done", p.kernel_launches())
