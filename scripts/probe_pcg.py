"""PCG kernel probe (dev aid): per-kernel time of the device PCG loop for each
preconditioner at a fixed linearisation point (isolates the sweep chains)."""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1607_00531_b200 import abi, synth  # noqa: E402
from paper_1607_00531_b200.epicorr import Context  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
d = synth.make_config(name)
g = d.grid
ctx = Context(0)
b = np.zeros(g.faces)
grad = ctx.objective_gn(g, d.iplus, d.iminus, b)["grad"]
nf = g.faces
for kind, kname in ((0, "none"), (1, "jacobi"), (2, "block")):
    ctx.pcg(g, d.iplus, d.iminus, b, grad, 1e-12, 5, kind=kind)
    ctx.profile(True)
    ctx.profile_reset()
    r = ctx.pcg(g, d.iplus, d.iminus, b, grad, 1e-12, 50, kind=kind)
    prof = ctx.profile_read()
    ctx.profile(False)
    line = [f"{kname:7s} iters={r['iters']:3d}"]
    for k in ("pcg_hvp", "pcg_update"):
        ms, n = prof.get(k, (0.0, 1))
        us = ms / n * 1e3
        line.append(f"{k}={us:6.1f}us")
    # bytes: p 24 B/face, hv 32 B/face (+neighbours), update 72 B/face (block) / 56 (none)
    print(" ".join(line), flush=True)
