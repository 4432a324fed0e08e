import sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_1607_00531_b200 import abi, synth
from paper_1607_00531_b200.epicorr import Context
d = synth.make_pair(synth.SynthSpec(m=(32, 24, 12), seed=5, scale=400.0))
g = d.grid
ctx = Context(0)
for iters in (5, 10, 20, 30):
    cfg = abi.AdmmConfig(max_iter=iters, eps_abs=1e-300, eps_rel=1e-300)
    r64 = ctx.admm_solve(g, d.iplus, d.iminus, cfg=cfg)
    ip32, im32 = d.iplus.astype(np.float32), d.iminus.astype(np.float32)
    r64q = ctx.admm_solve(g, ip32.astype(np.float64), im32.astype(np.float64), cfg=cfg)
    r32 = ctx.admm_solve_f32(g, ip32, im32, cfg=cfg)
    b = r64["b"]
    rel = lambda x: np.linalg.norm(np.asarray(x, np.float64) - b) / np.linalg.norm(b)
    diff = np.abs(r32["b"] - b).reshape(-1, g.n1).max(axis=1)
    print(iters, "rel64q %.2e rel32 %.2e" % (rel(r64q["b"]), rel(r32["b"])), "cols>1e-2:", int((diff > 1e-2).sum()), "of", diff.size,
          "lag", r64["rows"][-1]["lagrangian"], r32["rows"][-1]["lagrangian"], r64q["rows"][-1]["lagrangian"])
