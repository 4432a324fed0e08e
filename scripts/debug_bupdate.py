"""Dev aid: b_update on the small test case vs the oracle, per mode."""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from oracle import ffi  # noqa: E402
from paper_1607_00531_b200 import abi, synth  # noqa: E402
from paper_1607_00531_b200.epicorr import Context  # noqa: E402

d = synth.make_pair(synth.SynthSpec(m=(16, 12, 8), seed=7))
g, ip, im = d.grid, d.iplus, d.iminus
orc = ffi.load("oracle")
st = orc.admm_solve(g, ip, im, cfg=abi.AdmmConfig(max_iter=6, eps_abs=1e-300, eps_rel=1e-300))
ctx = Context(0)
for rho in (st["rho"], 1e6, 100.0):
    ref = orc.b_update(g, ip, im, st["b"], st["z"], st["u"], rho)
    for name, bits in (("prod", 0), ("diag", 1), ("chained", 1 | (1 << 13))):
        ctx.set_mode(bits)
        out = ctx.b_update(g, ip, im, st["b"], st["z"], st["u"], rho)
        diff = np.abs(out["b"] - ref["b"])
        bad = np.nonzero(diff)[0]
        cn = ctx.bstep_counters() if bits else {}
        print(f"rho={rho:g} {name:8s} maxdiff={diff.max():.3g} ncols_bad={len(set(bad // g.n1))} "
              f"first_bad_col={bad[0] // g.n1 if len(bad) else -1} sqp {out['sqp_iters']}/{ref['sqp_iters']} "
              f"qp {out['qp_iters']}/{ref['qp_iters']} {cn}", flush=True)
        ctx.set_mode(0)
