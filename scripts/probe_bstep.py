"""Fixed-state b-step micro benchmark (dev aid): run the GPU ADMM for
--warm iterations to get a state, then time epc_b_update on that state for
the certified-enclosure and the chained modes, and check they agree bitwise."""
import argparse
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1607_00531_b200 import abi, synth  # noqa: E402
from paper_1607_00531_b200.epicorr import Context  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--warm", type=int, default=3)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--modes", default="cert,chained")
a = ap.parse_args()

d = synth.make_config(a.config, scale=a.scale)
g = d.grid
ctx = Context(0)
st = ctx.admm_solve(g, d.iplus, d.iminus, cfg=abi.AdmmConfig(max_iter=a.warm, eps_abs=1e-300, eps_rel=1e-300))
print(f"{a.config} warm {a.warm} its, rho={st['rho']}", flush=True)
ref = None
for m in a.modes.split(","):
    bits = Context.MODE_BSTEP_TIMING | (Context.MODE_BSTEP_CHAINED if m == "chained" else 0)
    ctx.set_mode(bits)
    ctx.profile(True)
    ctx.profile_reset()
    for _ in range(a.reps):
        out = ctx.b_update(g, d.iplus, d.iminus, st["b"], st["z"], st["u"], st["rho"])
    prof = ctx.profile_read()
    ctx.profile(False)
    tm = ctx.bstep_timing()
    cn = ctx.bstep_counters()
    ms, n = prof["admm_bstep"]
    tt = sum(tm.values())
    same = True if ref is None else bool(np.array_equal(out["b"], ref))
    if ref is None:
        ref = out["b"]
    print(f"{m:8s}: {ms / n:.3f} ms/launch  Gcyc/launch={tt / a.reps / 1e9:.2f}  "
          f"sqp={out['sqp_iters']} qp={out['qp_iters']} same={same}  "
          + " ".join(f"{kk}={100 * v / tt:.0f}%" for kk, v in tm.items()), flush=True)
    print("          counters/launch: " + " ".join(f"{k}={v // a.reps}" for k, v in cn.items()),
          flush=True)
    ctx.set_mode(0)
