"""Dev aid: per-iteration b-step time, rho and counters along the C3 solve
(where along the trajectory the b-step's time goes)."""
import argparse
import sys

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1607_00531_b200 import abi, synth  # noqa: E402
from paper_1607_00531_b200.epicorr import Context  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--iters", type=int, default=100)
ap.add_argument("--scale", type=float, default=1.0)
a = ap.parse_args()
d = synth.make_config(a.config, scale=a.scale)
ctx = Context(0)
cfg = abi.AdmmConfig(max_iter=a.iters, eps_abs=1e-300, eps_rel=1e-300)
ctx.admm_solve(d.grid, d.iplus, d.iminus, cfg=abi.AdmmConfig(max_iter=2, eps_abs=1e-300, eps_rel=1e-300))
r = ctx.admm_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
rows = r["rows"]
tot = sum(x["b_update_s"] for x in rows)
print(f"{a.config} x{a.scale}: b-step total {tot * 1e3:.1f} ms over {len(rows)} iterations")
acc = 0.0
for x in rows:
    acc += x["b_update_s"]
    keys = [k for k in ("sqp_iterations", "qp_iterations", "ls_trials", "sqp_iters", "qp_iters") if k in x]
    print(f"it {x['iter']:3d} rho {x['rho']:.3g} b {x['b_update_s'] * 1e3:7.3f} ms cum {acc * 1e3:7.1f} "
          + " ".join(f"{k}={x[k]}" for k in keys))
