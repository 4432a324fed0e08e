"""Quick GPU probe: ADMM iteration timing + per-kernel split at C1/C3 and
bitwise agreement with the oracle for a few iterations (development aid)."""
import argparse
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1607_00531_b200 import abi, synth  # noqa: E402
from paper_1607_00531_b200.epicorr import Context  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C1")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--check", type=int, default=0, help="oracle iterations to compare (0 = skip)")
ap.add_argument("--prod", action="store_true", help="production kernel (no phase timing)")
ap.add_argument("--no-kkt", action="store_true", help="check_kkt = false (cost of the KKT check)")
a = ap.parse_args()

t = time.time()
d = synth.make_config(a.config, scale=a.scale)
print(f"generate {a.config}: {time.time() - t:.2f}s faces={d.grid.faces}", flush=True)
ctx = Context(0)
cfg = abi.AdmmConfig(max_iter=a.iters, eps_abs=1e-300, eps_rel=1e-300)
if a.no_kkt:
    cfg.check_kkt = 0
r = ctx.admm_solve(d.grid, d.iplus, d.iminus, cfg=abi.AdmmConfig(max_iter=2, eps_abs=1e-300, eps_rel=1e-300))
ctx.set_mode(0 if a.prod else 1)
ctx.profile(True)
ctx.profile_reset()
t = time.time()
r = ctx.admm_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
dt = time.time() - t
prof = ctx.profile_read()
if not a.prod:
    tm = ctx.bstep_timing()
    tt = sum(tm.values())
    print("b-step phases (lane-0 cycles, all warps):", {k: f"{100*v/tt:.1f}%" for k, v in tm.items()})
    print("  total Gcycles", tt / 1e9)
ctx.profile(False)
print(f"admm {a.iters} it: {dt:.3f}s  {dt / a.iters * 1e3:.2f} ms/it  "
      f"{d.grid.faces * a.iters / dt / 1e6:.1f} M face-it/s  stop={r['stop']}", flush=True)
tot = sum(v[0] for v in prof.values())
for k, (ms, n) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:20s} {ms:9.2f} ms  {n:5d} launches  {ms / max(n, 1):8.3f} ms/launch  {100 * ms / tot:5.1f}%")
print("rows:", [(x["iter"], x["rho"], round(x["lagrangian"], 6)) for x in r["rows"][-3:]])
if a.check:
    from oracle import ffi
    orc = ffi.load("oracle")
    c2 = abi.AdmmConfig(max_iter=a.check, eps_abs=1e-300, eps_rel=1e-300)
    t = time.time()
    ro = orc.admm_solve(d.grid, d.iplus, d.iminus, cfg=c2)
    print(f"oracle {a.check} it: {time.time() - t:.2f}s", flush=True)
    rg = ctx.admm_solve(d.grid, d.iplus, d.iminus, cfg=c2)
    print("bitwise b/z/u:", np.array_equal(rg["b"], ro["b"]), np.array_equal(rg["z"], ro["z"]),
          np.array_equal(rg["u"], ro["u"]),
          "rel b", np.linalg.norm(rg["b"] - ro["b"]) / max(np.linalg.norm(ro["b"]), 1e-300))
    for x, y in zip(rg["rows"], ro["rows"]):
        if x["lagrangian"] != y["lagrangian"]:
            print("  row", x["iter"], "lag rel", abs(x["lagrangian"] - y["lagrangian"]) / abs(y["lagrangian"]))
            break
