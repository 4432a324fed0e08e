"""b-step cost of the columns that hit the SQP cap vs the rest (dev aid).

Needs a library built with -DEPC_PROBE_HEAVY (scripts/build_variant.py
heavy -DEPC_PROBE_HEAVY; EPC_LIB=scripts/_var/heavy.so). Runs `warm`
production iterations of the C3 solve, then `iters` more in timing mode,
warm-started from the first call's state."""
import sys

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1607_00531_b200 import abi, synth  # noqa: E402
from paper_1607_00531_b200.epicorr import Context  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 60
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 10
d = synth.make_config(name, scale=scale)
ctx = Context(0)
ctx.set_mode(0)
cfg = lambda n: abi.AdmmConfig(max_iter=n, eps_abs=1e-300, eps_rel=1e-300)  # noqa: E731
st = dict(b=None, z=None, u=None, rho=0.0)
if warm:
    r = ctx.admm_solve(d.grid, d.iplus, d.iminus, cfg=cfg(warm))
    st = dict(b=r["b"], z=r["z"], u=r["u"], rho=r["rho"])
ctx.set_mode(Context.MODE_BSTEP_TIMING)
ctx.admm_solve(d.grid, d.iplus, d.iminus, cfg=cfg(iters), **st)
ph = ctx.bstep_timing()
c = list(ctx.bstep_counters())
cnt = ctx.bstep_counters()
vals = [cnt[k] for k in ctx.BSTEP_COUNTERS]
ctx.set_mode(0)
heavy_tot = sum(ph.values())
light_tot, ch_h, ch_l, n_h, n_l, tr_h, tr_l, un_h, un_l = vals[:9]
print(f"{name} x{scale} iterations {warm}..{warm + iters}")
print(f"heavy columns {n_h} ({100 * n_h / max(n_h + n_l, 1):.2f}%), light {n_l}")
print(f"cycles per heavy column {heavy_tot / max(n_h, 1):.0f}, per light column {light_tot / max(n_l, 1):.0f}")
print(f"heavy share of all column cycles {100 * heavy_tot / max(heavy_tot + light_tot, 1):.1f}%")
print("heavy phases:", {k: f"{100 * v / max(heavy_tot, 1):.1f}%" for k, v in ph.items()})
print(f"exact-chain trials: heavy {un_h} of {tr_h} trials ({tr_h / max(n_h, 1):.1f} trials per column), "
      f"chain cycles {100 * ch_h / max(heavy_tot, 1):.1f}% of heavy ({ch_h / max(un_h, 1):.0f} per trial)")
print(f"exact-chain trials: light {un_l} of {tr_l} trials ({tr_l / max(n_l, 1):.1f} per column), "
      f"chain cycles {100 * ch_l / max(light_tot, 1):.1f}% of light ({ch_l / max(un_l, 1):.0f} per trial)")
rj_h, rj_l, e3_h, e3_l, e6_h, e6_l, sf_h, sf_l = vals[9:17]
print(f"rejected trials heavy {rj_h}: over the threshold after 96 faces {e3_h}, after 192 {e6_h}")
print(f"rejected trials light {rj_l}: over the threshold after 96 faces {e3_l}, after 192 {e6_l}")
print(f"factor: segmented chains not agreeing heavy {sf_h} light {sf_l}")
