"""b-step line-search statistics (dev aid): the accepted-trial histogram and
trial counts over a C3 solve (EPC_MODE_BSTEP_TIMING counters)."""
import sys

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1607_00531_b200 import abi, synth  # noqa: E402
from paper_1607_00531_b200.epicorr import Context  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 100
d = synth.make_config(name, scale=scale)
ctx = Context(0)
ctx.set_mode(0)
ctx.set_mode(Context.MODE_BSTEP_TIMING)
c0 = ctx.admm_counters()
ctx.admm_solve(d.grid, d.iplus, d.iminus, cfg=abi.AdmmConfig(max_iter=iters, eps_abs=1e-300, eps_rel=1e-300))
c1 = ctx.admm_counters()
cnt = ctx.bstep_counters()
ctx.set_mode(0)
sqp, qp = c1[2] - c0[2], c1[3] - c0[3]
print(f"{name} x{scale} {iters} it: sqp {sqp} qp {qp} per column-iteration sqp "
      f"{sqp / (d.grid.faces // d.grid.n1 * iters):.2f}")
print(cnt)
print(f"trials per search {cnt['ls_trials'] / max(cnt['ls_searches'], 1):.2f}")
