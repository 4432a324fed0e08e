"""b-step cost of exactness (dev aid): C3 b-step time with every SQP /
line-search decision on exact chains (EPC_MODE_BSTEP_CHAINED) against the
certified decisions, both in the diagnostic build, plus phase splits."""
import sys
import time

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1607_00531_b200 import abi, synth  # noqa: E402
from paper_1607_00531_b200.epicorr import Context  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
d = synth.make_config("C3", scale=scale)
ctx = Context(0)
cfg = abi.AdmmConfig(max_iter=iters, eps_abs=1e-300, eps_rel=1e-300)
for name, bits in (("certified", Context.MODE_BSTEP_TIMING),
                   ("chained", Context.MODE_BSTEP_TIMING | Context.MODE_BSTEP_CHAINED)):
    ctx.set_mode(0)
    ctx.set_mode(bits)
    ctx.profile(True)
    ctx.profile_reset()
    t = time.time()
    ctx.admm_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
    dt = time.time() - t
    prof = ctx.profile_read()
    ctx.profile(False)
    tm = ctx.bstep_timing()
    tt = sum(tm.values())
    print(f"{name}: {dt:.3f}s, b-step {prof['admm_bstep'][0]:.1f} ms; phases",
          {k: f"{100 * v / tt:.1f}%" for k, v in tm.items()}, f"Gcycles {tt / 1e9:.1f}", flush=True)
ctx.set_mode(0)
