"""Dev aid: latency of one column QP (k_qp_batch, nqp = 1) vs its active-set
size, at n = 257 (the C3 column): the per-QP-iteration cost of the Schur
path (EPC_LIB selects an A/B build)."""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1607_00531_b200.epicorr import Context  # noqa: E402

ctx = Context(0)
n = 257
for amp in (5.0, 20.0, 40.0, 80.0, 200.0):
    rng = np.random.default_rng(1)
    gd = 3.0 + rng.uniform(0, 1, (1, n))
    go = np.zeros((1, n))
    go[:, :-1] = -1.0 + 0.2 * rng.uniform(-1, 1, (1, n - 1))
    c = amp * np.cumsum(rng.uniform(-1, 1, (1, n)), axis=1) / np.sqrt(n)
    x0 = np.zeros((1, n))
    ctx.qp_active_set_batch(n, 1.0, gd, go, c, x0, 6 * n + 10)
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        out = ctx.qp_active_set_batch(n, 1.0, gd, go, c, x0, 6 * n + 10)
        ts.append(time.perf_counter() - t)
    ctx.set_mode(0)
    ctx.set_mode(Context.MODE_BSTEP_TIMING)
    ctx.qp_active_set_batch(n, 1.0, gd, go, c, x0, 6 * n + 10)
    tm = list(ctx.bstep_timing().values())[:7]
    ctx.set_mode(0)
    tt = sum(tm) or 1
    names = ["factor", "g", "solves", "schur_form", "schur_solve", "p_update", "ratio"]
    it = int(out["iters"][0])
    na = int(np.count_nonzero(out["sign"][0]))
    print(f"amp {amp:6.1f}: iters {it:4d} active {na:4d}  {min(ts) * 1e3:8.3f} ms  "
          f"{min(ts) / max(it, 1) * 1e6:8.1f} us/iteration  " +
          " ".join(f"{k} {100 * v / tt:.0f}%" for k, v in zip(names, tm)), flush=True)
