"""fp32-variant solve time and per-kernel split at C3 (dev aid; device-resident inputs)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1607_00531_b200 import abi, synth  # noqa: E402
from paper_1607_00531_b200.epicorr import Context  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
d = synth.make_config(name)
g = d.grid
ctx = Context(0)
cfg = abi.AdmmConfig(max_iter=iters, eps_abs=1e-300, eps_rel=1e-300)
ipd = torch.from_numpy(d.iplus.astype(np.float32)).cuda()
imd = torch.from_numpy(d.iminus.astype(np.float32)).cuda()
ctx.admm_solve_f32(g, ipd, imd, cfg=cfg)
ts = []
for rep in range(3):
    torch.cuda.synchronize()
    t = time.time()
    ctx.admm_solve_f32(g, ipd, imd, cfg=cfg)
    torch.cuda.synchronize()
    ts.append(time.time() - t)
print(f"f32 {name} {iters} it: best {min(ts) * 1e3:.1f} ms  ({[round(x * 1e3, 1) for x in ts]})")
ctx.profile(True)
ctx.profile_reset()
ctx.admm_solve_f32(g, ipd, imd, cfg=cfg)
prof = ctx.profile_read()
ctx.profile(False)
tot = sum(v[0] for v in prof.values())
for k, (ms, n) in sorted(prof.items(), key=lambda kv: -kv[1][0])[:8]:
    print(f"  {k:20s} {ms:9.2f} ms  {n:5d} launches  {ms / max(n, 1):8.3f} ms/launch  {100 * ms / tot:5.1f}%")
