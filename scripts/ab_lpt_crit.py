"""A/B of the critical-column SM reservation (EPC_LPT_CRIT; 0 = off): C3 x400
over 30 iterations and C3 x1 over 30, time + the bitwise digest."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from ab_fuse_fwd2 import digest  # noqa: E402
from dataclasses import replace  # noqa: E402
from paper_1607_00531_b200 import abi, synth  # noqa: E402
from paper_1607_00531_b200.epicorr import Context  # noqa: E402

dev = torch.device("cuda:0")
stream = torch.cuda.current_stream(dev)
ctx = Context(0, stream=stream)
for name, scale, iters, reps in (("C3", 400.0, 30, 2), ("C3", 1.0, 30, 3), ("C2", 400.0, 30, 2)):
    d = synth.make_pair(replace(synth.CONFIGS[name], scale=scale))
    ip, im = torch.from_numpy(d.iplus).to(dev), torch.from_numpy(d.iminus).to(dev)
    cfg = abi.AdmmConfig(max_iter=iters, eps_abs=1e-300, eps_rel=1e-300)
    r = ctx.admm_solve(d.grid, ip, im, cfg=cfg)
    dg = digest(r)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        r2 = ctx.admm_solve(d.grid, ip, im, cfg=cfg)
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
        assert digest(r2) == dg
    print(f"crit={os.environ.get('EPC_LPT_CRIT', 'default')} {name} x{scale:g} {iters} it: min {min(ts):.2f} ms digest {dg}", flush=True)
ctx.close()
