"""Pipelined vs synchronous ADMM loop (dev aid): time per solve with the
inputs device-resident (torch), CUDA events around each solve, both modes
alternated, and the fields compared bitwise."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1607_00531_b200 import abi, synth  # noqa: E402
from paper_1607_00531_b200.epicorr import Context  # noqa: E402

for name, iters in (("C1", 50), ("C2", 50), ("C3", 100)):
    d = synth.make_config(name)
    ip = torch.from_numpy(d.iplus).cuda()
    im = torch.from_numpy(d.iminus).cuda()
    st = torch.cuda.Stream()
    ctx = Context(0, stream=st)
    cfg = abi.AdmmConfig(max_iter=iters, eps_abs=1e-300, eps_rel=1e-300)
    ctx.admm_solve(d.grid, ip, im, cfg=abi.AdmmConfig(max_iter=3, eps_abs=1e-300, eps_rel=1e-300))
    times = {0: [], Context.MODE_DEVICE_LOOP: []}
    outs = {}
    for rep in range(3):
        for mode in times:
            ctx.set_mode(mode)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            r = ctx.admm_solve(d.grid, ip, im, cfg=cfg)
            e1.record(st)
            torch.cuda.synchronize()
            times[mode].append(e0.elapsed_time(e1))
            outs[mode] = r["b"].cpu().numpy()
    ctx.set_mode(0)
    same = np.array_equal(outs[0], outs[Context.MODE_DEVICE_LOOP])
    print(f"{name} {iters} it: sync {min(times[0]):.2f} ms, device loop {min(times[Context.MODE_DEVICE_LOOP]):.2f} ms"
          f" per solve (min of 3); bitwise {same}", flush=True)
