"""GN-PCG probe (dev aid): C2 solve timing, per-kernel split, PCG counts."""
import argparse
import sys
import time

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1607_00531_b200 import abi, synth  # noqa: E402
from paper_1607_00531_b200.epicorr import Context  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--outer", type=int, default=10)
ap.add_argument("--ncu", action="store_true",
                help="one GN step only, no warm-up (for ncu -k regex:pcg_loop -c 1)")
a = ap.parse_args()
d = synth.make_config(a.config, scale=a.scale)
ctx = Context(0)
cfg = abi.GnConfig(eta=1e-2, max_pcg=50, max_outer=a.outer)
if a.ncu:
    r = ctx.gn_solve(d.grid, d.iplus, d.iminus, cfg=abi.GnConfig(eta=1e-2, max_pcg=50, max_outer=1))
    print("pcg_iters", r["rows"][1]["pcg_iters"], "faces", d.grid.faces)
    sys.exit(0)
ctx.gn_solve(d.grid, d.iplus, d.iminus, cfg=abi.GnConfig(eta=1e-2, max_pcg=5, max_outer=1))
ctx.profile(True)
ctx.profile_reset()
t = time.time()
r = ctx.gn_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
dt = time.time() - t
prof = ctx.profile_read()
ctx.profile(False)
npcg = sum(x["pcg_iters"] for x in r["rows"])
print(f"GN {a.config}: {dt:.3f}s wall, {npcg} PCG its, stop={r['stop']} "
      f"{d.grid.faces * npcg / dt / 1e6:.1f} M face-PCG-it/s")
tot = sum(v[0] for v in prof.values())
for k, (ms, n) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:18s} {ms:9.2f} ms {n:6d} launches {ms / max(n, 1) * 1e3:9.1f} us/launch {100 * ms / tot:5.1f}%")
print("device-kernel total ms", tot, "host/sync overhead ms", dt * 1e3 - tot)
print([(x["iter"], x["pcg_iters"], x["step"], round(x["j_value"], 3)) for x in r["rows"]])
import torch  # noqa: E402
ip_d = torch.from_numpy(d.iplus).cuda()
im_d = torch.from_numpy(d.iminus).cuda()
ts = []
for rep in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    r2 = ctx.gn_solve(d.grid, ip_d, im_d, cfg=cfg)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"unprofiled device-resident solve: min {ts[0]:.1f} ms, median {ts[len(ts) // 2]:.1f} ms, "
      f"{d.grid.faces * npcg / ts[0] * 1e3 / 1e6:.1f} M face-PCG-it/s (min)")
