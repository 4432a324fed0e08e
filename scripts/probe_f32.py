import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_1607_00531_b200 import abi, synth
from paper_1607_00531_b200.epicorr import Context
from oracle import ffi
cfgname = sys.argv[1] if len(sys.argv) > 1 else "C1"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
d = synth.make_config(cfgname)
g = d.grid
ctx = Context(0)
cfg = abi.AdmmConfig(max_iter=iters, eps_abs=1e-300, eps_rel=1e-300)
r64 = ctx.admm_solve(g, d.iplus, d.iminus, cfg=cfg)
ip32, im32 = d.iplus.astype(np.float32), d.iminus.astype(np.float32)
t = time.time()
r32 = ctx.admm_solve_f32(g, ip32, im32, cfg=cfg)
print("f32 wall", time.time() - t, "stop", r32["stop"], r32["message"])
b64 = r64["b"]; b32 = r32["b"].astype(np.float64)
# sensitivity reference: fp64 on the fp32-rounded images
r64q = ctx.admm_solve(g, ip32.astype(np.float64), im32.astype(np.float64), cfg=cfg)
print("fp64 on fp32-rounded images, rel L2 b vs fp64:", np.linalg.norm(r64q["b"] - b64) / np.linalg.norm(b64))
print("b-step seconds: f64 %.3f f32 %.3f" % (sum(x["b_update_s"] for x in r64["rows"]), sum(x["b_update_s"] for x in r32["rows"])))
print("|b| max", np.abs(b64).max(), "rms", np.sqrt((b64 ** 2).mean()))
print("rel L2 b:", np.linalg.norm(b32 - b64) / np.linalg.norm(b64))
print("rel L2 z:", np.linalg.norm(r32["z"] - r64["z"]) / np.linalg.norm(r64["z"]))
for a, b in list(zip(r64["rows"], r32["rows"]))[::max(1, iters // 10)]:
    print(a["iter"], a["rho"], b["rho"], "lag %.6e %.6e rel %.2e" % (a["lagrangian"], b["lagrangian"], abs(a["lagrangian"] - b["lagrangian"]) / abs(a["lagrangian"])),
          "pr %.3e %.3e kkt %.2e %.2e" % (a["primal_res"], b["primal_res"], a["kkt_violation"], b["kkt_violation"]))
import torch
ipd, imd = torch.from_numpy(ip32).cuda(), torch.from_numpy(im32).cuda()
for rep in range(2):
    torch.cuda.synchronize(); t = time.time()
    r = ctx.admm_solve_f32(g, ipd, imd, cfg=cfg)
    torch.cuda.synchronize(); dt = time.time() - t
print(f"f32 device solve {dt*1e3:.1f} ms, {g.faces*iters/dt/1e6:.1f} M face-it/s")
ipd64, imd64 = torch.from_numpy(d.iplus).cuda(), torch.from_numpy(d.iminus).cuda()
torch.cuda.synchronize(); t = time.time()
r = ctx.admm_solve(g, ipd64, imd64, cfg=cfg)
torch.cuda.synchronize(); dt = time.time() - t
print(f"f64 device solve {dt*1e3:.1f} ms, {g.faces*iters/dt/1e6:.1f} M face-it/s")
