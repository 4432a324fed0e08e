"""Small invocations of every device path, as a memory-safety check.
compute-sanitizer is refused on this GPU pool (profiles/r02_sanitizer_refused.log),
so the script is run instead with the library's own checks
(scripts/r02k_gpu.sh): EPC_GUARD=1 puts 4 KB guard zones around every device
scratch slot (checked at the end through epc_guard_check), and the
EPC_SMEM_CANARY build fills every pad between the b-step's shared-memory
vectors with NaN canaries that each column checks when it is done.

  * the b-step (warp-synchronous shared memory, segmented chains, the
    certified enclosures) and the z-step, in ADMM solves at unit intensity
    and x400 (active constraints: the Schur path);
  * the large-active-set column QPs (the warp Cholesky and substitutions);
  * GN-PCG with the cooperative persistent loop (bounded-spin grid barrier)
    and with the per-iteration kernels;
  * the slab kernels (k-slab ADMM, 2 ranks in lockstep on one GPU) and the
    C++ NCCL slab solve at world 1;
  * the fp32 variant.
Checks the results against the oracle so a sanitizer run also proves the
instrumented kernels still compute the reference's bits."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from oracle import ffi  # noqa: E402
from paper_1607_00531_b200 import abi, dist_admm, synth  # noqa: E402
from paper_1607_00531_b200.epicorr import Context  # noqa: E402

EX = dict(eps_abs=1e-300, eps_rel=1e-300)
orc = ffi.load("oracle")
ctx = Context(0)
m = (24, 16, 6)
for scale in (1.0, 400.0):
    d = synth.make_pair(synth.SynthSpec(m=m, seed=3, scale=scale))
    cfg = abi.AdmmConfig(max_iter=3, **EX)
    o = ctx.admm_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
    r = orc.admm_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
    assert np.array_equal(o["b"], r["b"]), "admm b"
    print("admm", scale, "ok", flush=True)
n = 60
rng = np.random.default_rng(1)
gd = 3.0 + rng.uniform(0, 1, (2, n))
go = np.zeros((2, n))
go[:, :-1] = -1.0 + 0.2 * rng.uniform(-1, 1, (2, n - 1))
c = 40.0 * np.cumsum(rng.uniform(-1, 1, (2, n)), axis=1) / np.sqrt(n)
q = ctx.qp_active_set_batch(n, 1.0, gd, go, c, np.zeros((2, n)), 6 * n + 10)
rq = orc.qp_active_set(n, 1.0, gd[0].copy(), go[0].copy(), c[0].copy(), np.zeros(n), 6 * n + 10)
assert np.array_equal(q["x"][0], rq["x"]), "qp"
print("qp ok", int(np.count_nonzero(rq["sign"])), "active", flush=True)
import os  # noqa: E402
d = synth.make_pair(synth.SynthSpec(m=(16, 12, 8), seed=4))
gcfg = abi.GnConfig(eta=1e-2, max_pcg=20, max_outer=2)
for loop in ("1", "0"):
    os.environ["EPC_PCG_LOOP"] = loop
    o = ctx.gn_solve(d.grid, d.iplus, d.iminus, cfg=gcfg)
    r = orc.gn_solve(d.grid, d.iplus, d.iminus, cfg=gcfg)
    assert np.linalg.norm(o["b"] - r["b"]) <= 1e-8 * np.linalg.norm(r["b"]), "gn"
    print("gn loop", loop, "ok", flush=True)
os.environ.pop("EPC_PCG_LOOP")
d = synth.make_pair(synth.SynthSpec(m=(16, 12, 8), seed=5))
g = d.grid
cfg = abi.AdmmConfig(max_iter=3, **EX)
slabs = dist_admm.Slabs(*g.m, 2)
dev = torch.device("cuda", 0)
cl = g.m[0] * g.m[1]
gens = []
for rk in range(2):
    k0, mk = slabs.k_range(rk)
    sip = torch.from_numpy(d.iplus[k0 * cl:(k0 + mk) * cl].copy()).to(dev)
    sim = torch.from_numpy(d.iminus[k0 * cl:(k0 + mk) * cl].copy()).to(dev)
    gens.append(dist_admm.admm_rank(dist_admm.DeviceBackend(ctx, dev), g, slabs, rk, sip, sim, cfg=cfg))
res = dist_admm.run_lockstep(gens, dist_admm.torch_cat, dist_admm.torch_split)
r = orc.admm_solve(g, d.iplus, d.iminus, cfg=cfg)
assert np.array_equal(torch.cat([x["b"] for x in res]).cpu().numpy(), r["b"]), "slab"
print("slab lockstep ok", flush=True)
o = ctx.slab_admm_solve(None, 0, 1, g, torch.from_numpy(d.iplus).cuda(), torch.from_numpy(d.iminus).cuda(),
                        cfg=cfg)
assert np.array_equal(o["b"].cpu().numpy(), r["b"]), "slab c++"
print("slab c++ ok", flush=True)
f = ctx.admm_solve_f32(g, d.iplus.astype(np.float32), d.iminus.astype(np.float32), cfg=cfg)
print("f32 ok", float(np.abs(f["b"] - r["b"]).max()), flush=True)
if os.environ.get("EPC_GUARD"):
    bad = ctx.guard_check()
    assert bad == -1, f"guard zone of scratch slot {bad} overwritten"
    print("guard zones intact", flush=True)
# determinism (the reference's own race check, test_admm.cpp:384-401): the
# same solve three times, bitwise
d = synth.make_pair(synth.SynthSpec(m=(40, 24, 12), seed=9, scale=400.0))
runs = [ctx.admm_solve(d.grid, d.iplus, d.iminus, cfg=abi.AdmmConfig(max_iter=4, **EX)) for _ in range(3)]
assert all(np.array_equal(runs[0][k], r[k]) for r in runs[1:] for k in ("b", "z", "u")), "nondeterministic"
print("repeat runs bitwise identical", flush=True)
print("SANITIZE SMOKE DONE")
