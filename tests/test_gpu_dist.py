"""Slab-distributed ADMM on the GPU: the epc_slab_* C ABI steps (DeviceBackend)
for world sizes 1-3, the ranks run in lockstep in one process on one GPU
(each rank's kernels in turn; collectives in memory). The distributed solve
must equal the single-GPU epc_admm_solve and the reference oracle bitwise in
b, z, u. Multi-process NCCL uses the same driver (dist_admm.run_torch)."""
import numpy as np
import pytest
import torch

from paper_1607_00531_b200 import abi, dist_admm, synth

pytestmark = pytest.mark.gpu

EXACT = dict(eps_abs=1e-300, eps_rel=1e-300)


@pytest.mark.parametrize("world,m", [(1, (16, 12, 8)), (2, (16, 12, 8)), (3, (20, 14, 9)),
                                     (4, (33, 40, 17))])
def test_device_slabs_match_single_gpu(ctx, oracle, world, m):
    d = synth.make_pair(synth.SynthSpec(m=m, seed=5))
    g, ip, im = d.grid, d.iplus, d.iminus
    cfg = abi.AdmmConfig(max_iter=8, **EXACT)
    dev = torch.device("cuda", 0)
    slabs = dist_admm.Slabs(*m, world)
    cl = g.m[0] * g.m[1]
    gens = []
    for r in range(world):
        k0, mk = slabs.k_range(r)
        sip = torch.from_numpy(ip[k0 * cl:(k0 + mk) * cl].copy()).to(dev)
        sim = torch.from_numpy(im[k0 * cl:(k0 + mk) * cl].copy()).to(dev)
        gens.append(dist_admm.admm_rank(dist_admm.DeviceBackend(ctx, dev), g, slabs, r, sip, sim,
                                        cfg=cfg))
    res = dist_admm.run_lockstep(gens, dist_admm.torch_cat, dist_admm.torch_split)
    single = ctx.admm_solve(g, ip, im, cfg=cfg)
    ref = oracle.admm_solve(g, ip, im, cfg=cfg)
    for key in ("b", "z", "u"):
        got = torch.cat([r[key] for r in res]).cpu().numpy()
        assert np.array_equal(got, single[key]), (key, np.abs(got - single[key]).max())
        assert np.array_equal(got, ref[key])
    for r in res:
        assert r["rho"] == single["rho"] and r["stop"] == single["stop"]
        for a, b in zip(r["rows"], single["rows"]):
            assert a.rho == b["rho"] and a.kkt_violation == b["kkt_violation"]
            assert a.lagrangian == pytest.approx(b["lagrangian"], rel=1e-11)
            if world == 1:  # same kernels, same reductions
                assert a.primal_res == b["primal_res"] and a.dual_res == b["dual_res"]
