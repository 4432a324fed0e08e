"""GN-PCG in k-slabs on the GPU (dist_gn over the epc_gnslab_* C ABI), world
sizes 1-4 in lockstep on one GPU, against the single-GPU epc_gn_solve and
the reference oracle. The cross-rank sums are taken in a different order
than the single-GPU device trees, so the comparison is at the north-star
tolerances (b to 1e-8 relative L2, j to 1e-9) - in practice ~1e-14."""
import numpy as np
import pytest
import torch

from paper_1607_00531_b200 import abi, dist_admm, dist_gn, synth
from paper_1607_00531_b200.epicorr import Context

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,m", [(1, (16, 12, 8)), (2, (16, 12, 8)), (3, (20, 14, 9)),
                                     (4, (24, 18, 12))])
def test_device_gn_slabs(ctx, oracle, world, m):
    d = synth.make_pair(synth.SynthSpec(m=m, seed=9))
    g, ip, im = d.grid, d.iplus, d.iminus
    cfg = abi.GnConfig(eta=1e-2, max_pcg=50, max_outer=4)
    dev = torch.device("cuda", 0)
    slabs = dist_admm.Slabs(*m, world)
    cl = g.m[0] * g.m[1]
    gens = []
    for r in range(world):
        k0, mk, lo, hi = dist_gn._ext_layout(g, slabs, r)
        a, b = (k0 - lo) * cl, (k0 + mk + hi) * cl
        sip = torch.from_numpy(ip[a:b].copy()).to(dev)
        sim = torch.from_numpy(im[a:b].copy()).to(dev)
        # one context per rank: the Hessian blocks and factor live in it
        gens.append(dist_gn.gn_rank(dist_gn.DeviceGnBackend(Context(0), dev), g, slabs, r, sip,
                                    sim, cfg=cfg))
    res = dist_admm.run_lockstep(gens, dist_admm.torch_cat, dist_admm.torch_split)
    single = ctx.gn_solve(g, ip, im, cfg=cfg)
    ref = oracle.gn_solve(g, ip, im, cfg=cfg)
    bb = torch.cat([r["b"] for r in res]).cpu().numpy()
    for other in (single, ref):
        rel = np.linalg.norm(bb - other["b"]) / np.linalg.norm(other["b"])
        assert rel <= 1e-10, rel
    for r in res:
        assert r["stop"] == single["stop"]
        assert len(r["rows"]) == len(single["rows"])
        for a, b in zip(r["rows"], single["rows"]):
            assert a.pcg_iters == b["pcg_iters"]
            assert a.j_value == pytest.approx(b["j_value"], rel=1e-10)
            assert a.step == pytest.approx(b["step"], rel=1e-10)
