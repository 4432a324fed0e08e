"""The multi-GPU variants of the drop-in boundary, through the
C ABI: the device-list batch solve (C4: pairs split over contexts, solved
concurrently from host threads) and the NCCL k-slab solve (C5: the C++ twin
of dist_admm.admm_rank, collectives on an NCCL communicator). The boxes have
one GPU: the device list runs several contexts on device 0 (the split and
the threads are the same code), the slab solve runs at world size 1 through
a real NCCL communicator and without one; the multi-rank slab logic is the
lockstep / gloo tests' (tests/test_dist_admm.py, tests/test_gpu_dist.py)."""
import numpy as np
import pytest

from paper_1607_00531_b200 import abi, synth

pytestmark = pytest.mark.gpu
EXACT = dict(eps_abs=1e-300, eps_rel=1e-300)


@pytest.mark.parametrize("ndev", [1, 2, 3])
def test_batch_devices_each_pair_bitwise(ctx, oracle, ndev):
    from paper_1607_00531_b200.epicorr import Context, admm_solve_batch_devices
    g, ip, im = synth.make_batch("C4", npairs=5, m=(16, 12, 8))
    nc, nf = g.cells, g.faces
    cfg = abi.AdmmConfig(max_iter=40)  # default eps: the pairs stop at different iterations
    ctxs = [ctx] + [Context(0) for _ in range(ndev - 1)]
    try:
        out = admm_solve_batch_devices(ctxs, g, 5, ip, im, cfg=cfg)
    finally:
        for c in ctxs[1:]:
            c.close()
    one = ctx.admm_solve_batch(g, 5, ip, im, cfg=cfg)
    for k in ("b", "z", "u"):
        assert np.array_equal(out[k], one[k]), k
    for q in range(5):
        r = oracle.admm_solve(g, ip[q * nc:(q + 1) * nc].copy(), im[q * nc:(q + 1) * nc].copy(), cfg=cfg)
        assert np.array_equal(out["b"][q * nf:(q + 1) * nf], r["b"]), q
        assert out["pairs"][q]["stop"] == r["stop"] and out["pairs"][q]["rho"] == r["rho"]
        assert len(out["pairs"][q]["rows"]) == len(r["rows"])


@pytest.mark.parametrize("use_nccl", [False, True])
def test_slab_solve_world1_bitwise(ctx, oracle, use_nccl):
    torch = pytest.importorskip("torch")
    from paper_1607_00531_b200.epicorr import NcclComm, nccl_unique_id
    d = synth.make_pair(synth.SynthSpec(m=(20, 12, 10), seed=21, scale=400.0))
    g = d.grid
    cfg = abi.AdmmConfig(max_iter=12, **EXACT)
    ref = oracle.admm_solve(g, d.iplus, d.iminus, cfg=cfg)
    comm = NcclComm(0, 1, 0, nccl_unique_id()) if use_nccl else None
    try:
        ip, im = torch.from_numpy(d.iplus).cuda(), torch.from_numpy(d.iminus).cuda()
        o = ctx.slab_admm_solve(comm, 0, 1, g, ip, im, cfg=cfg)
    finally:
        if comm is not None:
            comm.close()
    for k in ("b", "z", "u"):
        assert np.array_equal(o[k].cpu().numpy(), ref[k]), k
    assert o["rho"] == ref["rho"] and o["stop"] == ref["stop"]
    for a, b in zip(o["rows"], ref["rows"]):
        assert a["rho"] == b["rho"] and a["kkt_violation"] == b["kkt_violation"]
        assert a["lagrangian"] == pytest.approx(b["lagrangian"], rel=1e-11)


def test_slab_solve_warm_start_default_eps_and_errors(ctx, oracle):
    torch = pytest.importorskip("torch")
    d = synth.make_pair(synth.SynthSpec(m=(16, 12, 8), seed=5))
    g = d.grid
    ip, im = torch.from_numpy(d.iplus).cuda(), torch.from_numpy(d.iminus).cuda()
    # warm start from the oracle's state after 5 iterations, then default eps
    s5 = oracle.admm_solve(g, d.iplus, d.iminus, cfg=abi.AdmmConfig(max_iter=5, **EXACT))
    cfg = abi.AdmmConfig(max_iter=40)
    ref = oracle.admm_solve(g, d.iplus, d.iminus, b=s5["b"], z=s5["z"], u=s5["u"], rho=s5["rho"],
                            cfg=cfg)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    o = ctx.slab_admm_solve(None, 0, 1, g, ip, im, b=T(s5["b"]), z=T(s5["z"]), u=T(s5["u"]),
                            rho=s5["rho"], cfg=cfg)
    assert o["stop"] == ref["stop"] and len(o["rows"]) == len(ref["rows"])
    assert np.array_equal(o["b"].cpu().numpy(), ref["b"])
    # the reference's exceptions: infeasible start, 2D grid, missing communicator
    bad = np.zeros(g.faces)
    bad[3] = 5.0
    with pytest.raises(ValueError, match="infeasible starting field"):
        ctx.slab_admm_solve(None, 0, 1, g, ip, im, b=T(bad), cfg=cfg)
    with pytest.raises(ValueError, match="communicator"):
        ctx.slab_admm_solve(None, 0, 2, g, ip, im, cfg=cfg)
