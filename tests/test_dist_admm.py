"""Slab-distributed ADMM (SURVEY §8(e), C5 k-slabs): the decomposition
logic of paper_1607_00531_b200/dist_admm.py on CPU. The local steps run on
the oracle-based backend (tests/dist_cpu_backend.py); the collectives run in
lockstep in one process and, for world size 2, over torch.distributed gloo
in two processes. The distributed solve must reproduce the single-process
reference solve bitwise in b, z, u (the rho decisions see the same values)
and its rows to rounding."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1607_00531_b200 import abi, dist_admm, synth

M = (10, 8, 7)
ITERS = 6
EXACT = dict(eps_abs=1e-300, eps_rel=1e-300)


def _pair():
    d = synth.make_pair(synth.SynthSpec(m=M, seed=11))
    return d.grid, d.iplus, d.iminus


def _slab_inputs(g, ip, im, slabs, r):
    k0, mk = slabs.k_range(r)
    cl = g.m[0] * g.m[1]
    return (np.ascontiguousarray(ip[k0 * cl:(k0 + mk) * cl]),
            np.ascontiguousarray(im[k0 * cl:(k0 + mk) * cl]))


def test_slab_bookkeeping():
    for world in (1, 2, 3, 4, 7):
        s = dist_admm.Slabs(10, 8, 7, world)
        assert sum(s.k_range(r)[1] for r in range(world)) == 7
        assert sum(s.i_range(r)[1] for r in range(world)) == 11
        for r in range(world):
            assert sum(s.block(r, q) for q in range(world)) == s.slab_faces(r)
            assert sum(s.block(q, r) for q in range(world)) == s.islab_faces(r)


def _check_against_oracle(oracle, g, ip, im, results, slabs, cfg):
    ref = oracle.admm_solve(g, ip, im, cfg=cfg)
    for key in ("b", "z", "u"):
        got = np.concatenate([np.asarray(r[key]) for r in results])
        assert np.array_equal(got, ref[key]), (key, np.abs(got - ref[key]).max())
    for r in results:
        assert r["stop"] == ref["stop"] and r["rho"] == ref["rho"]
        assert len(r["rows"]) == len(ref["rows"])
        for a, b in zip(r["rows"], ref["rows"]):
            assert a.iter == b["iter"] and a.rho == b["rho"]
            assert a.kkt_violation == b["kkt_violation"]
            for f in ("primal_res", "dual_res", "lagrangian"):
                assert getattr(a, f) == pytest.approx(b[f], rel=1e-11, abs=1e-300)


@pytest.mark.parametrize("world", [1, 2, 3])
def test_lockstep_cpu_matches_reference(oracle, world):
    from dist_cpu_backend import OracleBackend, np_cat, np_split
    g, ip, im = _pair()
    cfg = abi.AdmmConfig(max_iter=ITERS, **EXACT)
    slabs = dist_admm.Slabs(*M, world)
    gens = []
    for r in range(world):
        sip, sim = _slab_inputs(g, ip, im, slabs, r)
        gens.append(dist_admm.admm_rank(OracleBackend(oracle, g), g, slabs, r, sip, sim, cfg=cfg))
    res = dist_admm.run_lockstep(gens, np_cat, np_split)
    _check_against_oracle(oracle, g, ip, im, res, slabs, cfg)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [1, 2, 3])
def test_lockstep_exact_sums_rows_bitwise(oracle, world):
    """Every decision on the reference's sequential sums, chained rank after
    rank in index order (decide.py fallback): the rows' residuals are then
    bitwise the reference's, and b, z, u still are."""
    from dist_cpu_backend import OracleBackend, np_cat, np_split
    g, ip, im = _pair()
    cfg = abi.AdmmConfig(max_iter=ITERS, **EXACT)
    slabs = dist_admm.Slabs(*M, world)
    gens = []
    for r in range(world):
        sip, sim = _slab_inputs(g, ip, im, slabs, r)
        gens.append(dist_admm.admm_rank(OracleBackend(oracle, g), g, slabs, r, sip, sim, cfg=cfg,
                                        exact_sums=True))
    res = dist_admm.run_lockstep(gens, np_cat, np_split)
    _check_against_oracle(oracle, g, ip, im, res, slabs, cfg)
    ref = oracle.admm_solve(g, ip, im, cfg=cfg)
    for r in res:
        assert r["decisions"] == [0, ITERS]
        for a, b in zip(r["rows"], ref["rows"]):
            for f in ("primal_res", "dual_res", "eps_pri", "eps_dual"):
                assert getattr(a, f) == b[f], f


def test_lockstep_default_tolerances_and_infeasible_start(oracle):
    """Default eps (the stop test fires at iteration 1) through
    the certified decisions; an infeasible starting field raises the
    reference's invalid_argument before iteration 1 (admm.cpp:501-502)."""
    from dist_cpu_backend import OracleBackend, np_cat, np_split
    g, ip, im = _pair()
    world = 2
    slabs = dist_admm.Slabs(*M, world)
    cfg = abi.AdmmConfig(max_iter=ITERS)
    gens = []
    for r in range(world):
        sip, sim = _slab_inputs(g, ip, im, slabs, r)
        gens.append(dist_admm.admm_rank(OracleBackend(oracle, g), g, slabs, r, sip, sim, cfg=cfg))
    res = dist_admm.run_lockstep(gens, np_cat, np_split)
    _check_against_oracle(oracle, g, ip, im, res, slabs, cfg)
    bad = np.zeros(g.faces)
    bad.reshape(-1, g.m[0] + 1)[3, 5] = 1.5  # |D1 b| = 1.5 > 1
    gens = []
    for r in range(world):
        sip, sim = _slab_inputs(g, ip, im, slabs, r)
        k0, mk = slabs.k_range(r)
        lay = (g.m[0] + 1) * g.m[1]
        st = (np.ascontiguousarray(bad[k0 * lay:(k0 + mk) * lay]), None, None)
        gens.append(dist_admm.admm_rank(OracleBackend(oracle, g), g, slabs, r, sip, sim, cfg=cfg,
                                        state=st))
    with pytest.raises(ValueError, match="infeasible starting field"):
        dist_admm.run_lockstep(gens, np_cat, np_split)


def _worker(rank, world, port, q, exact_sums=False):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from dist_cpu_backend import OracleBackend
        from oracle import ffi
        g, ip, im = _pair()
        cfg = abi.AdmmConfig(max_iter=ITERS, **EXACT)
        slabs = dist_admm.Slabs(*M, world)
        sip, sim = _slab_inputs(g, ip, im, slabs, rank)
        gen = dist_admm.admm_rank(OracleBackend(ffi.load("oracle"), g), g, slabs, rank, sip, sim,
                                  cfg=cfg, exact_sums=exact_sums)
        out = dist_admm.run_torch(gen, dist, torch.device("cpu"))
        rows = [(x.iter, x.rho, x.kkt_violation, x.primal_res, x.dual_res, x.lagrangian)
                for x in out["rows"]]
        q.put((rank, out["b"], out["z"], out["u"], out["rho"], out["stop"], rows))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exact_sums", [False, True])
def test_gloo_two_ranks_match_reference(oracle, exact_sums):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, exact_sums)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=240) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g, ip, im = _pair()
    cfg = abi.AdmmConfig(max_iter=ITERS, **EXACT)

    class R(dict):
        pass
    results = []
    for (_, b, z, u, rho, stop, rows) in got:
        rr = []
        for (it, rh, kkt, pr, du, lag) in rows:
            row = abi.AdmmRow()
            row.iter, row.rho, row.kkt_violation = it, rh, kkt
            row.primal_res, row.dual_res, row.lagrangian = pr, du, lag
            rr.append(row)
        results.append(dict(b=b, z=z, u=u, rho=rho, stop=stop, rows=rr))
    _check_against_oracle(oracle, g, ip, im, results, dist_admm.Slabs(*M, world), cfg)


# ---- the halo2 collective used by the GN slabs (dist_gn), gloo vs lockstep --
HL = 3  # layer length


def _halo_gen(rank, world, owned_layers=2):
    lo = 1 if rank > 0 else 0
    hi = 1 if rank + 1 < world else 0
    n = (lo + owned_layers + hi) * HL
    x = np.full(n, -1.0)
    o0, o1 = lo * HL, (lo + owned_layers) * HL
    x[o0:o1] = rank * 100 + np.arange(o1 - o0)
    yield ("halo2", x, o0, o1, HL, lo, hi)
    return x


def _halo_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = dist_admm.run_torch(_halo_gen(rank, world), dist, torch.device("cpu"))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_halo2_gloo_matches_lockstep():
    from dist_cpu_backend import np_cat, np_split
    world = 3
    want = dist_admm.run_lockstep([_halo_gen(r, world) for r in range(world)], np_cat, np_split)
    # the lockstep exchange itself: halos hold the neighbours' edge layers
    assert np.array_equal(want[0][-HL:], 100 + np.arange(HL))
    assert np.array_equal(want[1][:HL], 3 + np.arange(HL))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert np.array_equal(got[r], want[r])
