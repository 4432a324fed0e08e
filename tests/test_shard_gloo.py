"""Multi-process (world size 2, gloo, CPU) test of the pair sharding used
for the C4 batch: shards cover every pair exactly once, each rank solves its
own pairs, and the gathered results equal a single-process run. The per-pair
solver here is the CPU oracle (test infrastructure); on the GPU box the same
host logic drives epc_admm_solve_batch."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1607_00531_b200 import abi, shard, synth


def test_shard_ranges_cover_exactly():
    for n in (1, 7, 64, 65):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                f, c = shard.shard_range(n, r, world)
                seen.extend(range(f, f + c))
                for i in range(f, f + c):
                    assert shard.owner_of(i, n, world) == r
            assert seen == list(range(n))
            counts = [shard.shard_range(n, r, world)[1] for r in range(world)]
            assert max(counts) - min(counts) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


M = (10, 8, 6)
NPAIRS = 5
ITERS = 4


def _solve_pairs(first, count):
    from oracle import ffi
    g, ip, im = synth.make_batch("C4", npairs=count, first=first, m=M)
    orc = ffi.load("oracle")
    cfg = abi.AdmmConfig(max_iter=ITERS, eps_abs=1e-300, eps_rel=1e-300)
    out = []
    for p in range(count):
        sl = slice(p * g.cells, (p + 1) * g.cells)
        r = orc.admm_solve(g, np.ascontiguousarray(ip[sl]), np.ascontiguousarray(im[sl]), cfg=cfg)
        out.append(r["b"])
    return np.stack(out) if out else np.zeros((0, g.faces))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, count = shard.shard_range(NPAIRS, rank, world)
    b = _solve_pairs(first, count)
    t = shard.max_over_ranks(float(rank + 1), dist)
    tot = shard.sum_over_ranks(float(count), dist)
    # gather variable-size blocks via padding
    faces = (M[0] + 1) * M[1] * M[2]
    maxc = -(-NPAIRS // world)
    pad = np.zeros((maxc, faces))
    pad[:count] = b
    buf = [torch.zeros(maxc, faces, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(buf, torch.from_numpy(pad))
    if rank == 0:
        blocks = []
        for r in range(world):
            f, c = shard.shard_range(NPAIRS, r, world)
            blocks.append(buf[r].numpy()[:c])
        q.put((np.concatenate(blocks), t, tot))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_pair_sharding_matches_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, tmax, total = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert tmax == 2.0 and total == NPAIRS
    ref = _solve_pairs(0, NPAIRS)
    assert np.array_equal(got, ref)
