"""A/B of the forward axis-2 transform fused into the b-step's drain
(EPC_FUSE_FWD2=1, default) against the separate GEMM launch (=0).

Run once per mode (the switch is read once per process); prints the solve
time per config and a digest of b, z, u, rho and the rows' rho / kkt, which
must agree bitwise between the two modes.

    EPC_FUSE_FWD2=0 python scripts/ab_fuse_fwd2.py
    EPC_FUSE_FWD2=1 python scripts/ab_fuse_fwd2.py
"""
import hashlib
import os
import sys
from dataclasses import replace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1607_00531_b200 import abi, synth  # noqa: E402
from paper_1607_00531_b200.epicorr import Context  # noqa: E402


def digest(r):
    h = hashlib.sha256()
    for k in ("b", "z", "u"):
        h.update(r[k].cpu().numpy().tobytes())
    h.update(repr(r["rho"]).encode())
    h.update(repr([(row["rho"], row["kkt_violation"]) for row in r["rows"]]).encode())
    return h.hexdigest()[:16]


def main():
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)
    ctx = Context(0, stream=stream)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    mode = os.environ.get("EPC_FUSE_FWD2", "1")
    for name, scale, iters, reps in (("C3", 1.0, 100, 5), ("C3", 400.0, 20, 2), ("C1", 1.0, 50, 5)):
        spec = replace(synth.CONFIGS[name], scale=scale)
        d = synth.make_pair(spec)
        g = d.grid
        ip = torch.from_numpy(d.iplus).to(dev)
        im = torch.from_numpy(d.iminus).to(dev)
        cfg = abi.AdmmConfig(max_iter=iters, eps_abs=1e-300, eps_rel=1e-300)
        r = ctx.admm_solve(g, ip, im, cfg=cfg)
        dg = digest(r)
        ts = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            e0.record(stream)
            r2 = ctx.admm_solve(g, ip, im, cfg=cfg)
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
            assert digest(r2) == dg, "not deterministic"
        ts.sort()
        ctx.profile(True)
        ctx.profile_reset()
        ctx.admm_solve(g, ip, im, cfg=cfg)
        prof = ctx.profile_read()
        ctx.profile(False)
        per = " ".join(f"{k}={v[0] / v[1]:.4f}" for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])
                       if v[1] and v[0] / iters > 0.01)
        print(f"fuse={mode} lib={os.environ.get('EPC_LIB', 'main')} {name} x{scale:g} {iters} it: "
              f"median {ts[len(ts) // 2]:.2f} ms (min {ts[0]:.2f}) digest {dg} stop {r['stop']}\n"
              f"    ms/launch: {per}", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
