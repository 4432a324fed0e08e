#!/usr/bin/env python3
"""bench.py — ADMM time-to-solution and voxel-iterations/s on B200.

Workload (BASELINE.json configs[2], the config its metric is quoted on):
ADMM on the 256x256x96 synthetic volume pair, fp64, 100 outer iterations
from b = 0, reference-default alpha/rho schedule, eps_abs = eps_rel = 1e-300
so the iteration count is fixed. One "step" = one full solve.

  value  = faces x ADMM iterations x ranks / max-over-ranks device time,
           inputs resident in HBM (EPC_MEM_DEVICE through the C ABI);
  e2e    = the same through the C ABI with pinned host buffers: every step
           copies I+/I- in and b/z/u out inside the timed region.

Multi-GPU (torchrun, one process per GPU): ADMM does not shard a single
C3 volume (BASELINE runs C3 on 1 GPU), so each rank solves its own volume
pair (independent replicas, weak scaling, no data-path collective); the
barrier + max-over-ranks timing uses NCCL only for the timing plumbing.

--impl reference: the reference's own CPU implementation of this path
(oracle/_ref: proj/src compiled unmodified) on all host threads, same config
and metric, each step a bounded sample (a few ADMM iterations) of the solve.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1607_00531_b200 import abi, synth  # noqa: E402

METRIC = "voxel-iterations/s (ADMM, 256x256x96, fp64)"  # BASELINE.json metric (C3)


def metric_for(config):
    """BASELINE's metric string, naming the grid actually run (C3 unless --config)."""
    if config == "C3":
        return METRIC
    spec = synth.CONFIGS[config]
    return f"voxel-iterations/s (ADMM, {'x'.join(map(str, spec.m))}, fp64)"
UNIT = "face-iterations/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--iters", type=int, default=None, help="ADMM iterations per solve")
    ap.add_argument("--scale", type=float, default=1.0, help="intensity scale (x400 variant)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gn", action="store_true", help="skip the GN-PCG leg (configs[1])")
    ap.add_argument("--gn-config", default="C2")
    ap.add_argument("--no-f32", action="store_true", help="skip the fp32-variant leg")
    ap.add_argument("--no-gn-c3", action="store_true", help="skip the GN-PCG C3 leg")
    ap.add_argument("--no-x400", action="store_true", help="skip the amplitude-x400 C3 leg")
    ap.add_argument("--sharded", action="store_true",
                    help="run the C4 / C5 sharded legs even at one rank (they run by default at N > 1)")
    return ap.parse_args()


# fp64 DADD/DMUL issue rate measured on this pool (profiles/r01_ubench_fp64_tput.log)
FP64_PEAK_TOPS = 18.3
NCU_BSTEP_SUMMARY = "r02ff_bstep_c3_late_ncu.json"  # C3 b-step, launch 91 of 100, ncu --set full
# the GN-PCG kernels' ncu captures: C2 runs the persistent loop (L2-resident),
# C3 the per-iteration kernels (k_pcg_hvp, k_pcg_update_bj)
NCU_PCG_SUMMARY = {"C2": "r02fin_pcg_c2_ncu.json", "C3": "r02fin_pcg_parts_c3_ncu.json"}
DEFAULT_ITERS = {"C1": 50, "C2": 50, "C3": 100, "C4": 50, "C5": 50}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for n, v in zip(names, s[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


def dist_setup(n):
    if n <= 1 and "RANK" not in os.environ:
        return 0, 1, 0, None
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", n))
    local = int(os.environ.get("LOCAL_RANK", rank))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29511")
    import torch
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", local))
    else:
        dist.init_process_group("nccl", rank=rank, world_size=world)
    return rank, world, local, dist


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def ref_checker(threads):
    """The reference's CPU implementation: oracle/_ref (proj/src compiled
    unmodified) when built, else the single-threaded C port (oracle/_build).
    -> (checker, kind, cores)."""
    from oracle import ffi
    kind = "reference" if os.path.exists(ffi.PATHS["ref"]) else "port"
    chk = ffi.load("ref" if kind == "reference" else "oracle")
    cores = threads if kind == "reference" else 1
    if kind == "reference":
        chk.set_threads(cores)
    return chk, kind, cores


def admm_cfg(iters, threads=1):
    return abi.AdmmConfig(max_iter=iters, eps_abs=1e-300, eps_rel=1e-300, threads=threads)


def ref_admm_window(chk, cores, d, state, n):
    """n reference ADMM iterations warm-started from state (b, z, u, rho) via
    ADMMState init (admm.hpp:127-129; the mechanism multilevel.cpp:252 uses),
    which continues the trajectory exactly (eps = 1e-300: no stop test fires).
    -> (seconds, b_update seconds, result)."""
    kw = {} if state is None else dict(b=state["b"], z=state["z"], u=state["u"], rho=state["rho"])
    t = time.perf_counter()
    r = chk.admm_solve(d.grid, d.iplus, d.iminus, cfg=admm_cfg(n, cores), **kw)
    dt = time.perf_counter() - t
    return dt, sum(x["b_update_s"] for x in r["rows"]), r


def window_sizes(total, k):
    """k consecutive windows covering `total` iterations (cycled when k > total)."""
    if k <= total:
        return [(s * total) // k for s in range(k + 1)]
    return None


def ref_trajectory(chk, cores, d, iters, steps):
    """The whole iters-long solve timed as `steps` consecutive windows, each
    warm-started from the previous one's state: every timed step is a
    bounded slice and together they are exactly one full solve (restarted
    from b = 0 when steps > iters). -> (seconds, b_update seconds, faces x
    iterations, per-window list, mid-trajectory state, its iteration)."""
    bounds = window_sizes(iters, steps)
    sizes = ([bounds[s + 1] - bounds[s] for s in range(steps)] if bounds is not None
             else [1] * steps)
    state, done = None, 0
    tot = tb = 0.0
    units = 0
    wins = []
    mid, mid_it = None, 0
    for n in sizes:
        if done >= iters:
            state, done = None, 0
        if mid is None and done >= iters // 2:
            mid, mid_it = state, done
        dt, bt, r = ref_admm_window(chk, cores, d, state, n)
        state = r
        done += n
        tot += dt
        tb += bt
        units += d.grid.faces * n
        wins.append({"first_iter": done - n + 1, "iters": n, "s": round(dt, 4)})
    return tot, tb, units, wins, mid, mid_it


def run_reference_arm(a, iters):
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return 0
    d = synth.make_config(a.config, scale=a.scale)
    threads = os.cpu_count() or 1
    chk, kind, cores = ref_checker(threads)
    for _ in range(a.warmup):  # one iteration from b = 0 each (page-in, thread pools)
        ref_admm_window(chk, cores, d, None, 1)
    tot, tb, units, wins, mid, mid_it = ref_trajectory(chk, cores, d, iters, a.steps)
    value = units / tot
    # a 1-thread figure: the iteration after the mid-trajectory window boundary
    one = None
    if kind == "reference" and mid is not None:
        try:
            chk.set_threads(1)
            dt1, _, _ = ref_admm_window(chk, 1, d, mid, 1)
            one = {"value": d.grid.faces / dt1, "unit": UNIT, "cores": 1,
                   "sample": f"ADMM iteration {mid_it + 1} of the {a.config} solve, 1 thread"}
        except Exception as e:  # diagnostic only
            one = {"value": None, "sample": str(e)[:120]}
        finally:
            chk.set_threads(cores)
    line = {"metric": metric_for(a.config), "value": value, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": tot / a.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": admm_config_dict(a, d.grid, iters),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "cpu_model": cpu_model(),
                             "sample": (f"the whole {iters}-iteration {a.config} solve from b = 0, "
                                        f"timed as {a.steps} consecutive warm-started windows "
                                        f"(ADMMState init)"),
                             "time_to_solution_s": tot * iters / max(1, sum(w["iters"] for w in wins)),
                             "phase_split": {"b_update_s": tb, "z_dual_lagrangian_s": tot - tb,
                                             "b_update_frac": tb / tot},
                             "one_thread": one,
                             "windows": wins},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if not a.no_gn:
        dg = synth.make_config(a.gn_config)
        gt = gn_reference_trajectory(dg, threads, a.steps)
        line["gn"] = {"metric": f"voxel-iterations/s (GN-PCG, {'x'.join(map(str, dg.grid.dims()))}, fp64)",
                      "value": gt["value"], "unit": GN_UNIT,
                      "cpu_baseline": gt,
                      "e2e": {"value": gt["value"], "unit": GN_UNIT, "h2d_bytes_per_step": 0,
                              "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def admm_config_dict(a, g, iters):
    """The `config` object, identical in both arms (same workload)."""
    return {"workload": f"ADMM {a.config} {'x'.join(map(str, g.dims()))}, {iters} iterations, "
                        f"fp64, from b=0",
            "faces": g.faces, "iterations": iters, "intensity_scale": a.scale,
            "pairs": 64 if a.config == "C4" else 1,
            "parallelism": ("pairs sharded over ranks" if a.config == "C4"
                            else "one volume per GPU (replicas)"),
            "l2": "working set > L2 (126 MB); the GPU arm also writes 256 MB before every timed step"}


GN_UNIT = "face-PCG-iterations/s"


def gn_config():
    """BASELINE configs[1]: block-Jacobi GN-PCG, 10 GN steps x up to 50 PCG
    iterations at eta = 1e-2; the outer stopping tests are disabled
    (eps = 1e-300) so every run does exactly 10 GN steps."""
    return abi.GnConfig(eta=1e-2, max_outer=10, max_pcg=50, eps_obj=1e-300, eps_iter=1e-300,
                        eps_grad=1e-300, precond=abi.PRECOND_BLOCK_JACOBI)


def gn_reference_sample(d, threads, outer=1, b0=None):
    """The reference's GN (oracle/_ref, else the C port) for `outer` GN steps
    of the configs[1] solve from b0 -> (kind, seconds, cores, PCG iterations, b)."""
    chk, kind, cores = ref_checker(threads)
    cfg = gn_config()
    cfg.max_outer = outer
    cfg.threads = cores
    t = time.perf_counter()
    r = chk.gn_solve(d.grid, d.iplus, d.iminus, b0=b0, cfg=cfg)
    dt = time.perf_counter() - t
    npcg = sum(x["pcg_iters"] for x in r["rows"])
    return kind, dt, cores, npcg, r["b"]


def gn_reference_trajectory(d, threads, steps, outer_total=10):
    """The reference's whole 10-step GN solve, timed one GN step per window
    (warm-started from the previous b; the stopping tests are off, so the
    trajectory is the one-call solve's), cycled to fill `steps` windows."""
    b, done, tot, npcg = None, 0, 0.0, 0
    kind = cores = None
    for _ in range(max(steps, 1)):
        if done >= outer_total:
            b, done = None, 0
        kind, dt, cores, n, b = gn_reference_sample(d, threads, 1, b)
        done += 1
        tot += dt
        npcg += n
    return {"value": d.grid.faces * npcg / tot, "unit": GN_UNIT, "cores": cores, "kind": kind,
            "sample": (f"the {outer_total}-step {'x'.join(map(str, d.grid.dims()))} GN solve, one "
                       f"GN step per window, {max(steps, 1)} windows"),
            "pcg_iterations": npcg, "seconds": tot}


def run_gn_leg(a, ctx, dev, stream, flush, rank, dist, config_name, cpu_windows, min_solves=10):
    """GN-PCG (configs[1] on C2 128x128x64, and the north-star target on C3
    256x256x96): device-resident time to solution and face-PCG-iterations/s,
    e2e through the C ABI with host buffers, the PCG kernels against the HBM
    roof (with the ncu DRAM traffic when a capture summary is committed), and
    the reference CPU sample beside it (cpu_windows GN steps of the solve)."""
    import ctypes as C

    import torch
    from dataclasses import replace
    spec = synth.CONFIGS[config_name]
    spec = replace(spec, seed=spec.seed + 1000 * rank)
    d = synth.make_pair(spec)
    g = d.grid
    cfg = gn_config()
    ip_d, im_d = torch.from_numpy(d.iplus).to(dev), torch.from_numpy(d.iminus).to(dev)
    ip_h, im_h = torch.from_numpy(d.iplus).pin_memory(), torch.from_numpy(d.iminus).pin_memory()
    b0_h = torch.zeros(g.faces, dtype=torch.float64).pin_memory()
    bo_h = torch.empty(g.faces, dtype=torch.float64).pin_memory()
    torch.cuda.synchronize(dev)

    def solve_device():
        return ctx.gn_solve(g, ip_d, im_d, cfg=cfg)

    def solve_host():
        rows = (abi.GnRow * (cfg.max_outer + 1))()
        st = abi.SolveStatus()
        P = lambda t: C.c_void_p(t.data_ptr())
        rc = ctx.lib.epc_gn_solve(ctx.h, C.byref(g), abi.EPC_MEM_HOST, P(ip_h), P(im_h), P(b0_h),
                                  P(bo_h), C.byref(abi.ObjectiveParams()), C.byref(cfg), 0, rows,
                                  cfg.max_outer + 1, C.byref(st))
        assert rc == 0, ctx._err()
        return sum(rows[i].pcg_iters for i in range(min(st.nrows, cfg.max_outer + 1)))

    def timed(fn, k):
        tot, launches, npcg = 0.0, 0, 0
        for _ in range(k):
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ctx.reset_launch_count()
            e0.record(stream)
            r = fn()
            e1.record(stream)
            e1.synchronize()
            launches += ctx.launch_count()
            tot += e0.elapsed_time(e1) / 1e3
            npcg += r if isinstance(r, int) else sum(x["pcg_iters"] for x in r["rows"])
        return tot, launches, npcg

    # a GN solve is ~25 ms with 10 host round trips: time at least 10 solves
    # so host scheduling jitter averages out
    gk = max(a.steps, min_solves)
    for _ in range(max(a.warmup, 3)):
        solve_device()
    t_dev, launches, npcg = timed(solve_device, gk)
    t_e2e, _, npcg_h = timed(solve_host, gk)
    from paper_1607_00531_b200 import shard
    t_dev = shard.max_over_ranks(t_dev, dist, dev)
    t_e2e = shard.max_over_ranks(t_e2e, dist, dev)
    world = dist.get_world_size() if dist is not None else 1
    # per-kernel times of one profiled solve; algorithmic bytes per face per
    # launch: pcg_hvp reads z, p_old, diag, off and writes p, q
    # (48 B); pcg_update reads d, r, p, q, fd, fl and writes d, r, z (72 B).
    # The profiled solve is one solve; npcg counts gk solves.
    ctx.profile(True)
    ctx.profile_reset()
    solve_device()
    prof = ctx.profile_read()
    ctx.profile(False)
    per_face = {"pcg_update": 72, "pcg_hvp": 48}
    # the persistent loop kernel runs both phases (120 B/face per PCG
    # iteration) for all iterations of one PCG solve per launch
    loop_iters = npcg / gk / max(1, prof.get("pcg_loop", (0, 0))[1])
    kernels = []
    for name, (ms, n) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
        if not n:
            continue
        k = {"kernel": name, "launches": n, "ms_per_launch": ms / n,
             "share": ms / sum(v[0] for v in prof.values())}
        if name in per_face:
            gbs = per_face[name] * g.faces / (ms / n / 1e3) / 1e9
            k.update(alg_bytes=per_face[name] * g.faces, achieved_gbs=gbs)
        elif name == "pcg_loop":
            alg = 120 * g.faces * loop_iters
            k.update(alg_bytes=alg, pcg_iterations_per_launch=loop_iters,
                     achieved_gbs=alg / (ms / n / 1e3) / 1e9)
        kernels.append(k)
    roof = None
    top = next((k for k in kernels if "achieved_gbs" in k), None)
    fits_l2 = 15 * 8 * g.faces < 126e6
    if top is not None:
        try:
            peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
            src = "measured"
        except Exception:
            peak, src = 6650.0, "fallback"
        traffic, tsrc, tunit = None, None, None
        cap_name = NCU_PCG_SUMMARY.get(config_name)
        try:  # DRAM bytes from the committed ncu --set full capture of the same kernel
            cap = json.load(open(os.path.join(ROOT, "profiles", cap_name)))
            if top["kernel"] == "pcg_loop":
                traffic, tunit = float(cap["dram_bytes_per_pcg_iteration"]), "bytes per PCG iteration"
            else:
                traffic = float(cap["kernels"][top["kernel"]]["dram_bytes_per_launch"])
                tunit = "bytes per launch"
            tsrc = "profiles/" + cap_name
        except Exception:
            pass
        for k in kernels:  # every PCG kernel's own fraction of the roof
            if "achieved_gbs" in k:
                k["frac_hbm"] = k["achieved_gbs"] / peak
        roof = {"bound": "hbm", "kernel": top["kernel"], "achieved": top["achieved_gbs"], "peak": peak,
                "peak_source": src, "unit": "GB/s", "frac": top["achieved_gbs"] / peak,
                "traffic": traffic, "traffic_unit": tunit, "alg_bytes": top["alg_bytes"],
                "alg_bytes_per_pcg_iteration": 120 * g.faces, "traffic_source": tsrc,
                "note": ("algorithmic bytes (120 B/face per PCG iteration) / CUDA-event time; " +
                         ("the PCG vectors fit in L2 at this size" if fits_l2 else
                          "the PCG vectors (~15 face vectors) exceed L2: HBM-resident"))}
    out = {"metric": f"voxel-iterations/s (GN-PCG, {'x'.join(map(str, g.dims()))}, fp64)",
           "value": g.faces * npcg / t_dev * world, "unit": GN_UNIT,
           "steps": gk, "time_to_solution_s": t_dev / gk, "pcg_iterations_per_solve": npcg // gk,
           "workload": f"GN-PCG {config_name} block-Jacobi, 10 GN steps x <=50 PCG, eta 1e-2",
           "e2e": {"value": g.faces * npcg_h / t_e2e * world, "unit": GN_UNIT,
                   "h2d_bytes_per_step": (2 * g.cells + g.faces) * 8,
                   "d2h_bytes_per_step": g.faces * 8},
           "gpu_launches": launches, "roofline": roof, "kernels": kernels[:8],
           "l2": "256 MB flush write before every timed step"}
    if rank == 0 and not a.no_cpu_baseline:
        try:
            out["cpu_baseline"] = gn_reference_trajectory(d, os.cpu_count() or 1, cpu_windows)
        except Exception as e:
            out["cpu_baseline"] = {"value": None, "kind": "unavailable", "sample": str(e)[:120]}
    return out


def gpu_checkpoints(ctx, g, ip_d, im_d, starts, params=None):
    """Host copies of the ADMM state at the given iteration counts, from the
    device solve (b, z, u, rho are bitwise the reference's trajectory:
    tests/test_gpu_fullsize.py), so CPU windows can start mid-trajectory."""
    out, st, done = {}, None, 0
    for s_ in sorted(set(starts)):
        if s_ > done:
            kw = {} if st is None else dict(b=st["b"], z=st["z"], u=st["u"], rho=st["rho"])
            st = ctx.admm_solve(g, ip_d, im_d, cfg=admm_cfg(s_ - done), params=params, **kw)
            done = s_
        out[s_] = None if st is None else dict(
            b=st["b"].double().cpu().numpy(), z=st["z"].double().cpu().numpy(),
            u=st["u"].double().cpu().numpy(), rho=st["rho"])
    return out


def cpu_windows_baseline(ctx, d, ip_d, im_d, iters, config, starts, n):
    """cpu_baseline: the reference (oracle/_ref, all host threads) timed on n
    iterations starting at each of `starts` (states from gpu_checkpoints):
    a bounded sample spread evenly over the whole trajectory."""
    threads = os.cpu_count() or 1
    chk, kind, cores = ref_checker(threads)
    cps = gpu_checkpoints(ctx, d.grid, ip_d, im_d, starts)
    tot, units = 0.0, 0
    for s_ in starts:
        dt, _, _ = ref_admm_window(chk, cores, d, cps[s_], n)
        tot += dt
        units += d.grid.faces * n
    return {"value": units / tot, "unit": UNIT, "cores": cores, "kind": kind,
            "cpu_model": cpu_model(),
            "sample": (f"{n} ADMM iterations from each of iterations {[x + 1 for x in starts]} "
                       f"of the {iters}-iteration {config} solve (warm-started through "
                       f"ADMMState init), {units // d.grid.faces} iterations in all"),
            "seconds": tot}


def run_x400_leg(a, ctx, dev, stream, flush, iters, rank, dist):
    """The amplitude-x400 variant of C3 (image.hpp:87-90: the
    reference's phantoms use 400 so the distance term dominates alpha = 50):
    time per solve, b-step ms per launch, and the SQP / QP / line-search
    work counters, beside a reference CPU sample."""
    import torch
    from dataclasses import replace
    spec = synth.CONFIGS[a.config]
    spec = replace(spec, scale=400.0, seed=spec.seed + 1000 * rank)
    d = synth.make_pair(spec)
    g = d.grid
    ip_d, im_d = torch.from_numpy(d.iplus).to(dev), torch.from_numpy(d.iminus).to(dev)
    cfg = admm_cfg(iters)
    ctx.admm_solve(g, ip_d, im_d, cfg=cfg)
    k = max(1, min(a.steps, 5))
    tot = 0.0
    launches = 0
    c0 = ctx.admm_counters()
    for _ in range(k):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx.reset_launch_count()
        e0.record(stream)
        ctx.admm_solve(g, ip_d, im_d, cfg=cfg)
        e1.record(stream)
        e1.synchronize()
        launches += ctx.launch_count()
        tot += e0.elapsed_time(e1) / 1e3
    c1 = ctx.admm_counters()
    from paper_1607_00531_b200 import shard
    tmax = shard.max_over_ranks(tot, dist, dev)
    world = dist.get_world_size() if dist is not None else 1
    ctx.profile(True)
    ctx.profile_reset()
    ctx.admm_solve(g, ip_d, im_d, cfg=cfg)
    prof = ctx.profile_read()
    ctx.profile(False)
    bms, bn = prof.get("admm_bstep", (0.0, 0))
    # line-search counters from the diagnostic instantiation (one solve)
    from paper_1607_00531_b200.epicorr import Context
    ctx.set_mode(0)
    ctx.set_mode(Context.MODE_BSTEP_TIMING)
    ctx.admm_solve(g, ip_d, im_d, cfg=cfg)
    cnt = ctx.bstep_counters()
    ctx.set_mode(0)
    out = {"metric": f"voxel-iterations/s (ADMM x400, {'x'.join(map(str, g.dims()))}, fp64)",
           "value": g.faces * iters * k * world / tmax, "unit": UNIT,
           "time_to_solution_s": tmax / k, "steps": k, "gpu_launches": launches,
           "bstep_ms_per_launch": bms / max(bn, 1),
           "bstep_share": bms / max(1e-30, sum(v[0] for v in prof.values())),
           "sqp_iterations_per_solve": (c1[2] - c0[2]) // k,
           "qp_iterations_per_solve": (c1[3] - c0[3]) // k,
           "line_search": {kk: cnt[kk] for kk in ("ls_searches", "ls_trials", "ls_undecided",
                                                   "ls_failed", "acc0", "acc1", "acc2_3",
                                                   "acc4_7", "acc8_15", "acc16_31", "acc32_39")},
           "workload": f"ADMM {a.config} x400 intensity, {iters} iterations, fp64, from b=0"}
    if rank == 0 and not a.no_cpu_baseline:
        try:
            out["cpu_baseline"] = cpu_windows_baseline(ctx, d, ip_d, im_d, iters,
                                                       a.config + " x400",
                                                       starts=[0, iters // 2], n=1)
        except Exception as e:
            out["cpu_baseline"] = {"value": None, "kind": "unavailable", "sample": str(e)[:120]}
    return out


def run_f32_leg(a, ctx, dev, stream, flush, g, ipn, imn, iters, b64, dist):
    """fp32 variant (BASELINE configs[2] "fp64 and an fp32 variant"), reported
    separately: the same solve through epc_admm_solve_f32, device-resident
    throughput, e2e with host float32 buffers, and its deviation from the
    fp64 result (which is bitwise the reference's) on the same inputs."""
    import torch
    cfg = abi.AdmmConfig(max_iter=iters, eps_abs=1e-300, eps_rel=1e-300)
    ip32 = np.ascontiguousarray(ipn[:g.cells], dtype=np.float32)
    im32 = np.ascontiguousarray(imn[:g.cells], dtype=np.float32)
    ip_d, im_d = torch.from_numpy(ip32).to(dev), torch.from_numpy(im32).to(dev)
    ip_h, im_h = torch.from_numpy(ip32).pin_memory(), torch.from_numpy(im32).pin_memory()
    torch.cuda.synchronize(dev)

    def timed(fn, k):
        tot, launches, out = 0.0, 0, None
        for _ in range(k):
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ctx.reset_launch_count()
            e0.record(stream)
            out = fn()
            e1.record(stream)
            e1.synchronize()
            launches += ctx.launch_count()
            tot += e0.elapsed_time(e1) / 1e3
        return tot, launches, out

    for _ in range(a.warmup):
        ctx.admm_solve_f32(g, ip_d, im_d, cfg=cfg)
    t_dev, launches, r = timed(lambda: ctx.admm_solve_f32(g, ip_d, im_d, cfg=cfg), a.steps)
    t_e2e, _, rh = timed(lambda: ctx.admm_solve_f32(g, ip_h.numpy(), im_h.numpy(), cfg=cfg), a.steps)
    from paper_1607_00531_b200 import shard
    t_dev = shard.max_over_ranks(t_dev, dist, dev)
    t_e2e = shard.max_over_ranks(t_e2e, dist, dev)
    world = dist.get_world_size() if dist is not None else 1
    b32 = r["b"].double().cpu().numpy()
    ref = np.asarray(b64, dtype=np.float64)
    units = g.faces * iters * a.steps * world
    return {"metric": f"voxel-iterations/s (ADMM fp32 variant, {'x'.join(map(str, g.dims()))})",
            "value": units / t_dev, "unit": UNIT, "ms_per_step": t_dev / a.steps * 1e3,
            "dtype": "f32", "time_to_solution_s": t_dev / a.steps,
            "e2e": {"value": units / t_e2e, "unit": UNIT, "h2d_bytes_per_step": 2 * g.cells * 4,
                    "d2h_bytes_per_step": 3 * g.faces * 4},
            "gpu_launches": launches,
            "rel_l2_b_vs_fp64": float(np.linalg.norm(b32 - ref) / max(np.linalg.norm(ref), 1e-300)),
            "note": "fp32 storage and element arithmetic, fp64-accumulated sums, thresholds "
                    "rescaled for fp32; not bitwise (tolerance in tests/test_gpu_admm_f32.py)"}


def run_slabs(a, iters):
    """C5: one volume, k-slabs across the ranks; strong scaling.
    Each rank generates the same seeded volume and keeps its slab; the solve
    is paper_1607_00531_b200.dist_admm over the epc_slab_* C ABI, with NCCL
    all-to-all transposes, a one-layer halo and a scalar all-gather between
    the local steps. World size 1 runs the same driver without collectives."""
    import torch
    from paper_1607_00531_b200 import dist_admm
    from paper_1607_00531_b200.epicorr import Context
    rank, world, local, dist = dist_setup(a.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    ctx = Context(local, stream=stream)
    d = synth.make_config(a.config, scale=a.scale)
    g = d.grid
    slabs = dist_admm.Slabs(g.m[0], g.m[1], g.m[2], world)
    k0, mk = slabs.k_range(rank)
    cl = g.m[0] * g.m[1]
    ip_h = torch.from_numpy(np.ascontiguousarray(d.iplus[k0 * cl:(k0 + mk) * cl])).pin_memory()
    im_h = torch.from_numpy(np.ascontiguousarray(d.iminus[k0 * cl:(k0 + mk) * cl])).pin_memory()
    ip_d, im_d = ip_h.to(dev), im_h.to(dev)
    cfg = abi.AdmmConfig(max_iter=iters, eps_abs=1e-300, eps_rel=1e-300)
    backend = dist_admm.DeviceBackend(ctx, dev)
    nf = slabs.slab_faces(rank)
    out_h = [torch.empty(nf, dtype=torch.float64).pin_memory() for _ in range(3)]

    def solve(host):
        ip_, im_ = (ip_h.to(dev, non_blocking=True), im_h.to(dev, non_blocking=True)) if host \
            else (ip_d, im_d)
        torch.cuda.synchronize(dev)  # the H2D runs on torch's stream, the solve on ctx's
        gen = dist_admm.admm_rank(backend, g, slabs, rank, ip_, im_, cfg=cfg)
        if dist is None:
            r = dist_admm.run_lockstep([gen], dist_admm.torch_cat, dist_admm.torch_split)[0]
        else:
            r = dist_admm.run_torch(gen, dist, dev)
        if host:
            for o, key in zip(out_h, ("b", "z", "u")):
                o.copy_(r[key], non_blocking=True)
        return r

    def timed(host, k):
        tot, launches = 0.0, 0
        for _ in range(k):
            torch.cuda.synchronize(dev)
            if dist is not None:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            ctx.reset_launch_count()
            e0.record(stream)
            solve(host)
            torch.cuda.synchronize(dev)
            e1.record(stream)
            e1.synchronize()
            launches += ctx.launch_count()
            tot += e0.elapsed_time(e1) / 1e3
        return tot, launches

    for _ in range(a.warmup):
        solve(False)
    with ClockSampler(local) as clk:
        t_dev, launches = timed(False, a.steps)
    t_e2e, _ = timed(True, a.steps)
    from paper_1607_00531_b200 import shard
    t_dev = shard.max_over_ranks(t_dev, dist, dev)
    t_e2e = shard.max_over_ranks(t_e2e, dist, dev)
    units = g.faces * iters * a.steps
    ctx.profile(True)
    ctx.profile_reset()
    solve(False)
    prof = ctx.profile_read()
    ctx.profile(False)
    kernels = [{"kernel": k, "ms_per_launch": ms / n, "launches": n}
               for k, (ms, n) in sorted(prof.items(), key=lambda kv: -kv[1][0])[:8] if n]
    cpu = None
    if rank == 0 and not a.no_cpu_baseline:
        try:
            chk, kind, cores = ref_checker(os.cpu_count() or 1)
            dt, _, _ = ref_admm_window(chk, cores, d, None, 1)
            cpu = {"value": g.faces / dt, "unit": UNIT, "cores": cores, "kind": kind,
                   "cpu_model": cpu_model(),
                   "sample": f"ADMM iteration 1 of the full {a.config} volume"}
        except Exception as e:
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                   "sample": str(e)[:120]}
    if rank == 0:
        h2d = (ip_h.numel() + im_h.numel()) * 8 * world
        line = {"metric": metric_for(a.config), "value": units / t_dev, "unit": UNIT,
                "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
                "ms_per_step": t_dev / a.steps * 1e3, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"ADMM {a.config} {'x'.join(map(str, g.dims()))}, "
                                       f"{iters} iterations, fp64, from b=0, k-slabs over "
                                       f"{world} GPU(s)",
                           "faces": g.faces, "iterations": iters, "parallelism": f"kslab{world}",
                           "l2": "working set > L2 (126 MB)"},
                "e2e": {"value": units / t_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": 3 * g.faces * 8},
                "gpu_launches": launches, "clocks": clk.summary(),
                "roofline": {"bound": "hbm", "kernel": "admm_bstep", "achieved": None,
                             "peak": None, "unit": "GB/s", "frac": None, "traffic": None,
                             "note": "see the C3 line for the b-step roofline; per-kernel times "
                                     "of one solve on rank 0 below", "kernels": kernels},
                "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_sharded_legs(a, ctx, dev, stream, dist, rank, world, iters=10):
    """--gpus N > 1 (or --sharded): the configs that shard one workload over
    the ranks, beside the C3 replicas, so a scaling run measures
    communication:
      C4: the 64 pairs in contiguous blocks per rank (epc_admm_solve_batch),
          no collective; value = all pairs' face-iterations / max-over-ranks time;
      C5: one 512x512x256 volume in k-slabs (dist_admm over NCCL): the time
          of every collective kind (all-to-all transposes, halo, all-gather)
          measured per rank (max over ranks), strong scaling.
    `iters` ADMM iterations per solve (fixed count)."""
    import torch
    from paper_1607_00531_b200 import dist_admm, shard
    cfg = abi.AdmmConfig(max_iter=iters, eps_abs=1e-300, eps_rel=1e-300)
    out = {}
    # C4
    first, npairs = shard.shard_range(64, rank, world)
    g4, ip4, im4 = synth.make_batch("C4", npairs=npairs, first=first)
    ip4d, im4d = torch.from_numpy(ip4).to(dev), torch.from_numpy(im4).to(dev)
    ctx.admm_solve_batch(g4, npairs, ip4d, im4d, cfg=abi.AdmmConfig(max_iter=1, eps_abs=1e-300, eps_rel=1e-300))
    torch.cuda.synchronize(dev)
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.admm_solve_batch(g4, npairs, ip4d, im4d, cfg=cfg)
    e1.record(stream)
    e1.synchronize()
    t4 = shard.max_over_ranks(e0.elapsed_time(e1) / 1e3, dist, dev)
    out["C4"] = {"workload": f"ADMM C4 64 x 128x128x64 pairs, {iters} iterations, pairs sharded over "
                             f"{world} ranks", "value": g4.faces * 64 * iters / t4, "unit": UNIT,
                 "seconds": t4, "scaling": "weak per pair, strong per batch", "collectives": {}}
    del ip4d, im4d
    # C5
    d5 = synth.make_config("C5")
    g5 = d5.grid
    slabs = dist_admm.Slabs(g5.m[0], g5.m[1], g5.m[2], world)
    k0, mk = slabs.k_range(rank)
    cl = g5.m[0] * g5.m[1]
    ip5 = torch.from_numpy(np.ascontiguousarray(d5.iplus[k0 * cl:(k0 + mk) * cl])).to(dev)
    im5 = torch.from_numpy(np.ascontiguousarray(d5.iminus[k0 * cl:(k0 + mk) * cl])).to(dev)
    del d5
    backend = dist_admm.DeviceBackend(ctx, dev)

    def solve(n, timings=None):
        c = abi.AdmmConfig(max_iter=n, eps_abs=1e-300, eps_rel=1e-300)
        gen = dist_admm.admm_rank(backend, g5, slabs, rank, ip5, im5, cfg=c)
        return dist_admm.run_torch(gen, dist, dev, timings=timings)

    solve(1)
    torch.cuda.synchronize(dev)
    dist.barrier()
    t0 = time.perf_counter()
    solve(iters)
    torch.cuda.synchronize(dev)
    t5 = shard.max_over_ranks(time.perf_counter() - t0, dist, dev)
    tim = {}
    solve(iters, timings=tim)  # a second solve with every collective timed
    coll = {k: {"seconds_per_iteration": shard.max_over_ranks(v[0], dist, dev) / iters,
                "calls_per_iteration": v[1] / iters} for k, v in sorted(tim.items())}
    out["C5"] = {"workload": f"ADMM C5 512x512x256, {iters} iterations, k-slabs over {world} ranks",
                 "value": g5.faces * iters / t5, "unit": UNIT, "seconds": t5, "scaling": "strong",
                 "collectives": coll,
                 "note": "wall time (the slab driver synchronises between steps); collective times "
                         "from a second, instrumented solve, max over ranks"}
    return out


def main():
    a = parse()
    iters = a.iters or DEFAULT_ITERS.get(a.config, 50)
    if a.impl == "reference":
        return run_reference_arm(a, iters)
    if a.config == "C5":
        return run_slabs(a, iters)

    import torch
    rank, world, local, dist = dist_setup(a.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_1607_00531_b200.epicorr import Context
    stream = torch.cuda.Stream(device=dev)
    ctx = Context(local, stream=stream)

    from dataclasses import replace

    from paper_1607_00531_b200 import shard
    cfg = abi.AdmmConfig(max_iter=iters, eps_abs=1e-300, eps_rel=1e-300)
    if a.config == "C4":
        # 64 independent pairs sharded across ranks (no data-path collective)
        total_pairs = 64
        first, npairs = shard.shard_range(total_pairs, rank, world)
        g, ipn, imn = synth.make_batch("C4", npairs=npairs, first=first, scale=a.scale)
    else:
        # each rank: its own volume pair (replica) of the config
        spec = synth.CONFIGS[a.config]
        spec = replace(spec, scale=a.scale, seed=spec.seed + 1000 * rank)
        d = synth.make_pair(spec)
        g, ipn, imn = d.grid, d.iplus, d.iminus
        total_pairs, npairs = world, 1
    ip_d = torch.from_numpy(ipn).to(dev)
    im_d = torch.from_numpy(imn).to(dev)
    ip_h = torch.from_numpy(ipn).pin_memory()
    im_h = torch.from_numpy(imn).pin_memory()
    bo_h = torch.empty(g.faces * npairs, dtype=torch.float64).pin_memory()
    zo_h = torch.empty(g.faces * npairs, dtype=torch.float64).pin_memory()
    uo_h = torch.empty(g.faces * npairs, dtype=torch.float64).pin_memory()
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)

    def solve_device():
        if npairs == 1 and a.config != "C4":
            return ctx.admm_solve(g, ip_d, im_d, cfg=cfg)
        return ctx.admm_solve_batch(g, npairs, ip_d, im_d, cfg=cfg)

    def solve_host():
        # C ABI with pinned host buffers: H2D of I+/I-, D2H of b, z, u inside the call
        import ctypes as C
        rows = (abi.AdmmRow * (iters * npairs))()
        st = (abi.SolveStatus * npairs)()
        rho = (C.c_double * npairs)()
        P = lambda t: C.c_void_p(t.data_ptr())
        rc = ctx.lib.epc_admm_solve_batch(ctx.h, C.byref(g), npairs, abi.EPC_MEM_HOST, P(ip_h),
                                          P(im_h), None, None, None, P(bo_h), P(zo_h), P(uo_h),
                                          rho, C.byref(abi.ObjectiveParams()), C.byref(cfg), 0,
                                          rows, iters, st)
        assert rc == 0, ctx._err()
        return st

    def barrier():
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def timed(fn, k):
        """Device time of k steps (CUDA events on the launching stream),
        L2 flushed (256 MB write) before each step outside the events."""
        tot = 0.0
        launches = 0
        for _ in range(k):
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            ctx.reset_launch_count()
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            launches += ctx.launch_count()
            tot += e0.elapsed_time(e1) / 1e3
        return tot, launches

    for _ in range(a.warmup):
        solve_device()
    barrier()
    with ClockSampler(local) as clk:
        barrier()
        t_dev, launches = timed(solve_device, a.steps)
        barrier()
    t_max = t_dev
    if dist is not None:
        tt = torch.tensor([t_dev], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    faces_iters = g.faces * iters
    value = faces_iters * total_pairs * a.steps / t_max

    # e2e through the C ABI with pinned host buffers
    solve_host()
    barrier()
    t_e2e, _ = timed(solve_host, a.steps)
    if dist is not None:
        tt = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())
    e2e = faces_iters * total_pairs * a.steps / t_e2e

    # roofline: per-kernel CUDA-event timing of one profiled solve
    ctx.profile(True)
    ctx.profile_reset()
    r_last = solve_device()
    prof = ctx.profile_read()
    ctx.profile(False)
    last_b = r_last["b"][:g.faces].double().cpu().numpy() if a.config != "C4" else None
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    nf, nc = g.faces, g.cells
    # algorithmic bytes per launch: b-step reads I+,I-,b,z,u and
    # writes b; each DCT GEMM reads + writes one face field (rhs GEMM reads b,u).
    alg = {"admm_bstep": 8 * (2 * nc + 4 * nf), "dct_fwd2": 8 * 3 * nf, "dct_fwd3_div": 8 * 2 * nf,
           "dct_inv3": 8 * 2 * nf, "dct_inv2_dual": 8 * 7 * nf}
    # The DCT GEMMs are fp64-pipe bound: 2*M*K*N unfused mul+add per transform
    # (exact k order, no FMA), against the measured fp64 issue rate
    # (scripts/ubench_fp64_tput.cu -> profiles/r01_ubench_fp64_tput.log).
    # the forward axis-2 transform fused into the b-step's drain (the default
    # at C3, bstep.cu: bstep_drain_fwd2): its bytes belong to the b-step launch
    # (launches whose b-step ran long, the first high-rho iterations, keep the
    # separate GEMM: the launch counts give the fused share)
    n_b = prof.get("admm_bstep", (0.0, 0))[1]
    n_f2 = prof.get("dct_fwd2", (0.0, 0))[1]
    fwd2_fused_frac = (1.0 - n_f2 / n_b) if (n_b and g.m[2] > 1) else 0.0
    fwd2_fused = fwd2_fused_frac > 0.5
    alg_bstep_alone = alg["admm_bstep"]
    alg_bstep_fused = alg["admm_bstep"] + alg["dct_fwd2"]
    alg["admm_bstep"] = int(alg_bstep_alone + fwd2_fused_frac * alg["dct_fwd2"])
    if n_f2 == 0:
        alg.pop("dct_fwd2")
    m1_, m2_, m3_ = g.m
    n1_ = m1_ + 1
    pairs_ = npairs if a.config == "C4" else 1
    fp64_ops = {"dct_fwd2": 2 * m2_ * m2_ * n1_ * m3_ * pairs_,
                "dct_inv2_dual": 2 * m2_ * m2_ * n1_ * m3_ * pairs_,
                "dct_fwd3_div": 2 * m3_ * m3_ * n1_ * m2_ * pairs_,
                "dct_inv3": 2 * m3_ * m3_ * n1_ * m2_ * pairs_}
    fp64_peak = float(peaks.get("fp64_tops", FP64_PEAK_TOPS)) * 1e12
    kernels = []
    for name, (ms, n) in prof.items():
        if name in alg and n:
            per = ms / n / 1e3
            gbs = alg[name] / per / 1e9
            k = {"kernel": name, "ms_per_launch": ms / n, "alg_bytes": alg[name],
                 "achieved_gbs": gbs, "frac_hbm": gbs / hbm_peak}
            if name in fp64_ops:
                k["fp64_tops"] = fp64_ops[name] / per / 1e12
                k["frac_fp64"] = fp64_ops[name] / per / fp64_peak
            kernels.append(k)
    top = max(prof.items(), key=lambda kv: kv[1][0])
    bname, (bms, bn) = top
    b_per = bms / bn / 1e3
    b_ach = alg.get(bname, 0) / b_per / 1e9
    # DRAM traffic of one b-step launch from the committed ncu --set full
    # capture summary (scripts/summarize_ncu.py), bytes per launch
    traffic, traffic_src, pipe = None, None, None
    try:
        cap = json.load(open(os.path.join(ROOT, "profiles", NCU_BSTEP_SUMMARY)))
        mb = float(cap["dram__bytes_read.sum"][0]) + float(cap["dram__bytes_write.sum"][0])
        if cap["dram__bytes_read.sum"][1] == "Mbyte":
            traffic, traffic_src = mb * 1e6, "profiles/" + NCU_BSTEP_SUMMARY
        # what does bound it: issue and fp64-pipe activity and the stall mix
        stalls = cap.get("stall_mix_pct", {})
        pipe = {"issue_active_frac": float(cap["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]) / 100,
                "fp64_pipe_active_frac":
                    float(cap["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"][0]) / 100,
                "top_stall": max(stalls.items(), key=lambda kv: kv[1])[0] if stalls else None,
                "source": "profiles/" + NCU_BSTEP_SUMMARY}
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": bname, "achieved": b_ach, "peak": hbm_peak,
                "peak_source": peak_src, "unit": "GB/s", "frac": b_ach / hbm_peak,
                "traffic": traffic, "traffic_source": traffic_src, "share_of_step": bms / sum(v[0] for v in prof.values()),
                "note": "b-step is fp64-latency bound (serial SQP/QP chains), not HBM bound"
                        + ("; the forward axis-2 DCT runs in its drain (bytes included)" if fwd2_fused else ""),
                "fwd2_fused": fwd2_fused, "fwd2_fused_frac": fwd2_fused_frac,
                # the captured launch (iteration 91) is a fused one when any are:
                # compare its DRAM traffic with that launch's algorithmic bytes
                "traffic_alg_bytes": alg_bstep_fused if fwd2_fused_frac > 0 else alg_bstep_alone,
                "traffic_over_alg": (traffic / (alg_bstep_fused if fwd2_fused_frac > 0 else alg_bstep_alone)
                                     if traffic else None),
                "bstep_pipes": pipe,
                "kernels": kernels}

    cpu = None
    if rank == 0 and not a.no_cpu_baseline and a.config != "C4":
        try:
            one = synth.VolumePairData(g, np.ascontiguousarray(ipn[:g.cells]),
                                       np.ascontiguousarray(imn[:g.cells]), None)
            cpu = cpu_windows_baseline(ctx, one, ip_d, im_d, iters, a.config,
                                       starts=[int(iters * f) for f in (0, .2, .4, .6, .8)], n=3)
        except Exception as e:  # the checker is optional on a bench box
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                   "sample": str(e)[:120]}

    gn = gn3 = x400 = None
    if not a.no_gn and a.config != "C4":
        gn = run_gn_leg(a, ctx, dev, stream, flush, rank, dist, a.gn_config, cpu_windows=10)
        if a.config == "C3" and not a.no_gn_c3:
            gn3 = run_gn_leg(a, ctx, dev, stream, flush, rank, dist, "C3", cpu_windows=1,
                             min_solves=3)
    if a.config == "C3" and not a.no_x400 and a.scale == 1.0:
        x400 = run_x400_leg(a, ctx, dev, stream, flush, iters, rank, dist)
    sharded = None
    if a.config == "C3" and (world > 1 or a.sharded) and dist is not None:
        try:  # the headline line must survive a failure in the sharded legs
            sharded = run_sharded_legs(a, ctx, dev, stream, dist, rank, world)
        except Exception as e:
            sharded = {"error": f"{type(e).__name__}: {e}"[:300]}
            print(f"[bench] sharded legs failed on rank {rank}: {e}", file=sys.stderr, flush=True)
    f32 = None
    if not a.no_f32 and a.config != "C4":
        f32 = run_f32_leg(a, ctx, dev, stream, flush, g, ipn, imn, iters, last_b, dist)

    if rank == 0:
        line = {"metric": metric_for(a.config), "value": value, "unit": UNIT, "n_gpus": world,
                "steps": a.steps, "warmup": a.warmup, "ms_per_step": t_max / a.steps * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": admm_config_dict(a, g, iters),
                "time_to_solution_s": t_max / a.steps,
                "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 2 * nc * 8 * npairs,
                        "d2h_bytes_per_step": 3 * nf * 8 * npairs},
                "gpu_launches": launches, "clocks": clk.summary(),
                "roofline": roofline, "cpu_baseline": cpu}
        if gn is not None:
            line["gn"] = gn
        if gn3 is not None:
            line["gn_c3"] = gn3
        if x400 is not None:
            line["x400"] = x400
        if sharded is not None:
            line["sharded"] = sharded
        if f32 is not None:
            line["fp32"] = f32
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
