"""Summaries for profiles/ (dev aid):
  launches <ncu --csv launch list> <out.csv>   per-kernel count / total ms / share
  capture  <.ncu-rep> <out.json>               key metrics + stall mix of one capture
"""
import collections
import csv
import json
import subprocess
import sys


def launches(src, dst):
    rows = [r for r in csv.reader(open(src)) if r]
    hdr = next(r for r in rows if "Kernel Name" in r)
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    unit = hdr.index("Metric Unit")
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
                 "nsecond": 1e-6}.get(r[unit], 1.0)
        name = r[ik].split("(")[0]
        tot[name] += float(r[iv].replace(",", "")) * scale
        cnt[name] += 1
    s = sum(tot.values())
    with open(dst, "w") as f:
        f.write("kernel,launches,total_ms,share\n")
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            f.write(f"{k},{cnt[k]},{v:.3f},{v / s:.4f}\n")


def capture(src, dst):
    out = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u = r[0], r[1]
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "launch__grid_size", "launch__block_size",
            "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]
    out_list = []
    for v in r[2:]:
        d = {}
        for k in keys:
            if k in h:
                i = h.index(k)
                d[k] = [v[i], u[i]]
        stalls = {}
        for i, n in enumerate(h):
            if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
                try:
                    x = float(v[i].replace(",", ""))
                except ValueError:
                    continue
                if x > 0:
                    stalls[n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = x
        t = sum(stalls.values()) or 1.0
        d["stall_mix_pct"] = {k: round(100 * x / t, 1) for k, x in
                              sorted(stalls.items(), key=lambda kv: -kv[1])}
        out_list.append(d)
    d = out_list[0] if len(out_list) == 1 else out_list  # one capture: a dict (bench reads it)
    json.dump(d, open(dst, "w"), indent=1)


def pcg(src, dst, pcg_iters, faces):
    """capture of one k_pcg_loop launch (one PCG solve of pcg_iters
    iterations): adds DRAM bytes per PCG iteration against the algorithmic
    120 B/face per iteration."""
    capture(src, dst)
    d = json.load(open(dst))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = sum(float(d[k][0].replace(",", "")) * scale[d[k][1]]
              for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    tu = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6,
          "ms": 1e-3}
    t = float(d["gpu__time_duration.sum"][0].replace(",", "")) * tu[d["gpu__time_duration.sum"][1]]
    n, f = int(pcg_iters), int(faces)
    d["pcg_iterations"] = n
    d["faces"] = f
    d["dram_bytes_per_pcg_iteration"] = tot / n
    d["alg_bytes_per_pcg_iteration"] = 120 * f
    d["traffic_over_alg"] = tot / n / (120 * f)
    d["dram_gbs_under_ncu"] = tot / t / 1e9
    json.dump(d, open(dst, "w"), indent=1)


def parts(src, dst, faces):
    """captures of the per-iteration PCG kernels (k_pcg_hvp, k_pcg_update_bj):
    DRAM bytes and time per launch against their algorithmic bytes (48 and
    72 B/face)."""
    capture(src, dst)
    d = json.load(open(dst))
    d = d if isinstance(d, list) else [d]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tu = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "us": 1e-6, "ms": 1e-3}
    out = {"faces": int(faces), "kernels": {}, "captures": d}
    for x in d:
        name = "pcg_hvp" if "pcg_hvp" in x["Kernel Name"][0] else "pcg_update"
        b = sum(float(x[k][0].replace(",", "")) * scale[x[k][1]]
                for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        t = float(x["gpu__time_duration.sum"][0].replace(",", "")) * tu[x["gpu__time_duration.sum"][1]]
        alg = (48 if name == "pcg_hvp" else 72) * int(faces)
        out["kernels"][name] = {"dram_bytes_per_launch": b, "alg_bytes_per_launch": alg,
                                "traffic_over_alg": b / alg, "seconds_under_ncu": t,
                                "dram_gbs_under_ncu": b / t / 1e9}
    json.dump(out, open(dst, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "parts":
        parts(*sys.argv[2:5])
        sys.exit(0)
    if sys.argv[1] == "pcg":
        pcg(*sys.argv[2:6])
    else:
        {"launches": launches, "capture": capture}[sys.argv[1]](sys.argv[2], sys.argv[3])
